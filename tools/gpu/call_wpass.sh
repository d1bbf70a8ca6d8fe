# warp pass (m = 1024): GPU suite subset + per-pass times
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_operators.py tests/test_gpu_bounds.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/x_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/x_pytest.txt
for sz in 512 1024; do timeout 300 python tools/pass_times.py --size $sz > gpurun_out/x_pass${sz}.json 2>&1; done
