timeout 600 python -m pytest tests/test_gpu_variants.py tests/test_gpu_bounds.py -m gpu -q -x -p no:cacheprovider > gpurun_out/z_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/z_pytest.txt
for sz in 512 1024; do timeout 300 python tools/pass_times.py --size $sz > gpurun_out/z_pass${sz}.json 2>&1; done
