# bench (default run) + the new GPU tests
timeout 600 python -m pytest tests/test_gpu_bounds.py tests/test_gpu_sharded.py -m gpu -q -p no:cacheprovider > gpurun_out/b_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/b_pytest.txt
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/b_clocks.csv &
SMI=$!
timeout 1200 python bench.py > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err; echo "rc=$?" >> gpurun_out/b_bench.err
kill $SMI
timeout 900 python bench.py --impl reference > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err; echo "rc=$?" >> gpurun_out/b_ref.err
