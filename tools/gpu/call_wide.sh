timeout 600 python -m pytest tests/test_gpu_variants.py -m gpu -q -x -p no:cacheprovider > gpurun_out/w_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/w_pytest.txt
FL_WIDE=1 timeout 600 python -m pytest tests/test_gpu_variants.py tests/test_gpu_operators.py -m gpu -q -x -p no:cacheprovider > gpurun_out/w_pytest_wide.txt 2>&1; echo "rc=$?" >> gpurun_out/w_pytest_wide.txt
FL_WIDE=1 timeout 300 python tools/pass_times.py --size 512 > gpurun_out/w_pass512_wide.json 2>&1
FL_WIDE=0 timeout 300 python tools/pass_times.py --size 512 > gpurun_out/w_pass512_mirror.json 2>&1
