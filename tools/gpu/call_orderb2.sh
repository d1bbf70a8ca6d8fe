FL_ORDER=1 timeout 300 python tools/pass_times.py --size 1024 > gpurun_out/b3_pass1024.json 2>&1
FL_ORDER=1 timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider > gpurun_out/b3_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/b3_pytest.txt
