timeout 600 python -m pytest tests/test_gpu_variants.py tests/test_gpu_bounds.py tests/test_gpu_operators.py -m gpu -q -x -p no:cacheprovider > gpurun_out/z_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/z_pytest.txt
FL_W16=1 timeout 300 python tools/pass_times.py --size 512 > gpurun_out/z_pass512_w16.json 2>&1
FL_W16=0 timeout 300 python tools/pass_times.py --size 512 > gpurun_out/z_pass512_grp.json 2>&1
