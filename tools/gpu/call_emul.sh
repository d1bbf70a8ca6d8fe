timeout 600 python -m pytest tests/test_gpu_sharded.py -m gpu -q -x -k weak_scaling -p no:cacheprovider > gpurun_out/e_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/e_pytest.txt
timeout 900 python bench.py --emulate 2 --size 512 --steps 5 --warmup 3 > gpurun_out/e_emul2.json 2> gpurun_out/e_emul2.err; echo "rc=$?" >> gpurun_out/e_emul2.err
timeout 900 python bench.py --emulate 4 --size 256 --steps 5 --warmup 3 > gpurun_out/e_emul4.json 2> gpurun_out/e_emul4.err; echo "rc=$?" >> gpurun_out/e_emul4.err
