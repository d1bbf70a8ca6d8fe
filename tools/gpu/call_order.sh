# A/B: operator pass order B (contiguous synthesis first, fused mask pass on strided axis 0, KKT epilogue fused into the last contiguous analysis)
FL_ORDER=1 timeout 900 python -m pytest tests/test_gpu_operators.py tests/test_gpu_fullsize.py tests/test_gpu_solver.py -m gpu -q -x -p no:cacheprovider > gpurun_out/o_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/o_pytest.txt
for sz in 512 1024; do
for o in 0 1; do FL_ORDER=$o timeout 300 python tools/pass_times.py --size $sz > gpurun_out/o_pass${sz}_$o.json 2>&1; done
done
