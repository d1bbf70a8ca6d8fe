# A/B of library variants (variants/*.so) on the emulated sharded bench path, then the sharded tests on TESTV
L=paper_2502_04217_b200/libfftlasso_b200.so
for rep in 1 2; do
for v in ${VARIANTS:-variants/*.so}; do
  b=$(basename $v .so); cp $v $L
  timeout 900 python bench.py --emulate ${EMU:-8} --size ${SIZE:-512} --steps 3 --warmup 2 --no-solve --no-cpu-baseline > gpurun_out/ve_${b}_${rep}.json 2>&1
done
done
if [ -n "$TESTV" ]; then cp $TESTV $L; timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_bounds.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ve_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/ve_pytest.txt; fi
