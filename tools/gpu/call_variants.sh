# A/B of library variants built into variants/*.so (per-pass times at 512^3 and 1024^3, then the families tests on the last)
L=paper_2502_04217_b200/libfftlasso_b200.so
for v in ${VARIANTS:-variants/*.so}; do
  b=$(basename $v .so); cp $v $L
  for sz in ${SIZES:-512 1024}; do timeout 300 python tools/pass_times.py --size $sz > gpurun_out/v_${b}_${sz}.json 2>&1; done
done
for v in ${VARIANTS:-variants/*.so}; do
  b=$(basename $v .so); cp $v $L
  for sz in ${SIZES:-512 1024}; do timeout 300 python tools/pass_times.py --size $sz > gpurun_out/v2_${b}_${sz}.json 2>&1; done
done
if [ -n "$TESTV" ]; then cp $TESTV $L; timeout 900 python -m pytest ${TESTS:-tests/test_gpu_variants.py tests/test_gpu_bounds.py} -m gpu -q -x -p no:cacheprovider > gpurun_out/v_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/v_pytest.txt; fi
