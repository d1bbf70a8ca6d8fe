# round-2 closing evidence on the final library: GPU suite, smoke, default bench, reference arm,
# the reference's own suite, launch list
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/g_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/g_smoke.txt
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/g_clocks.csv &
SMI=$!
timeout 1200 python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo "rc=$?" >> gpurun_out/g_bench.err
kill $SMI
timeout 900 python bench.py --impl reference > gpurun_out/g_ref.json 2> gpurun_out/g_ref.err; echo "rc=$?" >> gpurun_out/g_ref.err
if [ -d reference_suite ]; then timeout 900 python tools/run_reference_suite.py run -q -rf > gpurun_out/g_refsuite.txt 2>&1; echo "rc=$?" >> gpurun_out/g_refsuite.txt; fi
python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline > gpurun_out/g_k_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline > gpurun_out/g_k_ncu.log 2>&1
