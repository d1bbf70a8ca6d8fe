# round-2 final evidence: GPU suite, smoke, default bench (+ clocks), the reference's own suite
# against the drop-in (needs reference_suite/ from `tools/run_reference_suite.py fetch`),
# and the ncu launch list of the bench's matvec part
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/f_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/f_smoke.txt
timeout 1200 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "rc=$?" >> gpurun_out/f_bench.err
if [ -d reference_suite ]; then timeout 900 python tools/run_reference_suite.py run -q -rf > gpurun_out/f_refsuite.txt 2>&1; echo "rc=$?" >> gpurun_out/f_refsuite.txt; fi
python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline > gpurun_out/f_k_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline > gpurun_out/f_k_ncu.log 2>&1
# ncu --set full of the five 512^3 matvec launches (order B) for the traffic / stall summary
python tools/profile_kkt.py --size 512 --reps 2 > gpurun_out/f_plain2.log 2>&1 && \
ncu --set full --clock-control none -k regex:"pass|epilogue" -s 5 -c 5 -o /tmp/f_full python tools/profile_kkt.py --size 512 --reps 2 > gpurun_out/f_ncu_full.log 2>&1
ncu -i /tmp/f_full.ncu-rep --page raw --csv > gpurun_out/f_full_raw.csv 2>&1
