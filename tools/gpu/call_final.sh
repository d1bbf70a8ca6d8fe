# full GPU suite + smoke + default bench + reference arm (round-2 evidence)
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/f_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/f_smoke.txt
timeout 1200 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "rc=$?" >> gpurun_out/f_bench.err
