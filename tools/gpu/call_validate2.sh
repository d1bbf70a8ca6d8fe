# Validation after the variant pruning: GPU suite + per-pass times + memcheck of the small sweep
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/w_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/w_pytest.txt
for sz in 512 1024; do timeout 300 python tools/pass_times.py --size $sz > gpurun_out/w_pass$sz.json 2>&1; done
timeout 600 python tools/sanitize_small.py > gpurun_out/w_sanitize_plain.txt 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_small.py > gpurun_out/w_memcheck.txt 2>&1; echo "rc=$?" >> gpurun_out/w_memcheck.txt
