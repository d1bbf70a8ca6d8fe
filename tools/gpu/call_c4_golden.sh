mkdir -p gpurun_out/golden
nohup python oracle/make_golden_fullsize.py --engine oracle c4 --out-dir gpurun_out/golden > gpurun_out/c4_oracle.log 2>&1 &
OPID=$!
nvidia-smi --query-gpu=name,memory.total --format=csv > gpurun_out/smi.txt; free -g >> gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python tools/pass_times.py --size 512 > gpurun_out/pass512.json 2>&1
timeout 300 python tools/pass_times.py --size 1024 > gpurun_out/pass1024.json 2>&1
wait $OPID; echo "oracle rc=$?" >> gpurun_out/c4_oracle.log
