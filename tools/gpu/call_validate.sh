# Round-2 validation call: GPU suite, default bench, sharded bench paths.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/v_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/v_pytest.txt
timeout 900 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; echo "rc=$?" >> gpurun_out/v_bench.err
timeout 600 python bench.py --emulate 8 --size 128 --steps 5 --warmup 3 > gpurun_out/v_emul8.json 2> gpurun_out/v_emul8.err; echo "rc=$?" >> gpurun_out/v_emul8.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --sharded --size 256 --steps 5 --warmup 3 > gpurun_out/v_tr1.json 2> gpurun_out/v_tr1.err; echo "rc=$?" >> gpurun_out/v_tr1.err
for sz in 512 1024; do
  timeout 300 python tools/pass_times.py --size $sz > gpurun_out/v_pass$sz.json 2>&1
done
