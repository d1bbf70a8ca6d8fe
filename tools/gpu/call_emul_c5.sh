# the N = 8 (C5, 1024^3) bench code path emulated on one GPU: 8 slab ranks in one process
timeout 1500 python bench.py --emulate 8 --size 512 --steps 3 --warmup 2 > gpurun_out/c5_emul8.json 2> gpurun_out/c5_emul8.err; echo "rc=$?" >> gpurun_out/c5_emul8.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --sharded --size 256 --steps 5 --warmup 3 > gpurun_out/c5_tr1.json 2> gpurun_out/c5_tr1.err; echo "rc=$?" >> gpurun_out/c5_tr1.err
