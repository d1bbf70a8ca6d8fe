# launch list of the emulated N = 8 (C5 1024^3) sharded matvec bench path (one process, 8 slab ranks)
python bench.py --emulate 8 --size 512 --steps 1 --warmup 1 --no-solve > gpurun_out/el_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/el_launches.csv \
    python bench.py --emulate 8 --size 512 --steps 1 --warmup 1 --no-solve > gpurun_out/el_ncu.log 2>&1
