# round-2 launch list of the bench's matvec part + --set full of the matvec kernels at 512^3 (order B: five passes)
python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline > gpurun_out/k_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/k_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline > gpurun_out/k_ncu_launch.log 2>&1
python tools/profile_kkt.py --size 512 --reps 2 > gpurun_out/k_plain2.log 2>&1 && \
ncu --set full --clock-control none -k regex:"pass|epilogue" -s 5 -c 5 -o /tmp/k_full python tools/profile_kkt.py --size 512 --reps 2 > gpurun_out/k_ncu_full.log 2>&1
ncu -i /tmp/k_full.ncu-rep --page raw --csv > gpurun_out/k_full_raw.csv 2>&1
