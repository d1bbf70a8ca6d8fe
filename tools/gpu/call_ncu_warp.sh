# ncu --set full of the m = 1024 warp-owned fused gram pass (1024^3)
python tools/profile_kkt.py --size 1024 --reps 2 > gpurun_out/y_plain1024.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:warp_pass -s 1 -c 1 -o /tmp/y_w1024 python tools/profile_kkt.py --size 1024 --reps 2 > gpurun_out/y_ncu1024.log 2>&1
ncu -i /tmp/y_w1024.ncu-rep --page raw --csv > gpurun_out/y_w1024_raw.csv 2>&1
ncu -i /tmp/y_w1024.ncu-rep --page details --csv > gpurun_out/y_w1024_details.csv 2>&1
ncu -i /tmp/y_w1024.ncu-rep --page source --csv > gpurun_out/y_w1024_source.csv 2>&1
