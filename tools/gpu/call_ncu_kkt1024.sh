# ncu --set full of the six launches of one 1024^3 KKT matvec (order A) with the final library
python tools/profile_kkt.py --size 1024 --reps 2 > gpurun_out/k1024_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:"pass|epilogue" -s 6 -c 6 -f -o /tmp/k1024_full python tools/profile_kkt.py --size 1024 --reps 2 > gpurun_out/k1024_ncu.log 2>&1
ncu -i /tmp/k1024_full.ncu-rep --page raw --csv > gpurun_out/k1024_raw.csv 2>&1
