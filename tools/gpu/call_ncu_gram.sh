# ncu --set full of the group-decoupled fused gram pass (512^3) and the 1024^3 matvec passes;
# raw/source pages exported as CSV on the box (the .ncu-rep files exceed the 64 MiB return limit)
python tools/profile_kkt.py --size 512 --reps 2 > gpurun_out/n_plain512.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:group_pass -s 1 -c 1 -o /tmp/n_gram512 python tools/profile_kkt.py --size 512 --reps 2 > gpurun_out/n_ncu512.log 2>&1
ncu -i /tmp/n_gram512.ncu-rep --page raw --csv > gpurun_out/n_gram512_raw.csv 2>&1
ncu -i /tmp/n_gram512.ncu-rep --page source --csv > gpurun_out/n_gram512_source.csv 2>&1
ncu -i /tmp/n_gram512.ncu-rep --page details --csv > gpurun_out/n_gram512_details.csv 2>&1
python tools/profile_kkt.py --size 1024 --reps 2 > gpurun_out/n_plain1024.log 2>&1 && \
ncu --set full --clock-control none -k regex:"group_pass|split_pass|fast_pass" -s 5 -c 5 -o /tmp/n_kkt1024 python tools/profile_kkt.py --size 1024 --reps 2 > gpurun_out/n_ncu1024.log 2>&1
ncu -i /tmp/n_kkt1024.ncu-rep --page raw --csv > gpurun_out/n_kkt1024_raw.csv 2>&1
ncu -i /tmp/n_kkt1024.ncu-rep --page details --csv > gpurun_out/n_kkt1024_details.csv 2>&1
ls -la gpurun_out > gpurun_out/n_ls.txt
