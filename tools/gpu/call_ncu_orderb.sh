# order B kernels: per-pass times and ncu --set full of the strided fused gram (mirror) and the contiguous analysis + KKT epilogue
FL_ORDER=1 timeout 300 python tools/pass_times.py --size 512 > gpurun_out/b_pass512.json 2>&1
FL_ORDER=1 python tools/profile_kkt.py --size 512 --reps 2 > gpurun_out/b_plain512.log 2>&1 && \
FL_ORDER=1 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"mirror_passILi512ELb1ELi2|group_passILi512ELi1ELb1" -c 2 -o /tmp/b_ob512 python tools/profile_kkt.py --size 512 --reps 2 > gpurun_out/b_ncu512.log 2>&1
ncu -i /tmp/b_ob512.ncu-rep --page raw --csv > gpurun_out/b_ob512_raw.csv 2>&1
ncu -i /tmp/b_ob512.ncu-rep --page details --csv > gpurun_out/b_ob512_details.csv 2>&1
ncu -i /tmp/b_ob512.ncu-rep --page source --csv > gpurun_out/b_ob512_source.csv 2>&1
