# ncu --set full of the strided fused gram (512^3, order B) of the library in place; raw/source/details as CSV
python tools/profile_kkt.py --size 512 --reps 2 > gpurun_out/s_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on ${NCUARGS} -k regex:"${KREGEX:-sgram_pass}" -s ${KSKIP:-1} -c 1 -f -o /tmp/s_gram python tools/profile_kkt.py --size 512 --reps 2 > gpurun_out/s_ncu.log 2>&1
ncu -i /tmp/s_gram.ncu-rep --page raw --csv > gpurun_out/s_raw.csv 2>&1
ncu -i /tmp/s_gram.ncu-rep --page source --csv > gpurun_out/s_source.csv 2>&1
ncu -i /tmp/s_gram.ncu-rep --page details --csv > gpurun_out/s_details.csv 2>&1
