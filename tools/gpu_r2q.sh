# round 2, box 17: ncu --set full of one k_line_solve_rt launch on c4 (source-mapped)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_line_solve_rt -s 4 -c 1 \
  -o gpurun_out/r2q_rt_c4 python tools/profile_case.py c4 0 > gpurun_out/r2q_ncu.log 2>&1
tail -2 gpurun_out/r2q_ncu.log
ncu -i gpurun_out/r2q_rt_c4.ncu-rep --page raw --csv > gpurun_out/r2q_raw.csv 2>&1
ncu -i gpurun_out/r2q_rt_c4.ncu-rep --page source --csv --print-source sass > gpurun_out/r2q_src.csv 2>&1
ncu -i gpurun_out/r2q_rt_c4.ncu-rep --page details > gpurun_out/r2q_details.txt 2>&1
ls -la gpurun_out/r2q*
