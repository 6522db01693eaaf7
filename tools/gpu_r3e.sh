# round 2 (re-entry), box 5: source-level ncu of one k_line_solve_rt launch on c4 (instruction counts per SASS line)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_line_solve_rt -s 4 -c 1 \
  -o gpurun_out/r3e_rt_c4 python tools/profile_case.py c4 0 > gpurun_out/r3e_ncu.log 2>&1
tail -2 gpurun_out/r3e_ncu.log
ncu -i gpurun_out/r3e_rt_c4.ncu-rep --page source --csv --print-source sass > gpurun_out/r3e_src.csv 2>&1
ncu -i gpurun_out/r3e_rt_c4.ncu-rep --page details > gpurun_out/r3e_details.txt 2>&1
ls -la gpurun_out/r3e*
