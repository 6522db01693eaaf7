# round 2 (re-entry), box 8: c4 bench line with the table-driven rt solve + ncu --set full of one application
( time timeout 900 python bench.py ) > gpurun_out/r3h_bench_c4.json 2> gpurun_out/r3h_bench_c4.err; echo "bench rc $?"
cut -c1-200 gpurun_out/r3h_bench_c4.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_line_solve_rt -s 4 -c 1 \
  -o gpurun_out/r3h_rt_c4 python tools/profile_case.py c4 0 > gpurun_out/r3h_ncu.log 2>&1
ncu -i gpurun_out/r3h_rt_c4.ncu-rep --page source --csv --print-source sass > gpurun_out/r3h_src.csv 2>&1
ncu -i gpurun_out/r3h_rt_c4.ncu-rep --page details > gpurun_out/r3h_details.txt 2>&1
bash tools/ncu_summary.sh gpurun_out/r3h_rt_c4.ncu-rep > gpurun_out/r3h_rt_c4_summary.txt
cat gpurun_out/r3h_rt_c4_summary.txt
