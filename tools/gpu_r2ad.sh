# round 2, box 29: instruction count of one c5 ring-solve launch after chunk_end_from
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_lsu.sum --clock-control none -k regex:k_line_solve -s 4 -c 2 python tools/profile_case.py c5 0 > gpurun_out/r2ad.txt 2>&1
grep -E "duration|inst_executed" gpurun_out/r2ad.txt
