# round 2, box 8: the c4 bench line with the CPU leg, the reference arm, the c4 launch list, and
# ncu --set full captures of the two dominant kernels on c4
timeout 900 python bench.py > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo "bench rc $?" >> gpurun_out/r2h_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2h_ref.json 2> gpurun_out/r2h_ref.err; echo "ref rc $?" >> gpurun_out/r2h_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_launches_c4.csv python tools/profile_case.py c4 > gpurun_out/r2h_launch_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_line_solve -s 6 -c 1 -o gpurun_out/r2h_solve_c4 python tools/profile_case.py c4 0 > gpurun_out/r2h_ncu_solve.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_line_factor -c 1 -o gpurun_out/r2h_factor_c4 python tools/profile_case.py c4 0 > gpurun_out/r2h_ncu_factor.log 2>&1
cut -c1-1500 gpurun_out/r2h_bench.json; tail -2 gpurun_out/r2h_bench.err; cat gpurun_out/r2h_ref.json; tail -2 gpurun_out/r2h_ref.err; tail -2 gpurun_out/r2h_launch_run.log; tail -2 gpurun_out/r2h_ncu_solve.log; tail -2 gpurun_out/r2h_ncu_factor.log; ls -la gpurun_out/ | grep r2h
