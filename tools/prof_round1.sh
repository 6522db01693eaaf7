# ncu evidence for profiles/: launch list of one c2 solve + full capture of the solve and factor kernels
set -x
python tools/profile_case.py c2 1 > gpurun_out/r1_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches_c2.csv python tools/profile_case.py c2 1 > gpurun_out/r1_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_line_solve -s 4 -c 2 -o gpurun_out/r1_solve_c2 python tools/profile_case.py c2 0 > gpurun_out/r1_ncu_solve.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_line_factor -c 1 -o gpurun_out/r1_factor_c2 python tools/profile_case.py c2 0 > gpurun_out/r1_ncu_factor.log 2>&1
python tools/profile_case.py c3 0 > gpurun_out/r1_plain_c3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_line_solve -s 4 -c 2 -o gpurun_out/r1_solve_c3 python tools/profile_case.py c3 0 > gpurun_out/r1_ncu_solve_c3.log 2>&1
ls -la gpurun_out/
