# source-level ncu captures of the c2 solve and factor kernels (stall reasons per line)
set -x
ncu --set full --clock-control none --import-source on -k regex:k_line_solve -s 120 -c 2 -o gpurun_out/s3_solve_c2 python tools/solve_probe.py c2 > gpurun_out/s3_ncu_solve_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_line_factor -c 1 -o gpurun_out/s3_factor_c2 python tools/profile_case.py c2 0 > gpurun_out/s3_ncu_factor.log 2>&1
ls -la gpurun_out/ | grep s3_
