# ncu evidence for profiles/ (round 1, final state): bench lines (c2 default, c3), the launch
# list of the c2 bench, full captures of one preconditioner application (forward + backward
# k_line_solve) for c2 and c3 and of the c2 factor kernel
set -x
python bench.py > gpurun_out/r1c_bench_c2.json 2> gpurun_out/r1c_bench_c2.err &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1c_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1c_ncu_launch.log 2>&1
python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1c_bench_c3.json 2> gpurun_out/r1c_bench_c3.err
python tools/solve_probe.py c2 > gpurun_out/r1c_probe_c2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_line_solve -s 120 -c 2 -o gpurun_out/r1c_solve_c2 python tools/solve_probe.py c2 > gpurun_out/r1c_ncu_solve_c2.log 2>&1
python tools/solve_probe.py c3 > gpurun_out/r1c_probe_c3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_line_solve -s 120 -c 2 -o gpurun_out/r1c_solve_c3 python tools/solve_probe.py c3 > gpurun_out/r1c_ncu_solve_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_line_factor -c 1 -o gpurun_out/r1c_factor_c2 python tools/profile_case.py c2 0 > gpurun_out/r1c_ncu_factor.log 2>&1
ls -la gpurun_out/ | grep r1c
