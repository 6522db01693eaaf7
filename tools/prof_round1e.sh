# ncu evidence for profiles/ (round 1, after the diagonal-tile fix): bench lines (c2
# and of the c2 factor kernel. Each ncu command runs only after the same command exited 0.
set -x
timeout 600 python bench.py > gpurun_out/r1e_bench_c2.json 2> gpurun_out/r1e_bench_c2.err &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1e_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1e_ncu_launch.log 2>&1
timeout 300 python bench.py --config c1 > gpurun_out/r1e_bench_c1.json 2> gpurun_out/r1e_bench_c1.err
timeout 120 python tools/solve_probe.py c2 > gpurun_out/r1e_probe_c2.log 2>&1 &&
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_line_solve -s 120 -c 2 -o gpurun_out/r1e_solve_c2 python tools/solve_probe.py c2 > gpurun_out/r1e_ncu_solve_c2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_line_factor -c 1 -o gpurun_out/r1e_factor_c2 python tools/profile_case.py c2 0 > gpurun_out/r1e_ncu_factor.log 2>&1
ls -la gpurun_out/ | grep r1e
