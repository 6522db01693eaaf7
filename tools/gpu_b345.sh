timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1e_bench_c3.json 2> gpurun_out/r1e_bench_c3.err
timeout 900 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r1e_bench_c4.json 2> gpurun_out/r1e_bench_c4.err
timeout 900 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r1e_bench_c5.json 2> gpurun_out/r1e_bench_c5.err
timeout 300 python tools/solve_probe.py c3 > gpurun_out/r1e_probe_c3.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_line_solve -s 120 -c 2 -o gpurun_out/r1e_solve_c3 python tools/solve_probe.py c3 > gpurun_out/r1e_ncu_solve_c3.log 2>&1
ls gpurun_out | grep r1e
