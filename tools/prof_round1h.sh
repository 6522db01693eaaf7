# round 1, final state after the tile-solve owner changes: GPU tests, smoke, c1/c2 bench
# lines, the c2 launch list and an ncu --set full capture of the c2 tile solve (each ncu
# command only after the same command exited 0 without ncu)
set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r1h_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r1h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1h_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r1h_smoke.log
timeout 600 python bench.py > gpurun_out/r1h_bench_c2.json 2> gpurun_out/r1h_bench_c2.err
timeout 300 python bench.py --config c1 > gpurun_out/r1h_bench_c1.json 2> gpurun_out/r1h_bench_c1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1h_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1h_ncu_launch.log 2>&1
timeout 120 python tools/solve_probe.py c2 > gpurun_out/r1h_probe_c2.log 2>&1 &&
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_line_solve -s 120 -c 2 -o gpurun_out/r1h_solve_c2 python tools/solve_probe.py c2 > gpurun_out/r1h_ncu_solve_c2.log 2>&1
ls -la gpurun_out/ | grep r1h
