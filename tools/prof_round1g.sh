# round 1, last state: the same captures as prof_round1f.sh after the pivot and accumulator changes
# an ncu --set full capture of the factor kernel on c2 and c3 (each ncu command only after
# the same command exited 0 without ncu)
set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r1g_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r1g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1g_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r1g_smoke.log
timeout 600 python bench.py > gpurun_out/r1g_bench_c2.json 2> gpurun_out/r1g_bench_c2.err
timeout 300 python bench.py --config c1 > gpurun_out/r1g_bench_c1.json 2> gpurun_out/r1g_bench_c1.err
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1g_bench_c3.json 2> gpurun_out/r1g_bench_c3.err
timeout 900 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r1g_bench_c4.json 2> gpurun_out/r1g_bench_c4.err
timeout 600 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r1g_bench_c5.json 2> gpurun_out/r1g_bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1g_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1g_ncu_launch.log 2>&1
timeout 120 python tools/profile_case.py c2 0 > gpurun_out/r1g_case_c2.log 2>&1 &&
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_line_factor -c 1 -o gpurun_out/r1g_factor_c2 python tools/profile_case.py c2 0 > gpurun_out/r1g_ncu_factor_c2.log 2>&1
ls -la gpurun_out/ | grep r1f
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1g_ref.json 2> gpurun_out/r1g_ref.err
