# round 2, last validation (box 21): GPU suite, smoke, default bench, reference arm
( time timeout 1500 python -m pytest tests -x -q -m gpu ) > gpurun_out/r3t_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3t_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3t_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r3t_smoke.log
( time timeout 900 python bench.py ) > gpurun_out/r3t_bench_c4.json 2> gpurun_out/r3t_bench_c4.err; echo "bench rc $?" >> gpurun_out/r3t_bench_c4.err
( time timeout 900 python bench.py --impl reference ) > gpurun_out/r3t_ref_c4.json 2> gpurun_out/r3t_ref_c4.err; echo "ref rc $?" >> gpurun_out/r3t_ref_c4.err
tail -6 gpurun_out/r3t_pytest.log; cat gpurun_out/r3t_smoke.log; cut -c1-200 gpurun_out/r3t_bench_c4.json; tail -4 gpurun_out/r3t_bench_c4.err; cut -c1-200 gpurun_out/r3t_ref_c4.json; tail -4 gpurun_out/r3t_ref_c4.err
