# round 2 (re-entry), box 1: full round-end style check at HEAD + ncu launch list of the bench command
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 ) > gpurun_out/r3a_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3a_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r3a_smoke.log
( time timeout 900 python bench.py ) > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err; echo "bench rc $?" >> gpurun_out/r3a_bench.err
( time timeout 900 python bench.py --impl reference ) > gpurun_out/r3a_ref.json 2> gpurun_out/r3a_ref.err; echo "ref rc $?" >> gpurun_out/r3a_ref.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3a_launches_c4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r3a_ncu.log 2>&1; echo "ncu rc $?" >> gpurun_out/r3a_ncu.log
tail -25 gpurun_out/r3a_pytest.log; cat gpurun_out/r3a_smoke.log; cut -c1-400 gpurun_out/r3a_bench.json; tail -5 gpurun_out/r3a_bench.err; cut -c1-600 gpurun_out/r3a_ref.json; tail -5 gpurun_out/r3a_ref.err; tail -3 gpurun_out/r3a_ncu.log
