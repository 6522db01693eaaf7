# round-end style check: GPU tests, smoke, default bench, reference arm
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r1h_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r1h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1h_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r1h_smoke.log
timeout 600 python bench.py > gpurun_out/r1h_bench.json 2> gpurun_out/r1h_bench.err; echo "bench rc $?" >> gpurun_out/r1h_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1h_ref.json 2> gpurun_out/r1h_ref.err; echo "ref rc $?" >> gpurun_out/r1h_ref.err
tail -2 gpurun_out/r1h_pytest.log; cat gpurun_out/r1h_smoke.log; cut -c1-300 gpurun_out/r1h_bench.json; tail -1 gpurun_out/r1h_bench.err; cat gpurun_out/r1h_ref.json; tail -2 gpurun_out/r1h_ref.err
