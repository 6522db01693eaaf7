# round 2, session 3: round-end style check at HEAD (GPU tests, smoke, default c4 bench, reference arm)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2ae_smi.txt
( time timeout 1500 python -m pytest tests -x -q -m gpu ) > gpurun_out/r2ae_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2ae_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ae_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r2ae_smoke.log
( time timeout 1200 python bench.py ) > gpurun_out/r2ae_bench.json 2> gpurun_out/r2ae_bench.err; echo "bench rc $?" >> gpurun_out/r2ae_bench.err
( time timeout 1200 python bench.py --impl reference ) > gpurun_out/r2ae_ref.json 2> gpurun_out/r2ae_ref.err; echo "ref rc $?" >> gpurun_out/r2ae_ref.err
tail -3 gpurun_out/r2ae_pytest.log; cat gpurun_out/r2ae_smoke.log; cut -c1-400 gpurun_out/r2ae_bench.json; tail -4 gpurun_out/r2ae_bench.err; cut -c1-300 gpurun_out/r2ae_ref.json; tail -4 gpurun_out/r2ae_ref.err
