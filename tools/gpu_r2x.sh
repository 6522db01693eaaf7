# round 2, box 23: the whole -m gpu suite with durations, then smoke()
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/r2x_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/r2x_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
