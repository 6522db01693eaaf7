# round 2, box 16: row-group tile ring kernel (k_line_solve_rt) — parity tests, then the
# preconditioner application A/B against the row-batch ring (FFB_SOLVE=ring) on c3 / c4
timeout 900 python -m pytest tests/test_gpu_tile_solve.py -x -q > gpurun_out/r2p_tests.log 2>&1
tail -3 gpurun_out/r2p_tests.log
for c in c3 c4; do
  timeout 300 python tools/solve_probe.py $c 0 >> gpurun_out/r2p_probe.log 2>&1
  FFB_SOLVE=ring timeout 300 python tools/solve_probe.py $c 0 >> gpurun_out/r2p_probe.log 2>&1
done
cat gpurun_out/r2p_probe.log
