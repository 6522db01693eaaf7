# round 2, box 28: ring solve chunk ends without the square root (chunk_end_from) — c5 solve
# time (4-CTA clusters) and the solve tests
timeout 900 python -m pytest tests/test_gpu_tile_solve.py tests/test_gpu_fullsize.py -x -q -k "c5 or ring or persistent or row_group" > gpurun_out/r2ac_tests.log 2>&1; tail -2 gpurun_out/r2ac_tests.log
for i in 1 2; do timeout 300 python tools/profile_case.py c5 0 | tail -1; done
FFB_SOLVE=ring timeout 300 python tools/solve_probe.py c4 0
timeout 300 python tools/solve_probe.py c4 0
