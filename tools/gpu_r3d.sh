# round 2 (re-entry), box 4: table-driven rt solve: tests touching it, sustained probe on c4, c3 application time
timeout 900 python -m pytest tests/test_gpu_tile_solve.py tests/test_gpu_fullsize.py tests/test_gpu_multi.py tests/test_gpu_ras.py -x -q -m gpu 2>&1 | tail -5
timeout 300 python tools/power_probe.py c4 300 2>&1 | grep solve
timeout 300 python tools/solve_probe.py c3 0 2>&1 | tail -1
