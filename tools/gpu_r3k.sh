# round 2 (re-entry), box 12: cluster row-group tile solve: tests, rank-share probe (8-GPU and 4-GPU shares of c4, c3 shares)
timeout 600 python -m pytest tests/test_gpu_tile_solve.py -x -q -m gpu 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ras.py tests/test_gpu_fullsize.py -x -q -m gpu 2>&1 | tail -5
timeout 200 python tools/rank_share_probe.py 270 3840 32 1 2 4 2>&1 | tail -3
timeout 200 python tools/rank_share_probe.py 540 3840 64 1 2 2>&1 | tail -2
timeout 200 python tools/rank_share_probe.py 270 1920 16 1 2 4 8 2>&1 | tail -4
