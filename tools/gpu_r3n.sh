# stress: the tile-solve test file 12 times with a per-test timeout (an intermittent hang was seen once)
for i in $(seq 1 12); do
  timeout 300 python -m pytest tests/test_gpu_tile_solve.py -q -m gpu --timeout 45 -x 2>&1 | tail -2 | tr '\n' ' '; echo " [run $i]"
done
for i in 1 2 3; do timeout 120 python tools/rank_share_probe.py 270 3840 32 2 4 2>&1 | tail -2; done
