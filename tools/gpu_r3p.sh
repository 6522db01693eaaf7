# round 2 (re-entry), box 15: single-precision factor copy: tests, then c4/c3 chains with FFB_FACTOR_F32=0/1
timeout 300 python -m pytest tests/test_gpu_tile_solve.py -x -q -m gpu 2>&1 | tail -4
timeout 300 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "c3" 2>&1 | tail -4
for v in 0 1; do
  echo "== c4 FFB_FACTOR_F32=$v"; FFB_FACTOR_F32=$v timeout 300 python tools/profile_case.py c4 2>&1 | tail -1
  echo "== c3 FFB_FACTOR_F32=$v"; FFB_FACTOR_F32=$v timeout 300 python tools/profile_case.py c3 2>&1 | tail -1
done
