# round 2 (re-entry), box 17: factor tile update with the tile as the accumulators' initial value (FFB_ACCX=1, built in) vs the read-modify-write after the products (variant lib)
timeout 600 python -m pytest tests/test_gpu_factor_variants.py tests/test_gpu_parity.py tests/test_gpu_linsolve.py -x -q -m gpu 2>&1 | tail -3
for rep in 1 2; do
for c in c4 c3 c2 c5; do
  unset FFB_LIB; echo "== $c accx=1"; timeout 300 python tools/profile_case.py $c 2>&1 | tail -1 | cut -c1-110
  export FFB_LIB=$PWD/paper_1508_02977_b200/_variants/lib_ACCX_0.so; echo "== $c accx=0"; timeout 300 python tools/profile_case.py $c 2>&1 | tail -1 | cut -c1-110
done
done
