# round 2, box 29: early start of the factor's look-ahead path (FFB_EARLYPIV=1, built in) vs the Z barrier for everybody (variant lib)
timeout 600 python -m pytest tests/test_gpu_factor_variants.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
for rep in 1 2; do
for c in c4 c3 c2; do
  unset FFB_LIB; echo "== $c early=1"; timeout 300 python tools/profile_case.py $c 2>&1 | tail -1 | cut -c1-110
  export FFB_LIB=$PWD/paper_1508_02977_b200/_variants/lib_EARLYPIV_0.so; echo "== $c early=0"; timeout 300 python tools/profile_case.py $c 2>&1 | tail -1 | cut -c1-110
done
done
