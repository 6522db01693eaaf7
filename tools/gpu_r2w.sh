# round 2, box 22: factor tile read-modify-write targets prefetched into L1 before the DMMA
# products (FFB_RPF=1, default) vs not (lib_rpf0); one full factorisation, same box
V=$PWD/paper_1508_02977_b200/_variants
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2w_tests.log 2>&1; tail -2 gpurun_out/r2w_tests.log
for i in 1 2; do
  for c in c2 c5 c4; do
    echo "rpf1 $(timeout 300 python tools/profile_case.py $c 0)" >> gpurun_out/r2w.log 2>&1
    echo "rpf0 $(FFB_LIB=$V/lib_rpf0.so timeout 300 python tools/profile_case.py $c 0)" >> gpurun_out/r2w.log 2>&1
  done
done
sed -e 's/ terms.*factor/ factor/' -e 's/ pcg.*//' gpurun_out/r2w.log
