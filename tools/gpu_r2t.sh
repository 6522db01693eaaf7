# round 2, box 20: factor — pivot chain on its own SM sub-partition (FFB_PIVSM 1 / 2) vs the
# previous warp roles (0); full factorisation time on c2, c4, c5 (first pass), same box
V=$PWD/paper_1508_02977_b200/_variants
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2t_tests.log 2>&1; tail -2 gpurun_out/r2t_tests.log
for i in 1 2; do
  for c in c2 c5 c4; do
    echo "pivsm1 $(timeout 300 python tools/profile_case.py $c 0)" >> gpurun_out/r2t.log 2>&1
    echo "pivsm0 $(FFB_LIB=$V/lib_pivsm0.so timeout 300 python tools/profile_case.py $c 0)" >> gpurun_out/r2t.log 2>&1
    echo "pivsm2 $(FFB_LIB=$V/lib_pivsm2.so timeout 300 python tools/profile_case.py $c 0)" >> gpurun_out/r2t.log 2>&1
  done
done
sed -e 's/ terms.*factor/ factor/' -e 's/ pcg.*//' gpurun_out/r2t.log
