# round 2, box 24: lagged factor experiment (FFB_LAG_FACTOR=1: factor once per chain, keep
# the factors across alpha updates) vs refactoring after every update; full chains
for c in c2 c3 c5 c4; do
  echo "refactor $(timeout 600 python tools/profile_case.py $c)" >> gpurun_out/r2y.log 2>&1
  echo "lagged   $(FFB_LAG_FACTOR=1 timeout 600 python tools/profile_case.py $c)" >> gpurun_out/r2y.log 2>&1
done
cat gpurun_out/r2y.log
