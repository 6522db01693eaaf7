# repeat the c3 two-rank test until it fails (intermittent failure seen once in three suite runs)
for i in $(seq 1 12); do
  timeout 300 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "c3_two_ranks" > gpurun_out/r3x_run.log 2>&1
  rc=$?
  echo "run $i rc $rc"
  if [ $rc -ne 0 ]; then grep -n "Error\|assert\|^E " gpurun_out/r3x_run.log | head -30; cp gpurun_out/r3x_run.log gpurun_out/r3x_fail_$i.log; fi
done
