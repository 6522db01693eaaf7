# repeat the suite prefix up to the multi-GPU tests until the intermittent failure shows, keep its log
for i in $(seq 1 8); do
  timeout 600 python -m pytest tests/test_gpu_cpp.py tests/test_gpu_factor_variants.py tests/test_gpu_fullsize.py tests/test_gpu_known_answers.py tests/test_gpu_linsolve.py tests/test_gpu_metrics.py tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/r3y_run.log 2>&1
  rc=$?
  echo "run $i rc $rc: $(tail -1 gpurun_out/r3y_run.log)"
  if [ $rc -ne 0 ]; then grep -n "^E \|Error\|^tests.*Error\|FAILED" gpurun_out/r3y_run.log | head -40; cp gpurun_out/r3y_run.log gpurun_out/r3y_fail_$i.log; break; fi
done
