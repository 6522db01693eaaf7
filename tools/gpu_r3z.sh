# repeat the whole GPU suite until the intermittent failure shows; keep the failing log
for i in $(seq 1 8); do
  timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r3z_run.log 2>&1
  rc=$?
  echo "run $i rc $rc: $(tail -1 gpurun_out/r3z_run.log)"
  if [ $rc -ne 0 ]; then cp gpurun_out/r3z_run.log gpurun_out/r3z_fail_$i.log; grep -n "^E \|FAILED\|Error" gpurun_out/r3z_run.log | head -40; break; fi
done
