# round 2, box 15: what bounds the c4 ring solve — FFB_SOLVE_DBG decomposition (1 skip the row
# arithmetic, 2 skip the line exchange, 4 skip the bulk copies; timing only)
timeout 600 python tools/solve_probe.py c4 0 4 1 5 > gpurun_out/r2o_probe_c4.log 2>&1
timeout 600 python tools/solve_probe.py c3 0 4 1 5 > gpurun_out/r2o_probe_c3.log 2>&1
cat gpurun_out/r2o_probe_c4.log gpurun_out/r2o_probe_c3.log
