# round 2, box 13: unmasked full blocks in the ring solve's row loop (c3/c4 line widths)
timeout 300 python tools/profile_case.py c4 0 > gpurun_out/r2m_c4.log 2>&1
timeout 300 python tools/profile_case.py c4 0 >> gpurun_out/r2m_c4.log 2>&1
timeout 300 python tools/profile_case.py c3 0 > gpurun_out/r2m_c3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tile_solve.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_multi.py -q -m gpu -x > gpurun_out/r2m_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2m_tests.log
cat gpurun_out/r2m_c4.log gpurun_out/r2m_c3.log; tail -3 gpurun_out/r2m_tests.log
