# round 2, box 12: whole GPU suite with the extrapolated warm start; the 20-warp ring-solve
# variant (paper_1508_02977_b200/_variants, FFB_SOLVE_WARPS=20) against the default on c4
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2l_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2l_pytest.log
timeout 300 python tools/profile_case.py c4 0 > gpurun_out/r2l_w16.log 2>&1
FFB_LIB=$PWD/paper_1508_02977_b200/_variants/libflowfem_b200_w20.so timeout 300 python tools/profile_case.py c4 0 > gpurun_out/r2l_w20.log 2>&1
timeout 300 python tools/profile_case.py c4 0 >> gpurun_out/r2l_w16.log 2>&1
tail -8 gpurun_out/r2l_pytest.log; for f in gpurun_out/r2l_w*.log; do echo $f; cat $f; done
