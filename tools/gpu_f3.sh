for i in 1 2; do timeout 120 python tools/profile_case.py c2 2>&1 | tail -1; done > gpurun_out/f3.log 2>&1
FFB_LIB=$PWD/paper_1508_02977_b200/libflowfem_b200_prof.so timeout 120 python tools/factor_timeline.py c2 > gpurun_out/f3_tl.log 2>&1
timeout 300 python -m pytest tests -x -q -m gpu > gpurun_out/f3_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/f3_pytest.log
cat gpurun_out/f3.log; tail -2 gpurun_out/f3_pytest.log
