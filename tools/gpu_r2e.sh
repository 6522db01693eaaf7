# round 2, box 5: multi-rank protocol (in-process communicator), C++ drop-in + the reference's
# acceptance gate, then the whole GPU suite
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_cpp.py -q -m gpu -s > gpurun_out/r2e_new.log 2>&1; echo "rc $?" >> gpurun_out/r2e_new.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2e_pytest.log
tail -40 gpurun_out/r2e_new.log; tail -8 gpurun_out/r2e_pytest.log
