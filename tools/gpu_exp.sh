# branch-free pivot rsqrt: pivot microbench, parity tests, c2/c3/c5 timings
set -x
(cd tools/microbench && timeout 60 ./pivot > ../../gpurun_out/e_pivot_mb.log 2>&1)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tile_solve.py -x -q -m gpu > gpurun_out/e_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/e_pytest.log
for c in c2 c2 c3 c5; do timeout 300 python tools/profile_case.py $c >> gpurun_out/e_cases.log 2>&1; done
