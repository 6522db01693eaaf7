# quick factor/solve check: band tests + timing of c2, c3, c5 (one adaptive solve each)
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tile_solve.py -x -q -m gpu > gpurun_out/q_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/q_pytest.log
for c in c2 c2 c3 c5; do timeout 300 python tools/profile_case.py $c >> gpurun_out/q_cases.log 2>&1; done
tail -3 gpurun_out/q_pytest.log; cat gpurun_out/q_cases.log
bash tools/gpu_ftl.sh c2
