timeout 120 python tools/profile_case.py c2 > gpurun_out/f1_case.log 2>&1
timeout 300 python -m pytest tests -x -q -m gpu > gpurun_out/f1_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/f1_pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/f1_bench_c2.json 2> gpurun_out/f1_bench_c2.err
cat gpurun_out/f1_case.log; tail -2 gpurun_out/f1_pytest.log; cat gpurun_out/f1_bench_c2.json
