set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/s3_pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/s3_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s3_bench_c2.json 2> gpurun_out/s3_bench_c2.err
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s3_bench_c3.json 2> gpurun_out/s3_bench_c3.err
tail -3 gpurun_out/s3_pytest_gpu.log; cat gpurun_out/s3_smoke.log gpurun_out/s3_bench_c2.json gpurun_out/s3_bench_c3.json
