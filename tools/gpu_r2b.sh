# round 2, box 2: new GPU tests (CG literal mode, stats, energy, full-size c3/c5), FP64 peak,
# c4 bench line with the factor roofline
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/microbench/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/r2b_fp64_peak.json
timeout 1500 python -m pytest tests -q -m gpu -k "not c4_chain" > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2b_pytest.log
timeout 600 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_c4.json 2> gpurun_out/r2b_bench_c4.err
cat gpurun_out/r2b_fp64_peak.json; tail -30 gpurun_out/r2b_pytest.log; cat gpurun_out/r2b_bench_c4.json; tail -3 gpurun_out/r2b_bench_c4.err
