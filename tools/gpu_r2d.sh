# round 2, box 4: full GPU suite incl. multi-rank (in-process communicator) and c4 parity,
# c4 bench line, c3 full-field dump for the full-resolution comparison in the build container
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2d_pytest.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_bench_c4.json 2> gpurun_out/r2d_bench_c4.err
timeout 300 python tools/dump_chain.py c3 gpurun_out/r2d_c3_u3.npy > gpurun_out/r2d_dump.log 2>&1
tail -30 gpurun_out/r2d_pytest.log; cut -c1-600 gpurun_out/r2d_bench_c4.json; tail -3 gpurun_out/r2d_bench_c4.err; cat gpurun_out/r2d_dump.log
