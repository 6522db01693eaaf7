# round 2, first box: GPU tests, bench lines on c4/c3/c5 (no CPU leg), c5 full-field dump
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv
nproc; grep -m1 "model name" /proc/cpuinfo
timeout 1100 python -m pytest tests -x -q -m gpu > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2a_pytest.log
for c in c4 c3 c5; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_$c.json 2> gpurun_out/r2a_bench_$c.err
done
timeout 300 python tools/dump_chain.py c5 gpurun_out/r2a_c5_u3.npy > gpurun_out/r2a_dump.log 2>&1
tail -3 gpurun_out/r2a_pytest.log; for c in c4 c3 c5; do cut -c1-400 gpurun_out/r2a_bench_$c.json; tail -2 gpurun_out/r2a_bench_$c.err; done; cat gpurun_out/r2a_dump.log
