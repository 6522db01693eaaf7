# round 2, box 7: persistent chain queue (correctness + c4 timing), full c4 parity
timeout 900 python -m pytest tests/test_gpu_tile_solve.py tests/test_gpu_fullsize.py tests/test_gpu_multi.py -q -m gpu -x > gpurun_out/r2g_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2g_tests.log
for b in 0 1 0; do
  if [ $b = 1 ]; then export FFB_NO_BALANCE=1; else unset FFB_NO_BALANCE; fi
  timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline >> gpurun_out/r2g_bench_c4.jsonl 2>> gpurun_out/r2g_bench_c4.err
done
tail -6 gpurun_out/r2g_tests.log
python - <<'PY'
import json
for line in open("gpurun_out/r2g_bench_c4.jsonl"):
    d=json.loads(line); s=d["solver"]
    print(round(d["value"],3), "asm ms", round(d["roofline"]["ms_per_launch"],3), "frac", round(d["roofline"]["frac"],3), "pcg", round(s["ms_pcg"]), "factor", round(s["ms_factor"]), s["pcg_iterations_per_step"], d["clocks"]["sm_mhz"])
PY
tail -3 gpurun_out/r2g_bench_c4.err
