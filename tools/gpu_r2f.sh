# round 2, box 6: multi-rank fixes, new CSR/Cholesky tests, balanced chain schedule (parity + c4 timing)
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_linsolve.py tests/test_gpu_tile_solve.py tests/test_gpu_fullsize.py -q -m gpu -x > gpurun_out/r2f_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2f_tests.log
for b in 0 1; do
  if [ $b = 1 ]; then export FFB_NO_BALANCE=1; fi
  timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench_c4_nobal$b.json 2> gpurun_out/r2f_bench_c4_nobal$b.err
done
unset FFB_NO_BALANCE
tail -15 gpurun_out/r2f_tests.log
python - <<'PY'
import json
for b in (0,1):
    try:
        d=json.load(open(f"gpurun_out/r2f_bench_c4_nobal{b}.json")); s=d["solver"]
        print("no_balance", b, round(d["value"],3), "asm ms", round(d["roofline"]["ms_per_launch"],3), "frac", round(d["roofline"]["frac"],3), "pcg", round(s["ms_pcg"]), "factor", round(s["ms_factor"]), s["iters"], d["clocks"]["sm_mhz"])
    except Exception as e: print(b, "ERR", e)
PY
tail -3 gpurun_out/r2f_bench_c4_nobal0.err
