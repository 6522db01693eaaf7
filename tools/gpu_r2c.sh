# round 2, box 3: two-level (coarse space) vs one-level Schwarz-PCG, iteration counts and times
for c in c4 c3 c2 c5; do
  for k in 1 0; do
    FFB_COARSE=$k timeout 600 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_${c}_coarse$k.json 2> gpurun_out/r2c_${c}_coarse$k.err
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -q -m gpu -k "not c4_chain" > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2c_pytest.log
python - <<'PY'
import json
for c in ["c4","c3","c2","c5"]:
    for k in (1,0):
        try:
            d=json.load(open(f"gpurun_out/r2c_{c}_coarse{k}.json"))
            s=d["solver"]; print(c, "coarse", k, round(d["value"],3), "Mpx/s", s["pcg_iterations_per_step"], s["iters"], "pcg ms", round(s["ms_pcg"]), "factor ms", round(s["ms_factor"]))
        except Exception as e: print(c,k,"ERR",e)
PY
tail -5 gpurun_out/r2c_pytest.log; tail -3 gpurun_out/r2c_c4_coarse1.err
