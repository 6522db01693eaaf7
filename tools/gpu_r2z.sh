# round 2, box 25: bench lines of every config with the row-group tile solve (no CPU leg)
for c in c2 c3 c5 c1; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2z_bench_$c.json 2> gpurun_out/r2z_bench_$c.err
done
python - <<'PY'
import json
for c in ["c1", "c2", "c3", "c5"]:
    d = json.loads(open(f"gpurun_out/r2z_bench_{c}.json").read().strip().splitlines()[-1])
    s = d["solver"]; r = d["roofline"]; f = d.get("roofline_factor") or {}
    print(c, f"{d['value']:.3f} Mpx/s e2e {d['e2e']['value']:.3f}", f"factor {s['ms_factor']:.0f} ms pcg {s['ms_pcg']:.0f} ms iters {s['pcg_iterations_per_step']}",
          f"solve frac {r['frac']:.3f} ({r['kernel']})", f"factor frac {f.get('frac')}", d["clocks"])
PY
