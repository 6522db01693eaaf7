"""CPU-2 of BASELINE.md §3: the reference's own Schwarz path (schwarz_solve, adapt off, solver
per pick_method, workers = host cores) — seconds per Schwarz iteration, and for the small
configs the iterations it needs to reach the converged solution within 1e-8 relative L2
(checked against the reference's monolithic CG at tol 1e-12). Builder probe; writes
profiles/r2_cpu2_reference_schwarz.json.

    python tools/ref_schwarz_cost.py [c1 c2 c5 c3 c4]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as po  # noqa: E402
from paper_1508_02977_b200 import synth, flowfem as ff  # noqa: E402

OUT = os.path.join(ROOT, "profiles", "r2_cpu2_reference_schwarz.json")


def pick(cfg, px, py, nc=3):
    """pick_method (pipeline.cpp:16-28): Cholesky up to 20000 unknowns per extended rectangle"""
    P = ff.build_partition(cfg.W, cfg.H, px, py, cfg.overlap)
    most = max(p.ext.w() * p.ext.h() * nc for p in P.parts)
    return (1, "cholesky") if most <= 20000 else (0, "cg")


def run(name, threads):
    R = po.REF
    R.set_threads(threads)
    f0, f1, _, cfg = synth.make(name)
    t10 = R.frames_to_terms(f0, f1, cfg.sigma, cfg.rho)
    sp = ff.choose_split(cfg.W, cfg.H, cfg.parts)
    method, mname = pick(cfg, sp.parts_x, sp.parts_y)
    nt = 2 * (cfg.W - 1) * (cfg.H - 1)
    a, l = np.full(nt, cfg.alpha0), np.full(nt, cfg.lambda0)
    out = dict(config=cfg.name, solver=mname, threads=threads, workers=threads)
    n_it = 2
    t = time.time()
    po.ref_schwarz_solve(t10, a, l, sp.parts_x, sp.parts_y, cfg.overlap, n_it, workers=threads,
                         method=method, cg_tol=cfg.tol)
    out["s_per_iter_first2"] = (time.time() - t) / n_it
    if name in ("c1", "c2"):
        mono, _, _ = R.cg_solve(t10, a, l, 3, 1e-12)
        errs = []
        for k in (10, 20, 40, 80, 160, 320):
            t = time.time()
            r = po.ref_schwarz_solve(t10, a, l, sp.parts_x, sp.parts_y, cfg.overlap, k,
                                     workers=threads, method=method, cg_tol=cfg.tol)
            dt = time.time() - t
            e = max(np.linalg.norm(r["u3"][c] - mono[c]) / np.linalg.norm(mono[c])
                    for c in range(3))
            errs.append(dict(iters=k, rel_l2=e, seconds=dt))
            print(name, k, e, dt, flush=True)
            if e < 1e-8:
                break
        out["convergence"] = errs
    print(name, out, flush=True)
    return out


if __name__ == "__main__":
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    thr = int(os.environ.get("FFB_THREADS", os.cpu_count() or 1))
    for n in sys.argv[1:] or ["c1", "c2", "c5", "c3", "c4"]:
        res[n] = run(n, thr)
        res["_cpu"] = next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo")
                            if l.startswith("model name")), "unknown")
        json.dump(res, open(OUT, "w"), indent=1)
