"""Golden fixtures for the full-size configurations c3, c4, c5 from the UNMODIFIED reference
(oracle/_ref, compiled from /root/reference/proj/src by oracle/Makefile). Run in the build
container (hours of CPU: monolithic Jacobi-CG at tol 1e-12 on up to 24.9M unknowns):

    make -C oracle && python tests/golden/make_golden_large.py [c5 c3 c4]

Protocol: the converged-pass chain (proj/src/pipeline.cpp:38-78 with
the reference's own `solve` / `cg_solve` per pass, proj/src/linsolve.cpp:298-361,
`error_indicator` / `update_alpha`, proj/src/adapt.cpp:9-112), n_passes alpha updates then a
final solve, tol 1e-12 (chain error ~1e-11, SURVEY probe7), on the synthetic inputs of
paper_1508_02977_b200/synth.py (seed 0).

The full fields (c3: 50 MB, c4: 200 MB of u3) are too large for the repository, so the
committed fixture `<cfg>_chain_sample.npz` holds:
  u3s       u1, u2, mt on the pixel grid subsampled with stride S (both axes)
  alphas    the final alpha of the cells of that grid ((H-1, W-1, 2) view, same stride)
  norms     full-field L2 norms of u1, u2, mt and alpha
  sha_u3    SHA-256 of the full u3 (float64 little-endian, planes), sha_alpha likewise
  eta_max, iters, seconds, f0_sha, f1_sha, stride
  energy_ref  energy (assembly.cpp:201-238) of the final state at the final alpha
The full outputs are kept beside the sample in $FFB_GOLDEN_FULL (default
/tmp/ffb_golden_full) for builder-side full-resolution comparisons.
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
import pyoracle as po  # noqa: E402
from paper_1508_02977_b200 import synth  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
FULL = os.environ.get("FFB_GOLDEN_FULL", "/tmp/ffb_golden_full")
STRIDE = {"c3": 7, "c4": 14, "c5": 5}


def sample_fields(u3, alpha, H, W, s):
    a = alpha.reshape(H - 1, W - 1, 2)
    return np.ascontiguousarray(u3[:, ::s, ::s]), np.ascontiguousarray(a[::s, ::s, :])


def run(name):
    R = po.REF
    if R is None:
        raise SystemExit("oracle/_ref not built (make -C oracle with /root/reference present)")
    R.set_threads(int(os.environ.get("FFB_GOLDEN_THREADS", os.cpu_count() or 1)))
    f0, f1, _, cfg = synth.make(name)
    t = time.time()
    r = R.converged_chain(f0, f1, cfg.sigma, rho=cfg.rho, alpha0=cfg.alpha0,
                          lambda0=cfg.lambda0, nc=3, n_passes=cfg.n_passes, kappa=cfg.kappa,
                          thr=cfg.eta_threshold, tol=1e-12)
    s = STRIDE[name]
    u3s, als = sample_fields(r["u3"], r["alpha"], cfg.H, cfg.W, s)
    norms = np.array([np.linalg.norm(r["u3"][c]) for c in range(3)] + [np.linalg.norm(r["alpha"])])
    meta = dict(eta_max=r["eta_max"], iters=r["iters"], seconds=r["seconds"], stride=s,
                norms=norms,
                sha_u3=hashlib.sha256(r["u3"].astype("<f8").tobytes()).hexdigest(),
                sha_alpha=hashlib.sha256(r["alpha"].astype("<f8").tobytes()).hexdigest(),
                f0_sha=hashlib.sha256(f0.tobytes()).hexdigest(),
                f1_sha=hashlib.sha256(f1.tobytes()).hexdigest())
    np.savez_compressed(os.path.join(OUT, f"{name}_chain_sample.npz"), u3s=u3s, alphas=als, **meta)
    os.makedirs(FULL, exist_ok=True)
    np.savez(os.path.join(FULL, f"{name}_chain_full.npz"), u3=r["u3"], alpha=r["alpha"], **meta)
    print(f"{name}: iters {list(r['iters'])} chain {r['seconds']:.0f} s (wall {time.time() - t:.0f} s)",
          flush=True)
    add_energy(name)


def add_energy(name):
    """energy (assembly.cpp:201-238) of the reference's final state at its final alpha, computed
    by the reference itself from the full outputs kept in $FFB_GOLDEN_FULL, added to the sample
    fixture as `energy_ref` (a size-independent scalar for the GPU parity tests)."""
    R = po.REF
    f0, f1, _, cfg = synth.make(name)
    full = np.load(os.path.join(FULL, f"{name}_chain_full.npz"))
    terms = R.frames_to_terms(f0, f1, cfg.sigma, cfg.rho)
    ntri = 2 * (cfg.W - 1) * (cfg.H - 1)
    e = R.energy(terms, full["alpha"], np.full(ntri, cfg.lambda0), full["u3"], 3)
    path = os.path.join(OUT, f"{name}_chain_sample.npz")
    d = dict(np.load(path))
    d["energy_ref"] = np.float64(e)
    np.savez_compressed(path, **d)
    print(name, "energy_ref", e, flush=True)


def chain_iters(names):
    """tests/golden/ref_chain_iters.json: the reference's converged-pass chain at each config's
    own tolerance (cfg.tol, 1e-10), per-solve CG iteration counts and wall time. bench.py
    extrapolates its bounded CPU-baseline sample (ref_chain_sample) with these counts."""
    import json
    R = po.REF
    threads = R.set_threads(int(os.environ.get("FFB_GOLDEN_THREADS", os.cpu_count() or 1)))
    path = os.path.join(OUT, "ref_chain_iters.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    cpu = next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo")
                if l.startswith("model name")), "unknown")
    for name in names:
        f0, f1, _, cfg = synth.make(name)
        r = R.converged_chain(f0, f1, cfg.sigma, rho=cfg.rho, alpha0=cfg.alpha0,
                              lambda0=cfg.lambda0, nc=3, n_passes=cfg.n_passes, kappa=cfg.kappa,
                              thr=cfg.eta_threshold, tol=cfg.tol)
        out[cfg.name] = dict(iters=[int(i) for i in r["iters"]], seconds=r["seconds"], tol=cfg.tol,
                             threads=threads, cpu=cpu)
        print(name, out[cfg.name], flush=True)
        json.dump(out, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--energy":
        for n in args[1:]:
            add_energy(n)
    elif args and args[0] == "--iters":
        chain_iters(args[1:] or ["c1", "c2", "c5", "c3", "c4"])
    else:
        for n in (args or ["c5", "c3", "c4"]):
            run(n)
