"""Generates the committed golden fixtures from the UNMODIFIED reference (oracle/_ref,
compiled from /root/reference/proj/src by oracle/Makefile). Run in the build container:

    make -C oracle && python tests/golden/make_golden.py

Fixtures (the reference ships no golden files):
  stages_small.npz   per-stage outputs on a seeded 23x31 pair (smoothing, derivatives,
                     data terms, y = A x and b, eta/eta_max, alpha update)
  c1_chain.npz       config c1 converged-pass chain (3 alpha passes + final solve,
                     reference monolithic CG at tol 1e-12): u3, alpha,
                     eta_max, iterations
  partitions.json    SHA-256 of the reference's flat Partition for every configured split
                     plus the split choices
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
import pyoracle as po  # noqa: E402
from paper_1508_02977_b200 import synth  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def small_stages(R):
    rng = np.random.default_rng(1234)
    H, W = 23, 31
    f0 = rng.uniform(0, 255, (H, W))
    f1 = np.clip(f0 + rng.normal(0, 8, (H, W)), 0, 255)
    s0 = R.gaussian_smooth(f0, 1.0)
    s1 = R.gaussian_smooth(f1, 1.0)
    fx, fy, ft, f = R.compute_derivatives(s0, s1)
    terms = R.build_data_terms(fx, fy, ft, f, 2.5)
    ntri = 2 * (W - 1) * (H - 1)
    alpha = rng.uniform(10, 1000, ntri)
    lam = np.full(ntri, 1000.0)
    x3 = rng.normal(size=(3, H, W))
    y3, b3 = R.assemble_apply(terms, alpha, lam, 3, x3)
    y2, b2 = R.assemble_apply(terms, alpha, lam, 2, x3)
    eta, em = R.error_indicator(terms, alpha, lam, x3, 3)
    eta2, em2 = R.error_indicator(terms, alpha, lam, x3, 2)
    a_new = R.update_alpha(alpha, lam, eta, em, 10.0, 0.1, 10.0)
    np.savez_compressed(os.path.join(OUT, "stages_small.npz"), f0=f0, f1=f1, s0=s0, s1=s1, fx=fx,
                        fy=fy, ft=ft, f=f, terms=terms, alpha=alpha, lam=lam, x3=x3, y3=y3, b3=b3,
                        y2=y2, b2=b2, eta=eta, eta_max=em, eta2=eta2, eta_max2=em2, alpha_new=a_new)


def c1_chain(R):
    f0, f1, _, cfg = synth.make("c1")
    r = R.converged_chain(f0, f1, cfg.sigma, rho=cfg.rho, alpha0=cfg.alpha0,
                          lambda0=cfg.lambda0, nc=3, n_passes=cfg.n_passes, kappa=cfg.kappa,
                          thr=cfg.eta_threshold, tol=1e-12)
    np.savez_compressed(os.path.join(OUT, "c1_chain.npz"), u3=r["u3"], alpha=r["alpha"],
                        eta_max=r["eta_max"], iters=r["iters"],
                        f0_sha=hashlib.sha256(f0.tobytes()).hexdigest(),
                        f1_sha=hashlib.sha256(f1.tobytes()).hexdigest())
    print("c1 chain iters", r["iters"], "seconds", r["seconds"])


def partitions(R):
    out = {"splits": {}, "partitions": {}}
    for name, cfg in synth.CONFIGS.items():
        px, py, ratio = R.choose_split(cfg.W, cfg.H, cfg.parts)
        out["splits"][name] = [px, py, ratio]
        for ov in (cfg.overlaps or (cfg.overlap,)):
            flat = R.build_partition(cfg.W, cfg.H, px, py, ov)
            out["partitions"][f"{name}_ov{ov}"] = dict(
                W=cfg.W, H=cfg.H, px=px, py=py, ov=ov, length=int(flat.size),
                sha256=hashlib.sha256(flat.astype("<i4").tobytes()).hexdigest())
    with open(os.path.join(OUT, "partitions.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    R = po.REF
    if R is None:
        raise SystemExit("build the reference oracle first: make -C oracle")
    R.set_threads(os.cpu_count())
    small_stages(R)
    partitions(R)
    c1_chain(R)
