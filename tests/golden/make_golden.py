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
  linsolve.npz       the linsolve boundary: SparseSystems from the
                     reference's assemble() (random frames/alpha, optional Dirichlet row,
                     as test_linsolve.cpp:16-33 builds them), the reference's rcm_order,
                     cg_solve (x, iterations, residual) and direct solve() on each, and
                     the outcome on an indefinite system
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


LINSOLVE_CASES = [  # (W, H, components, seed, dirichlet)
    (7, 6, 2, 1, False), (7, 6, 3, 5, True), (10, 9, 3, 3, False), (24, 18, 3, 11, True),
    (40, 30, 2, 4, False), (33, 21, 3, 8, False)]


def linsolve_system(R, W, H, nc, seed, dirichlet):
    rng = np.random.default_rng(seed)
    f0 = rng.uniform(0, 255, (H, W))
    f1 = np.clip(np.roll(f0, 1, axis=1) + rng.normal(0, 6, (H, W)), 0, 255)
    terms = R.frames_to_terms(f0, f1, 1.0, 2.5)
    nt = 2 * (W - 1) * (H - 1)
    alpha = rng.uniform(5.0, 150.0, nt)
    lam = np.full(nt, 35.0)
    dv = dval = None
    if dirichlet:
        dv = np.arange(W)  # bottom row, test_linsolve.cpp:25-30
        dval = rng.uniform(-1.0, 1.0, (W, nc))
    return po.ref_assemble_system(terms, alpha, lam, nc, dv, dval)


def linsolve(R):
    out = {}
    for k, (W, H, nc, seed, dirichlet) in enumerate(LINSOLVE_CASES):
        s = linsolve_system(R, W, H, nc, seed, dirichlet)
        xc, it, res = po.csr_cg_solve(R, s, 1e-12)
        xd, _, resd = po.ref_csr_solve(s, 1)
        out.update({f"{k}_row_ptr": s.row_ptr, f"{k}_cols": s.cols, f"{k}_vals": s.vals,
                    f"{k}_rhs": s.rhs, f"{k}_nc": nc, f"{k}_perm": po.rcm_order(R, s),
                    f"{k}_cg_x": xc, f"{k}_cg_iters": it, f"{k}_cg_res": res,
                    f"{k}_direct_x": xd, f"{k}_direct_res": resd})
        print("linsolve case", k, "n", s.n, "cg iters", it)
    # an indefinite system: one neighbour coupling made larger than the geometric mean of
    # its diagonals (both triangles)
    s = linsolve_system(R, 9, 8, 3, 21, False)
    vals = s.vals.copy()
    r = 40
    q = next(q for q in range(s.row_ptr[r], s.row_ptr[r + 1]) if s.cols[q] == r + 3)
    c = s.cols[q]
    dr = vals[next(q2 for q2 in range(s.row_ptr[r], s.row_ptr[r + 1]) if s.cols[q2] == r)]
    dc = vals[next(q2 for q2 in range(s.row_ptr[c], s.row_ptr[c + 1]) if s.cols[q2] == c)]
    v = 3.0 * np.sqrt(dr * dc)
    vals[q] = v
    vals[next(q2 for q2 in range(s.row_ptr[c], s.row_ptr[c + 1]) if s.cols[q2] == r)] = v
    bad = po.CsrSystem(s.row_ptr, s.cols, vals, s.rhs, 3)
    msgs = []
    for method in (1, 0):
        try:
            po.ref_csr_solve(bad, method, 1e-12)
            msgs.append("")
        except po.OracleError as e:
            msgs.append(str(e))
    out.update({"bad_row_ptr": bad.row_ptr, "bad_cols": bad.cols, "bad_vals": bad.vals,
                "bad_rhs": bad.rhs, "bad_msg_cholesky": msgs[0], "bad_msg_cg": msgs[1]})
    print("indefinite:", msgs)
    np.savez_compressed(os.path.join(OUT, "linsolve.npz"), **out)


if __name__ == "__main__":
    R = po.REF
    if R is None:
        raise SystemExit("build the reference oracle first: make -C oracle")
    R.set_threads(os.cpu_count())
    if len(sys.argv) > 1 and sys.argv[1] == "linsolve":
        linsolve(R)
        raise SystemExit(0)
    small_stages(R)
    partitions(R)
    c1_chain(R)
    linsolve(R)
