"""Development probe (uses the oracle's imaging for the inputs, so it lives under tests/): repeats
the row-batch ring solve (FFB_SOLVE=ring) and the row-group tile solve on the tile-solve test's
cases with a bounded iteration count, and reports any run whose iteration count or residual
differs from the first — an intermittent stall of that test showed up twice in ~20 suite runs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import pyoracle  # noqa: E402
from paper_1508_02977_b200 import flowfem as ff  # noqa: E402

CASES = [(40, 32, 1, 1, 0, 3, "2"), (12, 9, 1, 1, 0, 3, "4"), (50, 44, 3, 2, 4, 2, "4"),
         (130, 160, 2, 2, 3, 3, "2"), (149, 160, 1, 1, 0, 3, "2"), (149, 160, 1, 1, 0, 3, "4"),
         (149, 160, 1, 1, 0, 3, "1"), (130, 160, 2, 2, 3, 3, "1"), (149, 160, 1, 1, 0, 3, "8")]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
port = pyoracle.PORT


def rand_pair(H, W, seed):
    rng = np.random.default_rng(seed)
    f0 = rng.uniform(0, 255, (H, W))
    f1 = np.clip(np.roll(f0, 1, axis=1) * 1.02 + rng.normal(0, 3, (H, W)), 0, 255)
    return f0, f1


for H, W, px, py, ov, nc, cl in CASES:
    f0, f1 = rand_pair(H, W, 5 * H + W)
    t = port.frames_to_terms(f0, f1, 1.0, 2.5)
    rng = np.random.default_rng(H * W)
    ntri = 2 * (W - 1) * (H - 1)
    a = rng.uniform(20, 1000, ntri)
    l = np.full(ntri, 1000.0)
    os.environ["FFB_CLUSTER"] = cl
    for mode in ("ring", "rt"):
        os.environ["FFB_SOLVE"] = mode
        first = None
        bad = 0
        for rep in range(reps):
            ctx = ff.Context(0)
            try:
                s = ff.SchwarzSolver(ctx)
                s.set_terms(ff.DataTerms(t)); s.set_reg(ff.RegField(a, l)); s.set_partition(px, py, ov)
                try:
                    u, it, res = s.solve(components=nc, tol=1e-12, max_iters=400)
                    sig = (it, float(res), bool(np.isfinite(u.planes()).all()))
                except Exception as e:  # noqa: BLE001
                    sig = ("error", str(e)[:80])
            finally:
                ctx.close()
            if first is None:
                first = sig
            elif sig != first:
                bad += 1
                print(f"  MISMATCH {H}x{W} {px}x{py} ov{ov} nc{nc} C={cl} {mode} rep {rep}: {sig} vs {first}", flush=True)
        print(f"{H}x{W} {px}x{py} ov{ov} nc{nc} C={cl} {mode}: first {first}, {bad} deviating of {reps}", flush=True)
