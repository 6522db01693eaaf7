"""One full adaptive solve of a configuration through the C-ABI (for ncu / timing probes).

    python tools/profile_case.py c2 [n_passes]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1508_02977_b200 import flowfem as ff  # noqa: E402
from paper_1508_02977_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
f0, f1, _, cfg = synth.make(name)
n_passes = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_passes
rc = ff.RunConfig(sigma=cfg.sigma, rho=cfg.rho, parts=cfg.parts, overlap=cfg.overlap,
                  adapt_iters=n_passes, cg_tolerance=cfg.tol)
ctx = ff.Context(0)
t = time.perf_counter()
r = ff.run_on_frames(f0, f1, rc, ctx)
dt = time.perf_counter() - t
s = r.stats
print(f"{name}: {dt*1e3:.1f} ms wall, total {s.ms_total:.1f} ms: terms {s.ms_terms:.2f} "
      f"factor {s.ms_factor:.1f} pcg {s.ms_pcg:.1f} adapt {s.ms_adapt:.2f}; iters {s.iters}; "
      f"asm {s.ms_asm_per_iter:.3f} ms/launch = "
      f"{8*s.factor_doubles/(s.ms_asm_per_iter*1e-3)/1e9 if s.ms_asm_per_iter else 0:.0f} GB/s")
