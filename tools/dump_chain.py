"""Builder probe: one full run_on_frames of a configuration on cuda:0; saves u3 (and
optionally alpha) to an .npy for a full-resolution comparison with the reference golden
(tests/golden/make_golden_large.py keeps the full reference outputs in the build container).

    python tools/dump_chain.py c5 gpurun_out/c5_u3.npy [--alpha gpurun_out/c5_alpha.npy] [--overlap K]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1508_02977_b200 import flowfem as ff, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("out")
ap.add_argument("--alpha")
ap.add_argument("--overlap", type=int)
a = ap.parse_args()
f0, f1, _, cfg = synth.make(a.config)
rc = ff.RunConfig(sigma=cfg.sigma, rho=cfg.rho, parts=cfg.parts,
                  overlap=a.overlap if a.overlap is not None else cfg.overlap,
                  adapt_iters=cfg.n_passes, cg_tolerance=cfg.tol)
r = ff.run_on_frames(f0, f1, rc, ff.Context(0))
np.save(a.out, r.flow.planes())
if a.alpha:
    np.save(a.alpha, r.reg.alpha)
print(a.config, "iters", list(r.stats.iters), "ms", r.stats.ms_total, flush=True)
