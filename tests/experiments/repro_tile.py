import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle")); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import pyoracle
from paper_1508_02977_b200 import flowfem as ff
H, W, px, py, ov, nc = [int(x) for x in sys.argv[1:7]]
rng = np.random.default_rng(7 * H + W)
f0 = rng.uniform(0, 255, (H, W)); f1 = np.clip(np.roll(f0, 1, axis=1) * 1.02 + rng.normal(0, 3, (H, W)), 0, 255)
t = pyoracle.PORT.frames_to_terms(f0, f1, 1.0, 2.5)
ntri = 2 * (W - 1) * (H - 1)
a = np.random.default_rng(H + W).uniform(20, 1000, ntri); l = np.full(ntri, 1000.0)
ctx = ff.Context(0)
s = ff.SchwarzSolver(ctx); s.set_terms(ff.DataTerms(t)); s.set_reg(ff.RegField(a, l)); s.set_partition(px, py, ov)
u, it, res = s.solve(components=nc, tol=1e-12)
print("ok", it, res)
