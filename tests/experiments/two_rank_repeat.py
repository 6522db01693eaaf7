"""Development probe: repeat the two-rank c3 run of tests/test_gpu_multi.py (fresh contexts every
time, per-rank cluster sizing) and compare every repetition with the first bit for bit.
Usage: two_rank_repeat.py [reps] [FFB_SOLVE]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from paper_1508_02977_b200 import flowfem as ff, parallel as par, synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
if len(sys.argv) > 2:
    os.environ["FFB_SOLVE"] = sys.argv[2]
f0, f1, _, c = synth.make("c3")
cfg = ff.RunConfig(sigma=c.sigma, parts=c.parts, overlap=c.overlap, adapt_iters=1, cg_tolerance=c.tol)
ref1 = ff.run_on_frames(f0, f1, cfg, ff.Context(0))
first = None
bad = 0
for k in range(reps):
    res = par.run_local(f0, f1, cfg, 2)
    u = res[0].flow.planes()
    assert np.array_equal(u, res[1].flow.planes())
    d1 = max(np.linalg.norm(u[i] - ref1.flow.planes()[i]) / np.linalg.norm(ref1.flow.planes()[i]) for i in range(3))
    if first is None:
        first = (u.copy(), list(res[0].stats.iters))
    same = np.array_equal(u, first[0]) and list(res[0].stats.iters) == first[1]
    bad += 0 if same else 1
    print(f"rep {k}: iters {list(res[0].stats.iters)} (world 1: {list(ref1.stats.iters)}), rel diff to world 1 {d1:.2e}, "
          f"{'same as rep 0' if same else 'DIFFERS from rep 0'}", flush=True)
print(f"{bad} of {reps} repetitions differ from the first")
