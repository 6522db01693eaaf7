"""Development probe: is the subdomain solve deterministic when two contexts run it concurrently
on one GPU (SMs oversubscribed, as in the two-rank test)? Two host threads each repeat one
Schwarz-PCG solve of a c3-share frame pair; every repetition must reproduce the first bit for
bit. Usage: cluster_race.py <FFB_CLUSTER> <FFB_SOLVE or -> [reps]"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from paper_1508_02977_b200 import flowfem as ff, synth  # noqa: E402

os.environ["FFB_CLUSTER"] = sys.argv[1]
if sys.argv[2] != "-":
    os.environ["FFB_SOLVE"] = sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
H, W, parts = 540, 1920, 32  # half of c3: 8x4 subdomains
f0, f1, _ = synth.gen_c3(0, H, W)
cfg = ff.RunConfig(sigma=1.5, parts=parts, overlap=4, adapt_iters=1, cg_tolerance=1e-10)
out = {}


def work(r):
    ctx = ff.Context(0)
    res = []
    for k in range(reps):
        rr = ff.run_on_frames(f0, f1, cfg, ctx)
        res.append((rr.flow.planes().copy(), list(rr.stats.iters)))
    out[r] = res


th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
[t.start() for t in th]
[t.join() for t in th]
ref_u, ref_it = out[0][0]
bad = 0
for r in range(2):
    for k, (u, it) in enumerate(out[r]):
        if not np.array_equal(u, ref_u) or it != ref_it:
            bad += 1
            d = np.linalg.norm(u - ref_u) / np.linalg.norm(ref_u)
            print(f"  thread {r} rep {k}: iters {it} vs {ref_it}, rel diff {d:.2e}")
print(f"cluster {sys.argv[1]} solve {sys.argv[2]}: {bad} of {2 * reps} runs differ from the first (iters {ref_it})")
