"""CPU prototype (scipy + the oracle assembly; test infrastructure, not product code): weighted
(partition-of-unity scaled, symmetric) additive Schwarz against plain ASM on a c3-like pair —
PCG iteration counts to 1e-10. Usage: python precond_weighted_asm.py H W PX PY OV"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, scipy.sparse as sp, scipy.sparse.linalg as spl
import pyoracle
from paper_1508_02977_b200.synth import gen_c3
H, W, PX, PY, OV = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
f0, f1, _ = gen_c3(0, H, W)
P = pyoracle.PORT
terms = P.frames_to_terms(f0, f1, 1.5, 2.5)
ntri = 2 * (H - 1) * (W - 1)
alpha = np.full(ntri, 1000.0); lam = np.full(ntri, 1000.0)
S = pyoracle.ref_assemble_system(terms, alpha, lam, 3)
A = sp.csr_matrix((S.vals, S.cols, S.row_ptr), shape=(S.n, S.n)); b = S.rhs
part = pyoracle.parse_partition(P.build_partition(W, H, PX, PY, OV))
subs = []
cnt = np.zeros((H, W))
for p in part["parts"]:
    x0, y0, x1, y1 = p["ext"]  # assume [x0,x1) etc
    fx0 = x0 + (1 if x0 > 0 else 0); fy0 = y0 + (1 if y0 > 0 else 0)
    fx1 = x1 - (1 if x1 < W else 0); fy1 = y1 - (1 if y1 < H else 0)
    subs.append((fx0, fy0, fx1, fy1)); cnt[fy0:fy1, fx0:fx1] += 1
print("ext0", part["parts"][0]["ext"], part["parts"][0]["core"], "free0", subs[0], "cnt max", cnt.max())
def ramp(n, lo_in, hi_in, d):
    # smooth weight along one axis: 1 in the interior, ramps over the overlap width d at interior sides
    w = np.ones(n)
    if lo_in:
        w[:d] = (np.arange(d) + 0.5) / d
    if hi_in:
        w[n - d:] = (np.arange(d)[::-1] + 0.5) / d
    return w
facs = []; idxs = []; wraw = []
for (fx0, fy0, fx1, fy1) in subs:
    ys, xs = np.mgrid[fy0:fy1, fx0:fx1]
    v = (ys * W + xs).ravel()
    idx = (v[:, None] * 3 + np.arange(3)[None, :]).ravel()
    idxs.append(idx)
    Ai = A[idx][:, idx].tocsc()
    facs.append(spl.splu(Ai))
    d = 2 * OV - 1  # width of the free overlap between neighbours
    wx = ramp(fx1 - fx0, fx0 > 0, fx1 < W, d); wy = ramp(fy1 - fy0, fy0 > 0, fy1 < H, d)
    wraw.append(np.outer(wy, wx))
# normalise smooth weights to a POU
tot = np.zeros((H, W))
for (fx0, fy0, fx1, fy1), w in zip(subs, wraw): tot[fy0:fy1, fx0:fx1] += w
modes = {}
modes["asm"] = [np.ones(len(i)) for i in idxs]
modes["count"] = [np.repeat(1.0 / np.sqrt(cnt[fy0:fy1, fx0:fx1]).ravel(), 3) for (fx0, fy0, fx1, fy1) in subs]
modes["smooth"] = [np.repeat(np.sqrt(w / tot[fy0:fy1, fx0:fx1]).ravel(), 3) for (fx0, fy0, fx1, fy1), w in zip(subs, wraw)]
def pcg(mode, tol=1e-10, x0=None):
    D = modes[mode]
    def M(r):
        z = np.zeros_like(r)
        for idx, f, d in zip(idxs, facs, D): z[idx] += d * f.solve(d * r[idx])
        return z
    x = np.zeros_like(b) if x0 is None else x0.copy(); r = b - A @ x; nb = np.linalg.norm(b)
    z = M(r); p = z.copy(); rz = r @ z; k = 0; hist = []
    while True:
        q = A @ p; a = rz / (p @ q); x += a * p; r -= a * q; k += 1
        res = np.linalg.norm(r) / nb; hist.append(res)
        if res <= tol or k > 500: break
        z = M(r); rz2 = r @ z; p = z + (rz2 / rz) * p; rz = rz2
    return x, k, hist
for m in ["asm", "count", "smooth"]:
    t = time.time(); x, k, h = pcg(m); print(m, "iters", k, "t", round(time.time() - t, 1), "res@10,20,30", [f"{h[min(i,len(h)-1)]:.1e}" for i in (9, 19, 29)])
