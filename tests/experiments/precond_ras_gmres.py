"""CPU prototype (scipy + the oracle assembly; test infrastructure, not product code): restricted
additive Schwarz with GMRES / BiCGStab against ASM on a c3-like 540x960 pair, 4x4 parts, ov 4."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, scipy.sparse as sp, scipy.sparse.linalg as spl
import pyoracle
from paper_1508_02977_b200.synth import gen_c3
H, W, PX, PY, OV = 540, 960, 4, 4, 4
f0, f1, _ = gen_c3(0, H, W)
P = pyoracle.PORT
terms = P.frames_to_terms(f0, f1, 1.5, 2.5)
ntri = 2 * (H - 1) * (W - 1)
alpha = np.full(ntri, 1000.0); lam = np.full(ntri, 1000.0)
S = pyoracle.ref_assemble_system(terms, alpha, lam, 3)
A = sp.csr_matrix((S.vals, S.cols, S.row_ptr), shape=(S.n, S.n)); b = S.rhs
part = pyoracle.parse_partition(P.build_partition(W, H, PX, PY, OV))
idxs=[]; facs=[]; cores=[]
for p in part["parts"]:
    x0, y0, x1, y1 = p["ext"]
    fx0 = x0 + (1 if x0 > 0 else 0); fy0 = y0 + (1 if y0 > 0 else 0)
    fx1 = x1 - (1 if x1 < W else 0); fy1 = y1 - (1 if y1 < H else 0)
    ys, xs = np.mgrid[fy0:fy1, fx0:fx1]
    v = (ys * W + xs).ravel(); idx = (v[:, None] * 3 + np.arange(3)[None, :]).ravel()
    cx0, cy0, cx1, cy1 = p["core"]
    incore = ((xs >= cx0) & (xs < cx1) & (ys >= cy0) & (ys < cy1)).ravel()
    idxs.append(idx); cores.append(np.repeat(incore.astype(float), 3))
    facs.append(spl.splu(A[idx][:, idx].tocsc()))
def M_asm(r):
    z = np.zeros_like(r)
    for idx, f in zip(idxs, facs): z[idx] += f.solve(r[idx])
    return z
def M_ras(r):
    z = np.zeros_like(r)
    for idx, f, c in zip(idxs, facs, cores): z[idx] += c * f.solve(r[idx])
    return z
nb = np.linalg.norm(b)
class Cnt:
    def __init__(s): s.k=0
    def __call__(s, x): s.k+=1
for name, M in (("asm", M_asm), ("ras", M_ras)):
    c = Cnt(); t=time.time()
    x, info = spl.gmres(A, b, M=spl.LinearOperator(A.shape, M), rtol=1e-10, atol=0, restart=200, maxiter=200, callback=c, callback_type="pr_norm")
    print(name, "gmres iters", c.k, "true res", np.linalg.norm(b - A @ x) / nb, round(time.time()-t,1))
    c = Cnt(); t=time.time()
    x, info = spl.bicgstab(A, b, M=spl.LinearOperator(A.shape, M), rtol=1e-10, atol=0, maxiter=200, callback=c)
    print(name, "bicgstab iters (2 precond applies each)", c.k, "true res", np.linalg.norm(b - A @ x) / nb, round(time.time()-t,1))
