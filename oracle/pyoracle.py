"""TEST INFRASTRUCTURE (oracle) — not product code.

ctypes wrappers for the two CPU checkers built by ``oracle/Makefile``:

* ``PORT`` — ``_port/libflowfem_port.so``, our plain-C restatement of the
  reference hot path (``oracle/flowfem_port.c``);
* ``REF``  — ``_ref/libflowfem_ref.so``, the unmodified reference
  (``/root/reference/proj/src``) compiled out of tree, driven through
  ``oracle/ref_capi.cpp``. ``None`` when it was not built.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module, and only as the checker.

Both libraries expose the same call shapes; ``Oracle`` hides the prefix.
Arrays are numpy float64 / int32, C-contiguous, in the conventions of
``include/flowfem_b200.h``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_vp = C.c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    pass


class Oracle:
    """One of the two CPU checkers (prefix ``fp_`` for the port, ``ref_`` for the reference)."""

    def __init__(self, path: str, prefix: str, kind: str):
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.kind = kind  # "port" | "reference"
        self.path = path
        L = self.lib
        for name, res in (("last_error", C.c_char_p), ("set_threads", C.c_int)):
            f = getattr(L, prefix + name)
            f.restype = res
        getattr(L, prefix + "build_partition").restype = C.c_long

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    def _call(self, name, *args):
        rc = self._f(name)(*args)
        if rc != 0:
            raise OracleError(self._f("last_error")().decode())

    def set_threads(self, n: int) -> int:
        return self._f("set_threads")(int(n))

    # ---- imaging -----------------------------------------------------------
    def gaussian_smooth(self, img, sigma):
        img = _f64(img)
        H, W = img.shape
        out = np.empty_like(img)
        self._call("gaussian_smooth", W, H, _ptr(img), C.c_double(sigma), _ptr(out))
        return out

    def compute_derivatives(self, f0, f1):
        f0, f1 = _f64(f0), _f64(f1)
        H, W = f0.shape
        outs = [np.empty_like(f0) for _ in range(4)]
        self._call("compute_derivatives", W, H, _ptr(f0), _ptr(f1), *[_ptr(o) for o in outs])
        return outs  # fx, fy, ft, f

    def build_data_terms(self, fx, fy, ft, f, rho):
        fx, fy, ft, f = map(_f64, (fx, fy, ft, f))
        H, W = fx.shape
        out = np.empty((10, H, W))
        self._call("build_data_terms", W, H, _ptr(fx), _ptr(fy), _ptr(ft), _ptr(f),
                   C.c_double(rho), _ptr(out))
        return out

    def frames_to_terms(self, f0, f1, sigma, rho):
        f0, f1 = _f64(f0), _f64(f1)
        H, W = f0.shape
        out = np.empty((10, H, W))
        self._call("frames_to_terms", W, H, _ptr(f0), _ptr(f1), C.c_double(sigma),
                   C.c_double(rho), _ptr(out))
        return out

    # ---- partition ---------------------------------------------------------
    def choose_split(self, W, H, n_parts):
        px, py, ratio = C.c_int(), C.c_int(), C.c_double()
        self._call("choose_split", W, H, n_parts, C.byref(px), C.byref(py), C.byref(ratio))
        return px.value, py.value, ratio.value

    def build_partition(self, W, H, px, py, ov) -> np.ndarray:
        f = self._f("build_partition")
        need = f(W, H, px, py, ov, None, C.c_long(0))
        if need < 0:
            raise OracleError(self._f("last_error")().decode())
        buf = np.zeros(need, dtype=np.int32)
        got = f(W, H, px, py, ov, _ptr(buf), C.c_long(need))
        assert got == need
        return buf

    # ---- operator / solver -------------------------------------------------
    def assemble_apply(self, terms, alpha, lam, nc, x3):
        terms, alpha, lam, x3 = map(_f64, (terms, alpha, lam, x3))
        _, H, W = terms.shape
        y3 = np.zeros((3, H, W))
        b3 = np.zeros((3, H, W))
        self._call("assemble_apply", W, H, _ptr(terms), _ptr(alpha), _ptr(lam), nc, _ptr(x3),
                   _ptr(y3), _ptr(b3))
        return y3, b3

    def cg_solve(self, terms, alpha, lam, nc, tol, warm3=None, max_iters=0):
        terms, alpha, lam = map(_f64, (terms, alpha, lam))
        _, H, W = terms.shape
        out = np.zeros((3, H, W))
        it, res = C.c_int(), C.c_double()
        if self.prefix == "fp_":
            self._call("cg_solve", W, H, _ptr(terms), _ptr(alpha), _ptr(lam), nc,
                       C.c_double(tol), max_iters, _ptr(None if warm3 is None else _f64(warm3)),
                       _ptr(out), C.byref(it), C.byref(res))
        else:
            self._call("solve_monolithic", W, H, _ptr(terms), _ptr(alpha), _ptr(lam), nc, 0,
                       C.c_double(tol), _ptr(None if warm3 is None else _f64(warm3)),
                       _ptr(out), C.byref(it), C.byref(res))
        return out, it.value, res.value

    def error_indicator(self, terms, alpha, lam, u3, nc=3):
        terms, alpha, lam, u3 = map(_f64, (terms, alpha, lam, u3))
        _, H, W = terms.shape
        eta = np.zeros(2 * (W - 1) * (H - 1))
        em = C.c_double()
        self._call("error_indicator", W, H, _ptr(terms), _ptr(alpha), _ptr(lam), _ptr(u3), nc,
                   _ptr(eta), C.byref(em))
        return eta, em.value

    def update_alpha(self, alpha, lam, eta, eta_max, kappa, thr, alpha_th):
        alpha, lam, eta = map(_f64, (alpha, lam, eta))
        out = np.zeros_like(alpha)
        if self.prefix == "fp_":
            self._call("update_alpha", alpha.size, _ptr(alpha), _ptr(eta), C.c_double(eta_max),
                       C.c_double(kappa), C.c_double(thr), C.c_double(alpha_th), _ptr(out))
        else:
            self._call("update_alpha", alpha.size, _ptr(alpha), _ptr(lam), _ptr(eta),
                       C.c_double(eta_max), C.c_double(kappa), C.c_double(thr),
                       C.c_double(alpha_th), _ptr(out))
        return out

    def energy(self, terms, alpha, lam, u3, nc=3):
        """energy (assembly.cpp:201-238)."""
        terms, alpha, lam, u3 = map(_f64, (terms, alpha, lam, u3))
        H, W = terms.shape[1:]
        e = C.c_double()
        self._call("energy", W, H, _ptr(terms), _ptr(alpha), _ptr(lam), _ptr(u3), nc, C.byref(e))
        return e.value

    def converged_chain(self, f0, f1, sigma, rho=2.5, alpha0=1000.0, lambda0=1000.0, nc=3,
                        n_passes=3, kappa=10.0, thr=0.1, alpha_th=None, tol=1e-10):
        """D2 converged-pass protocol; returns dict(u3, alpha, eta_max, iters, seconds)."""
        f0, f1 = _f64(f0), _f64(f1)
        H, W = f0.shape
        if alpha_th is None:
            alpha_th = alpha0 / 100.0
        out = np.zeros((3, H, W))
        alpha = np.zeros(2 * (W - 1) * (H - 1))
        em = np.zeros(max(n_passes, 1))
        iters = np.zeros(n_passes + 1, dtype=np.int32)
        sec = C.c_double()
        args = [W, H, _ptr(f0), _ptr(f1), C.c_double(sigma), C.c_double(rho),
                C.c_double(alpha0), C.c_double(lambda0), nc, n_passes, C.c_double(kappa),
                C.c_double(thr), C.c_double(alpha_th), C.c_double(tol)]
        if self.prefix == "ref_":
            args.append(0)  # method: CG
        args += [_ptr(out), _ptr(alpha), _ptr(em), _ptr(iters), C.byref(sec)]
        self._call("converged_chain", *args)
        return dict(u3=out, alpha=alpha, eta_max=em[:n_passes], iters=iters, seconds=sec.value)


class CsrSystem:
    """A SparseSystem in CSR form (proj/include/flowfem/assembly.hpp:43-53): both triangles
    stored, free vertex major / component minor."""

    def __init__(self, row_ptr, cols, vals, rhs, components=3):
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
        self.cols = np.ascontiguousarray(cols, dtype=np.int32)
        self.vals = _f64(vals)
        self.rhs = _f64(rhs)
        self.components = int(components)
        self.n = len(self.row_ptr) - 1

    def dense(self):
        A = np.zeros((self.n, self.n))
        for r in range(self.n):
            for q in range(self.row_ptr[r], self.row_ptr[r + 1]):
                A[r, self.cols[q]] = self.vals[q]
        return A


def ref_assemble_system(terms, alpha, lam, nc=3, dir_vertices=None, dir_values=None):
    """The reference's assemble() (assembly.cpp:32-166) as a CsrSystem, optionally with a
    Dirichlet set (dir_values: len(dir_vertices) x nc)."""
    if REF is None:
        raise OracleError("reference oracle not built")
    terms = _f64(terms)
    _, H, W = terms.shape
    alpha, lam = _f64(alpha), _f64(lam)
    dv = np.ascontiguousarray(dir_vertices if dir_vertices is not None else [], dtype=np.int32)
    dval = _f64(dir_values if dir_values is not None else np.zeros((0, nc)))
    n, nnz = C.c_int(), C.c_long()
    args = [W, H, _ptr(terms), _ptr(alpha), _ptr(lam), nc, len(dv), _ptr(dv), _ptr(dval)]
    REF._call("assemble_system", *args, C.byref(n), C.byref(nnz), None, None, None, None)
    rp = np.zeros(n.value + 1, dtype=np.int32)
    cols = np.zeros(nnz.value, dtype=np.int32)
    vals = np.zeros(nnz.value)
    rhs = np.zeros(n.value)
    REF._call("assemble_system", *args, C.byref(n), C.byref(nnz), _ptr(rp), _ptr(cols),
              _ptr(vals), _ptr(rhs))
    return CsrSystem(rp, cols, vals, rhs, nc)


def csr_cg_solve(oracle, sys: CsrSystem, tol=1e-10, max_iters=0, warm=None):
    """cg_solve (linsolve.cpp:298-361) of the port or the reference on a CsrSystem;
    returns (x, iterations, residual)."""
    x = np.zeros(sys.n)
    it, res = C.c_int(), C.c_double()
    w = None if warm is None else _f64(warm)
    if oracle.prefix == "ref_":
        oracle._call("csr_cg_solve", sys.n, sys.components, _ptr(sys.row_ptr), _ptr(sys.cols),
                     _ptr(sys.vals), _ptr(sys.rhs), C.c_double(tol), int(max_iters), _ptr(w),
                     _ptr(x), C.byref(it), C.byref(res))
    else:
        oracle._call("csr_cg_solve", sys.n, _ptr(sys.row_ptr), _ptr(sys.cols), _ptr(sys.vals),
                     _ptr(sys.rhs), C.c_double(tol), int(max_iters), _ptr(w), _ptr(x),
                     C.byref(it), C.byref(res))
    return x, it.value, res.value


def ref_csr_solve(sys: CsrSystem, method=1, tol=1e-10, max_iters=0, warm=None):
    """The reference's solve() (linsolve.cpp:363-399); method 1 Cholesky, 0 CG."""
    x = np.zeros(sys.n)
    it, res = C.c_int(), C.c_double()
    w = None if warm is None else _f64(warm)
    REF._call("csr_solve", sys.n, sys.components, _ptr(sys.row_ptr), _ptr(sys.cols),
              _ptr(sys.vals), _ptr(sys.rhs), int(method), C.c_double(tol), int(max_iters),
              _ptr(w), _ptr(x), C.byref(it), C.byref(res))
    return x, it.value, res.value


def csr_spmv(oracle, sys: CsrSystem, x):
    y = np.zeros(sys.n)
    oracle._call("csr_spmv", sys.n, _ptr(sys.row_ptr), _ptr(sys.cols), _ptr(sys.vals),
                 _ptr(_f64(x)), _ptr(y))
    return y


def rcm_order(oracle, sys: CsrSystem):
    perm = np.zeros(sys.n, dtype=np.int32)
    if oracle.prefix == "ref_":
        oracle._call("rcm_order", sys.n, sys.components, _ptr(sys.row_ptr), _ptr(sys.cols),
                     _ptr(perm))
    else:
        oracle._call("rcm_order", sys.n, sys.components, _ptr(sys.row_ptr), _ptr(sys.cols),
                     _ptr(perm))
    return perm


def ref_compute_metrics(flow3, tu, tv):
    """The reference's compute_metrics (metrics.cpp:75-100): (aae_deg, ee, valid)."""
    flow3 = _f64(flow3)
    _, H, W = flow3.shape
    tu = np.ascontiguousarray(tu, dtype=np.float32)
    tv = np.ascontiguousarray(tv, dtype=np.float32)
    a, e, k = C.c_double(), C.c_double(), C.c_long()
    REF._call("compute_metrics", W, H, _ptr(flow3), _ptr(tu), _ptr(tv), C.byref(a), C.byref(e),
              C.byref(k))
    return a.value, e.value, k.value


def ref_write_flo(path, tu, tv):
    tu = np.ascontiguousarray(tu, dtype=np.float32)
    tv = np.ascontiguousarray(tv, dtype=np.float32)
    H, W = tu.shape
    REF._call("write_flo", path.encode(), W, H, _ptr(tu), _ptr(tv))


def ref_to_flo(flow3):
    flow3 = _f64(flow3)
    _, H, W = flow3.shape
    u = np.zeros((H, W), np.float32)
    v = np.zeros((H, W), np.float32)
    REF._call("to_flo", W, H, _ptr(flow3), _ptr(u), _ptr(v))
    return u, v


def _load(sub, name, prefix, kind):
    p = os.path.join(HERE, sub, name)
    return Oracle(p, prefix, kind) if os.path.exists(p) else None


PORT = _load("_port", "libflowfem_port.so", "fp_", "port")
REF = _load("_ref", "libflowfem_ref.so", "ref_", "reference")


def ref_chain_sample(f0, f1, sigma, rho=2.5, alpha0=1000.0, lambda0=1000.0, nc=3, kappa=10.0,
                     thr=0.1, alpha_th=None, cap_lo=2, cap_hi=12):
    """A timed one-of-each-stage sample of the reference's converged-pass chain
    (ref_capi.cpp ref_chain_sample); returns the stage seconds as a dict."""
    if REF is None:
        raise OracleError("reference oracle not built")
    f0, f1 = _f64(f0), _f64(f1)
    H, W = f0.shape
    if alpha_th is None:
        alpha_th = alpha0 / 100.0
    t = np.zeros(8)
    REF._call("chain_sample", W, H, _ptr(f0), _ptr(f1), C.c_double(sigma), C.c_double(rho),
              C.c_double(alpha0), C.c_double(lambda0), nc, C.c_double(kappa), C.c_double(thr),
              C.c_double(alpha_th), int(cap_lo), int(cap_hi), _ptr(t))
    keys = ("imaging", "mesh_reg", "assemble", "cg_setup", "cg_iter", "expand", "adapt", "wall")
    return dict(zip(keys, t.tolist()))


def extrapolate_chain(sample: dict, iters) -> float:
    """Seconds of a full converged-pass chain from a ref_chain_sample and the per-solve CG
    iteration counts of a full reference run (len(iters) = n_passes + 1 solves)."""
    n_solves = len(iters)
    return (sample["imaging"] + sample["mesh_reg"]
            + n_solves * (sample["assemble"] + sample["cg_setup"] + sample["expand"])
            + sum(iters) * sample["cg_iter"] + (n_solves - 1) * sample["adapt"])


def ref_schwarz_solve(terms, alpha, lam, px, py, ov, n_iters, workers=1, nc=3, adapt=False,
                      n_adapt=10, kappa=10.0, thr=0.1, alpha_th=10.0, method=1, cg_tol=1e-10):
    """The reference's literal Schwarz loop (proj/src/schwarz.cpp:162-319)."""
    if REF is None:
        raise OracleError("reference oracle not built")
    terms = _f64(terms)
    _, H, W = terms.shape
    alpha, lam = _f64(alpha).copy(), _f64(lam).copy()
    out = np.zeros((3, H, W))
    inc = np.zeros(n_iters)
    em = np.zeros(n_iters)
    REF._call("schwarz_solve", W, H, _ptr(terms), _ptr(alpha), _ptr(lam), px, py, ov, n_iters,
              workers, nc, int(adapt), n_adapt, C.c_double(kappa), C.c_double(thr),
              C.c_double(alpha_th), method, C.c_double(cg_tol), _ptr(out), _ptr(inc), _ptr(em))
    n_upd = min(n_adapt, n_iters) if adapt else 0
    return dict(u3=out, alpha=alpha, lam=lam, increments=inc, eta_max=em[:n_upd])


def parse_partition(flat: np.ndarray) -> dict:
    """Decode the flat partition format (include/flowfem_b200.h) into Python structures."""
    f = [int(v) for v in flat]
    W, H, px, py, ov, npart = f[:6]
    parts = []
    for p in range(npart):
        h = f[6 + 10 * p: 16 + 10 * p]
        parts.append(dict(core=tuple(h[0:4]), ext=tuple(h[4:8]), nb=h[8], nn=h[9]))
    pos = 6 + 10 * npart
    for part in parts:
        part["boundary"] = f[pos: pos + part["nb"]]
        pos += part["nb"]
        nbs = []
        for _ in range(part["nn"]):
            q, bx0, by0, bx1, by1, g = f[pos: pos + 6]
            nbs.append(dict(part=q, band=(bx0, by0, bx1, by1), gamma=f[pos + 6: pos + 6 + g]))
            pos += 6 + g
        part["neighbors"] = nbs
    assert pos == len(f)
    return dict(width=W, height=H, parts_x=px, parts_y=py, overlap=ov, parts=parts)
