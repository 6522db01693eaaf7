"""Python mirror of the reference ``flowfem`` API for the hot path, over the C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/flowfem/*.hpp
(imaging.hpp, assembly.hpp, adapt.hpp, schwarz.hpp, pipeline.hpp): functions raise
``FlowfemError`` (a ``RuntimeError``) carrying the reference's ``"<module>.<op>: ..."``
message prefixes. Arrays are numpy float64, images (H, W) row-major, vertex id y*W + x.

Every numerical call runs in ``libflowfem_b200.so`` on the GPU; the decomposition helpers
(``enumerate_splits``, ``choose_split``, ``build_partition``, ``assign_workers``) are host
integer code in the same library, as in the reference.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib


class FlowfemError(RuntimeError):
    pass


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _check(rc):
    if rc != 0:
        raise FlowfemError(_lib.last_error())


# ------------------------------------------------------------------------- context
class Context:
    """One GPU (one process per GPU). Owns the device-resident solver state."""

    def __init__(self, device: int | None = None):
        lib = _lib.load()
        if device is None:
            device = int(os.environ.get("FFB_DEVICE", os.environ.get("LOCAL_RANK", "0")))
        h = C.c_void_p()
        _check(lib.ffb_create(C.byref(h), int(device)))
        self._h = h
        self.device = device
        self.lib = lib

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_handle: int | None):
        """Launch on an external CUDA stream (e.g. torch.cuda.current_stream().cuda_stream,
        where 0 is the legacy default stream); None restores the context's own stream."""
        own = stream_handle is None
        _check(self.lib.ffb_set_stream(self._h, C.c_void_p(0 if own else stream_handle),
                                       int(own)))

    def set_factor_storage(self, bits: int):
        """64 (default): the preconditioner streams the subdomain factors in double. 32: opt-in —
        the wide-line solve kernel (c3, c4) streams a single-precision copy, half the bytes per
        application; factorisation, products and the CG stay in double (same 1e-8 parity)."""
        _check(self.lib.ffb_set_factor_storage(self._h, int(bits)))

    def factor_storage(self):
        """(requested bits, bits in use with the resident partition)."""
        b, u = C.c_int(), C.c_int()
        _check(self.lib.ffb_get_factor_storage(self._h, C.byref(b), C.byref(u)))
        return b.value, u.value

    def close(self):
        if getattr(self, "_h", None):
            self.lib.ffb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context()
    return _default


def kernel_launches() -> int:
    """Device kernels this process has launched through the library."""
    return int(_lib.load().ffb_kernel_launches())


# ------------------------------------------------------------------------- imaging
def gaussian_smooth(img, sigma: float, ctx: Context | None = None) -> np.ndarray:
    """imaging.hpp:42-44 / imaging.cpp:33-63."""
    ctx = ctx or default_context()
    img = _f64(img)
    H, W = img.shape
    out = np.empty_like(img)
    _check(ctx.lib.ffb_gaussian_smooth(ctx.handle, W, H, _p(img), float(sigma), _p(out)))
    return out


@dataclass
class DerivativeField:
    fx: np.ndarray
    fy: np.ndarray
    ft: np.ndarray
    f: np.ndarray


def compute_derivatives(f0, f1, ctx: Context | None = None) -> DerivativeField:
    """imaging.hpp:54-56 / imaging.cpp:65-106."""
    ctx = ctx or default_context()
    f0, f1 = _f64(f0), _f64(f1)
    if f0.shape != f1.shape:
        raise FlowfemError("imaging.compute_derivatives: frame sizes differ")
    H, W = f0.shape
    outs = [np.empty_like(f0) for _ in range(4)]
    _check(ctx.lib.ffb_compute_derivatives(ctx.handle, W, H, _p(f0), _p(f1),
                                           *[_p(o) for o in outs]))
    return DerivativeField(*outs)


TERM_NAMES = ("a11", "a12", "a13", "a22", "a23", "a33", "f1", "f2", "f3", "c")


class DataTerms:
    """imaging.hpp:61-67: ten (H, W) planes, also reachable by name."""

    def __init__(self, planes: np.ndarray):
        self.planes = np.ascontiguousarray(planes, dtype=np.float64)
        assert self.planes.ndim == 3 and self.planes.shape[0] == 10

    @property
    def height(self):
        return self.planes.shape[1]

    @property
    def width(self):
        return self.planes.shape[2]

    def __getattr__(self, name):
        if name in TERM_NAMES:
            return self.planes[TERM_NAMES.index(name)]
        raise AttributeError(name)


def build_data_terms(d: DerivativeField, rho: float, ctx: Context | None = None) -> DataTerms:
    """imaging.hpp:69 / imaging.cpp:108-138."""
    ctx = ctx or default_context()
    fx, fy, ft, f = map(_f64, (d.fx, d.fy, d.ft, d.f))
    H, W = fx.shape
    out = np.empty((10, H, W))
    _check(ctx.lib.ffb_build_data_terms(ctx.handle, W, H, _p(fx), _p(fy), _p(ft), _p(f),
                                        float(rho), _p(out)))
    return DataTerms(out)


def frames_to_terms(f0, f1, sigma: float, rho: float, ctx: Context | None = None) -> DataTerms:
    """run_on_frames' imaging prefix (pipeline.cpp:49-52)."""
    ctx = ctx or default_context()
    f0, f1 = _f64(f0), _f64(f1)
    if f0.shape != f1.shape:
        raise FlowfemError("imaging.compute_derivatives: frame sizes differ")
    H, W = f0.shape
    out = np.empty((10, H, W))
    _check(ctx.lib.ffb_frames_to_terms(ctx.handle, W, H, _p(f0), _p(f1), float(sigma),
                                       float(rho), _p(out)))
    return DataTerms(out)


# ---------------------------------------------------------------------- decomposition
@dataclass
class SplitChoice:
    parts_x: int
    parts_y: int
    ratio: float


def enumerate_splits(width: int, height: int, n_parts: int) -> List[SplitChoice]:
    """schwarz.hpp:16 / schwarz.cpp:16-30."""
    lib = _lib.load()
    cap = max(int(n_parts), 1)
    px = np.zeros(cap, np.int32)
    py = np.zeros(cap, np.int32)
    ra = np.zeros(cap)
    n = lib.ffb_enumerate_splits(width, height, n_parts, _p(px), _p(py), _p(ra), cap)
    if n < 0:
        raise FlowfemError(_lib.last_error())
    return [SplitChoice(int(px[i]), int(py[i]), float(ra[i])) for i in range(n)]


def choose_split(width: int, height: int, n_parts: int) -> SplitChoice:
    """schwarz.hpp:19 / schwarz.cpp:32-44."""
    lib = _lib.load()
    px, py, ra = C.c_int(), C.c_int(), C.c_double()
    _check(lib.ffb_choose_split(width, height, n_parts, C.byref(px), C.byref(py), C.byref(ra)))
    return SplitChoice(px.value, py.value, ra.value)


def assign_workers(n_workers: int, n_parts: int) -> List[int]:
    """schwarz.hpp:56 / schwarz.cpp:46-52."""
    lib = _lib.load()
    out = np.zeros(max(n_workers, 1), np.int32)
    _check(lib.ffb_assign_workers(n_workers, n_parts, _p(out)))
    return [int(v) for v in out[:n_workers]]


@dataclass
class Rect:
    x0: int
    y0: int
    x1: int
    y1: int

    def w(self):
        return self.x1 - self.x0

    def h(self):
        return self.y1 - self.y0

    def contains(self, x, y):
        return self.x0 <= x < self.x1 and self.y0 <= y < self.y1


@dataclass
class Neighbor:
    part: int
    band: Rect
    gamma: List[int]


@dataclass
class Subdomain:
    core: Rect
    ext: Rect
    neighbors: List[Neighbor] = field(default_factory=list)
    boundary: List[int] = field(default_factory=list)


@dataclass
class Partition:
    width: int
    height: int
    parts_x: int
    parts_y: int
    overlap: int
    parts: List[Subdomain]
    flat: np.ndarray


def build_partition_flat(width, height, parts_x, parts_y, overlap) -> np.ndarray:
    lib = _lib.load()
    need = lib.ffb_build_partition(width, height, parts_x, parts_y, overlap, None, 0)
    if need < 0:
        raise FlowfemError(_lib.last_error())
    buf = np.zeros(need, np.int32)
    got = lib.ffb_build_partition(width, height, parts_x, parts_y, overlap, _p(buf), need)
    assert got == need
    return buf


def parse_partition(flat: np.ndarray) -> Partition:
    f = [int(v) for v in flat]
    W, H, px, py, ov, npart = f[:6]
    heads = [f[6 + 10 * p: 16 + 10 * p] for p in range(npart)]
    pos = 6 + 10 * npart
    parts = []
    for h in heads:
        s = Subdomain(Rect(*h[0:4]), Rect(*h[4:8]))
        s.boundary = f[pos: pos + h[8]]
        pos += h[8]
        for _ in range(h[9]):
            q, bx0, by0, bx1, by1, g = f[pos: pos + 6]
            s.neighbors.append(Neighbor(q, Rect(bx0, by0, bx1, by1), f[pos + 6: pos + 6 + g]))
            pos += 6 + g
        parts.append(s)
    assert pos == len(f)
    return Partition(W, H, px, py, ov, parts, np.asarray(flat, np.int32))


def build_partition(width, height, parts_x, parts_y, overlap) -> Partition:
    """schwarz.hpp:52 / schwarz.cpp:54-128 (bit-exact)."""
    return parse_partition(build_partition_flat(width, height, parts_x, parts_y, overlap))


# ------------------------------------------------------------------- operator / adapt
@dataclass
class RegField:
    alpha: np.ndarray
    lambda_: np.ndarray


def uniform_reg(width: int, height: int, alpha0: float, lambda0: float) -> RegField:
    """assembly.cpp:9-14."""
    nt = 2 * (width - 1) * (height - 1)
    return RegField(np.full(nt, float(alpha0)), np.full(nt, float(lambda0)))


@dataclass
class FlowState:
    u1: np.ndarray
    u2: np.ndarray
    mt: np.ndarray

    @staticmethod
    def from_planes(p3):
        p3 = np.asarray(p3)
        return FlowState(p3[0], p3[1], p3[2])

    def planes(self):
        return np.ascontiguousarray(np.stack([self.u1, self.u2, self.mt]), dtype=np.float64)


def assemble_apply(terms: DataTerms, reg: RegField, components: int, x: FlowState,
                   ctx: Context | None = None):
    """(A x, b) of the unconstrained global system: assemble + spmv (assembly.cpp:32-249)."""
    ctx = ctx or default_context()
    t = terms.planes
    _, H, W = t.shape
    x3 = x.planes()
    y3 = np.zeros((3, H, W))
    b3 = np.zeros((3, H, W))
    _check(ctx.lib.ffb_assemble_apply(ctx.handle, W, H, _p(t), _p(_f64(reg.alpha)),
                                      _p(_f64(reg.lambda_)), components, _p(x3), _p(y3),
                                      _p(b3)))
    return FlowState.from_planes(y3), FlowState.from_planes(b3)


# ---------------------------------------------------------------- I/O and evaluation
def load_image(path: str) -> np.ndarray:
    """imaging.hpp load_image (image_io.cpp:136-145): binary PGM or PNG -> H x W float64 in
    [0,1]."""
    lib = _lib.load()
    W, H = C.c_int(), C.c_int()
    _check(lib.ffb_load_image(os.fsencode(path), C.byref(W), C.byref(H), None))
    img = np.zeros((H.value, W.value))
    _check(lib.ffb_load_image(os.fsencode(path), C.byref(W), C.byref(H), _p(img)))
    return img


def save_pgm(path: str, img) -> None:
    """image_io.cpp:147-160 (clamped to [0,1], 8 bit)."""
    img = _f64(img)
    H, W = img.shape
    _check(_lib.load().ffb_save_pgm(os.fsencode(path), W, H, _p(img)))


@dataclass
class FloField:
    """metrics.hpp:13-23: float32 flow planes (H x W); |component| > 1e9 marks invalid."""
    u: np.ndarray
    v: np.ndarray

    @property
    def width(self) -> int:
        return self.u.shape[1]

    @property
    def height(self) -> int:
        return self.u.shape[0]


def read_flo(path: str) -> FloField:
    """metrics.cpp:22-45."""
    lib = _lib.load()
    W, H = C.c_int(), C.c_int()
    _check(lib.ffb_read_flo(os.fsencode(path), C.byref(W), C.byref(H), None, None))
    u = np.zeros((H.value, W.value), np.float32)
    v = np.zeros((H.value, W.value), np.float32)
    _check(lib.ffb_read_flo(os.fsencode(path), C.byref(W), C.byref(H), _p(u), _p(v)))
    return FloField(u, v)


def write_flo(path: str, f: FloField) -> None:
    """metrics.cpp:47-64."""
    u = np.ascontiguousarray(f.u, dtype=np.float32)
    v = np.ascontiguousarray(f.v, dtype=np.float32)
    H, W = u.shape
    _check(_lib.load().ffb_write_flo(os.fsencode(path), W, H, _p(u), _p(v)))


def to_flo(state: "FlowState") -> FloField:
    """metrics.cpp:66-73: (u1, u2) rounded to float32."""
    p = state.planes()
    return FloField(p[0].astype(np.float32), p[1].astype(np.float32))


@dataclass
class FlowMetrics:
    """metrics.hpp:33-37."""
    aae_deg: float = 0.0
    ee: float = 0.0
    valid: int = 0


def compute_metrics(flow: "FlowState", truth: FloField, ctx: Context | None = None) -> FlowMetrics:
    """metrics.cpp:75-100 as a device reduction: average angular error (degrees, (u, v, 1)
    normalisation) and endpoint error over pixels with valid truth."""
    ctx = ctx or default_context()
    p = flow.planes()
    if p.shape[1:] != truth.u.shape:
        raise FlowfemError("metrics.compute_metrics: flow and ground truth sizes differ")
    H, W = truth.u.shape
    u1 = np.ascontiguousarray(p[0])
    u2 = np.ascontiguousarray(p[1])
    tu = np.ascontiguousarray(truth.u, dtype=np.float32)
    tv = np.ascontiguousarray(truth.v, dtype=np.float32)
    a, e, k = C.c_double(), C.c_double(), C.c_longlong()
    _check(ctx.lib.ffb_compute_metrics(ctx.handle, W, H, _p(u1), _p(u2), _p(tu), _p(tv),
                                       C.byref(a), C.byref(e), C.byref(k)))
    return FlowMetrics(a.value, e.value, k.value)


# ---------------------------------------------------------------- linsolve boundary
class SolveMethod:
    """linsolve.hpp:10 (enum class SolveMethod)."""
    DirectCholesky = 0
    ConjugateGradient = 1


@dataclass
class SolverConfig:
    """linsolve.hpp:12-17."""
    method: int = SolveMethod.DirectCholesky
    cg_tolerance: float = 1e-10
    cg_max_iters: int = 0
    factor_workers: int = 1  # accepted for API parity; the factor runs on the device


@dataclass
class SolveReport:
    """linsolve.hpp:19-22."""
    iterations: int = 0
    residual: float = 0.0


@dataclass
class SparseSystem:
    """assembly.hpp:43-53: n scalar unknowns, CSR with both triangles, free vertex major /
    component minor (the Dirichlet bookkeeping of the reference is not needed here)."""
    row_ptr: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    rhs: np.ndarray
    components: int = 3

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int32)
        self.cols = np.ascontiguousarray(self.cols, dtype=np.int32)
        self.vals = _f64(self.vals)
        self.rhs = _f64(self.rhs)
        if len(self.rhs) != self.n:
            raise FlowfemError("linsolve: rhs length does not match the system size")

    @property
    def n(self) -> int:
        return len(self.row_ptr) - 1


def _ip(a):
    return a.ctypes.data_as(C.c_void_p)


def spmv(sys: SparseSystem, x, ctx: Context | None = None) -> np.ndarray:
    """y = A x (assembly.hpp:76, assembly.cpp:240-249), on the device, bitwise."""
    ctx = ctx or default_context()
    x = _f64(x)
    y = np.zeros(sys.n)
    _check(ctx.lib.ffb_csr_spmv(ctx.handle, sys.n, _ip(sys.row_ptr), _ip(sys.cols),
                                _p(sys.vals), _p(x), _p(y)))
    return y


def rcm_order(sys: SparseSystem) -> np.ndarray:
    """linsolve.hpp:22-24 / linsolve.cpp:37-83 (host integer work, bit-exact)."""
    lib = _lib.load()
    perm = np.zeros(sys.n, dtype=np.int32)
    _check(lib.ffb_rcm_order(sys.n, sys.components, _ip(sys.row_ptr), _ip(sys.cols), _ip(perm)))
    return perm


def cg_solve(sys: SparseSystem, cfg: SolverConfig = SolverConfig(), warm_start=None,
             report: SolveReport | None = None, ctx: Context | None = None) -> np.ndarray:
    """linsolve.hpp:53-56 / linsolve.cpp:298-361 on the device (bitwise the reference's)."""
    ctx = ctx or default_context()
    x = np.zeros(sys.n)
    it, res = C.c_int(), C.c_double()
    w = _f64(warm_start) if warm_start is not None and len(warm_start) == sys.n else None
    rc = ctx.lib.ffb_csr_cg_solve(ctx.handle, sys.n, _ip(sys.row_ptr), _ip(sys.cols),
                                  _p(sys.vals), _p(sys.rhs), float(cfg.cg_tolerance),
                                  int(cfg.cg_max_iters), _p(w) if w is not None else None,
                                  _p(x), C.byref(it), C.byref(res))
    if report is not None:
        report.iterations, report.residual = it.value, res.value
    _check(rc)
    return x


def solve(sys: SparseSystem, cfg: SolverConfig = SolverConfig(),
          report: SolveReport | None = None, warm_start=None,
          ctx: Context | None = None) -> np.ndarray:
    """linsolve.hpp:58-62 / linsolve.cpp:363-399: zero rhs -> 0; CG or the direct solve
    (band Cholesky of the RCM-ordered matrix on the device + one refinement step)."""
    ctx = ctx or default_context()
    x = np.zeros(sys.n)
    it, res = C.c_int(), C.c_double()
    w = _f64(warm_start) if warm_start is not None and len(warm_start) == sys.n else None
    rc = ctx.lib.ffb_csr_solve(ctx.handle, sys.n, sys.components, _ip(sys.row_ptr),
                               _ip(sys.cols), _p(sys.vals), _p(sys.rhs), int(cfg.method),
                               float(cfg.cg_tolerance), int(cfg.cg_max_iters),
                               _p(w) if w is not None else None, _p(x), C.byref(it),
                               C.byref(res))
    if report is not None:
        report.iterations, report.residual = it.value, res.value
    _check(rc)
    return x


def assemble(terms: DataTerms, reg: RegField, components: int = 3, dirichlet_vertices=None,
             dirichlet_values=None, ctx: Context | None = None) -> SparseSystem:
    """assemble (assembly.hpp:59-61, assembly.cpp:32-166) as an explicit CSR system, with an
    optional Dirichlet set (vertex ids, values (n, components)) eliminated into the rhs;
    values from the device operator, bitwise equal to the reference's."""
    ctx = ctx or default_context()
    t = terms.planes
    _, H, W = t.shape
    lib = ctx.lib
    nd = 0 if dirichlet_vertices is None else len(dirichlet_vertices)
    dv = np.ascontiguousarray(dirichlet_vertices, dtype=np.int32) if nd else None
    dval = _f64(np.asarray(dirichlet_values).reshape(nd, components)) if nd else None
    n, nnz = C.c_int(), C.c_longlong()
    args = [ctx.handle, W, H, _p(t), _p(_f64(reg.alpha)), _p(_f64(reg.lambda_)), components, nd,
            _ip(dv) if nd else None, _p(dval) if nd else None, C.byref(n), C.byref(nnz)]
    _check(lib.ffb_assemble_system(*args, None, None, None, None, None, None))
    rp = np.zeros(n.value + 1, dtype=np.int32)
    cols = np.zeros(nnz.value, dtype=np.int32)
    vals = np.zeros(nnz.value)
    rhs = np.zeros(n.value)
    _check(lib.ffb_assemble_system(*args, _ip(rp), _ip(cols), _p(vals), _p(rhs), None, None))
    return SparseSystem(rp, cols, vals, rhs, components)


class SparseCholesky:
    """SparseCholesky (linsolve.hpp:32-48) on the device: analyze = the reference's RCM order
    (bit-exact) + band width, factorize = band Cholesky of the permuted matrix, solve."""

    def __init__(self, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        _check(self.ctx.lib.ffb_chol_create(self.ctx.handle, C.byref(h)))
        self._h = h
        self.n = 0

    def analyze(self, sys: SparseSystem):
        _check(self.ctx.lib.ffb_chol_analyze(self._h, sys.n, sys.components, _ip(sys.row_ptr),
                                             _ip(sys.cols)))
        self.n = sys.n

    def factorize(self, sys: SparseSystem, workers: int = 1):
        _check(self.ctx.lib.ffb_chol_factorize(self._h, sys.n, _p(sys.vals)))

    def solve(self, b) -> np.ndarray:
        b = _f64(b)
        x = np.zeros(self.n)
        _check(self.ctx.lib.ffb_chol_solve(self._h, len(b), _p(b), _p(x)))
        return x

    def bandwidth(self) -> int:
        bw = C.c_int()
        _check(self.ctx.lib.ffb_chol_info(self._h, C.byref(bw), None))
        return bw.value

    def __del__(self):
        try:
            if self._h:
                self.ctx.lib.ffb_chol_destroy(self._h)
        except Exception:
            pass


@dataclass
class IndicatorField:
    eta: np.ndarray
    eta_max: float


def error_indicator(terms: DataTerms, reg: RegField, state: FlowState, components: int = 3,
                    ctx: Context | None = None) -> IndicatorField:
    """adapt.hpp:20-23 / adapt.cpp:9-99."""
    ctx = ctx or default_context()
    t = terms.planes
    _, H, W = t.shape
    eta = np.zeros(2 * (W - 1) * (H - 1))
    em = C.c_double()
    _check(ctx.lib.ffb_error_indicator(ctx.handle, W, H, _p(t), _p(_f64(reg.alpha)),
                                       _p(_f64(reg.lambda_)), _p(state.planes()), components,
                                       _p(eta), C.byref(em)))
    return IndicatorField(eta, em.value)


@dataclass
class AdaptConfig:
    enabled: bool = True
    kappa: float = 10.0
    eta_threshold: float = 0.1
    alpha_th: float = 10.0
    n_adapt: int = 10


def update_alpha(reg: RegField, ind: IndicatorField, cfg: AdaptConfig,
                 ctx: Context | None = None) -> RegField:
    """adapt.hpp:34-35 / adapt.cpp:101-112; lambda untouched."""
    ctx = ctx or default_context()
    a = _f64(reg.alpha)
    out = np.empty_like(a)
    _check(ctx.lib.ffb_update_alpha(ctx.handle, a.size, _p(a), _p(_f64(ind.eta)),
                                    float(ind.eta_max), float(cfg.kappa),
                                    float(cfg.eta_threshold), float(cfg.alpha_th), _p(out)))
    return RegField(out, reg.lambda_.copy())


# ------------------------------------------------------------------------- solver
class SchwarzSolver:
    """Device-resident global system + additive-Schwarz-preconditioned CG.

    The stateful form of the converged-pass loop: set_terms / set_reg / set_partition,
    then solve (warm-started), adapt, solve, ...
    """

    def __init__(self, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.shape = None

    def set_terms(self, terms: DataTerms):
        t = terms.planes
        _, H, W = t.shape
        self.shape = (H, W)
        _check(self.ctx.lib.ffb_set_terms(self.ctx.handle, W, H, _p(t)))

    def set_frames(self, f0, f1, sigma, rho):
        f0, f1 = _f64(f0), _f64(f1)
        H, W = f0.shape
        self.shape = (H, W)
        _check(self.ctx.lib.ffb_set_frames(self.ctx.handle, W, H, _p(f0), _p(f1), float(sigma),
                                           float(rho)))

    def set_reg(self, reg: RegField):
        _check(self.ctx.lib.ffb_set_reg(self.ctx.handle, _p(_f64(reg.alpha)),
                                        _p(_f64(reg.lambda_))))

    def get_reg(self) -> RegField:
        H, W = self.shape
        nt = 2 * (W - 1) * (H - 1)
        a, l = np.zeros(nt), np.zeros(nt)
        _check(self.ctx.lib.ffb_get_reg(self.ctx.handle, _p(a), _p(l)))
        return RegField(a, l)

    def set_partition(self, parts_x: int, parts_y: int, overlap: int):
        _check(self.ctx.lib.ffb_set_partition(self.ctx.handle, parts_x, parts_y, overlap))

    def solve(self, components=3, tol=1e-10, max_iters=0, warm: FlowState | None = None):
        H, W = self.shape
        u3 = warm.planes() if warm is not None else np.zeros((3, H, W))
        it, res = C.c_int(), C.c_double()
        _check(self.ctx.lib.ffb_pcg_solve(self.ctx.handle, components, float(tol), max_iters,
                                          int(warm is not None), _p(u3), C.byref(it),
                                          C.byref(res)))
        return FlowState.from_planes(u3), it.value, res.value

    def adapt(self, components=3, kappa=10.0, eta_threshold=0.1, alpha_th=10.0) -> float:
        em = C.c_double()
        _check(self.ctx.lib.ffb_adapt(self.ctx.handle, components, float(kappa),
                                      float(eta_threshold), float(alpha_th), C.byref(em)))
        return em.value


@dataclass
class SchwarzOptions:
    """schwarz.hpp:59-66 (workers only affects CPU threading in the reference and is accepted
    for signature compatibility). ``solver.method`` picks the subdomain solver: DirectCholesky
    (device factorisation + one refinement step) or ConjugateGradient (the reference's
    Jacobi-PCG per subdomain, warm-started, bitwise equal to the reference's)."""
    n_iters: int = 10
    workers: int = 1
    components: int = 3
    adapt: AdaptConfig = field(default_factory=AdaptConfig)
    solver: SolverConfig = field(default_factory=SolverConfig)
    record_alpha_history: bool = False


@dataclass
class SchwarzStats:
    """schwarz.hpp:68-73."""
    increments: List[float] = field(default_factory=list)
    seconds: List[float] = field(default_factory=list)
    eta_max: List[float] = field(default_factory=list)
    alpha_history: List[np.ndarray] = field(default_factory=list)


def schwarz_solve(terms: DataTerms, reg: RegField, parts_x: int, parts_y: int, overlap: int,
                  opt: SchwarzOptions, ctx: Context | None = None):
    """schwarz_solve (schwarz.hpp:79-81): the reference's synchronous RAS loop on the device.

    ``reg`` is updated in place when adapting (RegField& reg). Returns (FlowState, stats)."""
    ctx = ctx or default_context()
    t = terms.planes
    _, H, W = t.shape
    lib = ctx.lib
    _check(lib.ffb_set_terms(ctx.handle, W, H, _p(t)))
    reg.alpha = _f64(reg.alpha)
    _check(lib.ffb_set_reg(ctx.handle, _p(reg.alpha), _p(_f64(reg.lambda_))))
    _check(lib.ffb_set_partition(ctx.handle, parts_x, parts_y, overlap))
    u3 = np.zeros((3, H, W))
    n = max(opt.n_iters, 1)
    inc, sec = np.zeros(n), np.zeros(n)
    a = opt.adapt
    n_upd = min(a.n_adapt, opt.n_iters) if a.enabled else 0
    em = np.zeros(max(n_upd, 1))
    ntri = 2 * (W - 1) * (H - 1)
    hist = np.zeros((max(n_upd, 1), ntri)) if opt.record_alpha_history else None
    o = _lib.SchwarzOptionsC(opt.n_iters, opt.workers, opt.components, int(a.enabled),
                             a.n_adapt, float(a.kappa), float(a.eta_threshold), float(a.alpha_th),
                             int(opt.solver.method), int(opt.solver.cg_max_iters),
                             float(opt.solver.cg_tolerance), int(opt.record_alpha_history))
    st = _lib.SchwarzStatsC(inc.ctypes.data, sec.ctypes.data, em.ctypes.data,
                            hist.ctypes.data if hist is not None else None, 0)
    _check(lib.ffb_schwarz_run(ctx.handle, C.byref(o), _p(u3), C.byref(st)))
    if a.enabled:
        _check(lib.ffb_get_reg(ctx.handle, _p(reg.alpha), None))
    stats = SchwarzStats(list(inc[:opt.n_iters]), list(sec[:opt.n_iters]), list(em[:st.n_updates]),
                         [hist[k].copy() for k in range(st.n_updates)] if hist is not None else [])
    return FlowState.from_planes(u3), stats


def energy(terms: DataTerms, reg: RegField, state: FlowState, components: int = 3,
           ctx: Context | None = None) -> float:
    """energy (assembly.hpp:70-73, assembly.cpp:201-238): the discrete energy whose gradient
    is A x - b; a deterministic device reduction."""
    ctx = ctx or default_context()
    t = terms.planes
    _, H, W = t.shape
    e = C.c_double()
    _check(ctx.lib.ffb_energy(ctx.handle, W, H, _p(t), _p(_f64(reg.alpha)), _p(_f64(reg.lambda_)),
                              _p(_f64(state.planes())), components, C.byref(e)))
    return e.value


def resident_energy(components: int = 3, ctx: Context | None = None) -> float:
    """energy of the context's resident solution (the last solve) at the resident alpha."""
    ctx = ctx or default_context()
    e = C.c_double()
    _check(ctx.lib.ffb_energy_resident(ctx.handle, components, C.byref(e)))
    return e.value


# ------------------------------------------------------------------------- pipeline
@dataclass
class RunConfig:
    """pipeline.hpp:15-33 (solver-relevant fields; file/CLI fields are out of scope)."""
    sigma: float = 1.0
    rho: float = 2.5
    alpha0: float = 1000.0
    lambda0: float = 1000.0
    illumination: bool = True
    parts: int = 4
    overlap: int = 5
    adapt: bool = True
    kappa: float = 10.0
    eta_threshold: float = 0.1
    alpha_th: Optional[float] = None
    adapt_iters: int = 10
    cg_tolerance: float = 1e-10
    max_iters: int = 0

    def to_c(self) -> _lib.RunConfigC:
        return _lib.RunConfigC(self.sigma, self.rho, self.alpha0, self.lambda0,
                               int(self.illumination), self.parts, self.overlap, int(self.adapt),
                               self.adapt_iters, self.kappa, self.eta_threshold,
                               float("nan") if self.alpha_th is None else self.alpha_th,
                               self.cg_tolerance, self.max_iters)


@dataclass
class RunStats:
    parts_x: int
    parts_y: int
    iters: List[int]
    residual: List[float]
    eta_max: List[float]
    pcg_iterations: int
    ms_terms: float
    ms_factor: float
    ms_pcg: float
    ms_adapt: float
    ms_total: float
    factor_doubles: float
    iter_bytes: float
    ms_asm_per_iter: float
    ms_factor_full: float = 0.0
    factor_flops: float = 0.0

    @staticmethod
    def from_c(s: _lib.RunStatsC, n_passes: int):
        n = s.n_solves
        return RunStats(s.parts_x, s.parts_y, list(s.iters[:n]), list(s.residual[:n]),
                        list(s.eta_max[:max(n - 1, 0)]), s.pcg_iterations, s.ms_terms,
                        s.ms_factor, s.ms_pcg, s.ms_adapt, s.ms_total, s.factor_doubles,
                        s.iter_bytes, s.ms_asm_per_iter, s.ms_factor_full, s.factor_flops)


@dataclass
class RunResult:
    flow: FlowState
    reg: RegField
    stats: RunStats
    width: int
    height: int


def run_on_frames(f0, f1, cfg: RunConfig, ctx: Context | None = None) -> RunResult:
    """pipeline.hpp:53 / pipeline.cpp:38-78 under the converged-pass protocol."""
    ctx = ctx or default_context()
    f0, f1 = _f64(f0), _f64(f1)
    if f0.shape != f1.shape:
        raise FlowfemError("cli.run: frame sizes differ")
    if f0.ndim != 2 or f0.shape[0] < 2 or f0.shape[1] < 2:
        raise FlowfemError("cli.run: frames must be at least 2x2")
    H, W = f0.shape
    u3 = np.zeros((3, H, W))
    alpha = np.zeros(2 * (W - 1) * (H - 1))
    st = _lib.RunStatsC()
    c = cfg.to_c()
    _check(ctx.lib.ffb_run_on_frames(ctx.handle, W, H, _p(f0), _p(f1), C.byref(c), _p(u3),
                                     _p(alpha), C.byref(st)))
    lam = np.full_like(alpha, cfg.lambda0)
    return RunResult(FlowState.from_planes(u3), RegField(alpha, lam),
                     RunStats.from_c(st, cfg.adapt_iters), W, H)


@dataclass
class PipelineConfig:
    """The file-level fields of pipeline.hpp:15-33 used by run_pipeline; the solver fields
    are a RunConfig. Visualisations (out_png, dump_alpha, dump_mt) are out of scope."""
    frame0: str = ""
    frame1: str = ""
    ground_truth: str = ""
    out_flo: str = ""
    out_metrics: str = ""
    run: RunConfig = field(default_factory=RunConfig)
    scale_255: bool = False  # multiply the [0,1] images by 255 (SURVEY D3 frames)


@dataclass
class PipelineResult:
    result: RunResult
    metrics: Optional[FlowMetrics]


def run_pipeline(cfg: PipelineConfig, ctx: Context | None = None) -> PipelineResult:
    """run_pipeline (pipeline.cpp:110-120): load both frames, run_on_frames, compute_metrics
    against the ground truth if given, write the .flo and the metrics CSV (pipeline.cpp:82-98)."""
    if not cfg.frame0 or not cfg.frame1:
        raise FlowfemError("cli.run: both frames are required")
    f0, f1 = load_image(cfg.frame0), load_image(cfg.frame1)
    if cfg.scale_255:
        f0, f1 = f0 * 255.0, f1 * 255.0
    res = run_on_frames(f0, f1, cfg.run, ctx)
    metrics = None
    if cfg.ground_truth:
        metrics = compute_metrics(res.flow, read_flo(cfg.ground_truth), ctx)
    if cfg.out_flo:
        write_flo(cfg.out_flo, to_flo(res.flow))
    if cfg.out_metrics:
        try:
            with open(cfg.out_metrics, "w") as fh:
                fh.write("mode,aae_deg,ee,valid_pixels\n")
                if metrics is not None:
                    fh.write(f"{'illum_on' if cfg.run.illumination else 'illum_off'},"
                             f"{metrics.aae_deg:g},{metrics.ee:g},{metrics.valid}\n")
        except OSError:
            raise FlowfemError("cli.out_metrics: cannot open " + cfg.out_metrics)
    return PipelineResult(res, metrics)


def run_on_frames_device(f0_ptr: int, f1_ptr: int, W: int, H: int, u3_ptr: int, cfg: RunConfig,
                         ctx: Context | None = None) -> RunStats:
    """Same with device pointers (e.g. torch CUDA tensors' data_ptr()); inputs stay in HBM."""
    ctx = ctx or default_context()
    st = _lib.RunStatsC()
    c = cfg.to_c()
    _check(ctx.lib.ffb_run_on_frames_dev(ctx.handle, W, H, C.c_void_p(f0_ptr),
                                         C.c_void_p(f1_ptr), C.byref(c), C.c_void_p(u3_ptr),
                                         C.byref(st)))
    return RunStats.from_c(st, cfg.adapt_iters)
