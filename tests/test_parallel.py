"""Multi-GPU path on CPU: the sharded host driver
(paper_1508_02977_b200/parallel.py) with world_size 1 and 2 over gloo.

The device stages are emulated by ``EmuBackend`` (numpy; the operator comes from the oracle
port, subdomain solves are dense) implementing the same staged protocol as the C-ABI
(ffb_pcg_begin / stage 0 / all-reduce z / stage 1 / status / end): only this rank's
subdomains contribute to z, vectors and CG scalars are replicated. Checks: the shard rule
equals the library's, every subdomain is owned exactly once, and the 2-rank result equals
the 1-rank result and the oracle's converged chain.
"""
import os
import socket
import tempfile

import numpy as np
import pytest

from conftest import rel_l2
from paper_1508_02977_b200 import flowfem as ff
from paper_1508_02977_b200 import parallel as par


def test_shard_rule_matches_library():
    from paper_1508_02977_b200 import _lib
    import ctypes as C
    lib = _lib.load()
    for npart in (1, 4, 16, 64, 256, 7):
        for world in (1, 2, 3, 4, 8):
            owned = []
            for rank in range(world):
                lo, hi = C.c_int(), C.c_int()
                assert lib.ffb_shard_range(npart, rank, world, C.byref(lo), C.byref(hi)) == 0
                assert (lo.value, hi.value) == par.shard_range(npart, rank, world)
                owned += list(range(lo.value, hi.value))
            assert owned == list(range(npart))


def free_rect(P, p):
    e = P.parts[p].ext
    return (e.x0 + (e.x0 > 0), e.y0 + (e.y0 > 0), e.x1 - (e.x1 < P.width), e.y1 - (e.y1 < P.height))


class EmuBackend:
    """numpy emulation of one rank's device stages (test infrastructure)."""

    def __init__(self, port, rank, world):
        self.port, self.rank, self.world = port, rank, world

    def setup(self, f0, f1, cfg):
        H, W = f0.shape
        self.H, self.W, self.N = H, W, H * W
        self.t10 = self.port.frames_to_terms(f0, f1, cfg.sigma, cfg.rho)
        nt = 2 * (W - 1) * (H - 1)
        self.alpha = np.full(nt, cfg.alpha0)
        self.lam = np.full(nt, cfg.lambda0)
        sp = ff.choose_split(W, H, cfg.parts)
        self.P = ff.build_partition(W, H, sp.parts_x, sp.parts_y, cfg.overlap)
        lo, hi = par.shard_range(len(self.P.parts), self.rank, self.world)
        self.own = range(lo, hi)
        self.x = np.zeros(3 * self.N)
        return sp

    def _apply(self, v):  # interleaved (vertex-major, component-minor) -> A v
        p3 = v.reshape(self.N, 3).T.reshape(3, self.H, self.W)
        y3, b3 = self.port.assemble_apply(self.t10, self.alpha, self.lam, 3, p3)
        return y3.reshape(3, self.N).T.ravel(), b3.reshape(3, self.N).T.ravel()

    def _factor(self):
        # probe A with 27 coloured vectors (stencil reach is one pixel)
        n = 3 * self.N
        A = np.zeros((n, n))
        ys, xs = np.divmod(np.arange(self.N), self.W)
        for cy in range(3):
            for cx in range(3):
                verts = np.flatnonzero((xs % 3 == cx) & (ys % 3 == cy))
                for c in range(3):
                    e = np.zeros(n)
                    e[3 * verts + c] = 1.0
                    col = self._apply(e)[0]
                    for v in verts:
                        x, y = xs[v], ys[v]
                        for yy in range(max(0, y - 1), min(self.H, y + 2)):
                            for xx in range(max(0, x - 1), min(self.W, x + 2)):
                                w = yy * self.W + xx
                                A[3 * w:3 * w + 3, 3 * v + c] = col[3 * w:3 * w + 3]
        self.blocks = []
        for p in self.own:
            x0, y0, x1, y1 = free_rect(self.P, p)
            verts = [y * self.W + x for y in range(y0, y1) for x in range(x0, x1)]
            idx = np.array([3 * v + c for v in verts for c in range(3)])
            self.blocks.append((idx, np.linalg.inv(A[np.ix_(idx, idx)])))

    def _asm_partial(self):
        z = np.zeros(3 * self.N)
        for idx, Ainv in self.blocks:
            z[idx] += Ainv @ self.r[idx]
        self.z[:] = z

    def begin(self, nc, tol, max_iters, warm):
        import torch
        self._factor()
        if not warm:
            self.x[:] = 0.0
        self.tol = tol
        ax, self.b = self._apply(self.x)
        self.r = self.b - ax
        self.normb = np.sqrt(self.b @ self.b)
        self.res = np.sqrt(self.r @ self.r) / self.normb
        self.done = self.res <= tol
        self.k = 0
        self.iters = 0
        self.z = np.zeros(3 * self.N)
        self.zt = torch.from_numpy(self.z)
        self.p = np.zeros(3 * self.N)
        if not self.done:
            self._asm_partial()

    def z_buffer(self):
        return self.zt

    def stage(self, s):
        if self.done:
            return
        if s == 1:
            rz = self.r @ self.z
            self.rz_old, self.rz = getattr(self, "rz", 0.0), rz
            self.k += 1
            return
        beta = 0.0 if self.k == 1 else self.rz / self.rz_old
        self.p = self.z + beta * self.p
        q = self._apply(self.p)[0]
        alpha = self.rz / (self.p @ q)
        self.x += alpha * self.p
        self.r -= alpha * q
        self.res = np.sqrt(self.r @ self.r) / self.normb
        self.iters = self.k
        if self.res <= self.tol:
            self.done = True
            return
        self._asm_partial()

    def status(self):
        return self.done, self.iters, self.res, False

    def end(self):
        if hasattr(self, "rz"):
            del self.rz
        return self.x.reshape(self.N, 3).T.reshape(3, self.H, self.W).copy(), self.iters, self.res

    def adapt(self, nc, kappa, thr, alpha_th):
        u3 = self.x.reshape(self.N, 3).T.reshape(3, self.H, self.W)
        eta, em = self.port.error_indicator(self.t10, self.alpha, self.lam, u3, nc)
        self.alpha = self.port.update_alpha(self.alpha, self.lam, eta, em, kappa, thr, alpha_th)
        return em

    def reg(self):
        return ff.RegField(self.alpha.copy(), self.lam.copy())


def _frames():
    rng = np.random.default_rng(5)
    yy, xx = np.mgrid[0:20, 0:24].astype(float)
    f0 = 120 + 60 * np.sin(xx / 3.0 + 0.5 * yy / 2.0) + rng.normal(0, 4, xx.shape)
    f1 = 120 + 60 * np.sin((xx - 0.7) / 3.0 + 0.5 * (yy - 0.3) / 2.0) + rng.normal(0, 4, xx.shape)
    return f0, f1


CFG = dict(sigma=1.0, parts=4, overlap=2, adapt_iters=2, cg_tolerance=1e-11)


def _worker(rank, world, port_path, out_dir, master_port):
    import torch.distributed as dist
    import sys
    sys.path.insert(0, os.path.dirname(port_path))
    import pyoracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(master_port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    f0, f1 = _frames()
    pyoracle.PORT.set_threads(1)
    be = EmuBackend(pyoracle.PORT, rank, world)
    res = par.sharded_run_on_frames(be, f0, f1, ff.RunConfig(**CFG), par.torch_allreduce())
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), u3=res.flow.planes(), alpha=res.reg.alpha,
             iters=np.array(res.iters))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2])
def test_sharded_driver_gloo(port, world):
    import torch.multiprocessing as mp
    import pyoracle
    out = tempfile.mkdtemp()
    mp.start_processes(_worker, args=(world, os.path.abspath(pyoracle.__file__), out, _free_port()),
                       nprocs=world, start_method="spawn", join=True)
    f0, f1 = _frames()
    o = port.converged_chain(f0, f1, CFG["sigma"], n_passes=CFG["adapt_iters"], tol=1e-13)
    results = [np.load(os.path.join(out, f"r{r}.npz")) for r in range(world)]
    for r in results:  # every rank ends with the same replicated solution
        assert np.array_equal(r["u3"], results[0]["u3"])
    for c in range(3):
        assert rel_l2(results[0]["u3"][c], o["u3"][c]) < 1e-8
    assert rel_l2(results[0]["alpha"], o["alpha"]) < 1e-7
    assert all(it > 0 for it in results[0]["iters"])
