"""Multi-GPU protocol on CPU: the row-band exchange sets of the library
(ffb_comm_rows, host-only) and a numpy emulation of the distributed Schwarz-PCG over gloo
with world_size 1 and 2.

The emulation (``EmuRank``; the operator from the oracle port, subdomain solves dense)
follows the device protocol of capi.cpp / pcg.cu step by step: a rank owns a band of
subdomain rows; every vector is valid only on the rows the protocol makes valid (all other
rows are NaN, so a missing or misplaced halo poisons the result); per iteration it exchanges
the residual on the rows its subdomains reach into, the partial subdomain sums of z on the
neighbours' rows, one row of z (for p), and all-reduces the per-subdomain-row reduction units.
Checks: the exchange sets pair up, every row is owned once, the 2-rank run equals the 1-rank
run bitwise and the oracle's converged chain to 1e-8.
"""
import os
import socket
import tempfile

import numpy as np
import pytest

from conftest import rel_l2
from paper_1508_02977_b200 import flowfem as ff
from paper_1508_02977_b200 import parallel as par


def test_rank_rows_consistent():
    """The exchange sets pair up between neighbouring ranks; owned rows tile the image."""
    for (W, H, px, py, ov) in ((3840, 2160, 16, 16, 4), (1920, 1080, 8, 8, 4),
                               (584, 388, 4, 4, 2), (128, 128, 2, 2, 4), (1024, 1024, 4, 4, 1)):
        for world in (1, 2, 3, 4, 8):
            rows = [par.rank_rows(W, H, px, py, ov, r, world) for r in range(world)]
            assert rows[0]["y0"] == 0 and rows[-1]["y1"] == H
            assert [g["j1"] - g["j0"] for g in rows] == [
                (r + 1) * py // world - r * py // world for r in range(world)]
            for a, b in zip(rows, rows[1:]):
                assert a["y1"] == b["y0"]
            live = [g for g in rows if g["j1"] > g["j0"]]
            for a, b in zip(live, live[1:]):
                assert (a["fb0"], a["fb1"]) == (b["ra0"], b["ra1"])  # my partial z -> its rows
                assert (a["rb0"], a["rb1"]) == (b["fa0"], b["fa1"])  # my r rows -> its halo
                assert a["fb1"] - a["fb0"] == max(ov - 1, 0)


def free_rect(P, p):
    e = P.parts[p].ext
    return (e.x0 + (e.x0 > 0), e.y0 + (e.y0 > 0), e.x1 - (e.x1 < P.width), e.y1 - (e.y1 < P.height))


class EmuRank:
    """numpy emulation of one rank of the row-band protocol (test infrastructure)."""

    def __init__(self, port, rank, world, dist):
        self.port, self.rank, self.world, self.dist = port, rank, world, dist

    def setup(self, f0, f1, cfg):
        H, W = f0.shape
        self.H, self.W, self.N = H, W, H * W
        self.t10 = self.port.frames_to_terms(f0, f1, cfg.sigma, cfg.rho)
        nt = 2 * (W - 1) * (H - 1)
        self.alpha = np.full(nt, cfg.alpha0)
        self.lam = np.full(nt, cfg.lambda0)
        sp = ff.choose_split(W, H, cfg.parts)
        self.px, self.py = sp.parts_x, sp.parts_y
        self.P = ff.build_partition(W, H, self.px, self.py, cfg.overlap)
        self.g = par.rank_rows(W, H, self.px, self.py, cfg.overlap, self.rank, self.world)
        live = [q for q in range(self.world)
                if par.rank_rows(W, H, self.px, self.py, cfg.overlap, q, self.world)["j1"] >
                par.rank_rows(W, H, self.px, self.py, cfg.overlap, q, self.world)["j0"]]
        me = self.g["j1"] > self.g["j0"]  # a rank without subdomains exchanges nothing
        self.up = max([q for q in live if q < self.rank], default=-1) if me else -1
        self.dn = min([q for q in live if q > self.rank], default=-1) if me else -1
        self.ys = np.array(self.P.ys if hasattr(self.P, "ys") else
                           [self.P.parts[j * self.px].core.y0 for j in range(self.py)] + [H])
        self.x = np.zeros((H, W, 3))

    # ---- rows helpers (vectors are (H, W, 3): row-major pixels, interleaved components)
    def nan_except(self, v, a, b):
        out = np.full_like(v, np.nan)
        out[a:b] = v[a:b]
        return out

    def exchange(self, v_send, rows_send, rows_recv, peer, v_recv):
        import torch
        import torch.distributed as dist
        if peer < 0:
            return
        s = torch.from_numpy(np.ascontiguousarray(v_send[rows_send[0]:rows_send[1]]))
        r = torch.empty((rows_recv[1] - rows_recv[0], self.W, 3), dtype=torch.float64)
        ops = [dist.P2POp(dist.isend, s, peer), dist.P2POp(dist.irecv, r, peer)]
        if s.numel() or r.numel():
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        v_recv[rows_recv[0]:rows_recv[1]] = r.numpy()

    def reduce(self, unit_vals):
        """unit values -> all-reduce (exact: each unit non-zero on one rank) -> j-order sum"""
        import torch
        import torch.distributed as dist
        t = torch.from_numpy(unit_vals.copy())
        if self.world > 1:
            dist.all_reduce(t)
        s = 0.0
        for v in t.numpy():
            s += v
        return s

    def units(self, a, b=None):
        u = np.zeros(self.py)
        for j in range(self.g["j0"], self.g["j1"]):
            sl = slice(self.ys[j], self.ys[j + 1])
            u[j] = float(np.sum(a[sl] * (a[sl] if b is None else b[sl])))
        return u

    # ---- operator and subdomains
    def apply(self, v):
        p3 = np.moveaxis(v, 2, 0)
        y3, b3 = self.port.assemble_apply(self.t10, self.alpha, self.lam, 3, np.ascontiguousarray(p3))
        return np.moveaxis(y3, 0, 2), np.moveaxis(b3, 0, 2)

    def factor(self):
        H, W = self.H, self.W
        n = 3 * self.N
        A = np.zeros((n, n))
        ys, xs = np.divmod(np.arange(self.N), W)
        for cy in range(3):
            for cx in range(3):
                verts = np.flatnonzero((xs % 3 == cx) & (ys % 3 == cy))
                for c in range(3):
                    e = np.zeros((H, W, 3))
                    e.reshape(-1, 3)[verts, c] = 1.0
                    col = self.apply(e)[0].ravel()
                    for v in verts:
                        x, y = xs[v], ys[v]
                        for yy in range(max(0, y - 1), min(H, y + 2)):
                            for xx in range(max(0, x - 1), min(W, x + 2)):
                                w = yy * W + xx
                                A[3 * w:3 * w + 3, 3 * v + c] = col[3 * w:3 * w + 3]
        self.blocks = {}
        for j in range(self.g["j0"], self.g["j1"]):
            for i in range(self.px):
                x0, y0, x1, y1 = free_rect(self.P, j * self.px + i)
                verts = [y * W + x for y in range(y0, y1) for x in range(x0, x1)]
                idx = np.array([3 * v + c for v in verts for c in range(3)])
                self.blocks[(j, i)] = (idx, np.linalg.inv(A[np.ix_(idx, idx)]))

    def row_sums(self, r):
        """S_j for this rank's subdomain rows: sum over the row's subdomains, ascending i"""
        S = {}
        for j in range(self.g["j0"], self.g["j1"]):
            s = np.zeros(3 * self.N)
            for i in range(self.px):
                idx, Ainv = self.blocks[(j, i)]
                s[idx] += Ainv @ r.ravel()[idx]
            S[j] = s.reshape(self.H, self.W, 3)
        return S

    def precondition(self, r):
        g = self.g
        # r halo: the rows my subdomains reach into, from the neighbours
        self.exchange(r, (g["ra0"], g["ra1"]), (g["fa0"], g["fa1"]), self.up, r)
        self.exchange(r, (g["rb0"], g["rb1"]), (g["fb0"], g["fb1"]), self.dn, r)
        S = self.row_sums(r)
        # partial sums on the neighbours' rows
        recv_up = np.full((self.H, self.W, 3), np.nan)
        recv_dn = np.full((self.H, self.W, 3), np.nan)
        if g["j1"] > g["j0"]:
            self.exchange(S[g["j0"]], (g["fa0"], g["fa1"]), (g["ra0"], g["ra1"]), self.up, recv_up)
            self.exchange(S[g["j1"] - 1], (g["fb0"], g["fb1"]), (g["rb0"], g["rb1"]), self.dn, recv_dn)
        z = np.full((self.H, self.W, 3), np.nan)
        for y in range(g["y0"], g["y1"]):
            acc = None
            for j in range(self.py):  # the <= 2 subdomain rows covering y, ascending
                fr = free_rect(self.P, j * self.px)
                if not fr[1] <= y < fr[3]:
                    continue
                sj = S[j][y] if j in S else (recv_up[y] if j < g["j0"] else recv_dn[y])
                acc = sj.copy() if acc is None else acc + sj
            z[y] = acc
        rz = self.reduce(self.units(r, z))
        # one row of z each side
        self.exchange(z, (g["y0"], g["y0"] + 1), (g["y0"] - 1, g["y0"]), self.up, z)
        self.exchange(z, (g["y1"] - 1, g["y1"]), (g["y1"], g["y1"] + 1), self.dn, z)
        return z, rz

    def solve(self, tol, warm):
        g = self.g
        self.factor()
        if not warm:
            self.x[:] = 0.0
        ax, b = self.apply(self.x)
        r = self.nan_except(b - ax, g["y0"], g["y1"])
        normb = np.sqrt(self.reduce(self.units(b)))
        res = np.sqrt(self.reduce(self.units(r))) / normb
        it = 0
        p = np.full_like(r, np.nan)
        z, rz = self.precondition(r)
        k = 1
        rz_old = None
        while res > tol:
            beta = 0.0 if k == 1 else rz / rz_old
            lo, hi = max(g["y0"] - 1, 0), min(g["y1"] + 1, self.H)
            pn = np.full_like(p, np.nan)
            pn[lo:hi] = z[lo:hi] if k == 1 else z[lo:hi] + beta * p[lo:hi]
            p = pn
            q = self.nan_except(self.apply(p)[0], g["y0"], g["y1"])
            pap = self.reduce(self.units(p, q))
            alpha = rz / pap
            own = slice(g["y0"], g["y1"])
            self.x[own] += alpha * p[own]
            r[own] -= alpha * q[own]
            res = np.sqrt(self.reduce(self.units(r))) / normb
            it = k
            if res <= tol:
                break
            z, rz_new = self.precondition(r)
            rz_old, rz = rz, rz_new
            k += 1
        # all-gather x (owned rows of every rank)
        import torch
        import torch.distributed as dist
        if self.world > 1:
            t = torch.from_numpy(np.where(np.arange(self.H)[:, None, None] >= g["y0"],
                                          np.where(np.arange(self.H)[:, None, None] < g["y1"],
                                                   self.x, 0.0), 0.0))
            dist.all_reduce(t)
            self.x = t.numpy().copy()
        return it, res

    def adapt(self, kappa, thr, alpha_th):
        u3 = np.ascontiguousarray(np.moveaxis(self.x, 2, 0))
        eta, em = self.port.error_indicator(self.t10, self.alpha, self.lam, u3, 3)
        self.alpha = self.port.update_alpha(self.alpha, self.lam, eta, em, kappa, thr, alpha_th)
        return em


def _frames():
    rng = np.random.default_rng(5)
    yy, xx = np.mgrid[0:28, 0:24].astype(float)
    f0 = 120 + 60 * np.sin(xx / 3.0 + 0.5 * yy / 2.0) + rng.normal(0, 4, xx.shape)
    f1 = 120 + 60 * np.sin((xx - 0.7) / 3.0 + 0.5 * (yy - 0.3) / 2.0) + rng.normal(0, 4, xx.shape)
    return f0, f1


CFG = dict(sigma=1.0, parts=4, overlap=3, adapt_iters=2, cg_tolerance=1e-11)


def _worker(rank, world, port_path, out_dir, master_port):
    import sys
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(port_path))
    import pyoracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(master_port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    f0, f1 = _frames()
    pyoracle.PORT.set_threads(1)
    cfg = ff.RunConfig(**CFG)
    em = EmuRank(pyoracle.PORT, rank, world, dist)
    em.setup(f0, f1, cfg)
    iters = []
    for p in range(cfg.adapt_iters + 1):
        it, _ = em.solve(cfg.cg_tolerance, p > 0)
        iters.append(it)
        if p < cfg.adapt_iters:
            em.adapt(cfg.kappa, cfg.eta_threshold, cfg.alpha0 / 100.0)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), x=em.x, alpha=em.alpha, iters=np.array(iters))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def emu_runs():
    import torch.multiprocessing as mp
    import pyoracle
    out = {}
    for world in (1, 2):
        d = tempfile.mkdtemp()
        mp.start_processes(_worker, args=(world, os.path.abspath(pyoracle.__file__), d,
                                          _free_port()), nprocs=world, start_method="spawn",
                           join=True)
        out[world] = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(world)]
    return out


def test_row_band_protocol_gloo_bitwise(emu_runs):
    """world 2 over gloo == world 1, bitwise (x, alpha, iteration counts)."""
    one = emu_runs[1][0]
    for r in emu_runs[2]:
        np.testing.assert_array_equal(r["x"], one["x"])
        np.testing.assert_array_equal(r["alpha"], one["alpha"])
        np.testing.assert_array_equal(r["iters"], one["iters"])
        assert np.isfinite(r["x"]).all()


def test_row_band_protocol_matches_oracle(emu_runs, port):
    f0, f1 = _frames()
    o = port.converged_chain(f0, f1, CFG["sigma"], n_passes=CFG["adapt_iters"], tol=1e-13)
    x = emu_runs[2][0]["x"]
    for c in range(3):
        assert rel_l2(x[:, :, c], o["u3"][c]) < 1e-8
    assert rel_l2(emu_runs[2][0]["alpha"], o["alpha"]) < 1e-7
