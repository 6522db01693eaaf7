"""Multi-GPU run_on_frames: the Schwarz subdomains are sharded over the ranks of one node
(one process per GPU, torch.distributed for the plumbing).

Rank r factors and solves only subdomains [lo, hi) (ffb_shard_range: contiguous blocks in
partition order), so the band-factor memory and the two dominant kernels (factorisation,
subdomain solves) split across GPUs. The CG vectors are replicated: every rank applies the
operator and updates x, r, p on the whole image, and the CG scalars are computed identically
everywhere from identical vectors, so they need no collective. The one exchange per
iteration is the additive-Schwarz sum z = sum_i R_i^T A_i^-1 R_i r, whose per-rank partial
sums are all-reduced between the two device stages of an iteration.

The driver is written against a small backend interface so that the same host logic runs on
B200s (``DeviceBackend``, the C-ABI) and, for the multi-process CPU tests, on an emulation
backend (tests/test_parallel.py).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Callable, List

import numpy as np

from . import _lib
from .flowfem import (Context, FlowfemError, FlowState, RegField, RunConfig, _check, _f64, _p,
                      choose_split, uniform_reg)


def shard_range(n_parts: int, rank: int, world: int):
    """Subdomains [lo, hi) owned by ``rank`` (same rule as the library's ffb_shard_range)."""
    if world < 1 or not 0 <= rank < world:
        raise FlowfemError("schwarz: invalid shard rank/world")
    return rank * n_parts // world, (rank + 1) * n_parts // world


class DeviceBackend:
    """The B200 path of one rank (C-ABI staged solve)."""

    def __init__(self, ctx: Context, rank: int, world: int):
        self.ctx, self.rank, self.world = ctx, rank, world
        self.lib = ctx.lib
        _check(self.lib.ffb_set_shard(ctx.handle, rank, world))
        self._z = None

    # -- problem setup (replicated on every rank)
    def setup(self, f0, f1, cfg: RunConfig):
        f0, f1 = _f64(f0), _f64(f1)
        H, W = f0.shape
        self.shape = (H, W)
        _check(self.lib.ffb_set_frames(self.ctx.handle, W, H, _p(f0), _p(f1), float(cfg.sigma),
                                       float(cfg.rho)))
        reg = uniform_reg(W, H, cfg.alpha0, cfg.lambda0)
        _check(self.lib.ffb_set_reg(self.ctx.handle, _p(reg.alpha), _p(reg.lambda_)))
        sp = choose_split(W, H, cfg.parts)
        _check(self.lib.ffb_set_partition(self.ctx.handle, sp.parts_x, sp.parts_y, cfg.overlap))
        return sp

    # -- staged CG
    def begin(self, nc, tol, max_iters, warm):
        _check(self.lib.ffb_pcg_begin(self.ctx.handle, nc, float(tol), int(max_iters), int(warm),
                                      None))

    def stage(self, s):
        _check(self.lib.ffb_pcg_stage(self.ctx.handle, int(s)))

    def status(self):
        d, it, err = C.c_int(), C.c_int(), C.c_int()
        res = C.c_double()
        _check(self.lib.ffb_pcg_status(self.ctx.handle, C.byref(d), C.byref(it), C.byref(res),
                                       C.byref(err)))
        return bool(d.value), it.value, res.value, bool(err.value)

    def end(self):
        it, res = C.c_int(), C.c_double()
        H, W = self.shape
        u3 = np.zeros((3, H, W))
        _check(self.lib.ffb_pcg_end(self.ctx.handle, _p(u3), C.byref(it), C.byref(res)))
        return u3, it.value, res.value

    def z_buffer(self, which: int = 0):
        """torch CUDA view (zero copy) of the device z vector, the operand of the collective
        (which = 1..4: r, x and the two p buffers, for diagnostics)."""
        import torch
        ptr, n = C.c_void_p(), C.c_longlong()
        _check(self.lib.ffb_device_buffer(self.ctx.handle, which, C.byref(ptr), C.byref(n)))

        class _Arr:  # __cuda_array_interface__ shim
            __cuda_array_interface__ = {"shape": (n.value,), "typestr": "<f8",
                                        "data": (ptr.value, False), "version": 3}

        return torch.as_tensor(_Arr(), device=f"cuda:{self.ctx.device}")

    def adapt(self, nc, kappa, thr, alpha_th):
        em = C.c_double()
        _check(self.lib.ffb_adapt(self.ctx.handle, nc, float(kappa), float(thr), float(alpha_th),
                                  C.byref(em)))
        return em.value

    def reg(self):
        H, W = self.shape
        nt = 2 * (W - 1) * (H - 1)
        a, l = np.zeros(nt), np.zeros(nt)
        _check(self.lib.ffb_get_reg(self.ctx.handle, _p(a), _p(l)))
        return RegField(a, l)


@dataclass
class ShardedResult:
    flow: FlowState
    reg: RegField
    iters: List[int]
    residual: List[float]
    eta_max: List[float]


def sharded_solve(backend, nc: int, tol: float, max_iters: int, warm: bool,
                  allreduce: Callable, chunk: int = 8):
    """One Schwarz-preconditioned CG solve with the subdomains sharded over the ranks.

    allreduce(buf) sums ``backend.z_buffer()`` over the ranks in place (same stream)."""
    z = None
    backend.begin(nc, tol, max_iters, warm)
    z = backend.z_buffer()
    allreduce(z)
    backend.stage(1)
    while True:
        for _ in range(chunk):
            backend.stage(0)
            allreduce(z)
            backend.stage(1)
        done, it, res, err = backend.status()
        if done or err:
            break
    return backend.end()


def sharded_run_on_frames(backend, f0, f1, cfg: RunConfig, allreduce: Callable) -> ShardedResult:
    """run_on_frames (pipeline.cpp:38-78) under the converged-pass protocol, sharded."""
    backend.setup(f0, f1, cfg)
    nc = 3 if cfg.illumination else 2
    n_passes = cfg.adapt_iters if cfg.adapt else 0
    alpha_th = cfg.alpha_th if cfg.alpha_th is not None else cfg.alpha0 / 100.0
    iters, resid, etas = [], [], []
    u3 = None
    for p in range(n_passes + 1):
        u3, it, res = sharded_solve(backend, nc, cfg.cg_tolerance, cfg.max_iters, p > 0, allreduce)
        iters.append(it)
        resid.append(res)
        if p < n_passes:
            etas.append(backend.adapt(nc, cfg.kappa, cfg.eta_threshold, alpha_th))
    return ShardedResult(FlowState.from_planes(u3), backend.reg(), iters, resid, etas)


def torch_allreduce(group=None):
    """all-reduce(sum) over the default process group, on the current CUDA stream."""
    import torch.distributed as dist

    def f(t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return f


def run_distributed(f0, f1, cfg: RunConfig) -> ShardedResult:
    """Entry point under torchrun: one rank per GPU (RANK/WORLD_SIZE/LOCAL_RANK)."""
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = Context(local)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    backend = DeviceBackend(ctx, rank, world)
    reduce = torch_allreduce() if world > 1 else (lambda t: None)
    return sharded_run_on_frames(backend, f0, f1, cfg, reduce)
