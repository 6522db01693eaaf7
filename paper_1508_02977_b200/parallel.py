"""Multi-GPU run_on_frames: one rank per GPU, the exchange inside the library.

Rank r of `world` owns a band of subdomain rows (and the pixel rows of their cores); the
library factors and solves only that band's subdomains, runs the CG kernels on its rows, and
exchanges with the neighbouring ranks — over NCCL P2P (ncclSend/ncclRecv on NVLink) for the
overlap halos, ncclAllReduce for the CG reduction units — so a whole multi-pass solve is ONE
C-ABI call per rank (ffb_run_on_frames_dev). The reductions are organised per subdomain row
and summed in a fixed order: iterates and results are bitwise identical for any world size at
equal subdomain-solve cluster size (each rank sizes its clusters from its own subdomains).

This module only wires the communicator:
  * ``init_nccl(ctx, rank, world)`` under torch.distributed (rank 0 makes the NCCL unique id,
    torch broadcasts it);
  * ``LocalHub`` / ``run_local`` — N contexts on N host threads (possibly on one device) with
    the in-process communicator: the same protocol for tests on a single GPU.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from typing import List, Optional

import numpy as np

from . import _lib
from .flowfem import Context, FlowfemError, RunConfig, RunResult, _check, run_on_frames


def rank_rows(width: int, height: int, parts_x: int, parts_y: int, overlap: int, rank: int,
              world: int) -> dict:
    """Row geometry of `rank` (ffb_comm_rows, host-only): owned pixel rows y0..y1, subdomain
    rows j0..j1, rows its subdomains cover above (fa) / below (fb), its rows covered by the
    rank above (ra) / below (rb); every range half-open."""
    out = np.zeros(12, dtype=np.int32)
    _check(_lib.load().ffb_comm_rows(width, height, parts_x, parts_y, overlap, rank, world,
                                     out.ctypes.data))
    k = ("y0", "y1", "j0", "j1", "fa0", "fa1", "fb0", "fb1", "ra0", "ra1", "rb0", "rb1")
    return dict(zip(k, (int(v) for v in out)))


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(_lib.load().ffb_comm_nccl_id(buf))
    return bytes(buf)


def init_nccl(ctx: Context, rank: int, world: int, group=None) -> None:
    """NCCL communicator of the library for this rank (torch.distributed shares the id)."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    buf = (C.c_ubyte * 128).from_buffer_copy(obj[0])
    _check(ctx.lib.ffb_comm_init_nccl(ctx.handle, rank, world, buf))


class LocalHub:
    """In-process communicator shared by `world` contexts (ffb_comm_local_hub)."""

    def __init__(self, world: int):
        self.lib = _lib.load()
        h = C.c_void_p()
        _check(self.lib.ffb_comm_local_hub(world, C.byref(h)))
        self._h = h
        self.world = world

    def attach(self, ctx: Context, rank: int) -> None:
        _check(ctx.lib.ffb_comm_init_local(ctx.handle, self._h, rank))

    def close(self):
        if self._h:
            self.lib.ffb_comm_local_hub_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def comm_info(ctx: Context):
    rank, world = C.c_int(), C.c_int()
    _check(ctx.lib.ffb_comm_info(ctx.handle, C.byref(rank), C.byref(world), None))
    return rank.value, world.value


def run_local(f0, f1, cfg: RunConfig, world: int, devices: Optional[List[int]] = None
              ) -> List[RunResult]:
    """run_on_frames on `world` contexts driven by `world` host threads over the in-process
    communicator (devices default to [0] * world: every rank on GPU 0). Returns the per-rank
    results (each rank holds the whole solution)."""
    devices = devices or [0] * world
    ctxs = [Context(d) for d in devices]
    hub = LocalHub(world)
    for r, c in enumerate(ctxs):
        hub.attach(c, r)
    out: List[Optional[RunResult]] = [None] * world
    err: List[Optional[BaseException]] = [None] * world

    def work(r):
        try:
            out[r] = run_on_frames(f0, f1, cfg, ctxs[r])
        except BaseException as e:  # noqa: BLE001 - surfaced below
            err[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise FlowfemError(f"rank failed: {e}") from e
    for c in ctxs:
        c.close()
    hub.close()
    return out  # type: ignore[return-value]


def run_distributed(f0, f1, cfg: RunConfig) -> RunResult:
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
    if world > 1:
        init_nccl(ctx, rank, world)
    return run_on_frames(f0, f1, cfg, ctx)
