"""Multi-GPU protocol of the library (paper_1508_02977_b200/parallel.py) on one
B200: `world` contexts driven by `world` host threads over the in-process communicator run
the same row-band protocol as NCCL ranks on separate GPUs — per CG iteration the residual
halo (overlap rows), the partial subdomain sums of z on the neighbours' rows, one row of z,
and the all-reduced reduction units. No kernel waits on another: the ranks meet at host
rendezvous between enqueued stages, so this is safe on one device.

The claim checked: the result (u, alpha, per-pass iteration counts, eta_max) is BITWISE
identical for world 1, 2, 3, 4, including ranks without subdomains (world > subdomain rows),
whenever the ranks run the subdomain solves with the same cluster size as one GPU (always for
the register-tiled solve of c1/c2; pinned with FFB_CLUSTER for the ring solve of c3), and
equal to the oracle's converged chain."""
import numpy as np
import pytest

from conftest import rel_l2
from paper_1508_02977_b200 import flowfem as ff
from paper_1508_02977_b200 import parallel as par
from paper_1508_02977_b200 import synth

pytestmark = pytest.mark.gpu


def run_world(f0, f1, cfg, world):
    if world == 1:
        return [ff.run_on_frames(f0, f1, cfg, ff.Context(0))]
    return par.run_local(f0, f1, cfg, world)


def same(a, b):
    np.testing.assert_array_equal(a.flow.planes(), b.flow.planes())
    np.testing.assert_array_equal(a.reg.alpha, b.reg.alpha)
    assert a.stats.iters == b.stats.iters
    np.testing.assert_array_equal(a.stats.eta_max, b.stats.eta_max)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_c2_bitwise_across_world_sizes(world):
    """c2 (388x584, 4x4 subdomains, overlap 2), 2 adaptive passes."""
    f0, f1, _, c = synth.make("c2")
    cfg = ff.RunConfig(sigma=c.sigma, parts=c.parts, overlap=c.overlap, adapt_iters=2,
                       cg_tolerance=1e-10)
    ref = run_world(f0, f1, cfg, 1)[0]
    res = run_world(f0, f1, cfg, world)
    for r in res:
        same(r, ref)


def test_empty_ranks_and_block_jacobi(port):
    """World larger than the subdomain rows (c1: 2 rows, world 3 -> one rank owns nothing)
    and overlap 1 (free rectangles = cores: no halo rows at all); against the oracle."""
    f0, f1, _, c = synth.make("c1")
    for ov, world in ((c.overlap, 3), (1, 2)):
        cfg = ff.RunConfig(sigma=c.sigma, parts=c.parts, overlap=ov, adapt_iters=1,
                           cg_tolerance=1e-11)
        ref = run_world(f0, f1, cfg, 1)[0]
        for r in run_world(f0, f1, cfg, world):
            same(r, ref)
    o = port.converged_chain(f0, f1, c.sigma, n_passes=1, tol=1e-13)
    for k in range(3):
        assert rel_l2(ref.flow.planes()[k], o["u3"][k]) < 1e-8


def test_c3_two_ranks_match_single(ctx, monkeypatch):
    """c3 at full size (1080x1920, 8x8, overlap 4), 1 adaptive pass, world 2 vs world 1.
    Each rank sizes its subdomain-solve clusters from its own subdomain count (c3: 1 CTA per
    chain on one GPU, 2-CTA clusters for the 32 subdomains of a rank), which changes the
    summation order inside the ring solve: the solutions then agree to the solve tolerance.
    With the cluster size pinned (FFB_CLUSTER=1) the ranks reproduce one GPU bit for bit."""
    f0, f1, _, c = synth.make("c3")
    cfg = ff.RunConfig(sigma=c.sigma, parts=c.parts, overlap=c.overlap, adapt_iters=1,
                       cg_tolerance=c.tol)
    ref = run_world(f0, f1, cfg, 1)[0]
    for r in run_world(f0, f1, cfg, 2):
        for k in range(3):
            assert rel_l2(r.flow.planes()[k], ref.flow.planes()[k]) < 1e-9
        assert abs(sum(r.stats.iters) - sum(ref.stats.iters)) <= 2
    monkeypatch.setenv("FFB_CLUSTER", "1")
    ref = run_world(f0, f1, cfg, 1)[0]
    for r in run_world(f0, f1, cfg, 2):
        same(r, ref)
