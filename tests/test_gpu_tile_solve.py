"""The register-tiled subdomain solve (k_line_solve_tile, band.cu) against the shared-memory
ring kernel (k_line_solve) and the oracle CG, on line widths that exercise its edge cases:
a last tile row of full height (kd a multiple of 32), short last rows, one-tile lines, two
components, and every cluster size the placement tables cover (FFB_CLUSTER = 1, 2, 4, 8).
Both kernels apply the same block LDL^T preconditioner with different summation orders, so
the converged fields agree to the solve tolerance, and each equals the oracle's.
"""
import ctypes as C

import numpy as np
import pytest

from conftest import rel_l2
from paper_1508_02977_b200 import flowfem as ff

pytestmark = pytest.mark.gpu


def rand_pair(H, W, seed):
    rng = np.random.default_rng(seed)
    f0 = rng.uniform(0, 255, (H, W))
    f1 = np.clip(np.roll(f0, 1, axis=1) * 1.02 + rng.normal(0, 3, (H, W)), 0, 255)
    return f0, f1


def solve(t, a, l, px, py, ov, nc, factor_bits=64):
    ctx = ff.Context(0)
    try:
        ctx.set_factor_storage(factor_bits)
        s = ff.SchwarzSolver(ctx)
        s.set_terms(ff.DataTerms(t))
        s.set_reg(ff.RegField(a, l))
        s.set_partition(px, py, ov)
        u, it, res = s.solve(components=nc, tol=1e-12)
        fn = ctx.lib.ffb_debug_solve_kernel
        fn.restype, fn.argtypes = C.c_int, [C.c_void_p]
        return u.planes()[:nc], it, res, fn(ctx.handle)
    finally:
        ctx.close()


# (H, W, px, py, ov, nc, cluster): kd = nc * short side of the free rectangle
CASES = [
    (40, 32, 1, 1, 0, 3, None),   # kd 96: three full tile rows, C = 8
    (40, 32, 1, 1, 0, 3, "1"),    # one CTA: every block and tile local
    (40, 32, 1, 1, 0, 2, "2"),    # kd 64, two components
    (12, 9, 1, 1, 0, 3, None),    # kd 27: one diagonal tile, short
    (96, 80, 4, 4, 2, 3, None),   # 16 subdomains, C = 4
    (130, 160, 2, 2, 3, 3, None),  # kd ~ 200: seven tile rows, short last row, C = 8
    (130, 160, 2, 2, 3, 3, "2"),  # the same on 2-CTA clusters (28 tiles on 32 warps)
    (50, 44, 3, 2, 4, 2, "4"),    # two components on 4-CTA clusters
]


@pytest.mark.parametrize("H,W,px,py,ov,nc,cluster", CASES)
def test_tile_solve_matches_ring_and_oracle(monkeypatch, port, H, W, px, py, ov, nc, cluster):
    f0, f1 = rand_pair(H, W, 7 * H + W)
    t = port.frames_to_terms(f0, f1, 1.0, 2.5)
    rng = np.random.default_rng(H + W)
    ntri = 2 * (W - 1) * (H - 1)
    a = rng.uniform(20, 1000, ntri)
    l = np.full(ntri, 1000.0)
    if cluster:
        monkeypatch.setenv("FFB_CLUSTER", cluster)
    monkeypatch.delenv("FFB_SOLVE", raising=False)
    u_t, it_t, res_t, kind_t = solve(t, a, l, px, py, ov, nc)
    monkeypatch.setenv("FFB_SOLVE", "ring")
    u_r, it_r, res_r, kind_r = solve(t, a, l, px, py, ov, nc)
    assert kind_t == 1, "the register-tiled kernel was not selected"
    assert kind_r == 0
    assert res_t <= 1e-12 and res_r <= 1e-12
    assert abs(it_t - it_r) <= 2  # same preconditioner up to rounding
    ref_u, _, _ = port.cg_solve(t, a, l, nc, 1e-13)
    for c in range(nc):
        assert rel_l2(u_t[c], u_r[c]) < 1e-9, c
        assert rel_l2(u_t[c], ref_u[c]) < 1e-9, c


# k_line_solve_rt (row-group tiles; one CTA per chain or a cluster of 2 / 4 CTAs, each with its
# run of row groups): (H, W, px, py, ov, nc, FFB_SOLVE, FFB_CLUSTER)
RT_CASES = [
    (40, 32, 1, 1, 0, 3, "rt", "1"),    # kd 96: six 16-row groups, three diagonal tiles
    (12, 9, 1, 1, 0, 3, "rt", "1"),     # kd 27: one partial group, rows past the line
    (50, 44, 3, 2, 4, 2, "rt", "1"),    # two components, six subdomains
    (130, 160, 2, 2, 3, 3, None, "1"),  # kd ~200: the default choice at one CTA per chain
    (149, 160, 1, 1, 0, 3, None, "1"),  # kd 447: the widest line, odd, one group split over stages
    (40, 32, 1, 1, 0, 3, "rt", "2"),    # 2-CTA clusters: groups 0-3 / 4-5
    (12, 9, 1, 1, 0, 3, "rt", "4"),     # two groups on four CTAs: two CTAs only exchange zeros
    (50, 44, 3, 2, 4, 2, "rt", "4"),    # two components, 4-CTA clusters
    (130, 160, 2, 2, 3, 3, "rt", "2"),  # kd ~200 on 2-CTA clusters
    (149, 160, 1, 1, 0, 3, None, "2"),  # kd 447 on 2-CTA clusters: the default choice there
    (149, 160, 1, 1, 0, 3, None, "4"),  # and on 4
]


@pytest.mark.parametrize("H,W,px,py,ov,nc,force,cluster", RT_CASES)
def test_row_group_tiles_match_ring_and_oracle(monkeypatch, port, H, W, px, py, ov, nc, force,
                                               cluster):
    f0, f1 = rand_pair(H, W, 5 * H + W)
    t = port.frames_to_terms(f0, f1, 1.0, 2.5)
    rng = np.random.default_rng(H * W)
    ntri = 2 * (W - 1) * (H - 1)
    a = rng.uniform(20, 1000, ntri)
    l = np.full(ntri, 1000.0)
    monkeypatch.setenv("FFB_CLUSTER", cluster)
    if force:
        monkeypatch.setenv("FFB_SOLVE", force)
    else:
        monkeypatch.delenv("FFB_SOLVE", raising=False)
    u_t, it_t, res_t, kind_t = solve(t, a, l, px, py, ov, nc)
    monkeypatch.setenv("FFB_SOLVE", "ring")
    u_r, it_r, res_r, kind_r = solve(t, a, l, px, py, ov, nc)
    assert kind_t == 2, "the row-group tile kernel was not selected"
    assert kind_r == 0
    assert res_t <= 1e-12 and res_r <= 1e-12
    assert abs(it_t - it_r) <= 2
    ref_u, _, _ = port.cg_solve(t, a, l, nc, 1e-13)
    for c in range(nc):
        assert rel_l2(u_t[c], u_r[c]) < 1e-9, c
        assert rel_l2(u_t[c], ref_u[c]) < 1e-9, c


@pytest.mark.parametrize("H,W,px,py,ov,nc,cluster", [
    (149, 160, 1, 1, 0, 3, "1"),  # kd 447 (odd, line size 2 mod 4: the copy's padded stride)
    (139, 150, 1, 1, 0, 3, "1"),  # kd 417
    (130, 160, 2, 2, 3, 3, "1"),
    (149, 160, 1, 1, 0, 3, "2"),  # clusters
    (50, 44, 3, 2, 4, 2, "4"),
])
def test_row_group_tiles_f32_factor_copy(monkeypatch, port, H, W, px, py, ov, nc, cluster):
    """The opt-in single-precision factor copy (ffb_set_factor_storage 32) streamed by the
    row-group tile kernel: same converged solution as the double factors and the oracle."""
    f0, f1 = rand_pair(H, W, 11 * H + W)
    t = port.frames_to_terms(f0, f1, 1.0, 2.5)
    rng = np.random.default_rng(H * W + 1)
    ntri = 2 * (W - 1) * (H - 1)
    a = rng.uniform(20, 1000, ntri)
    l = np.full(ntri, 1000.0)
    monkeypatch.setenv("FFB_CLUSTER", cluster)
    monkeypatch.setenv("FFB_SOLVE", "rt")
    u_d, it_d, res_d, kind_d = solve(t, a, l, px, py, ov, nc)
    u_f, it_f, res_f, kind_f = solve(t, a, l, px, py, ov, nc, factor_bits=32)
    assert kind_d == 2 and kind_f == 2
    assert res_d <= 1e-12 and res_f <= 1e-12
    assert abs(it_d - it_f) <= 2
    ref_u, _, _ = port.cg_solve(t, a, l, nc, 1e-13)
    for c in range(nc):
        assert rel_l2(u_f[c], u_d[c]) < 1e-9, c
        assert rel_l2(u_f[c], ref_u[c]) < 1e-9, c
    assert not np.array_equal(u_f, u_d)  # the copy really was used


def test_tile_solve_deterministic(port):
    H, W = 96, 80
    f0, f1 = rand_pair(H, W, 3)
    t = port.frames_to_terms(f0, f1, 1.0, 2.5)
    ntri = 2 * (W - 1) * (H - 1)
    a, l = np.full(ntri, 300.0), np.full(ntri, 1000.0)
    u1, it1, _, k1 = solve(t, a, l, 4, 4, 2, 3)
    u2, it2, _, k2 = solve(t, a, l, 4, 4, 2, 3)
    assert k1 == k2 == 1 and it1 == it2
    assert np.array_equal(u1, u2)  # fixed-order reductions: bitwise run to run


def test_persistent_chain_queue_bitwise(ctx, monkeypatch):
    """The persistent ring solve (capi.cpp balance_chains: one CTA per SM pulls the forward
    and then the backward chains of every subdomain from a queue, a backward chain waiting for
    its subdomain's forward chains) computes exactly what the two launches per application do
    (FFB_NO_BALANCE=1): same chains, same arithmetic, only the schedule differs — bitwise equal,
    on a 16x16 partition with more chains than SMs (1600x900: 512 chains)."""
    import numpy as np
    rng = np.random.default_rng(3)
    H, W = 900, 1600
    yy, xx = np.mgrid[0:H, 0:W].astype(float)
    f0 = 120 + 50 * np.sin(xx / 9.0) * np.cos(yy / 7.0) + rng.normal(0, 3, (H, W))
    f1 = 120 + 50 * np.sin((xx - 0.8) / 9.0) * np.cos((yy - 0.5) / 7.0) + rng.normal(0, 3, (H, W))
    cfg = ff.RunConfig(sigma=1.5, parts=256, overlap=4, adapt_iters=1, cg_tolerance=1e-10)
    a = ff.run_on_frames(f0, f1, cfg, ff.Context(0))
    monkeypatch.setenv("FFB_NO_BALANCE", "1")
    b = ff.run_on_frames(f0, f1, cfg, ff.Context(0))
    np.testing.assert_array_equal(a.flow.planes(), b.flow.planes())
    assert a.stats.iters == b.stats.iters
    assert max(a.stats.residual) <= 1e-10
