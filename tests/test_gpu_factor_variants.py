"""The factor kernel's schedule variants (band.cu line_factor / sweep_invert) against the
default schedule and the oracle CG: factor clusters of 1, 2 and 8 CTAs (FFB_FCLUSTER — with
look-ahead the Z row blocks are split between CTA pairs, so 2 and 8 exercise the pair
grouping), no look-ahead (FFB_LOOKAHEAD=0), and FFMA instead of DMMA tile updates
(FFB_FACTOR_MMA=0). Every variant factors the same line matrices, so the converged fields
agree to the solve tolerance."""
import numpy as np
import pytest

from conftest import rel_l2
from paper_1508_02977_b200 import flowfem as ff

pytestmark = pytest.mark.gpu


def solve(t, a, l, px, py, ov, nc):
    ctx = ff.Context(0)
    try:
        s = ff.SchwarzSolver(ctx)
        s.set_terms(ff.DataTerms(t))
        s.set_reg(ff.RegField(a, l))
        s.set_partition(px, py, ov)
        u, it, res = s.solve(components=nc, tol=1e-12)
        return u.planes()[:nc], it, res
    finally:
        ctx.close()


VARIANTS = [
    {"FFB_FCLUSTER": "1"},
    {"FFB_FCLUSTER": "2"},
    {"FFB_FCLUSTER": "8"},
    {"FFB_LOOKAHEAD": "0"},
    {"FFB_FACTOR_MMA": "0"},
]


@pytest.mark.parametrize("H,W,px,py,ov,nc", [(130, 160, 2, 2, 3, 3), (96, 80, 4, 4, 2, 2)])
def test_factor_variants_agree(monkeypatch, port, H, W, px, py, ov, nc):
    rng = np.random.default_rng(H * W)
    f0 = rng.uniform(0, 255, (H, W))
    f1 = np.clip(np.roll(f0, 1, axis=0) * 0.98 + rng.normal(0, 3, (H, W)), 0, 255)
    t = port.frames_to_terms(f0, f1, 1.0, 2.5)
    ntri = 2 * (W - 1) * (H - 1)
    a = rng.uniform(20, 1000, ntri)
    l = np.full(ntri, 1000.0)
    for k in ("FFB_FCLUSTER", "FFB_LOOKAHEAD", "FFB_FACTOR_MMA"):
        monkeypatch.delenv(k, raising=False)
    u0, it0, res0 = solve(t, a, l, px, py, ov, nc)
    ref_u, _, _ = port.cg_solve(t, a, l, nc, 1e-13)
    for c in range(nc):
        assert rel_l2(u0[c], ref_u[c]) < 1e-9
    for v in VARIANTS:
        with monkeypatch.context() as m:
            for k, x in v.items():
                m.setenv(k, x)
            u, it, res = solve(t, a, l, px, py, ov, nc)
        assert res <= 1e-12, v
        assert abs(it - it0) <= 2, v
        for c in range(nc):
            assert rel_l2(u[c], u0[c]) < 1e-9, (v, c)
