"""The reference's literal Schwarz loop on the device (ffb_schwarz_solve)
against the reference's own schwarz_solve (oracle/_ref, Cholesky subdomain solves) and the
known answers of test_schwarz.cpp:149-200."""
import numpy as np
import pytest

from conftest import rel_l2
from paper_1508_02977_b200 import flowfem as ff

pytestmark = pytest.mark.gpu


def pair(H, W, seed):
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:H, 0:W].astype(float)
    f0 = 120 + 60 * np.sin(xx / 4.0 + yy / 5.0) + 20 * np.cos(yy / 3.0) + rng.normal(0, 3, xx.shape)
    f1 = 120 + 60 * np.sin((xx - 1.2) / 4.0 + (yy - 0.4) / 5.0) + 20 * np.cos((yy - 0.4) / 3.0) \
        + rng.normal(0, 3, xx.shape)
    return f0, f1


def test_single_part_equals_monolithic(ctx, port):
    """test_schwarz.cpp:149-169: one part is the monolithic solve; increments after the first
    iteration are exactly zero."""
    f0, f1 = pair(30, 36, 1)
    t = port.frames_to_terms(f0, f1, 1.0, 2.5)
    reg = ff.uniform_reg(36, 30, 1000.0, 1000.0)
    opt = ff.SchwarzOptions(n_iters=3, adapt=ff.AdaptConfig(enabled=False))
    u, st = ff.schwarz_solve(ff.DataTerms(t), reg, 1, 1, 0, opt, ctx)
    assert st.increments[0] > 0 and st.increments[1] == 0.0 and st.increments[2] == 0.0
    ref_u, _, _ = port.cg_solve(t, reg.alpha, reg.lambda_, 3, 1e-13)
    for c in range(3):
        assert rel_l2(u.planes()[c], ref_u[c]) < 1e-10


def test_converges_to_monolithic(ctx, port):
    """test_schwarz.cpp:171-200 / acceptance C3: 2x2, overlap 5 converges to the monolithic
    solution."""
    f0, f1 = pair(40, 44, 2)
    t = port.frames_to_terms(f0, f1, 1.0, 2.5)
    reg = ff.uniform_reg(44, 40, 1000.0, 1000.0)
    u, st = ff.schwarz_solve(ff.DataTerms(t), reg, 2, 2, 5,
                             ff.SchwarzOptions(n_iters=60, adapt=ff.AdaptConfig(enabled=False)), ctx)
    ref_u, _, _ = port.cg_solve(t, reg.alpha, reg.lambda_, 3, 1e-13)
    for c in range(3):
        assert rel_l2(u.planes()[c], ref_u[c]) < 1e-6
    assert st.increments[-1] < st.increments[0] * 1e-4


@pytest.mark.parametrize("H,W,px,py,ov,adapt,nc", [(40, 44, 2, 2, 3, True, 3), (36, 50, 3, 2, 2, False, 3),
                                                   (32, 32, 2, 2, 3, True, 2)])
def test_matches_reference_schwarz_loop(ctx, port, ref, H, W, px, py, ov, adapt, nc):
    """The same loop as the reference's schwarz_solve (Cholesky + refinement per subdomain,
    interleaved alpha updates for the first n_adapt iterations): field, increments, alpha and
    eta_max agree to rounding."""
    import pyoracle
    f0, f1 = pair(H, W, H + W)
    t = port.frames_to_terms(f0, f1, 1.0, 2.5)
    nt = 2 * (W - 1) * (H - 1)
    alpha, lam = np.full(nt, 1000.0), np.full(nt, 1000.0)
    n_iters, n_adapt = 8, 3
    r = pyoracle.ref_schwarz_solve(t, alpha, lam, px, py, ov, n_iters, workers=1, nc=nc,
                                   adapt=adapt, n_adapt=n_adapt, method=1)
    reg = ff.RegField(alpha.copy(), lam.copy())
    opt = ff.SchwarzOptions(n_iters=n_iters, components=nc,
                            adapt=ff.AdaptConfig(enabled=adapt, n_adapt=n_adapt, alpha_th=10.0))
    u, st = ff.schwarz_solve(ff.DataTerms(t), reg, px, py, ov, opt, ctx)
    for c in range(nc):
        assert rel_l2(u.planes()[c], r["u3"][c]) < 1e-9, c
    inc = np.array(st.increments)
    np.testing.assert_allclose(inc, r["increments"], rtol=1e-6, atol=1e-9 * inc.max())
    if adapt:
        assert rel_l2(reg.alpha, r["alpha"]) < 1e-9
        np.testing.assert_allclose(st.eta_max, r["eta_max"], rtol=1e-8)
