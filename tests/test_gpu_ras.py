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


@pytest.mark.parametrize("H,W,px,py,ov,adapt,nc", [(40, 44, 2, 2, 3, True, 3), (36, 50, 3, 2, 2, False, 3),
                                                   (32, 40, 2, 2, 3, True, 2)])
def test_cg_subdomain_mode_matches_reference_bitwise(ctx, port, ref, H, W, px, py, ov, adapt, nc):
    """SolveMethod::ConjugateGradient subdomain solves (schwarz.cpp:248-252, picked by
    pick_method for c2-c5, pipeline.cpp:16-28): the reference's Jacobi-PCG per subdomain,
    warm-started from the previous iteration. Same unknown order, det_dot chunking and CSR
    row order as the reference, so field, increments, alpha and eta_max are bitwise equal."""
    import pyoracle
    f0, f1 = pair(H, W, 7 * H + W)
    t = port.frames_to_terms(f0, f1, 1.0, 2.5)
    nt = 2 * (W - 1) * (H - 1)
    alpha, lam = np.full(nt, 1000.0), np.full(nt, 1000.0)
    n_iters, n_adapt, tol = 7, 3, 1e-10
    r = pyoracle.ref_schwarz_solve(t, alpha, lam, px, py, ov, n_iters, workers=1, nc=nc,
                                   adapt=adapt, n_adapt=n_adapt, method=0, cg_tol=tol)
    reg = ff.RegField(alpha.copy(), lam.copy())
    opt = ff.SchwarzOptions(n_iters=n_iters, components=nc,
                            adapt=ff.AdaptConfig(enabled=adapt, n_adapt=n_adapt, alpha_th=10.0),
                            solver=ff.SolverConfig(method=ff.SolveMethod.ConjugateGradient,
                                                   cg_tolerance=tol))
    u, st = ff.schwarz_solve(ff.DataTerms(t), reg, px, py, ov, opt, ctx)
    np.testing.assert_array_equal(u.planes()[:nc], r["u3"][:nc])
    np.testing.assert_array_equal(np.array(st.increments), r["increments"])
    if adapt:
        np.testing.assert_array_equal(reg.alpha, r["alpha"])
        np.testing.assert_array_equal(st.eta_max, r["eta_max"])


def test_schwarz_stats_seconds_and_alpha_history(ctx, port):
    """SchwarzStats (schwarz.hpp:68-73): one wall time per iteration, one alpha snapshot per
    update when record_alpha_history is set (schwarz.cpp:303-316)."""
    f0, f1 = pair(36, 40, 5)
    t = port.frames_to_terms(f0, f1, 1.0, 2.5)
    reg = ff.uniform_reg(40, 36, 1000.0, 1000.0)
    opt = ff.SchwarzOptions(n_iters=5, adapt=ff.AdaptConfig(enabled=True, n_adapt=3, alpha_th=10.0),
                            record_alpha_history=True)
    _, st = ff.schwarz_solve(ff.DataTerms(t), reg, 2, 2, 3, opt, ctx)
    assert len(st.seconds) == 5 and all(s > 0 for s in st.seconds)
    assert len(st.eta_max) == 3 and len(st.alpha_history) == 3
    np.testing.assert_array_equal(st.alpha_history[-1], reg.alpha)
    assert (st.alpha_history[0] >= st.alpha_history[1]).all()  # alpha never grows
    assert not np.array_equal(st.alpha_history[0], st.alpha_history[1])


def test_literal_loop_c1_cholesky(ctx, port, ref):
    """SURVEY §8f-1 on config c1 itself: the reference's schwarz_solve with the Cholesky
    subdomain solver (pick_method's choice for c1: ext 68x68x3 = 13872 <= 20000 unknowns,
    pipeline.cpp:14-28), 10 iterations with 3 interleaved alpha updates, increments
    included."""
    import pyoracle
    from paper_1508_02977_b200 import synth
    f0, f1, _, cfg = synth.make("c1")
    t = port.frames_to_terms(f0, f1, cfg.sigma, cfg.rho)
    nt = 2 * (cfg.W - 1) * (cfg.H - 1)
    alpha, lam = np.full(nt, cfg.alpha0), np.full(nt, cfg.lambda0)
    r = pyoracle.ref_schwarz_solve(t, alpha, lam, 2, 2, cfg.overlap, 10, workers=4, nc=3,
                                   adapt=True, n_adapt=cfg.n_passes, alpha_th=cfg.alpha0 / 100,
                                   method=1)
    reg = ff.RegField(alpha.copy(), lam.copy())
    opt = ff.SchwarzOptions(n_iters=10, adapt=ff.AdaptConfig(enabled=True, n_adapt=cfg.n_passes,
                                                             alpha_th=cfg.alpha0 / 100))
    u, st = ff.schwarz_solve(ff.DataTerms(t), reg, 2, 2, cfg.overlap, opt, ctx)
    for c in range(3):
        assert rel_l2(u.planes()[c], r["u3"][c]) < 1e-9, c
    inc = np.array(st.increments)
    np.testing.assert_allclose(inc, r["increments"], rtol=1e-6, atol=1e-9 * inc.max())
    assert rel_l2(reg.alpha, r["alpha"]) < 1e-9
    np.testing.assert_allclose(st.eta_max, r["eta_max"], rtol=1e-8)


@pytest.mark.parametrize("nc", [2, 3])
def test_energy_matches_reference(ctx, port, ref, nc):
    """a25: energy (assembly.cpp:201-238) as a device reduction, against the reference and the
    bitwise-pinned port (summation order differs: 1e-13 relative)."""
    rng = np.random.default_rng(11 + nc)
    H, W = 41, 57
    f0, f1 = pair(H, W, nc)
    t = port.frames_to_terms(f0, f1, 1.0, 2.5)
    nt = 2 * (W - 1) * (H - 1)
    reg = ff.RegField(rng.uniform(10, 1000, nt), rng.uniform(10, 1000, nt))
    u3 = rng.normal(0, 2, (3, H, W))
    e_dev = ff.energy(ff.DataTerms(t), reg, ff.FlowState.from_planes(u3), nc, ctx)
    e_ref = ref.energy(t, reg.alpha, reg.lambda_, u3, nc)
    assert e_ref == port.energy(t, reg.alpha, reg.lambda_, u3, nc)
    assert abs(e_dev - e_ref) <= 1e-13 * abs(e_ref)


def test_energy_gradient_is_residual(ctx, port):
    """Acceptance C2 (acceptance.cpp:145-181) / test_assembly.cpp:100-133: the central
    finite-difference gradient of the device energy equals A x - b of the device operator."""
    rng = np.random.default_rng(5)
    H, W = 10, 10
    f0, f1 = rng.uniform(0, 1, (H, W)), rng.uniform(0, 1, (H, W))
    t = port.frames_to_terms(f0, f1, 1.0, 1.5)
    nt = 2 * (W - 1) * (H - 1)
    reg = ff.RegField(np.full(nt, 0.7), np.full(nt, 1.3))
    x3 = rng.uniform(-1, 1, (3, H, W))
    dt = ff.DataTerms(t)
    y3, b3 = ff.assemble_apply(dt, reg, 3, ff.FlowState.from_planes(x3), ctx)
    grad = (y3.planes() - b3.planes()).ravel()
    h = 1e-6
    fd = np.zeros_like(grad)
    xf = x3.ravel()
    for i in range(xf.size):
        keep = xf[i]
        xf[i] = keep + h
        ep = ff.energy(dt, reg, ff.FlowState.from_planes(xf.reshape(3, H, W)), 3, ctx)
        xf[i] = keep - h
        em = ff.energy(dt, reg, ff.FlowState.from_planes(xf.reshape(3, H, W)), 3, ctx)
        xf[i] = keep
        fd[i] = (ep - em) / (2 * h)
    assert np.linalg.norm(fd - grad) / np.linalg.norm(grad) <= 1e-5
