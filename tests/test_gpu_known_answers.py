"""The reference's analytic known-answer and property tests of the imaging, indicator and
alpha-update stages, run through the C-ABI on the B200 (SURVEY §8c "port them as B200 tests").
Each case names the reference test it restates (paths under /root/reference/proj/tests); the
inputs are rebuilt here from the closed forms those tests describe, not from reference data.
The bitwise parity tests (test_gpu_parity.py) pin the same kernels against the oracle; these
pin them against mathematics.
"""
import numpy as np
import pytest

from paper_1508_02977_b200 import flowfem as ff

pytestmark = pytest.mark.gpu


def rand_image(H, W, seed):
    return np.random.default_rng(seed).uniform(0.0, 1.0, (H, W))


def gauss_taps(sigma):
    """imaging.cpp:19-29: exp(-k^2 / 2 sigma^2) on [-ceil(3 sigma), ceil(3 sigma)], renormalised."""
    r = int(np.ceil(3.0 * sigma))
    k = np.arange(-r, r + 1)
    t = np.exp(-(k * k) / (2.0 * sigma * sigma))
    return t / t.sum(), r


def fold(i, n):
    """imaging.cpp:11-17: symmetric reflection -1-i / 2n-1-i, repeated until inside."""
    while i < 0 or i >= n:
        i = -1 - i if i < 0 else 2 * n - 1 - i
    return i


def smooth_direct(img, sigma):
    """Dense 2-D convolution with the outer product of the taps (the reference's
    ref::gaussian_smooth_direct, restated)."""
    t, r = gauss_taps(sigma)
    H, W = img.shape
    out = np.zeros_like(img)
    for y in range(H):
        for x in range(W):
            s = 0.0
            for dy in range(-r, r + 1):
                yy = fold(y + dy, H)
                for dx in range(-r, r + 1):
                    s += t[dy + r] * t[dx + r] * img[yy, fold(x + dx, W)]
            out[y, x] = s
    return out


# ------------------------------------------------------------------ test_imaging.cpp
def test_sigma_zero_is_a_bitwise_copy(ctx):
    # test_imaging.cpp:25-29
    img = rand_image(9, 13, 7)
    assert np.array_equal(ff.gaussian_smooth(img, 0.0, ctx), img)


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_smoothing_preserves_the_mean(ctx, seed):
    # test_imaging.cpp:31-39 (symmetric reflection + renormalised taps)
    img = rand_image(11, 17, seed)
    for sigma in (0.5, 1.0, 2.5):
        assert abs(ff.gaussian_smooth(img, sigma, ctx).mean() - img.mean()) <= 1e-10


def test_constant_stays_constant_and_range_shrinks(ctx):
    # test_imaging.cpp:41-53
    out = ff.gaussian_smooth(np.full((12, 12), 0.37), 1.7, ctx)
    assert np.allclose(out, 0.37, rtol=1e-13, atol=0)
    noisy = rand_image(20, 20, 11)
    sm = ff.gaussian_smooth(noisy, 2.0, ctx)
    assert sm.min() >= noisy.min() - 1e-12 and sm.max() <= noisy.max() + 1e-12


@pytest.mark.parametrize("seed,sigma", [(3, 0.8), (3, 1.9), (9, 0.8), (9, 1.9)])
def test_separable_smoothing_matches_dense_2d(ctx, seed, sigma):
    # test_imaging.cpp:55-64
    img = rand_image(14, 15, seed)
    assert np.max(np.abs(ff.gaussian_smooth(img, sigma, ctx) - smooth_direct(img, sigma))) < 1e-13


def test_derivatives_exact_on_affine_frames(ctx):
    # test_imaging.cpp:76-94
    H, W = 8, 11
    a, b, c, d = 0.2, 0.03, -0.015, 0.05
    y, x = np.mgrid[0:H, 0:W]
    f0 = a + b * x + c * y
    f1 = f0 + d
    der = ff.compute_derivatives(f0, f1, ctx)
    assert np.allclose(der.fx, b, rtol=1e-12, atol=0)
    assert np.allclose(der.fy, c, rtol=1e-12, atol=0)
    assert np.allclose(der.ft, d, rtol=1e-12, atol=0)
    assert np.array_equal(der.f, f0)


def test_derivatives_use_the_frame_average(ctx):
    # test_imaging.cpp:96-108: f0 flat, f1 a ramp of slope 0.1 -> fx is half the slope
    H, W = 6, 6
    x = np.mgrid[0:H, 0:W][1]
    der = ff.compute_derivatives(np.full((H, W), 0.5), 0.5 + 0.1 * x, ctx)
    assert np.allclose(der.fx, 0.05, rtol=1e-12, atol=0)


def test_data_terms_at_rho_zero_known_answer(ctx):
    # test_imaging.cpp:110-133: fx = 2, fy = 0, ft = 1, f = 3 on every pixel
    sh = (4, 4)
    d = ff.DerivativeField(np.full(sh, 2.0), np.zeros(sh), np.full(sh, 1.0), np.full(sh, 3.0))
    t = ff.build_data_terms(d, 0.0, ctx)
    want = dict(a11=4.0, a12=0.0, a13=-6.0, a22=0.0, a23=-0.0, a33=9.0, f1=-2.0, f2=-0.0, f3=3.0,
                c=1.0)
    for name, v in want.items():
        assert np.all(getattr(t, name) == v), name


def test_data_terms_with_rho_match_direct_smoothing_of_products(ctx):
    # test_imaging.cpp:135-151
    f0, f1 = rand_image(12, 14, 21), rand_image(12, 14, 22)
    d = ff.compute_derivatives(f0, f1, ctx)
    rho = 1.4
    t = ff.build_data_terms(d, rho, ctx)
    for name, prod in (("a11", d.fx * d.fx), ("a23", -d.fy * d.f), ("f3", d.f * d.ft),
                       ("c", d.ft * d.ft)):
        assert np.max(np.abs(getattr(t, name) - smooth_direct(prod, rho))) < 1e-13, name


def test_imaging_is_deterministic(ctx):
    # test_imaging.cpp:66-74 (worker counts there; repeated launches here)
    img = rand_image(21, 33, 5)
    assert np.array_equal(ff.gaussian_smooth(img, 1.3, ctx), ff.gaussian_smooth(img, 1.3, ctx))


# -------------------------------------------------------------------- test_adapt.cpp
def zero_terms(H, W):
    return ff.DataTerms(np.zeros((10, H, W)))


def test_zero_data_constant_state_gives_zero_indicator(ctx):
    # test_adapt.cpp:57-67
    H = W = 7
    st = ff.FlowState(np.full((H, W), 0.4), np.full((H, W), -1.3), np.full((H, W), 2.0))
    ind = ff.error_indicator(zero_terms(H, W), ff.uniform_reg(W, H, 100.0, 100.0), st, 3, ctx)
    assert ind.eta_max == 0.0
    assert np.all(ind.eta == 0.0)


def test_zero_data_linear_field_flags_only_boundary_triangles(ctx):
    # test_adapt.cpp:69-88: a globally linear field has a continuous constant flux, so only
    # the natural-condition mismatch on the outer edges survives. Cell (x, y): lower triangle
    # (v00, v10, v11) = 2 (y (W-1) + x), upper (v00, v11, v01) the next one (mesh.cpp:29).
    H, W = 6, 8
    y, x = np.mgrid[0:H, 0:W]
    st = ff.FlowState(0.5 + x + y, np.zeros((H, W)), np.zeros((H, W)))
    ind = ff.error_indicator(zero_terms(H, W), ff.uniform_reg(W, H, 50.0, 50.0), st, 3, ctx)
    assert ind.eta_max > 0.0
    eta = ind.eta.reshape(H - 1, W - 1, 2)
    for cy in range(H - 1):
        for cx in range(W - 1):
            lower_on_boundary = cy == 0 or cx == W - 2      # edges v00-v10 (bottom), v10-v11 (right)
            upper_on_boundary = cy == H - 2 or cx == 0      # edges v11-v01 (top), v01-v00 (left)
            assert (eta[cy, cx, 0] > 0.0) == lower_on_boundary, (cx, cy, "lower")
            assert (eta[cy, cx, 1] > 0.0) == upper_on_boundary, (cx, cy, "upper")


def test_alpha_update_threshold_floor_and_quiet_field(ctx):
    # test_adapt.cpp:90-120 with the reference's own numbers
    reg = ff.RegField(np.full(4, 1000.0), np.full(4, 1000.0))
    ind = ff.IndicatorField(np.array([1.0, 0.05, 0.1, 0.55]), 1.0)
    upd = ff.update_alpha(reg, ind, ff.AdaptConfig(kappa=10.0, eta_threshold=0.1, alpha_th=10.0), ctx)
    assert upd.alpha[0] == pytest.approx(100.0, rel=1e-14)          # 1000 / (1 + 10 * 0.9)
    assert upd.alpha[1] == 1000.0                                    # below the threshold
    assert upd.alpha[2] == 1000.0                                    # exactly at it: zero excess
    assert upd.alpha[3] == pytest.approx(1000.0 / 5.5, rel=1e-14)
    assert np.array_equal(upd.lambda_, reg.lambda_)
    floored = ff.update_alpha(reg, ind, ff.AdaptConfig(kappa=1e6, eta_threshold=0.1, alpha_th=10.0), ctx)
    assert floored.alpha[0] == 10.0
    quiet = ff.update_alpha(reg, ff.IndicatorField(np.zeros(4), 0.0),
                            ff.AdaptConfig(kappa=1e6, eta_threshold=0.1, alpha_th=10.0), ctx)
    assert np.array_equal(quiet.alpha, reg.alpha) and np.array_equal(quiet.lambda_, reg.lambda_)


def test_alpha_non_increasing_under_repeated_updates(ctx):
    # test_adapt.cpp:122-140
    H, W = 10, 12
    rng = np.random.default_rng(77)
    terms = ff.DataTerms(rng.uniform(-1.0, 1.0, (10, H, W)))
    st = ff.FlowState(*rng.uniform(-1.0, 1.0, (3, H, W)))
    reg = ff.uniform_reg(W, H, 500.0, 500.0)
    cfg = ff.AdaptConfig(alpha_th=5.0)
    for _ in range(4):
        ind = ff.error_indicator(terms, reg, st, 3, ctx)
        upd = ff.update_alpha(reg, ind, cfg, ctx)
        assert np.all(upd.alpha <= reg.alpha) and np.all(upd.alpha >= cfg.alpha_th)
        assert np.array_equal(upd.lambda_, reg.lambda_)
        reg = upd


def test_indicator_is_deterministic(ctx):
    # test_adapt.cpp:142-158 (thread counts there; repeated launches here)
    H, W = 13, 17
    rng = np.random.default_rng(5)
    terms = ff.DataTerms(rng.uniform(-1.0, 1.0, (10, H, W)))
    st = ff.FlowState(*rng.uniform(-1.0, 1.0, (3, H, W)))
    reg = ff.uniform_reg(W, H, 300.0, 900.0)
    reg.alpha += (np.arange(reg.alpha.size) % 11) * 40.0
    a = ff.error_indicator(terms, reg, st, 3, ctx)
    b = ff.error_indicator(terms, reg, st, 3, ctx)
    assert np.array_equal(a.eta, b.eta) and a.eta_max == b.eta_max


# ------------------------------------------------------------------ test_assembly.cpp
@pytest.mark.parametrize("nc", [3, 2])
def test_assembled_matrix_bitwise_symmetric_positive_diagonal(ctx, nc):
    # test_assembly.cpp:74-98, on the device CSR assembly (ffb_assemble_system)
    H, W = 9, 12
    terms = ff.frames_to_terms(255.0 * rand_image(H, W, 5), 255.0 * rand_image(H, W, 6), 1.0, 2.5, ctx)
    s = ff.assemble(terms, ff.uniform_reg(W, H, 1000.0, 1000.0), nc, ctx=ctx)
    assert s.n == nc * W * H
    entries = {}
    for r in range(s.n):
        cols = s.cols[s.row_ptr[r]:s.row_ptr[r + 1]]
        assert np.all(np.diff(cols) > 0)  # sorted columns (assembly.hpp:43-53)
        assert r in cols
        for q in range(s.row_ptr[r], s.row_ptr[r + 1]):
            entries[(r, int(s.cols[q]))] = s.vals[q]
            if s.cols[q] == r:
                assert s.vals[q] > 0.0
    for (r, c), v in entries.items():
        assert (c, r) in entries
        assert np.float64(v).tobytes() == np.float64(entries[(c, r)]).tobytes()


def test_dirichlet_rows_are_eliminated_into_the_rhs(ctx):
    # test_assembly.cpp:147-167 (constrained solve): fixing vertices removes their unknowns and
    # the constrained solution, expanded, satisfies the free rows of the unconstrained system
    H, W, nc = 7, 9, 3
    terms = ff.frames_to_terms(255.0 * rand_image(H, W, 8), 255.0 * rand_image(H, W, 9), 1.0, 2.5, ctx)
    reg = ff.uniform_reg(W, H, 200.0, 300.0)
    dv = np.array([0, 5, W * H - 1], dtype=np.int32)
    dvals = np.array([[0.3, -0.2, 0.1], [1.0, 0.5, -0.4], [-0.7, 0.0, 0.2]])
    full = ff.assemble(terms, reg, nc, ctx=ctx)
    con = ff.assemble(terms, reg, nc, dv, dvals, ctx=ctx)
    assert con.n == full.n - nc * len(dv)
    x = ff.solve(con, ff.SolverConfig(method=ff.SolveMethod.DirectCholesky), ctx=ctx)
    free = np.setdiff1d(np.arange(W * H), dv)
    xf = np.zeros((W * H, nc))
    xf[free] = np.asarray(x).reshape(-1, nc)
    xf[dv] = dvals
    r = ff.spmv(full, xf.ravel(), ctx) - full.rhs
    rfree = r.reshape(-1, nc)[free]
    assert np.max(np.abs(rfree)) <= 1e-8 * np.max(np.abs(full.rhs))


# ------------------------------------------------------------------ test_pipeline.cpp
def pattern_frame(H, W, sx=0.0, sy=0.0):
    """fixtures.hpp:23-33: a two-sinusoid texture clamped to [0, 1], shifted by (sx, sy)."""
    y, x = np.mgrid[0:H, 0:W].astype(float)
    x, y = x - sx, y - sy
    v = (0.45 + 0.25 * np.sin(2 * np.pi * x / 7.3 + 1.1) * np.cos(2 * np.pi * y / 9.7)
         + 0.15 * np.sin(2 * np.pi * (x + y) / 13.1))
    return np.clip(v, 0.0, 1.0)


def smooth_frame(H, W, sx, sy):
    """test_pipeline.cpp:24-35: long-wavelength texture bounded to [0.1, 0.7]."""
    y, x = np.mgrid[0:H, 0:W].astype(float)
    x, y = x - sx, y - sy
    return (0.4 + 0.2 * np.sin(2 * np.pi * x / 11.3 + 0.7) * np.cos(2 * np.pi * y / 14.7)
            + 0.1 * np.sin(2 * np.pi * (x + y) / 17.9))


def const_truth(H, W, tu, tv):
    return ff.FloField(np.full((H, W), tu, np.float32), np.full((H, W), tv, np.float32))


def small_config(**kw):
    # test_pipeline.cpp:37-47: [0, 1] frames, alpha0 = lambda0 = 0.05, 2x2 parts, overlap 5, no
    # adaptation (here the converged solve the reference's 15 Schwarz iterations approach)
    return ff.RunConfig(alpha0=0.05, lambda0=0.05, parts=4, overlap=5, adapt=False, adapt_iters=0,
                        **kw)


def test_plain_translation_is_recovered(ctx):
    # test_pipeline.cpp:55-67
    H = W = 48
    r = ff.run_on_frames(pattern_frame(H, W), pattern_frame(H, W, 1.0, 0.0), small_config(), ctx)
    m = ff.compute_metrics(r.flow, const_truth(H, W, 1.0, 0.0), ctx)
    assert m.valid == H * W
    assert m.ee < 0.3
    assert m.aae_deg < 8.0


def test_modelling_illumination_pays_off_under_a_gain(ctx):
    # test_pipeline.cpp:69-83 (acceptance criterion 7): brightness x1.2, shift (0.25, 0.1)
    H = W = 48
    f0 = smooth_frame(H, W, 0.0, 0.0)
    f1 = np.clip(1.2 * smooth_frame(H, W, 0.25, 0.1), 0.0, 1.0)
    truth = const_truth(H, W, 0.25, 0.1)
    on = ff.run_on_frames(f0, f1, ff.RunConfig(alpha0=0.05, lambda0=5.0, parts=4, overlap=5,
                                               adapt=False, adapt_iters=0, illumination=True), ctx)
    off = ff.run_on_frames(f0, f1, ff.RunConfig(alpha0=0.05, lambda0=5.0, parts=4, overlap=5,
                                                adapt=False, adapt_iters=0, illumination=False), ctx)
    ee_on = ff.compute_metrics(on.flow, truth, ctx).ee
    ee_off = ff.compute_metrics(off.flow, truth, ctx).ee
    assert ee_on < 0.6 * ee_off


# ------------------------------------------------------------------ test_linsolve.cpp
def dense_of(s):
    A = np.zeros((s.n, s.n))
    for r in range(s.n):
        A[r, s.cols[s.row_ptr[r]:s.row_ptr[r + 1]]] = s.vals[s.row_ptr[r]:s.row_ptr[r + 1]]
    return A


def test_refactorization_reuses_the_symbolic_pattern(ctx):
    # test_linsolve.cpp:135-158: analyze once, factorize twice with new values of one pattern
    H = W = 9
    terms = ff.frames_to_terms(255.0 * rand_image(H, W, 17), 255.0 * rand_image(H, W, 18), 1.0, 2.5, ctx)
    reg = ff.uniform_reg(W, H, 80.0, 60.0)
    s = ff.assemble(terms, reg, 3, ctx=ctx)
    chol = ff.SparseCholesky(ctx)
    chol.analyze(s)
    chol.factorize(s, 2)
    x0 = chol.solve(s.rhs)
    reg.alpha *= 0.25  # same pattern, new values
    s = ff.assemble(terms, reg, 3, ctx=ctx)
    chol.factorize(s, 2)
    x1 = chol.solve(s.rhs)
    fresh = ff.SparseCholesky(ctx)
    fresh.analyze(s)
    fresh.factorize(s, 1)
    assert np.array_equal(x1, fresh.solve(s.rhs))
    xd = np.linalg.solve(dense_of(s), s.rhs)
    assert np.linalg.norm(x1 - xd) / np.linalg.norm(xd) < 1e-10
    assert np.linalg.norm(x0 - x1) / np.linalg.norm(x1) > 1e-6  # the values really changed


def test_strongly_mixed_scales_stay_solvable(ctx):
    # test_linsolve.cpp:224-237: lambda = 1e12 next to alpha = 1e3 (condition ~1e9): backward
    # stability is the guarantee, forward agreement with the dense solve only to kappa * eps
    H = W = 8
    terms = ff.frames_to_terms(255.0 * rand_image(H, W, 33), 255.0 * rand_image(H, W, 34), 1.0, 2.5, ctx)
    s = ff.assemble(terms, ff.uniform_reg(W, H, 1e3, 1e12), 3, ctx=ctx)
    rep = ff.SolveReport()
    x = ff.solve(s, ff.SolverConfig(), rep, ctx=ctx)
    A = dense_of(s)
    scale = np.linalg.norm(A, np.inf) * np.linalg.norm(x, np.inf) + np.linalg.norm(s.rhs, np.inf)
    assert np.linalg.norm(A @ x - s.rhs, np.inf) < 1e-12 * scale
    xd = np.linalg.solve(A, s.rhs)
    assert np.linalg.norm(x - xd) / np.linalg.norm(xd) < 1e-3
