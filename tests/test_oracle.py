"""Pins the CPU oracle before it is trusted as the checker: the plain-C restatement
(oracle/flowfem_port.c) must reproduce the reference's committed golden vectors bit for
bit, and (where the reference was compiled here) the reference itself on fresh inputs."""
import hashlib

import numpy as np
import pytest

from conftest import rel_l2
from paper_1508_02977_b200 import synth


def test_port_matches_golden_stages(port, golden):
    g = golden("stages_small.npz")
    assert np.array_equal(port.gaussian_smooth(g["f0"], 1.0), g["s0"])
    assert np.array_equal(port.gaussian_smooth(g["f1"], 1.0), g["s1"])
    fx, fy, ft, f = port.compute_derivatives(g["s0"], g["s1"])
    for a, k in ((fx, "fx"), (fy, "fy"), (ft, "ft"), (f, "f")):
        assert np.array_equal(a, g[k]), k
    assert np.array_equal(port.build_data_terms(fx, fy, ft, f, 2.5), g["terms"])
    y3, b3 = port.assemble_apply(g["terms"], g["alpha"], g["lam"], 3, g["x3"])
    assert np.array_equal(y3, g["y3"]) and np.array_equal(b3, g["b3"])
    y2, b2 = port.assemble_apply(g["terms"], g["alpha"], g["lam"], 2, g["x3"])
    assert np.array_equal(y2, g["y2"]) and np.array_equal(b2, g["b2"])
    eta, em = port.error_indicator(g["terms"], g["alpha"], g["lam"], g["x3"], 3)
    assert np.array_equal(eta, g["eta"]) and em == g["eta_max"]
    eta2, em2 = port.error_indicator(g["terms"], g["alpha"], g["lam"], g["x3"], 2)
    assert np.array_equal(eta2, g["eta2"]) and em2 == g["eta_max2"]
    a_new = port.update_alpha(g["alpha"], g["lam"], g["eta"], float(g["eta_max"]), 10.0, 0.1, 10.0)
    assert np.array_equal(a_new, g["alpha_new"])


def test_port_matches_golden_c1_chain(port, golden):
    g = golden("c1_chain.npz")
    f0, f1, _, cfg = synth.make("c1")
    assert hashlib.sha256(f0.tobytes()).hexdigest() == str(g["f0_sha"])
    assert hashlib.sha256(f1.tobytes()).hexdigest() == str(g["f1_sha"])
    r = port.converged_chain(f0, f1, cfg.sigma, n_passes=cfg.n_passes, tol=1e-12)
    # same algorithm, same operation order: identical iteration counts and bits
    assert list(r["iters"]) == list(g["iters"])
    assert np.array_equal(r["u3"], g["u3"])
    assert np.array_equal(r["alpha"], g["alpha"])


@pytest.mark.parametrize("H,W,sigma,nc", [(17, 29, 1.0, 3), (40, 33, 1.5, 3), (12, 9, 0.0, 2)])
def test_port_matches_reference_fresh(port, ref, H, W, sigma, nc):
    rng = np.random.default_rng(H * W)
    f0 = rng.uniform(0, 255, (H, W))
    f1 = np.clip(np.roll(f0, 1, axis=1) + rng.normal(0, 3, (H, W)), 0, 255)
    t_p = port.frames_to_terms(f0, f1, sigma, 2.5)
    t_r = ref.frames_to_terms(f0, f1, sigma, 2.5)
    assert np.array_equal(t_p, t_r)
    cp = port.converged_chain(f0, f1, sigma, nc=nc, n_passes=2, tol=1e-10)
    cr = ref.converged_chain(f0, f1, sigma, nc=nc, n_passes=2, tol=1e-10)
    assert np.array_equal(cp["u3"], cr["u3"]) and list(cp["iters"]) == list(cr["iters"])


def test_oracle_solution_is_converged(port, golden):
    """The golden c1 fixture is a converged solve: its true residual, evaluated with the
    reference operator at the final alpha, is below the generation tolerance."""
    g = golden("c1_chain.npz")
    f0, f1, _, cfg = synth.make("c1")
    t = port.frames_to_terms(f0, f1, cfg.sigma, cfg.rho)
    lam = np.full_like(g["alpha"], cfg.lambda0)
    y3, b3 = port.assemble_apply(t, g["alpha"], lam, 3, g["u3"])
    assert rel_l2(y3, b3) < 1e-11


# ------------------------------------------------------------------ linsolve boundary (§8f-2)
def _csr_case(golden, k):
    import pyoracle as po
    g = golden("linsolve.npz")
    return g, po.CsrSystem(g[f"{k}_row_ptr"], g[f"{k}_cols"], g[f"{k}_vals"], g[f"{k}_rhs"],
                           int(g[f"{k}_nc"]))


@pytest.mark.parametrize("k", range(6))
def test_port_csr_cg_and_rcm_pinned_to_reference(port, golden, k):
    """The port's CSR cg_solve and rcm_order equal the reference's (golden) bit for bit."""
    import pyoracle as po
    g, s = _csr_case(golden, k)
    x, it, res = po.csr_cg_solve(port, s, 1e-12)
    assert np.array_equal(x, g[f"{k}_cg_x"])
    assert it == int(g[f"{k}_cg_iters"]) and res == float(g[f"{k}_cg_res"])
    assert np.array_equal(po.rcm_order(port, s), g[f"{k}_perm"])


def test_port_cg_indefinite_message(port, golden):
    import pyoracle as po
    g = golden("linsolve.npz")
    bad = po.CsrSystem(g["bad_row_ptr"], g["bad_cols"], g["bad_vals"], g["bad_rhs"], 3)
    with pytest.raises(po.OracleError) as e:
        po.csr_cg_solve(port, bad, 1e-12)
    assert str(e.value) == str(g["bad_msg_cg"])


def test_library_rcm_order_bitwise(golden):
    """ffb_rcm_order is host integer work: checked here without a GPU."""
    from paper_1508_02977_b200 import flowfem as ff
    for k in range(6):
        g, s = _csr_case(golden, k)
        fs = ff.SparseSystem(s.row_ptr, s.cols, s.vals, s.rhs, s.components)
        assert np.array_equal(ff.rcm_order(fs), g[f"{k}_perm"])
    with pytest.raises(ff.FlowfemError, match="linsolve.rcm_order: system size not a multiple"):
        g, s = _csr_case(golden, 0)
        ff.rcm_order(ff.SparseSystem(s.row_ptr, s.cols, s.vals, s.rhs, 5))
