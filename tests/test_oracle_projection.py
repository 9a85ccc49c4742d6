"""Pins for oracle/projection.py: the a-priori projection error E_proj (Eq. 59, PAPER.md:439,
sampled as on P:362-364) and the adaptive degree selection (Eq. 65),
plus anisotropic projection spaces."""
import numpy as np
import pytest

from oracle import macro as M
from oracle import projection as PE
from oracle.bspline import bernstein, gauss_01
from synth import Spline, make_config


def stretch_problem(kappa, h0=2.0, h1=0.5):
    """One macro element F(ξ) = (h0 (ξ0 + κ ξ0²), h1 ξ1): degree (2, 1), control points at
    the Bernstein coefficients (blossoms) of F, so F is represented exactly."""
    prob = make_config(1)
    U2 = np.array([0.0, 0, 0, 1, 1, 1])
    U1 = np.array([0.0, 0, 1, 1])
    bx = h0 * np.array([0.0, 0.5, 1.0 + kappa])
    ctrl = np.array([[bx[i0], h1 * i1] for i1 in range(2) for i0 in range(3)])
    prob.macro = Spline([2, 1], [U2, U1], ctrl)
    prob.n_el = (1, 1)
    prob.young = np.ones(1)
    return prob


def stretch_closed_form(kappa, q0, n_s, nu, h0=2.0, h1=0.5):
    """E_proj of the stretch map with interpolation at q0+1 Gauss nodes in direction 0, in
    closed form.  J = diag(h0(1+cξ0), h1), c = 2κ, D = h0 h1 (1+cξ0), G = J⁻¹ diagonal, so the
    nonzero Ā entries are (λ+2μ, μ)·(h1/h0)·r with r = 1/(1+cξ0), (λ+2μ, μ)·(h0/h1)(1+cξ0),
    and the constants λ, μ (twice each).  The interpolant of the linear and constant parts is
    exact for q0 >= 1; that of r has the error (divided differences of 1/(1+cx))
        r(x) - p(x) = (-c)^{q0+1} ω(x) / ((1+cx) Π_k (1+c x_k)),  ω(x) = Π_k (x - x_k);
    for q0 = 0 the linear part adds the error c(x - x_0).  Direction 1 is exact for any q1."""
    lam = nu / ((1 + nu) * (1 - 2 * nu))
    mu = 1 / (2 * (1 + nu))
    c = 2 * kappa
    xk, _ = gauss_01(q0 + 1)
    x = np.linspace(0, 1, n_s)
    omega = np.prod([x - a for a in xk], axis=0)
    er = (-c) ** (q0 + 1) * omega / ((1 + c * x) * np.prod(1 + c * xk))
    el = c * (x - xk[0]) if q0 == 0 else 0.0 * x
    s2 = (lam + 2 * mu) ** 2 + mu ** 2
    num = np.sqrt(s2 * ((h1 / h0) ** 2 * er ** 2 + (h0 / h1) ** 2 * el ** 2))
    den = np.sqrt(s2 * ((h1 / h0) ** 2 / (1 + c * x) ** 2 + (h0 / h1) ** 2 * (1 + c * x) ** 2)
                  + 2 * lam ** 2 + 2 * mu ** 2)
    return float(np.max(num / den))


@pytest.mark.parametrize("kappa,q,n_s", [(0.2, (1, 0), 5), (0.4, (2, 1), 9), (0.4, (3, 0), 7), (0.3, (4, 2), 6),
                                         (0.25, (0, 0), 5), (0.35, 3, 8)])
def test_eproj_closed_form_stretch(kappa, q, n_s):
    prob = stretch_problem(kappa)
    e, per = PE.projection_error(prob, q, n_s)
    q0 = q if np.ndim(q) == 0 else q[0]
    ref = stretch_closed_form(kappa, q0, n_s, prob.nu)
    assert per.shape == (1,)
    assert abs(e - ref) <= 1e-9 * ref + 1e-15, (e, ref)


def test_eproj_zero_when_field_in_projection_space():
    """Affine elements: Ā constant -> E_proj = 0 at q = 0.  Shear map: Ā ∈ Q_{0,2} exactly ->
    0 at q = (0, 2) and at q = 2, > 0 at q = (2, 1)."""
    assert PE.projection_error(make_config(1, macro_amp=0.0), 0, 5)[0] < 1e-14
    sh = make_config(1, macro_kind="shear")
    assert PE.projection_error(sh, (0, 2), 6)[0] < 1e-13
    assert PE.projection_error(sh, 2, 6)[0] < 1e-13
    assert PE.projection_error(sh, (2, 1), 6)[0] > 1e-4


def test_eproj_decreases_with_q_and_l2_variant():
    prob = make_config(1)
    es = [PE.projection_error(prob, q, 6)[0] for q in range(5)]
    assert all(a > b for a, b in zip(es, es[1:])), es
    assert es[-1] < 1e-4
    # the m-point L2 projection (Eqs. 23-24) is a different projector with errors of the same order
    e_l2 = PE.projection_error(prob, 2, 6, m=5)[0]
    assert 0.2 * es[2] < e_l2 < 5 * es[2]


def test_eproj_vanishes_at_interpolation_nodes():
    """Interpolation (R1) reproduces Ā at the Gauss nodes: with the sample set = the nodes,
    the error is round-off; sampled elsewhere it is not."""
    prob = make_config(1)
    t, q = 5, 2
    lam, mu = M.lame(1.0, prob.nu)
    field = lambda X: M.A_closed(M.macro_jacobian(prob.macro, prob.macro.ctrl, t, X), lam, mu)
    coef = M.project_field(field, q, 2)
    X = M.interp_nodes(q, 2)
    assert np.abs(M.field_from_coefficients(coef, q, X) - field(X)).max() < 1e-13


@pytest.mark.parametrize("kappa", [0.3, 0.45])
def test_select_degree_matches_closed_form(kappa):
    """Eq. 65 with reading R19 on the stretch map: macro degrees (2, 1) enriched / coarsened
    uniformly; the answer is the smallest q0 whose closed-form E_proj <= tol."""
    prob = stretch_problem(kappa)
    n_s = 9
    E = {q0: stretch_closed_form(kappa, q0, n_s, prob.nu) for q0 in range(0, 8)}
    for q0_target in (1, 2, 4, 5):
        tol = float(np.sqrt(E[q0_target] * E[q0_target - 1]))   # between the two, far from both
        q, e = PE.select_degree(prob, tol, n_s=n_s)
        assert q == (q0_target, max(q0_target - 1, 0)), (tol, q)
        assert abs(e - E[q0_target]) <= 1e-9 * E[q0_target]


def test_select_degree_cfg1_and_twist_reading():
    """cfg1 (biquadratic macro): tol = 1e-3 (the paper's) selects q = 3 per direction;
    a tolerance above E(q = p_M) coarsens."""
    prob = make_config(1, n_el=(2, 2))
    q, e = PE.select_degree(prob, 1e-3, n_s=6)
    e_lower = PE.projection_error(prob, tuple(x - 1 for x in q), 6)[0]
    assert q == (3, 3) and e <= 1e-3 < e_lower
    q2, e2 = PE.select_degree(prob, 0.5, n_s=6)
    assert max(q2) < 2 and e2 <= 0.5


@pytest.mark.parametrize("q,d", [((1, 3), 2), ((0, 2), 2), ((2, 1, 3), 3), ((0, 0, 2), 3)])
def test_anisotropic_interpolation_exact_and_idempotent(q, d):
    """Interpolation at Π (q_k+1) Gauss nodes is exact on Q_{q0,...} and idempotent; the
    Bernstein basis is a partition of unity and a tensor product of 1D bases."""
    rng = np.random.default_rng(7)
    npi = int(np.prod([x + 1 for x in q]))
    nodes = M.interp_nodes(q, d)
    assert nodes.shape == (npi, d)
    N = bernstein(q, nodes)
    assert np.allclose(N.sum(0), 1.0, atol=1e-15)
    c = rng.standard_normal(npi)
    c2 = M.interpolate(N.T @ c, q, d)
    assert np.allclose(c2, c, atol=1e-12)
    X = rng.random((11, d))
    vals = bernstein(q, X).T @ c                                 # a polynomial in Q_q
    f = lambda Y: bernstein(q, Y).T @ c
    coef = M.project_field(f, q, d)
    assert np.allclose(M.field_from_coefficients(coef, q, X), vals, atol=1e-12)
    # L2 projection with more points per direction is also exact on Q_q
    coef_l2 = M.project_field(f, q, d, m=max(q) + 2)
    assert np.allclose(coef_l2, c, atol=1e-12)
