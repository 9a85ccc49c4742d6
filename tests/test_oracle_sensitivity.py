"""Pins for oracle/sensitivity.py: g = uᵀ(∂K^π/∂P)v (Eqs. 70-73; reading R13)."""
import numpy as np
import pytest

from oracle import sensitivity as S
from synth import draw_uv_seeded


@pytest.fixture(params=[(1, {}), (2, dict(n_el=(2, 1, 1)))], ids=["cfg1", "cfg2-small"])
def case(request, oracle_problem):
    c, kw = request.param
    ob = oracle_problem(c, **kw)
    u, v = draw_uv_seeded(c, ob["dm"].n_dof)
    g = S.sensitivity(ob["prob"], ob["tabs"], ob["pattern"], u, v)
    return ob, u, v, g


def test_adjoint_equals_whole_assembly_complex_step(case):
    ob, u, v, g = case
    prob = ob["prob"]
    rng = np.random.default_rng(3)
    ent = [(int(k), int(a)) for k, a in zip(rng.integers(0, len(g), 5), rng.integers(0, prob.d, 5))]
    brute = S.brute_complex_step(prob, ob["tabs"], ob["pattern"], u, v, ent)
    ref = np.array([g[k, a] for k, a in ent])
    assert np.allclose(ref, brute, rtol=1e-12, atol=1e-12 * np.abs(g).max())


def test_central_finite_differences(case):
    ob, u, v, g = case
    prob = ob["prob"]
    k = len(g) // 2 + 1
    for a in range(prob.d):
        h = 1e-6
        cp, cm = prob.macro.ctrl.copy(), prob.macro.ctrl.copy()
        cp[k, a] += h
        cm[k, a] -= h
        fd = (S.energy(prob, ob["tabs"], ob["pattern"], u, v, cp)
              - S.energy(prob, ob["tabs"], ob["pattern"], u, v, cm)) / (2 * h)
        assert abs(fd - g[k, a]) < 1e-6 * max(1.0, abs(g[k, a]))


def test_translation_invariance(case):
    ob, u, v, g = case
    assert np.abs(g.sum(axis=0)).max() < 1e-11 * np.abs(g).max() * len(g)


def test_euler_homogeneity(case):
    """K(sP) = s^{d-2} K(P)  =>  Σ_{k,α} P_kα g_kα = (d-2) uᵀK^πv (0 in 2D)."""
    ob, u, v, g = case
    prob = ob["prob"]
    E = S.energy(prob, ob["tabs"], ob["pattern"], u, v)
    lhs = np.sum(prob.macro.ctrl * g)
    assert abs(lhs - (prob.d - 2) * E) < 1e-10 * (np.abs(prob.macro.ctrl * g).sum())


def test_symmetry_in_u_v(case):
    ob, u, v, g = case
    g2 = S.sensitivity(ob["prob"], ob["tabs"], ob["pattern"], v, u)
    assert np.allclose(g, g2, rtol=1e-13, atol=1e-13 * np.abs(g).max())


def test_linearity_in_u(case):
    ob, u, v, g = case
    g2 = S.sensitivity(ob["prob"], ob["tabs"], ob["pattern"], 2.5 * u, v)
    assert np.allclose(g2, 2.5 * g, rtol=1e-12, atol=1e-12 * np.abs(g).max())


def test_batched_complex_step_equals_entrywise(case):
    """`sensitivity` evaluates the complex-step perturbations of one tile as a batch
    (macro.tile_coefficients_batch); the entry-by-entry evaluation gives the same values."""
    ob, u, v, g = case
    prob = ob["prob"]
    rng = np.random.default_rng(11)
    ent = [(int(k), int(a)) for k, a in zip(rng.integers(0, len(g), 6), rng.integers(0, prob.d, 6))]
    ref = S.sensitivity_entrywise(prob, ob["tabs"], ob["pattern"], u, v, ent)
    for k, a in ent:
        assert abs(g[k, a] - ref[k, a]) <= 1e-14 * np.abs(g).max(), (k, a)
