"""Pins for oracle/macro.py: the macro field Ā (Eq. 37, App. A) and
the interpolation onto Q_q (reading R1)."""
import json
import os

import numpy as np
import pytest

from oracle import macro as M
from oracle.bspline import bernstein, gauss_01

GOLD = os.path.join(os.path.dirname(__file__), "golden")
rng = np.random.default_rng(7)


def rand_J(d, n=6):
    return np.eye(d) * 1.5 + 0.4 * rng.standard_normal((n, d, d))


def test_cube_golden_eq98_100():
    g = json.load(open(os.path.join(GOLD, "cube_eq98_100.json")))
    L, E, nu = g["L"], g["E"], g["nu"]
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    vals = {"a1": (lam + 2 * mu) * L, "a2": mu * L, "a3": lam * L, 0: 0.0}
    J = np.eye(3)[None] * L                       # Eq. 98: M(ξ) = L ξ
    A = M.A_closed(J, *M.lame(E, nu))[0]
    for (i, j) in [(1, 1), (2, 2), (3, 3), (1, 2), (1, 3), (2, 3)]:
        ref = np.array([[vals[x] for x in row] for row in g[f"A{i}{j}"]])
        assert np.allclose(A[i - 1, j - 1], ref, rtol=1e-15, atol=1e-15), (i, j)
        assert np.allclose(A[j - 1, i - 1], ref.T, rtol=1e-15, atol=1e-15)
    # Voigt route (the paper's own Eqs. 89-97) gives the same cube
    Av = M.A_voigt(J, *M.lame(E, nu))[0]
    assert np.allclose(Av, A, rtol=1e-14, atol=1e-14)


@pytest.mark.parametrize("d", [2, 3])
def test_three_routes_agree(d):
    J = rand_J(d)
    lam, mu = 0.8, 0.45
    A = M.A_closed(J, lam, mu)
    assert np.allclose(M.A_voigt(J, lam, mu), A, rtol=0, atol=2e-14 * np.abs(A).max())
    assert np.allclose(M.A_tensor(J, lam, mu), A, rtol=0, atol=2e-14 * np.abs(A).max())


@pytest.mark.parametrize("d", [2, 3])
def test_block_symmetry_eq38(d):
    A = M.A_closed(rand_J(d), 1.1, 0.6)
    assert np.array_equal(A, np.transpose(A, (0, 2, 1, 4, 3))) or np.allclose(
        A, np.transpose(A, (0, 2, 1, 4, 3)), rtol=0, atol=1e-15 * np.abs(A).max())


@pytest.mark.parametrize("d", [2, 3])
def test_homogeneity(d):
    J = rand_J(d)
    A1 = M.A_closed(J, 1.0, 0.5)
    A2 = M.A_closed(2.0 * J, 1.0, 0.5)
    assert np.allclose(A2, 2.0 ** (d - 2) * A1, rtol=1e-14, atol=0)


@pytest.mark.parametrize("d", [2, 3])
def test_energy_form_equivalence(d):
    """Σ_ij u_{,ξi}ᵀ Ā_ij v_{,ξj} == det J σ(u):ε(v) computed componentwise from the
    physical gradients (Eqs. 28, 36)."""
    J = rand_J(d, 1)[0]
    lam, mu = 0.7, 0.3
    A = M.A_closed(J[None], lam, mu)[0]
    du = rng.standard_normal((d, d))     # du[a, i] = ∂u_a/∂ξ_i
    dv = rng.standard_normal((d, d))
    lhs = np.einsum("ai,ijab,bj->", du, A, dv)
    Jinv = np.linalg.inv(J)
    gu = du @ Jinv                        # ∂u_a/∂x_c
    gv = dv @ Jinv
    eu, ev = 0.5 * (gu + gu.T), 0.5 * (gv + gv.T)
    sig = lam * np.trace(eu) * np.eye(d) + 2 * mu * eu
    rhs = np.linalg.det(J) * np.sum(sig * ev)
    assert abs(lhs - rhs) < 1e-13 * abs(rhs) + 1e-14


@pytest.mark.parametrize("q,d", [(0, 2), (1, 2), (2, 2), (2, 3), (3, 3), (4, 2)])
def test_interpolation_exact_on_Qq_and_idempotent(q, d):
    c = rng.standard_normal((q + 1) ** d)
    nodes = M.interp_nodes(q, d)
    samples = bernstein(q, nodes).T @ c
    c2 = M.interpolate(samples, q, d)
    assert np.allclose(c2, c, atol=1e-12)
    # idempotent: interpolating the interpolant reproduces it
    c3 = M.interpolate(bernstein(q, nodes).T @ c2, q, d)
    assert np.allclose(c3, c2, atol=1e-12)


@pytest.mark.parametrize("q,d", [(1, 2), (2, 2), (2, 3), (3, 2)])
def test_interpolation_equals_gauss_discretised_L2(q, d):
    """Reading R1: interpolation at the (q+1) Gauss nodes == L2 projection (Eqs. 23-24)
    whose mass matrix and right-hand side use the (q+1)-point Gauss rule."""
    f = lambda x: np.exp(x[:, 0]) * np.cos(2 * x[:, -1]) + x[:, 0] ** 5
    nodes = M.interp_nodes(q, d)
    x1, w1 = gauss_01(q + 1)
    w = np.ones(len(nodes))
    n1 = q + 1
    for m in range(len(nodes)):
        for k in range(d):
            w[m] *= w1[(m // n1 ** k) % n1]
    N = bernstein(q, nodes)                      # (C, m)
    Mpi = (N * w) @ N.T                          # Eq. 24 (mass)
    r = (N * w) @ f(nodes)                       # Eq. 24 (rhs)
    c_l2 = np.linalg.solve(Mpi, r)
    c_int = M.interpolate(f(nodes), q, d)
    assert np.allclose(c_l2, c_int, atol=1e-12)


def test_affine_macro_field_is_constant():
    """Affine F -> Ā constant -> interpolation coefficients are equal for every C."""
    from synth import make_config
    p = make_config(2, macro_amp=0.0)
    coef = M.tile_coefficients(p, p.macro.ctrl, 5)
    assert np.allclose(coef, coef[0][None], rtol=0, atol=1e-13 * np.abs(coef).max())
    # box [0,4]x[0,1]^2 with 4x4x4 elements: J = diag(1, .25, .25)
    A = M.A_closed(np.diag([1.0, 0.25, 0.25])[None], *M.lame(1.0, 0.3))[0]
    assert np.allclose(coef[0], A, atol=1e-14)


# ---------------------------------------------------------------------------
# L2 projection with an m-point Gauss rule (Eqs. 23-24; NEXT N2)

def _exact_l2_1d(q, k):
    """Exact L2 projection of x^k onto the degree-q Bernstein basis on [0,1], in rational
    arithmetic: M_ij = C(q,i)C(q,j) B(i+j+1, 2q-i-j+1), r_i = C(q,i) B(i+k+1, q-i+1)."""
    from fractions import Fraction
    from math import comb, factorial

    def beta(a, b):                     # B(a, b) = (a-1)!(b-1)!/(a+b-1)! for integers
        return Fraction(factorial(a - 1) * factorial(b - 1), factorial(a + b - 1))
    n = q + 1
    Mx = [[comb(q, i) * comb(q, j) * beta(i + j + 1, 2 * q - i - j + 1) for j in range(n)] for i in range(n)]
    r = [comb(q, i) * beta(i + k + 1, q - i + 1) for i in range(n)]
    for c in range(n):                  # Gauss-Jordan in fractions
        piv = next(i for i in range(c, n) if Mx[i][c] != 0)
        Mx[c], Mx[piv] = Mx[piv], Mx[c]
        r[c], r[piv] = r[piv], r[c]
        f = Mx[c][c]
        Mx[c] = [v / f for v in Mx[c]]
        r[c] /= f
        for i in range(n):
            if i != c and Mx[i][c] != 0:
                g = Mx[i][c]
                Mx[i] = [a - g * b for a, b in zip(Mx[i], Mx[c])]
                r[i] -= g * r[c]
    return np.array([float(v) for v in r])


@pytest.mark.parametrize("q,k,m", [(2, 4, 4), (2, 5, 4), (3, 6, 5), (1, 3, 3)])
def test_l2_projection_matches_exact_rational_projection(q, k, m):
    """For f = x^k the m-point rule integrates N_i f exactly when 2m-1 >= q+k, so the
    projection equals the exact L2 projection computed in rational arithmetic."""
    X, _ = M.projection_nodes(m, 1)
    c = M.project_l2(X[:, 0] ** k, q, 1, m)
    assert np.allclose(c, _exact_l2_1d(q, k), rtol=0, atol=1e-13)


@pytest.mark.parametrize("d", [2, 3])
def test_l2_projection_tensor_product_of_1d(d):
    """A separable f = x^4 y^3 (z^2) projects to the tensor product of the 1D exact
    projections (Bernstein C direction-0 fastest)."""
    q, m = 2, 4
    ks = [4, 3, 2][:d]
    X, _ = M.projection_nodes(m, d)
    f = np.prod([X[:, k] ** ks[k] for k in range(d)], axis=0)
    c = M.project_l2(f, q, d, m)
    ref = _exact_l2_1d(q, ks[0])
    for k in range(1, d):
        ref = np.kron(_exact_l2_1d(q, ks[k]), ref)      # direction k slower
    assert np.allclose(c, ref, rtol=0, atol=1e-13)


@pytest.mark.parametrize("m", [3, 4, 6])
def test_l2_projection_properties(m):
    """Exact on Q_q, idempotent, residual orthogonal to Q_q in the m-point inner product,
    and m = q+1 equals interpolation at the Gauss nodes (reading R1)."""
    q, d = 2, 2
    X, w = M.projection_nodes(m, d)
    N = bernstein(q, X)
    c0 = np.random.default_rng(m).standard_normal(N.shape[0])
    assert np.allclose(M.project_l2(N.T @ c0, q, d, m), c0, atol=1e-13)          # exact on Q_q
    f = np.exp(X[:, 0]) * np.sin(3 * X[:, 1])
    c = M.project_l2(f, q, d, m)
    assert np.allclose(M.project_l2(N.T @ c, q, d, m), c, atol=1e-13)           # idempotent
    assert np.abs((N * w) @ (f - N.T @ c)).max() < 1e-14                          # orthogonality
    if m == q + 1:
        assert np.allclose(c, M.interpolate(f, q, d), atol=1e-13)


def test_tile_coefficients_projection_converges():
    """Curved macro map: the m-point projections converge (m -> large) to the L2
    projection; m = q+1 and m = q+2 differ (the field is not in Q_q)."""
    from synth import make_config
    p = make_config(2)
    cs = {m: M.tile_coefficients(p, p.macro.ctrl, 5, m=m) for m in (3, 4, 6, 8, 10)}
    assert np.abs(cs[3] - cs[4]).max() > 1e-10
    assert np.abs(cs[8] - cs[10]).max() < 1e-12 * np.abs(cs[10]).max() < np.abs(cs[4] - cs[10]).max()


def test_tile_coefficients_batch_equals_single():
    """The batched evaluation (one perturbed control net per batch entry) is the single
    evaluation applied to each net; also under the m-point L2 projection."""
    from synth import make_config
    p = make_config(2)
    rng = np.random.default_rng(7)
    nets = np.stack([p.macro.ctrl + 0.01 * rng.standard_normal(p.macro.ctrl.shape) for _ in range(3)])
    for m in (None, 5):
        got = M.tile_coefficients_batch(p, nets, 9, m=m)
        for b in range(3):
            ref = M.tile_coefficients(p, nets[b], 9, m=m)
            if m is None:    # interpolation: bit for bit
                assert np.array_equal(got[b], ref)
            else:            # L2: BLAS blocking of the multi-column M_π solve, κ(M_π)^d ≈ 1e3 at q = 2
                assert np.abs(got[b] - ref).max() <= 1e-12 * np.abs(ref).max()
