"""Pins for oracle/bspline.py (Eq. 2, Eq. 21)."""
import json
import os
from math import comb

import numpy as np
import pytest

from oracle.bspline import basis_1d, bernstein, bernstein_1d, elements_of, gauss_01
from synth import open_uniform_knots

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def nonuniform_knots():
    return np.array([0, 0, 0, 0, 0.1, 0.35, 0.35, 0.7, 1, 1, 1, 1.0])   # p=3, a double knot


@pytest.mark.parametrize("p,U", [(2, open_uniform_knots(2, 5)), (3, nonuniform_knots()), (1, open_uniform_knots(1, 3))])
def test_partition_of_unity_and_derivative_sum(p, U):
    for s in elements_of(U):
        u = np.linspace(U[s], U[s + 1], 7)[1:-1]
        N, dN = basis_1d(U, p, s, u)
        assert np.allclose(N.sum(0), 1.0, atol=1e-13)
        assert np.allclose(dN.sum(0), 0.0, atol=1e-11)
        assert np.all(N >= -1e-15)
        # only span-p..span are nonzero
        mask = np.ones(N.shape[0], bool)
        mask[s - p:s + 1] = False
        assert np.all(N[mask] == 0)


def test_bernstein_golden():
    g = json.load(open(os.path.join(GOLD, "bernstein_s42_s68.json")))
    assert np.allclose(bernstein_1d(2, np.array([0.5]))[:, 0], g["deg2_at_half"], rtol=0, atol=1e-16)
    assert np.allclose(bernstein_1d(4, np.array([0.5]))[:, 0], g["deg4_at_half"], rtol=0, atol=1e-16)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_bspline_single_element_is_bernstein(p):
    U = np.array([0.0] * (p + 1) + [1.0] * (p + 1))
    x = np.linspace(0.01, 0.99, 11)
    N, dN = basis_1d(U, p, p, x)
    assert np.allclose(N, bernstein_1d(p, x), atol=1e-14)
    # derivative closed form: p (B_{k-1}^{p-1} - B_k^{p-1})
    Bm = bernstein_1d(p - 1, x)
    ref = np.stack([p * ((Bm[k - 1] if k > 0 else 0) - (Bm[k] if k < p else 0)) for k in range(p + 1)])
    assert np.allclose(dN, ref, atol=1e-12)


def test_bspline_derivative_vs_fd():
    U, p = nonuniform_knots(), 3
    for s in elements_of(U):
        u = np.array([U[s] + 0.37 * (U[s + 1] - U[s])])
        h = 1e-6
        Np, _ = basis_1d(U, p, s, u + h)
        Nm, _ = basis_1d(U, p, s, u - h)
        _, dN = basis_1d(U, p, s, u)
        assert np.allclose(dN, (Np - Nm) / (2 * h), atol=1e-6 * max(1, np.abs(dN).max()))


def test_bspline_uniform_quadratic_known_values():
    # uniform quadratic B-spline at the middle of an interior span: (1/8, 3/4, 1/8)
    U = open_uniform_knots(2, 5)
    s = 4  # span [0.4, 0.6]
    N, _ = basis_1d(U, 2, s, np.array([0.5]))
    assert np.allclose(N[s - 2:s + 1, 0], [1 / 8, 3 / 4, 1 / 8], atol=1e-15)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_gauss_exactness(n):
    x, w = gauss_01(n)
    for k in range(2 * n):
        assert abs(np.sum(w * x ** k) - 1.0 / (k + 1)) < 1e-15 * 4
    # not exact at degree 2n
    assert abs(np.sum(w * x ** (2 * n)) - 1.0 / (2 * n + 1)) > 1e-8


def test_multivariate_bernstein_ordering():
    xi = np.array([[0.2, 0.7, 0.4]])
    N = bernstein(2, xi)
    b = [bernstein_1d(2, xi[:, k])[:, 0] for k in range(3)]
    for C in range(27):
        c0, c1, c2 = C % 3, (C // 3) % 3, C // 9
        assert np.isclose(N[C, 0], b[0][c0] * b[1][c1] * b[2][c2])
    assert np.isclose(N.sum(), 1.0)
    assert comb(2, 1) == 2
