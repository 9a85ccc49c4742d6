"""ORACLE (test infrastructure): spline primitives.

- B-spline basis by the Cox–de Boor recursion (Eq. 2; the
  "non-uniform tensor product partition" of the unit cube).  The recursion is
  started from N_{i,0} = [i == span], so it returns the polynomial piece of
  the chosen knot span (no half-open-interval convention is needed at the
  right end; evaluation points are always interior to spans).
- Multivariate Bernstein basis of degree q ("multivariate
  Bernstein basis polynomials of degree p_π", Eq. 21).
- Gauss–Legendre rules on [0,1] (numpy.polynomial.legendre.leggauss).

Pinned by tests/test_oracle_bspline.py (partition of unity, Bernstein closed
forms, B-spline == Bernstein on one element, finite differences, Gauss
exactness on monomials).
"""
from __future__ import annotations

from math import comb

import numpy as np


def elements_of(U: np.ndarray):
    """Non-degenerate knot spans i (U[i] < U[i+1]) — the elements (Eq. 5-6)."""
    return [i for i in range(len(U) - 1) if U[i] < U[i + 1]]


def basis_1d(U: np.ndarray, p: int, span: int, u):
    """All n = len(U)-p-1 basis functions N_{i,p} and first derivatives at
    points u, restricted to the polynomial piece of knot span `span`.

    Cox–de Boor: N_{i,r} = (u-U_i)/(U_{i+r}-U_i) N_{i,r-1}
                         + (U_{i+r+1}-u)/(U_{i+r+1}-U_{i+1}) N_{i+1,r-1}
    derivative:  N'_{i,p} = p/(U_{i+p}-U_i) N_{i,p-1} - p/(U_{i+p+1}-U_{i+1}) N_{i+1,p-1}
    with the convention 0/0 = 0.  Returns (N, dN), each (n, len(u)).
    """
    u = np.asarray(u)
    m = len(U)
    N = np.zeros((m - 1,) + u.shape, dtype=np.result_type(u, np.float64))
    N[span] = 1.0
    prev = N
    for r in range(1, p + 1):
        cur = np.zeros((m - 1 - r,) + u.shape, dtype=N.dtype)
        for i in range(m - 1 - r):
            d1 = U[i + r] - U[i]
            d2 = U[i + r + 1] - U[i + 1]
            a = (u - U[i]) / d1 * prev[i] if d1 > 0 else 0.0
            b = (U[i + r + 1] - u) / d2 * prev[i + 1] if d2 > 0 else 0.0
            cur[i] = a + b
        if r == p:
            lower = prev
        prev = cur
    n = m - 1 - p
    if p == 0:
        return prev[:n], np.zeros_like(prev[:n])
    dN = np.zeros_like(prev)
    for i in range(n):
        d1 = U[i + p] - U[i]
        d2 = U[i + p + 1] - U[i + 1]
        t1 = p / d1 * lower[i] if d1 > 0 else 0.0
        t2 = p / d2 * lower[i + 1] if d2 > 0 else 0.0
        dN[i] = t1 - t2
    return prev[:n], dN


def bernstein_1d(q: int, x):
    """B_k^q(x) = binom(q,k) x^k (1-x)^(q-k), k = 0..q; returns (q+1, len(x))."""
    x = np.asarray(x)
    return np.stack([comb(q, k) * x ** k * (1 - x) ** (q - k) for k in range(q + 1)])


def qvec(q, d):
    """Per-direction degrees (q_0, …, q_{d-1}) of the projection space: an int is the
    isotropic Q_q, a sequence the anisotropic space of the twist example, p_π = 3, 3, 4
    (§3.3.4)."""
    if np.ndim(q) == 0:
        return (int(q),) * d
    q = tuple(int(x) for x in q)
    if len(q) != d:
        raise ValueError(f"q has {len(q)} entries for d = {d}")
    return q


def n_pi(q, d):
    """Number of Bernstein functions Π_k (q_k + 1) (Eq. 21)."""
    return int(np.prod([x + 1 for x in qvec(q, d)]))


def bernstein(q, xi):
    """Multivariate Bernstein N_C(ξ) = Π_k B_{c_k}^{q_k}(ξ_k) (Eq. 21), C = c0 +
    (q0+1)(c1 + (q1+1)c2) (direction-0 fastest); q an int or per-direction degrees.
    xi: (n_pts, d) -> (n_pi, n_pts)."""
    xi = np.asarray(xi)
    d = xi.shape[1]
    qv = qvec(q, d)
    B = [bernstein_1d(qv[k], xi[:, k]) for k in range(d)]
    out = []
    for C in range(n_pi(qv, d)):
        c, r = [], C
        for k in range(d):
            c.append(r % (qv[k] + 1))
            r //= qv[k] + 1
        v = np.ones(xi.shape[0], dtype=xi.dtype)
        for k in range(d):
            v = v * B[k][c[k]]
        out.append(v)
    return np.stack(out)


def gauss_01(n: int):
    """n-point Gauss–Legendre rule on [0,1] (nodes ascending)."""
    t, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (t + 1.0), 0.5 * w


def multi_index(n_per_dir, A):
    """Control-point index A -> (i0, i1[, i2]) with direction 0 fastest."""
    out = []
    for n in n_per_dir:
        out.append(A % n)
        A //= n
    return tuple(out)


def tensor_basis(spline, spans, theta):
    """Tensor-product basis R_A and parametric gradient ∂R_A/∂θ_k for ALL
    control points of `spline` at points theta (n_pts, d) of the knot span
    tuple `spans`.  Returns R (n_ctrl, n_pts), dR (d, n_ctrl, n_pts)."""
    d = spline.dim
    vals, ders = [], []
    for k in range(d):
        N, dN = basis_1d(spline.knots[k], spline.degree[k], spans[k], theta[:, k])
        vals.append(N)
        ders.append(dN)
    n = spline.n_per_dir
    n_ctrl = int(np.prod(n))
    R = np.zeros((n_ctrl, theta.shape[0]), dtype=np.result_type(theta, np.float64))
    dR = np.zeros((d, n_ctrl, theta.shape[0]), dtype=R.dtype)
    for A in range(n_ctrl):
        ii = multi_index(n, A)
        r = np.ones(theta.shape[0], dtype=R.dtype)
        for k in range(d):
            r = r * vals[k][ii[k]]
        R[A] = r
        for m in range(d):
            g = np.ones(theta.shape[0], dtype=R.dtype)
            for k in range(d):
                g = g * (ders[k][ii[k]] if k == m else vals[k][ii[k]])
            dR[m, A] = g
    return R, dR


def active_1d(spline, k, span):
    """Indices of the basis functions of direction k nonzero on `span`: span-p..span."""
    p = spline.degree[k]
    return list(range(span - p, span + 1))
