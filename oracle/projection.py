"""ORACLE (test infrastructure): a-priori projection error and adaptive projection
degree.

E_proj (Eq. 59), evaluated "by a simple sampling-based approach where the
differences between the exact macro-quantities and their projections are evaluated at
each sample point ... a priori to the assembly":

    E_proj = max_t max_{ξ ∈ S} ‖Ā^(t)(ξ) − Π^H Ā^(t)(ξ)‖_F / ‖Ā^(t)(ξ)‖_F

with ‖·‖_F over all d⁴ components (i, j, a, b) and S the tensor grid of n_s equispaced
points per direction of the element-local cube, endpoints included (reading R18).
Ā ∝ E_t, so E_proj does not depend on E; it is evaluated with E = 1.

Degree selection (Eq. 65; strategy of P:364 and P:524): "initializing
the projection degrees by the ones of the underlying macro-geometry.  Then, the projection
space is enriched (or coarsened) until the projection error is below the chosen
tolerance".  Reading R19: enrichment / coarsening is uniform, q(s) = (max(p_M,k + s, 0))_k,
and the selected degree is the smallest such q(s) with E_proj ≤ tol (for the twist, macro
degrees 1, 1, 2 give 3, 3, 4 with s = 2, as printed on P:524).
"""
from __future__ import annotations

import itertools

import numpy as np

from . import macro as M
from .bspline import qvec


def sample_grid(n_s, d):
    """n_s equispaced points per direction on [0,1] (endpoints included), direction-0 fastest."""
    x = np.linspace(0.0, 1.0, n_s)
    return np.array([tuple(reversed(p)) for p in itertools.product(*([x] * d))])


def tile_projection_error(prob, ctrl, t, q, n_s, m=0):
    """max over the sample grid of ‖Ā − Π^H Ā‖_F / ‖Ā‖_F for tile t (Eq. 59's inner max)."""
    d = prob.d
    lam, mu = M.lame(1.0, prob.nu)
    field = lambda X: M.A_closed(M.macro_jacobian(prob.macro, ctrl, t, X), lam, mu)
    coef = M.project_field(field, q, d, m, check_tile=t, ctrl=ctrl, macro=prob.macro)
    S = sample_grid(n_s, d)
    exact = field(S)                                   # (n_s^d, d, d, d, d)
    approx = M.field_from_coefficients(coef, q, S)
    num = np.sqrt(np.sum((exact - approx) ** 2, axis=(1, 2, 3, 4)))
    den = np.sqrt(np.sum(exact ** 2, axis=(1, 2, 3, 4)))
    return float(np.max(num / den))


def projection_error(prob, q=None, n_s=8, m=0, ctrl=None, tiles=None):
    """E_proj (Eq. 59) and the per-tile maxima; q defaults to prob.q."""
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    q = prob.q if q is None else q
    tiles = range(prob.n_tiles) if tiles is None else tiles
    per = np.array([tile_projection_error(prob, ctrl, t, q, n_s, m) for t in tiles])
    return float(per.max()), per


def select_degree(prob, tol, n_s=8, m_extra=0, q_max=8, ctrl=None):
    """Eq. 65 with reading R19: returns (q, E_proj(q)).  m_extra > 0 uses the L2
    projection with q_k + 1 + m_extra Gauss points per direction."""
    d = prob.d
    pM = qvec(prob.macro.degree, d)
    q_of = lambda s: tuple(max(p + s, 0) for p in pM)
    m_of = lambda q: 0 if m_extra == 0 else tuple(x + 1 + m_extra for x in q)
    err = lambda s: projection_error(prob, q_of(s), n_s, m_of(q_of(s)), ctrl)[0]
    s = 0
    e = err(s)
    if e <= tol:
        while max(q_of(s)) > 0:
            e_down = err(s - 1)
            if e_down > tol:
                break
            s, e = s - 1, e_down
        return q_of(s), e
    while max(q_of(s)) < q_max:
        s += 1
        e = err(s)
        if e <= tol:
            return q_of(s), e
    raise ValueError(f"E_proj = {e:.3e} > tol = {tol:.1e} at q = {q_of(s)} (q_max = {q_max})")
