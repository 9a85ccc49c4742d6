"""ORACLE (test infrastructure): sparsity set I_coo and lookup tables 𝔎.

I_coo (Eq. 56): pairs (A, B), A ≤ B, whose supports share a
knot span of the patch (reading R8: overlap of support interiors), sorted by
(A, B).

𝔎 (Eqs. 51-52), matricised as in Eq. 57:
  mat𝔎[k=(A,B)][κ = (i·d + j)·n_π + C] =
    ∫_{Ω_T} ∂_{ξ_i}(R_A∘𝒯⁻¹) ∂_{ξ_j}(R_B∘𝒯⁻¹) N_C dξ
  evaluated by pull-back to the tile parameter θ (dξ = det J_T dθ,
  ∇_ξ R = J_T⁻ᵀ ∇_θ R) with n_g Gauss points per direction per knot span
  (reading R3), summed over spans in lexicographic order, then points.
"""
from __future__ import annotations

import itertools

import numpy as np

from .bspline import bernstein, elements_of, gauss_01, n_pi, tensor_basis


def patch_spans(spline):
    """All knot-span tuples of a patch, direction-0 fastest."""
    els = [elements_of(U) for U in spline.knots]
    return [tuple(reversed(s)) for s in itertools.product(*reversed(els))]


def active_functions(spline, spans):
    """Control points A whose tensor basis function is nonzero on span tuple `spans`."""
    d = spline.dim
    n = spline.n_per_dir
    ranges = [range(spans[k] - spline.degree[k], spans[k] + 1) for k in range(d)]
    out = []
    for ii in itertools.product(*reversed(ranges)):
        ii = tuple(reversed(ii))
        A = 0
        for k in reversed(range(d)):
            A = A * n[k] + ii[k]
        out.append(A)
    return sorted(out)


def icoo(spline):
    """I_coo as an (n_nz, 2) int array of (A, B), A ≤ B, sorted (Eq. 56)."""
    pairs = set()
    for s in patch_spans(spline):
        act = active_functions(spline, s)
        for A in act:
            for B in act:
                if A <= B:
                    pairs.add((A, B))
    return np.array(sorted(pairs), dtype=np.int64)


def gauss_points_span(spline, spans, n_g):
    """Tensor Gauss points θ (n_pts, d) and weights w·|span| on span tuple `spans`."""
    x, w = gauss_01(n_g)
    d = spline.dim
    pts, wts = [], []
    for idx in itertools.product(*([range(n_g)] * d)):
        idx = tuple(reversed(idx))          # direction 0 fastest
        th, ww = [], 1.0
        for k in range(d):
            U = spline.knots[k]
            s = spans[k]
            h = U[s + 1] - U[s]
            th.append(U[s] + h * x[idx[k]])
            ww *= w[idx[k]] * h
        pts.append(th)
        wts.append(ww)
    return np.array(pts), np.array(wts)


def tile_point_data(spline, spans, n_g):
    """At the Gauss points of one span: ξ = 𝒯(θ), det J_T, the physical
    (ξ-space) gradients G[A, n, i] = (J_T⁻ᵀ ∇_θ R_A)_i, and the weights.
    Raises on det J_T <= 0 (reading R5)."""
    th, w = gauss_points_span(spline, spans, n_g)
    R, dR = tensor_basis(spline, spans, th)            # (n_ctrl, n), (d, n_ctrl, n)
    xi = R.T @ spline.ctrl                              # (n, d)
    JT = np.einsum("kAn,Aa->nak", dR, spline.ctrl)      # JT[n, a, k] = ∂ξ_a/∂θ_k
    DT = np.linalg.det(JT)
    if np.any(DT <= 0):
        raise ValueError("degenerate tile Jacobian")
    JTinv = np.linalg.inv(JT)                           # [n, k, a]
    G = np.einsum("nka,kAn->Ana", JTinv, dR)            # ∂R_A/∂ξ_a
    return xi, DT, G, w


def lookup_table(spline, q, n_g):
    """mat𝔎 (n_nz × n_π d²) for one tile patch (Eqs. 52, 57); q an int or per-direction
    degrees of the projection space (n_π = Π_k (q_k+1))."""
    d = spline.dim
    pairs = icoo(spline)
    row_of = {(int(a), int(b)): r for r, (a, b) in enumerate(pairs)}
    npi = n_pi(q, d)
    T = np.zeros((len(pairs), d, d, npi))
    for s in patch_spans(spline):
        act = active_functions(spline, s)
        xi, DT, G, w = tile_point_data(spline, s, n_g)
        N = bernstein(q, xi)                             # (C, n)
        wD = w * DT
        Ga = G[act]                                      # (na, n, d)
        # local[A, B, i, j, C] = Σ_n wD_n G_A[n,i] G_B[n,j] N_C[n]
        loc = np.einsum("n,Ani,Bnj,Cn->ABijC", wD, Ga, Ga, N, optimize=True)
        for ia, A in enumerate(act):
            for ib, B in enumerate(act):
                if A <= B:
                    T[row_of[(A, B)]] += loc[ia, ib]
    return T.reshape(len(pairs), d * d * npi), pairs
