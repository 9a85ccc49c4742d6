"""ORACLE (test infrastructure): lookup assembly K^π and standard assembly K^•.

Lookup (§3.2.4, 418-427):
  1. coefficients ⟨Ā_ij⟩_C per tile (macro.tile_coefficients; Eq. 42, reading R1)
  2. the tables mat𝔎_p (tables.lookup_table; Eqs. 52, 57), stacked over patches
  3. local = mat𝔎 · mat⟨Ā⟩ (Eq. 58) — one matmul per tile
  4. scatter into the full symmetric CSR (reading R9):
     block L = local[t, row] of pair (A, B) -> global (I, J):
       A < B:  K[(I,a),(J,b)] += L[a,b]  and  K[(J,b),(I,a)] += L[a,b]
       A = B:  K[(I,a),(I,b)] += L[min(a,b), max(a,b)]
     accumulated in the order t, then row (np.add.at is sequential).

Standard ("element loops with full Gauss quadrature"; Eq. 49
with the composed map Eq. 10): at each tile quadrature point,
J = J_F(𝒯(θ)) J_T(θ), ∇_x R = J⁻ᵀ ∇_θ R and
  K_AB[a,b] += w D (λ ∂_aR_A ∂_bR_B + μ ∂_bR_A ∂_aR_B + μ δ_ab ∇R_A·∇R_B).
`local_quadrature_Aform` evaluates Eq. 49 in the Ā form with any macro
field (exact Ā, or its interpolant Π_qĀ).
"""
from __future__ import annotations

import numpy as np

from . import macro as M
from .tables import active_functions, lookup_table, patch_spans, tile_point_data


class Tables:
    """Stacked lookup tables of all tile patches: T (n_rows_tile × d² n_π)."""

    def __init__(self, prob):
        self.per_patch = [lookup_table(s, prob.q, prob.n_gauss) for s in prob.tile]
        self.T = np.concatenate([t for t, _ in self.per_patch], axis=0)
        self.pairs = [pr for _, pr in self.per_patch]


def coef_matrix(coef):
    """mat⟨Ā⟩ for one tile (Eq. 58): rows κ = (i·d+j)·n_π + C, columns a·d + b."""
    npi, d = coef.shape[0], coef.shape[1]
    return np.transpose(coef, (1, 2, 0, 3, 4)).reshape(d * d * npi, d * d)


def local_lookup(prob, tabs: Tables, ctrl, tiles, coefs=None):
    """K^π element matrices (Eq. 50/58): (len(tiles), n_rows_tile, d, d)."""
    d = prob.d
    out = []
    for n, t in enumerate(tiles):
        coef = M.tile_coefficients(prob, ctrl, t) if coefs is None else coefs[n]
        out.append((tabs.T @ coef_matrix(coef)).reshape(-1, d, d))
    return np.stack(out)


def scatter(prob, pattern, local, tiles=None, out=None, bmap=None, nodes=None):
    """CSR values of K from element matrices (reading R9).  local (len(tiles), n_rows, d, d)
    of the given tiles (default all); `out`: add into this CSR value array instead of a
    new zero one (so that consecutive tile ranges accumulate in the order t, row);
    `bmap`: the tiles' block map (pattern.block_map(tiles)) if already at hand;
    `nodes` = (n0, n1): only the CSR rows of nodes n0 <= I < n1 (the same additions in
    the same order, restricted to those rows — for filling disjoint row ranges apart)."""
    d = prob.d
    nt = local.shape[0]
    tiles = np.arange(nt) if tiles is None else np.asarray(tiles)
    I, J = pattern.I[tiles].ravel(), pattern.J[tiles].ravel()
    L = local.reshape(-1, d, d)
    if bmap is None:
        fwd = pattern.pos(I, J)
        bwd = pattern.pos(J, I)
    else:
        fwd, bwd = bmap[:, 0], bmap[:, 1]
    rowlen = d * pattern.nnzb
    vals = np.zeros(pattern.nnz, dtype=local.dtype) if out is None else out
    off = I != J
    in1 = np.ones(len(I), dtype=bool) if nodes is None else (I >= nodes[0]) & (I < nodes[1])
    in2 = off if nodes is None else off & (J >= nodes[0]) & (J < nodes[1])
    n = len(I)
    idx = np.full((n, d, d, 2), -1, dtype=np.int64)
    val = np.zeros((n, d, d, 2), dtype=local.dtype)
    for a in range(d):
        for b in range(d):
            # (I,a),(J,b) for every block; diagonal blocks use the upper entry
            idx[in1, a, b, 0] = fwd[in1] + a * rowlen[I[in1]] + b
            val[in1, a, b, 0] = np.where(off[in1], L[in1, a, b], L[in1, min(a, b), max(a, b)])
            # mirrored (J,b),(I,a) for A < B
            idx[in2, a, b, 1] = bwd[in2] + b * rowlen[J[in2]] + a
            val[in2, a, b, 1] = L[in2, a, b]
    idx, val = idx.ravel(), val.ravel()          # C order: t, row, a, b, copy
    keep = idx >= 0
    np.add.at(vals, idx[keep], val[keep])
    return vals


def assemble_lookup(prob, tabs, pattern, ctrl=None):
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    local = local_lookup(prob, tabs, ctrl, range(prob.n_tiles))
    return scatter(prob, pattern, local), local


# --------------------------------------------------------------------------
# standard quadrature K^• (and the Ā-form with an arbitrary macro field)
# --------------------------------------------------------------------------
def _tile_points(prob, n_g):
    """Per patch, per span: (ξ, D_T, G (n_act, n, d) ξ-gradients of the functions
    active on the span, w, active list)."""
    out = []
    for s in prob.tile:
        lst = []
        for sp in patch_spans(s):
            act = active_functions(s, sp)
            xi, DT, G, w = tile_point_data(s, sp, n_g)
            lst.append((xi, DT, G[act], w, act))
        out.append(lst)
    return out


def local_standard(prob, t, pairs, ctrl=None, n_g=None, pts=None):
    """K^• element matrices of tile t in the pair-row layout: (n_rows_tile, d, d)."""
    d = prob.d
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    n_g = prob.n_gauss if n_g is None else n_g
    pts = _tile_points(prob, n_g) if pts is None else pts
    lam, mu = M.lame(prob.young[t], prob.nu)
    blocks = []
    for p, s in enumerate(prob.tile):
        K = np.zeros((s.n_ctrl, s.n_ctrl, d, d))
        for xi, DT, G, w, act in pts[p]:
            JF = M.macro_jacobian(prob.macro, ctrl, t, xi)          # ∂x/∂ξ
            # ∇_x R = J_F⁻ᵀ ∇_ξ R  (G already = J_T⁻ᵀ ∇_θ R); det J = det J_F det J_T
            JFinv = np.linalg.inv(JF)                                 # [n, i, a]
            gx = np.einsum("nia,Ani->Ana", JFinv, G)
            wD = w * DT * np.linalg.det(JF)
            loc = lam * np.einsum("n,Ana,Bnb->ABab", wD, gx, gx)
            loc += mu * np.einsum("n,Anb,Bna->ABab", wD, gx, gx)
            loc += mu * np.einsum("n,Anc,Bnc->AB", wD, gx, gx)[:, :, None, None] * np.eye(d)
            K[np.ix_(act, act)] += loc
        blocks.append(K[pairs[p][:, 0], pairs[p][:, 1]])
    return np.concatenate(blocks, axis=0)


def local_quadrature_Aform(prob, t, pairs, A_at, n_g=None, pts=None):
    """Eq. 49 evaluated by tile quadrature with a macro field A_at(ξ) -> (n, d, d, d, d)."""
    d = prob.d
    n_g = prob.n_gauss if n_g is None else n_g
    pts = _tile_points(prob, n_g) if pts is None else pts
    blocks = []
    for p, s in enumerate(prob.tile):
        K = np.zeros((s.n_ctrl, s.n_ctrl, d, d))
        for xi, DT, G, w, act in pts[p]:
            A = A_at(xi)
            K[np.ix_(act, act)] += np.einsum("n,Ani,Bnj,nijab->ABab", w * DT, G, G, A, optimize=True)
        blocks.append(K[pairs[p][:, 0], pairs[p][:, 1]])
    return np.concatenate(blocks, axis=0)


def exact_field(prob, t, ctrl=None):
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    lam, mu = M.lame(prob.young[t], prob.nu)
    return lambda xi: M.A_closed(M.macro_jacobian(prob.macro, ctrl, t, xi), lam, mu)


def interpolated_field(prob, t, ctrl=None):
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    coef = M.tile_coefficients(prob, ctrl, t)
    return lambda xi: M.field_from_coefficients(coef, prob.q, xi)
