"""ORACLE (test infrastructure): sensitivity g[k, α] = uᵀ (∂K^π/∂P_{k,α}) v.

PAPER.md §4.1.2 (562-598): ∂W_int^π/∂m is an integral of adjoint fields
living in the projection space against d/dm Ā (Eqs. 70-71), whose Bézier
coefficients come from "the product of the lookup table ... and the
displacement DOF" (Eq. 73).  Here u ≠ v in general and the
differentiated quantity is the assembled K^π (reading R13):

  uᵀK^πv = Σ_t ⟨W_t, mat⟨Ā⟩_t(P)⟩,   W_t = mat𝔎ᵀ X_t,
  X_t[row][a,b] = coefficient of local[t,row][a,b] in uᵀK^πv under the
                  scatter of reading R9:
     A < B:  u_{I,a} v_{J,b} + u_{J,b} v_{I,a}
     A = B:  a < b: u_{I,a} v_{I,b} + u_{I,b} v_{I,a};  a = b: u_{I,a} v_{I,a};  a > b: 0

W_t does not depend on P, so g[k, α] = Σ_{t ∋ k} ∂/∂P_{k,α} ⟨W_t, coef_t(P)⟩,
evaluated by the complex step (exact to round-off):
  ∂f/∂P ≈ Im f(P + i h e_{k,α}) / h,  h = 1e-30.

`brute_complex_step` differentiates the whole assembled uᵀK^π(P)v (no adjoint)
for tiny problems; it pins the adjoint route in tests.
"""
from __future__ import annotations

import numpy as np

from . import macro as M
from .assemble import coef_matrix, local_lookup, scatter

H = 1e-30


def adjoint_X(prob, pattern, u, v, t):
    """X_t (n_rows_tile, d, d) for tile t."""
    d = prob.d
    I, J = pattern.I[t], pattern.J[t]
    uI = u.reshape(-1, d)[I]
    uJ = u.reshape(-1, d)[J]
    vI = v.reshape(-1, d)[I]
    vJ = v.reshape(-1, d)[J]
    X = np.einsum("ra,rb->rab", uI, vJ) + np.einsum("rb,ra->rab", uJ, vI)
    diag = I == J
    Xd = np.einsum("ra,rb->rab", uI[diag], vI[diag])
    Xd = Xd + np.swapaxes(Xd, 1, 2)
    Xd = np.triu(np.ones((d, d)), 0)[None] * Xd
    for a in range(d):
        Xd[:, a, a] *= 0.5
    X[diag] = Xd
    return X


def tile_W(prob, tabs, pattern, u, v, t):
    """W_t = mat𝔎ᵀ X_t (n_k × d²)."""
    d = prob.d
    X = adjoint_X(prob, pattern, u, v, t).reshape(-1, d * d)
    return tabs.T.T @ X


def macro_active(prob, t):
    return M._active(prob.macro, M.tile_element(prob.macro, t))


def sensitivity(prob, tabs, pattern, u, v, ctrl=None, entries=None, tiles=None):
    """g (n_cp, d).  `entries`: optional list of (k, α) to compute (others left 0);
    `tiles`: optional subset of tiles whose terms of Eq. 73's sum over t are taken."""
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    d = prob.d
    g = np.zeros_like(ctrl, dtype=np.float64)
    want = None if entries is None else set((int(k), int(a)) for k, a in entries)
    for t in (range(prob.n_tiles) if tiles is None else tiles):
        act = macro_active(prob, t)
        ent = [(k, a) for k in act for a in range(d) if want is None or (k, a) in want]
        if not ent:
            continue
        W = tile_W(prob, tabs, pattern, u, v, t)
        # one complex-step perturbed control net per entry (k, α), evaluated as a batch
        c = np.broadcast_to(ctrl.astype(np.complex128), (len(ent),) + ctrl.shape).copy()
        for n, (k, a) in enumerate(ent):
            c[n, k, a] += 1j * H
        coefs = M.tile_coefficients_batch(prob, c, t)
        for n, (k, a) in enumerate(ent):
            g[k, a] += np.imag(np.sum(W * coef_matrix(coefs[n]))) / H
    return g


def sensitivity_entrywise(prob, tabs, pattern, u, v, entries, ctrl=None):
    """The same complex step, one tile_coefficients call per (tile, k, α): pins the
    batched evaluation of `sensitivity`."""
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    g = np.zeros_like(ctrl, dtype=np.float64)
    want = set((int(k), int(a)) for k, a in entries)
    for t in range(prob.n_tiles):
        act = macro_active(prob, t)
        ent = [(k, a) for k in act for a in range(prob.d) if (k, a) in want]
        if not ent:
            continue
        W = tile_W(prob, tabs, pattern, u, v, t)
        for k, a in ent:
            c = ctrl.astype(np.complex128)
            c[k, a] += 1j * H
            g[k, a] += np.imag(np.sum(W * coef_matrix(M.tile_coefficients(prob, c, t)))) / H
    return g


def energy(prob, tabs, pattern, u, v, ctrl=None):
    """uᵀ K^π(P) v through the full assembly (complex-capable)."""
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    local = local_lookup(prob, tabs, ctrl, range(prob.n_tiles))
    vals = scatter(prob, pattern, local)
    col = pattern.col_idx()
    rows = np.repeat(np.arange(len(pattern.row_ptr) - 1), np.diff(pattern.row_ptr))
    return np.sum(u[rows] * vals * v[col])


def brute_complex_step(prob, tabs, pattern, u, v, entries, ctrl=None):
    """g[k, α] = Im uᵀK^π(P + i h e_{k,α})v / h through the whole assembly."""
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    out = []
    for k, a in entries:
        c = ctrl.astype(np.complex128)
        c[k, a] += 1j * H
        out.append(np.imag(energy(prob, tabs, pattern, u, v, c)) / H)
    return np.array(out)
