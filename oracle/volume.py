"""ORACLE (test infrastructure): volume, volume gradient and body-force load vector by
lookup (§3.1, Eqs. 14-19, 25-26; §3.3 Eq. 53 body part; §4.1 Eqs. 66-67) and
by standard composed-map quadrature (Eq. 14 itself).  SURVEY §8(f) N3.

  t^h_C       = ∫_{Ω̄_T} |det J_T| (N_C ∘ 𝒯) dθ                           (Eq. 18)
  𝔉[A][C]     = ∫_{Ω̄_T} R_A |det J_T| (N_C ∘ 𝒯) dθ   (per tile patch)        (Eq. 53)
  d^(t)       = Π^H |det J_ℳ(t)| coefficients (interpolation, or the L2 projection
                of Eqs. 23-24 with m points)                                 (Eq. 15)
  V^π         = Σ_t t^h · d^(t)                                              (Eq. 19)
  f_{node(t,A), a} += b_a Σ_C 𝔉[A][C] d^(t)_C      (constant body force b)    (Eq. 53)
  dV^π/dP     by complex step of V^π (Eqs. 66-67 are its adjoint form).
Only the tests, smoke() and bench's cpu legs may import this.
"""
from __future__ import annotations

import numpy as np

from . import macro as M
from .bspline import bernstein, n_pi, tensor_basis
from .tables import gauss_points_span, patch_spans

H = 1e-30


def _span_data(spline, s, n_g):
    th, w = gauss_points_span(spline, s, n_g)
    R, dR = tensor_basis(spline, s, th)
    xi = R.T @ spline.ctrl
    JT = np.einsum("kAn,Aa->nak", dR, spline.ctrl)
    DT = np.linalg.det(JT)
    if np.any(DT <= 0):
        raise ValueError("degenerate tile Jacobian")
    return R, xi, DT, w


def volume_table(prob):
    """t^h (n_π): Eq. 18, summed over the tile patches."""
    t = 0.0
    for sp in prob.tile:
        for s in patch_spans(sp):
            _, xi, DT, w = _span_data(sp, s, prob.n_gauss)
            t = t + bernstein(prob.q, xi) @ (w * DT)
    return np.asarray(t)


def load_tables(prob):
    """𝔉 per patch (n_ctrl_p, n_π): Eq. 53's body-force integrals, stacked over patches
    in the tile-local control-point order."""
    out = []
    for sp in prob.tile:
        F = np.zeros((sp.ctrl.shape[0], n_pi(prob.q, prob.d)))
        for s in patch_spans(sp):
            R, xi, DT, w = _span_data(sp, s, prob.n_gauss)
            F += (R * (w * DT)) @ bernstein(prob.q, xi).T
        out.append(F)
    return np.concatenate(out, axis=0)


def det_coefficients(prob, ctrl, t, m=None):
    """d^(t): projection coefficients of |det J_ℳ(t)| (Eq. 15; interpolation at the
    q+1 Gauss nodes, reading R1, or the m-point L2 projection of Eqs. 23-24)."""
    def det(X):
        D = np.linalg.det(M.macro_jacobian(prob.macro, ctrl, t, X))
        if np.any(np.real(D) <= 0):
            raise ValueError(f"degenerate macro element: tile {t}")
        return D
    return M.project_field(det, prob.q, prob.d, m or getattr(prob, "n_proj", 0))


def volume_lookup(prob, ctrl=None, tiles=None, th=None):
    """V^π = Σ_t t^h · d^(t) (Eq. 19)."""
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    th = volume_table(prob) if th is None else th
    return sum(th @ det_coefficients(prob, ctrl, t) for t in (range(prob.n_tiles) if tiles is None else tiles))


def volume_standard(prob, ctrl=None, n_g=None, tiles=None):
    """V = Σ_t ∫ |det J_T| |det J_ℳ(t) ∘ 𝒯| dθ by Gauss quadrature of the composed map
    (Eq. 14)."""
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    n_g = n_g or prob.n_gauss
    V = 0.0
    for sp in prob.tile:
        for s in patch_spans(sp):
            _, xi, DT, w = _span_data(sp, s, n_g)
            for t in (range(prob.n_tiles) if tiles is None else tiles):
                V += np.sum(w * DT * np.linalg.det(M.macro_jacobian(prob.macro, ctrl, t, xi)))
    return V


def volume_gradient(prob, ctrl=None, tiles=None):
    """dV^π/dP (n_cp, d) by complex step (h = 1e-30) of V^π."""
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    th = volume_table(prob)
    tiles = list(range(prob.n_tiles)) if tiles is None else list(tiles)
    g = np.zeros(ctrl.shape)
    for t in tiles:
        for k in M._active(prob.macro, M.tile_element(prob.macro, t)):
            for a in range(prob.d):
                c = ctrl.astype(np.complex128)
                c[k, a] += 1j * H
                g[k, a] += np.imag(th @ det_coefficients(prob, c, t)) / H
    return g


def load_vector(prob, node, n_nodes, b, ctrl=None, tiles=None):
    """f (n_nodes, d) for a constant body force b (Eq. 53): the tile contributions
    b ⊗ (𝔉 d^(t)) added at node[t][A] (np.add.at)."""
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    F = load_tables(prob)
    f = np.zeros((n_nodes, prob.d))
    for t in (range(prob.n_tiles) if tiles is None else tiles):
        s = F @ det_coefficients(prob, ctrl, t)
        np.add.at(f, node[t], s[:, None] * np.asarray(b)[None, :])
    return f


def load_standard(prob, node, n_nodes, b, ctrl=None):
    """f by quadrature of the composed map: ∫ R_A b |det J_T| |det J_ℳ ∘ 𝒯| dθ."""
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    f = np.zeros((n_nodes, prob.d))
    off = np.cumsum([0] + [sp.ctrl.shape[0] for sp in prob.tile])
    for p, sp in enumerate(prob.tile):
        for s in patch_spans(sp):
            R, xi, DT, w = _span_data(sp, s, prob.n_gauss)
            for t in range(prob.n_tiles):
                dm = np.linalg.det(M.macro_jacobian(prob.macro, ctrl, t, xi))
                np.add.at(f, node[t][off[p]:off[p + 1]], (R @ (w * DT * dm))[:, None] * np.asarray(b)[None, :])
    return f
