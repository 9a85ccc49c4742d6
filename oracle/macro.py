"""ORACLE (test infrastructure): macro scale — Jacobian of F, macro field Ā,
interpolation onto the Bernstein space Q_q.

Ā_ij (Eq. 37; App. A.2 Eqs. 89-97) is
computed by three independent routes:
  A_closed  Ā_ij[a,b] = D (λ ǧ_i[a] ǧ_j[b] + μ ǧ_j[a] ǧ_i[b] + μ (ǧ_i·ǧ_j) δ_ab),
            ǧ_i = row i of J⁻¹ (contravariant vectors, Eqs. 80-81), D = det J
  A_voigt   Ā_ij = Ĝ_i Č Ĝ_jᵀ |det J| with Ĝ_i from Eq. 91 and Č from Eq. 84a / 93
  A_tensor  Ā_ij[a,b] = D Σ_kl J⁻¹[i,k] C[a,k,b,l] J⁻¹[j,l] (isotropic C)
Entry (a,b) multiplies u_a (trial, derivative ξ_i) against v_b (test,
derivative ξ_j): K_AB[a,b] = Σ_ij ∫ ∂_iR_A ∂_jR_B Ā_ij[a,b] (Eq. 49).

Interpolation (reading R1): the paper L2-projects (Eqs. 20-24, 42);
BASELINE.json mandates interpolation.  The oracle interpolates at the (q+1)^d
tensor Gauss–Legendre nodes by solving the full tensor Vandermonde system
V c = s (V[m, C] = N_C(x_m)); this equals the L2 projection with a
(q+1)-point Gauss right-hand side (pinned in tests).

J is ∂F/∂ξ in the element-local frame ξ ∈ [0,1]^d (Eq. 7):
∂F/∂u times the knot-span lengths (reading R4).
"""
from __future__ import annotations

import numpy as np

from .bspline import basis_1d, bernstein, elements_of, gauss_01, multi_index, qvec


def lame(E, nu):
    """λ = Eν/((1+ν)(1-2ν)), μ = E/(2(1+ν)) (plane strain in 2D, reading R11)."""
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    return lam, mu


# --------------------------------------------------------------------------
# macro map evaluation in the element-local frame
# --------------------------------------------------------------------------
def element_grid(macro):
    """Elements per direction (non-degenerate spans) of the macro patch."""
    return [elements_of(U) for U in macro.knots]


def tile_element(macro, t):
    """Tile t <-> macro element (e0, e1[, e2]) flattened direction-0 fastest (reading R9)."""
    els = element_grid(macro)
    n = [len(e) for e in els]
    ee = multi_index(n, t)
    return tuple(els[k][ee[k]] for k in range(len(n)))


def _active(macro, spans):
    """Macro control points whose basis function is nonzero on the element: span-p..span."""
    import itertools
    n = macro.n_per_dir
    rng = [range(spans[k] - macro.degree[k], spans[k] + 1) for k in range(macro.dim)]
    out = []
    for ii in itertools.product(*reversed(rng)):
        ii = tuple(reversed(ii))
        A = 0
        for k in reversed(range(macro.dim)):
            A = A * n[k] + ii[k]
        out.append(A)
    return out


def macro_jacobian(macro, ctrl, t, xi):
    """J[a, k] = ∂F_a/∂ξ_k at element-local points xi (n_pts, d) of tile t.

    F(u) = Σ_i R_i^H(u) m_i (Eq. 4); u_k = U_k[s_k] + h_k ξ_k; ∂/∂ξ_k = h_k ∂/∂u_k.
    NURBS (macro.weights, NEXT N4): R_i = w_i N_i / W with W = Σ_j w_j N_j, so
    ∂_k R_i = w_i (∂_k N_i W - N_i ∂_k W) / W².
    `ctrl` may be complex (complex-step sensitivity) and may carry leading batch axes
    (..., n_cp, d) — one control net per batch entry, e.g. one complex-step
    perturbation each.  Returns (..., n_pts, d, d)."""
    d = macro.dim
    spans = tile_element(macro, t)
    vals, ders = [], []
    for k in range(d):
        U = macro.knots[k]
        s = spans[k]
        h = U[s + 1] - U[s]
        u = U[s] + h * xi[:, k]
        N, dN = basis_1d(U, macro.degree[k], s, u)
        vals.append(N)
        ders.append(dN * h)
    n = macro.n_per_dir
    act = _active(macro, spans)               # basis functions nonzero on the element
    Nt, dNt = {}, {}
    for A in act:                             # tensor-product N_A and ∂_k N_A
        ii = multi_index(n, A)
        Nt[A] = np.prod([vals[m][ii[m]] for m in range(d)], axis=0)
        dNt[A] = [np.prod([ders[m][ii[m]] if m == k else vals[m][ii[m]] for m in range(d)], axis=0)
                  for k in range(d)]
    w = getattr(macro, "weights", None)
    if w is not None:
        W = sum(w[A] * Nt[A] for A in act)
        dW = [sum(w[A] * dNt[A][k] for A in act) for k in range(d)]
    ctrl = np.asarray(ctrl)
    J = np.zeros(ctrl.shape[:-2] + (xi.shape[0], d, d), dtype=np.result_type(ctrl, np.float64))
    for A in act:
        for k in range(d):
            g = dNt[A][k] if w is None else w[A] * (dNt[A][k] * W - Nt[A] * dW[k]) / W ** 2
            J[..., :, :, k] += g[:, None] * ctrl[..., A, None, :]
    return J


def macro_position(macro, ctrl, t, xi):
    """F at element-local points xi of tile t (used by the energy-identity pin)."""
    d = macro.dim
    spans = tile_element(macro, t)
    vals = []
    for k in range(d):
        U = macro.knots[k]
        s = spans[k]
        u = U[s] + (U[s + 1] - U[s]) * xi[:, k]
        vals.append(basis_1d(U, macro.degree[k], s, u)[0])
    n = macro.n_per_dir
    X = np.zeros((xi.shape[0], d))
    w = getattr(macro, "weights", None)
    W = 0.0
    if w is not None:
        for A in _active(macro, spans):
            ii = multi_index(n, A)
            W = W + w[A] * np.prod([vals[m][ii[m]] for m in range(d)], axis=0)
    for A in _active(macro, spans):
        ii = multi_index(n, A)
        g = np.ones(xi.shape[0]) if w is None else w[A] / W
        for m in range(d):
            g = g * vals[m][ii[m]]
        X += g[:, None] * ctrl[A][None, :]
    return X


# --------------------------------------------------------------------------
# macro field Ā (three routes)
# --------------------------------------------------------------------------
def _det_inv(J):
    D = np.linalg.det(J)
    G = np.linalg.inv(J)          # G[i, a] = ǧ_i[a] (row i of J⁻¹)
    return D, G


def A_closed(J, lam, mu):
    """Closed form of Eq. 37 (derivation in DESIGN.md §2).
    J (..., d, d) -> A (..., d, d, d, d) indexed [i, j, a, b]."""
    D, G = _det_inv(J)
    d = J.shape[-1]
    lam = np.asarray(lam)[..., None, None, None, None] if np.ndim(lam) else lam
    mu = np.asarray(mu)[..., None, None, None, None] if np.ndim(mu) else mu
    GiGj = np.einsum("...ia,...jb->...ijab", G, G)
    GjGi = np.einsum("...ja,...ib->...ijab", G, G)
    gg = np.einsum("...ic,...jc->...ij", G, G)
    eye = np.eye(d)
    A = lam * GiGj + mu * GjGi + mu * np.einsum("...ij,ab->...ijab", gg, eye)
    return D[..., None, None, None, None] * A


def _voigt_pairs(d):
    return [(0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1)] if d == 3 else [(0, 0), (1, 1), (0, 1)]


def A_voigt(J, lam, mu):
    """Paper route (App. A.2): Ā_ij = Ĝ_i Č Ĝ_jᵀ |det J| (Eq. 37, 97).

    ĝ_k = column k of J (Eq. 79); ǧ^{kl} = [ĝ_k·ĝ_l]⁻¹ (Eq. 81);
    Č_{ijkl} = λ ǧ^{ij} ǧ^{kl} + μ (ǧ^{ik} ǧ^{jl} + ǧ^{il} ǧ^{jk}) (Eq. 84a) in
    Voigt order (11,22,33,23,13,12) (Eq. 93); Ĝ_i (d × n_v) has column v equal
    to ĝ_l if Voigt pair v = {i, l} (l ≠ i or l = i), else 0 (Eq. 91)."""
    J = np.asarray(J)
    d = J.shape[-1]
    pairs = _voigt_pairs(d)
    nv = len(pairs)
    gcov = np.swapaxes(J, -1, -2)                     # gcov[..., k, :] = ĝ_k
    metric = np.einsum("...ka,...la->...kl", gcov, gcov)
    gcon = np.linalg.inv(metric)
    C = np.zeros(J.shape[:-2] + (nv, nv), dtype=J.dtype)
    for v, (i, j) in enumerate(pairs):
        for w, (k, l) in enumerate(pairs):
            C[..., v, w] = lam * gcon[..., i, j] * gcon[..., k, l] + mu * (
                gcon[..., i, k] * gcon[..., j, l] + gcon[..., i, l] * gcon[..., j, k])
    Gh = np.zeros(J.shape[:-2] + (d, d, nv), dtype=J.dtype)   # Gh[..., i, :, v] = Ĝ_i column v
    for i in range(d):
        for v, (a, b) in enumerate(pairs):
            if a == i:
                Gh[..., i, :, v] = gcov[..., b, :]
            elif b == i:
                Gh[..., i, :, v] = gcov[..., a, :]
    D = np.abs(np.linalg.det(J))
    A = np.einsum("...iav,...vw,...jbw->...ijab", Gh, C, Gh)
    return D[..., None, None, None, None] * A


def A_tensor(J, lam, mu):
    """Third route: Ā_ij[a,b] = D Σ_kl J⁻¹[i,k] C_{akbl} J⁻¹[j,l] with the isotropic
    C_{akbl} = λ δ_ak δ_bl + μ (δ_ab δ_kl + δ_al δ_kb)."""
    D, G = _det_inv(J)
    d = J.shape[-1]
    e = np.eye(d)
    C = lam * np.einsum("ak,bl->akbl", e, e) + mu * (np.einsum("ab,kl->akbl", e, e) + np.einsum("al,kb->akbl", e, e))
    return D[..., None, None, None, None] * np.einsum("...ik,akbl,...jl->...ijab", G, C, G)


# --------------------------------------------------------------------------
# interpolation onto Q_q (reading R1)
# --------------------------------------------------------------------------
def interp_nodes(q, d):
    """Π_k (q_k+1) tensor Gauss–Legendre nodes on [0,1]^d (q_k+1 per direction k),
    direction-0 fastest, ascending; q an int or per-direction degrees."""
    return projection_nodes(tuple(x + 1 for x in qvec(q, d)), d)[0]


def interpolate(samples, q, d):
    """Coefficients c_C with Σ_C c_C N_C(x_m) = samples[m] at the interpolation
    nodes: solves V c = s, V[m, C] = N_C(x_m) (plain definition).
    samples: (n_pi, ...) -> coefficients (n_pi, ...)."""
    V = bernstein(q, interp_nodes(q, d)).T      # (m, C)
    s = np.asarray(samples)
    flat = s.reshape(s.shape[0], -1)
    c = np.linalg.solve(V.astype(np.result_type(flat, np.float64)), flat)
    return c.reshape(s.shape)


def projection_nodes(m, d):
    """Tensor Gauss–Legendre nodes on [0,1]^d with m_k points in direction k (m an int or
    per-direction counts; direction-0 fastest) and their weights."""
    mv = qvec(m, d)
    rules = [gauss_01(mk) for mk in mv]
    n = int(np.prod(mv))
    pts = np.zeros((n, d))
    w = np.ones(n)
    for i in range(n):
        r = i
        for k in range(d):
            pts[i, k] = rules[k][0][r % mv[k]]
            w[i] *= rules[k][1][r % mv[k]]
            r //= mv[k]
    return pts, w


def project_l2(samples, q, d, m):
    """L2 projection onto Q_q (Eqs. 23-24): M_π d = r_π with [M_π]_kl = ∫ N_k N_l and
    (r_π)_k = ∫ N_k f, both integrated by the m-point Gauss rule per direction (q, m ints
    or per-direction); samples = f at projection_nodes(m, d).  Plain definition (full
    tensor mass matrix)."""
    X, w = projection_nodes(m, d)
    N = bernstein(q, X)                          # (C, m^d)
    Mpi = (N * w) @ N.T
    s = np.asarray(samples)
    flat = s.reshape(s.shape[0], -1)
    r = (N * w).astype(np.result_type(flat, np.float64)) @ flat
    c = np.linalg.solve(Mpi.astype(r.dtype), r)
    return c.reshape((N.shape[0],) + s.shape[1:])


def tile_coefficients(prob, ctrl, t, E=None, route=A_closed, m=None):
    """⟨Ā_ij⟩_C for tile t (Eq. 42): shape (n_pi, d, d, d, d) indexed [C, i, j, a, b].
    m (default prob.n_proj, 0 -> q+1): Gauss points per direction of the projection; q+1
    is interpolation at the Gauss nodes (reading R1), larger m the L2 projection of
    Eqs. 23-24 with that rule (NEXT N2).  Raises if det J <= 0 at a node (reading R5)."""
    d = prob.d
    E = prob.young[t] if E is None else E
    lam, mu = lame(E, prob.nu)

    def field(X):
        J = macro_jacobian(prob.macro, ctrl, t, X)
        if np.any(np.real(np.linalg.det(J)) <= 0):
            raise ValueError(f"degenerate macro element: tile {t}")
        return route(J, lam, mu)
    return project_field(field, prob.q, d, m or getattr(prob, "n_proj", 0))


def tile_coefficients_batch(prob, ctrls, t, E=None, route=A_closed, m=None):
    """tile_coefficients for a batch of control nets ctrls (B, n_cp, d) of the same tile:
    (B, n_pi, d, d, d, d).  The same arithmetic per batch entry (the batch rides along as
    extra columns of the projection's right-hand side); used by the complex-step
    sensitivity, one perturbed net per (k, α)."""
    d = prob.d
    E = prob.young[t] if E is None else E
    lam, mu = lame(E, prob.nu)

    def field(X):
        J = macro_jacobian(prob.macro, ctrls, t, X)             # (B, n, d, d)
        if np.any(np.real(np.linalg.det(J)) <= 0):
            raise ValueError(f"degenerate macro element: tile {t}")
        return np.moveaxis(route(J, lam, mu), 1, 0)              # (n, B, d, d, d, d)
    return np.moveaxis(project_field(field, prob.q, d, m or getattr(prob, "n_proj", 0)), 0, 1)


def projection_points(q, d, m=0):
    """m per direction: 0 -> q_k+1 (interpolation, R1); else m (>= q_k+1) points per
    direction for every k.  Returns (per-direction counts, interpolation?)."""
    qv = qvec(q, d)
    mv = tuple(x + 1 for x in qv) if not m else qvec(m, d)
    if any(mk < qk + 1 for mk, qk in zip(mv, qv)):
        raise ValueError(f"projection points {mv} < q+1 = {tuple(x + 1 for x in qv)}")
    return mv, all(mk == qk + 1 for mk, qk in zip(mv, qv))


def project_field(f, q, d, m=0, check_tile=None, ctrl=None, macro=None):
    """Π^H f (Eq. 20) for f evaluated at sample points X (n, d) -> (n, ...): interpolation
    at the Gauss nodes when every m_k = q_k+1 (R1), else the Gauss-discretised L2
    projection of Eqs. 23-24.  Raises on det J <= 0 at a node of tile check_tile (R5)."""
    mv, interp = projection_points(q, d, m)
    X = projection_nodes(mv, d)[0]
    if check_tile is not None:
        J = macro_jacobian(macro, ctrl, check_tile, X)
        if np.any(np.real(np.linalg.det(J)) <= 0):
            raise ValueError(f"degenerate macro element: tile {check_tile}")
    A = f(X)
    return interpolate(A, q, d) if interp else project_l2(A, q, d, mv)


def field_from_coefficients(coef, q, xi):
    """Π_q Ā at points xi: Σ_C N_C(ξ) coef[C] (Eq. 42)."""
    N = bernstein(q, xi)                        # (C, n_pts)
    return np.einsum("cp,c...->p...", N, coef)
