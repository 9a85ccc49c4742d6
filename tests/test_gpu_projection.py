"""GPU parity for SURVEY §8(f) N2 beyond the L2 projection: anisotropic projection spaces
(one degree per direction, the twist's p_π = 3, 3, 4 of P:524), the a-priori projection
error E_proj (Eq. 59, sampled as on P:362-364) and the adaptive degree selection (Eq. 65),
all through the C ABI against the oracle (and, for E_proj, a closed form)."""
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

TOL_TABLE, TOL_COEF, TOL_ELEM, TOL_K, TOL_SENS = 1e-13, 1e-12, 1e-12, 1e-11, 1e-11


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def kappa_tol(q, m=None):
    """Rounding bound of the projection inverse: 4 ε Π_k κ(Π1_k) (the 1D operator norms ×
    their inverses' norms), the same amplification the isotropic tests allow."""
    from oracle import macro as M
    from oracle.bspline import bernstein
    out = 1.0
    for k, qk in enumerate(q):
        mk = qk + 1 if m is None else m
        X, w = M.projection_nodes(mk, 1)
        N = bernstein(qk, X)
        out *= np.linalg.cond((N * w) @ N.T) if mk > qk + 1 else np.linalg.cond(N.T)
    return 4 * out * 2.0 ** -52


@pytest.mark.parametrize("c,kw", [
    (1, dict(q=(3, 1))),
    (2, dict(q=(1, 2, 3), n_el=(2, 2, 1))),
    (2, dict(q=(0, 2, 0), macro_kind="shear", n_el=(2, 2, 1))),
    (4, dict(q=(3, 3, 4), n_el=(2, 2, 2))),          # the twist's projection degrees
    (2, dict(q=(1, 2, 2), n_el=(2, 1, 1), n_proj=4)),  # anisotropic + the m-point L2 projection
])
def test_anisotropic_parity(c, kw):
    """Tables, coefficients, element matrices, K, the sensitivity, the matrix-free apply and
    the volume with one projection degree per direction, against the oracle."""
    from paper_2107_09568_b200 import Assembler
    from oracle import assemble as As, macro as M, sensitivity as S, volume as V
    from oracle.dofmap import DofMap, Pattern
    from synth import make_config, draw_uv_seeded
    kw = dict(kw)
    m = kw.pop("n_proj", 0)
    prob = make_config(c, **kw)
    if m:
        prob = dataclasses.replace(prob, n_proj=m)
    q = prob.q
    d = prob.d
    A = Assembler(prob)
    if m:
        A.set_projection(m)
    s = A.sizes
    assert list(s.q_dir)[:d] == list(q) and s.n_pi == int(np.prod([x + 1 for x in q]))
    assert list(s.m_dir)[:d] == ([m] * d if m else [x + 1 for x in q])
    tk = max(kappa_tol(q, m or None), 0.0)
    dev = torch.device("cuda")
    ctrl = torch.tensor(prob.macro.ctrl, device=dev)
    young = torch.tensor(prob.young, device=dev)
    tabs = As.Tables(prob)
    Tg = A.tables()
    off = 0
    for Tp, _ in tabs.per_patch:
        assert rel(Tg[off:off + len(Tp)], Tp) < TOL_TABLE
        off += len(Tp)
    coef = torch.zeros(s.n_tiles * d * d * s.k_stride, dtype=torch.float64, device=dev)
    A.interpolate(ctrl, young, prob.nu, coef)
    cg = coef.view(s.n_tiles, d * d, s.k_stride)[:, :, :s.n_k].cpu().numpy()
    for t in range(prob.n_tiles):
        ref = M.tile_coefficients(prob, prob.macro.ctrl, t)
        refm = np.transpose(ref, (3, 4, 1, 2, 0)).reshape(d * d, -1)
        assert rel(cg[t], refm) < max(TOL_COEF, tk), t
    dm = DofMap(prob)
    pt = Pattern(prob, dm, tabs.pairs)
    vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
    local = torch.empty(s.n_local_rows * s.n_tiles * d * d, dtype=torch.float64, device=dev)
    A.assemble(ctrl, young, prob.nu, vals, local)
    ref_vals, ref_local = As.assemble_lookup(prob, tabs, pt)
    L = local.view(s.n_local_rows, s.n_tiles, d, d).permute(1, 0, 2, 3).cpu().numpy()
    for t in range(prob.n_tiles):
        assert rel(L[t], ref_local[t]) < max(TOL_ELEM, tk), t
    assert rel(vals.cpu().numpy(), ref_vals) < max(TOL_K, tk)
    u, v = draw_uv_seeded(c + 40, s.n_dof)
    grad = torch.empty(s.n_macro_cp * d, dtype=torch.float64, device=dev)
    A.sensitivity(ctrl, young, prob.nu, torch.tensor(u, device=dev), torch.tensor(v, device=dev), grad)
    ref_g = S.sensitivity(prob, tabs, pt, u, v)
    assert rel(grad.cpu().numpy().reshape(-1, d), ref_g) < max(TOL_SENS, tk)
    y = torch.empty(s.n_dof, dtype=torch.float64, device=dev)
    A.apply(ctrl, young, prob.nu, torch.tensor(u, device=dev), y)
    import scipy.sparse as sp
    Kref = sp.csr_matrix((ref_vals, pt.col_idx(), pt.row_ptr), shape=(s.n_dof, s.n_dof))
    assert rel(y.cpu().numpy(), Kref @ u) < max(TOL_K, tk)
    vol = A.volume(ctrl)
    assert abs(vol - V.volume_lookup(prob)) < max(1e-13, tk) * vol


def test_anisotropic_shear_exact_against_standard():
    """The shear macro's Ā ∈ Q_{0,2,0}: the GPU K^π at q = (0, 2, 0) equals the oracle's
    standard quadrature K^• to round-off; at q = (2, 1, 2) it does not."""
    from paper_2107_09568_b200 import Assembler
    from oracle import assemble as As
    from synth import make_config
    for q, exact in (((0, 2, 0), True), ((2, 1, 2), False)):
        prob = make_config(2, macro_kind="shear", n_el=(2, 2, 1), q=q)
        A = Assembler(prob)
        s = A.sizes
        d = prob.d
        dev = torch.device("cuda")
        vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
        local = torch.empty(s.n_local_rows * s.n_tiles * d * d, dtype=torch.float64, device=dev)
        A.assemble(torch.tensor(prob.macro.ctrl, device=dev), torch.tensor(prob.young, device=dev), prob.nu, vals, local)
        tabs = As.Tables(prob)
        L = local.view(s.n_local_rows, s.n_tiles, d, d).permute(1, 0, 2, 3).cpu().numpy()
        std = np.stack([As.local_standard(prob, t, tabs.pairs) for t in range(prob.n_tiles)])
        err = rel(L, std)
        assert (err < 1e-13) if exact else (err > 1e-8), (q, err)


# ---------------------------------------------------------------------------
# E_proj (Eq. 59) and the degree selection (Eq. 65)

@pytest.mark.parametrize("c,kw,q,n_s,m_extra", [
    (1, {}, 2, 8, 0),
    (1, {}, (3, 1), 5, 0),
    (1, {}, (2, 2), 6, 2),                             # the L2 projection with q+3 points
    (2, dict(n_el=(2, 2, 1)), (1, 2, 3), 5, 0),
    (3, dict(n_el=(2, 2, 2), macro_kind="nurbs"), 2, 6, 0),   # rational F (N4)
    (4, dict(n_el=(2, 2, 2)), (3, 3, 4), 4, 0),
])
def test_projection_error_parity(c, kw, q, n_s, m_extra):
    from paper_2107_09568_b200 import projection_error
    from oracle import projection as PE
    from synth import make_config
    prob = make_config(c, **kw)
    d = prob.d
    qv = (q,) * d if np.ndim(q) == 0 else q
    e_tile = np.zeros(prob.n_tiles)
    e = projection_error(prob.macro, q, prob.nu, n_samples=n_s, m_extra=m_extra, e_tile=e_tile)
    m = 0 if m_extra == 0 else tuple(x + 1 + m_extra for x in qv)
    e_ref, per = PE.projection_error(prob, q, n_s, m=m)
    # |Δe| ≲ (rounding of Ā − Π Ā) / ‖Ā‖: a few ε κ(Π) per component
    tol = 10 * kappa_tol(qv) + 1e-14
    assert np.abs(e_tile - per).max() < tol, np.abs(e_tile - per).max()
    assert e == e_tile.max() and abs(e - e_ref) < tol
    # device output pointer
    et = torch.zeros(prob.n_tiles, dtype=torch.float64, device="cuda")
    projection_error(prob.macro, q, prob.nu, n_samples=n_s, m_extra=m_extra, e_tile=et)
    assert np.array_equal(et.cpu().numpy(), e_tile)


def test_projection_error_closed_form_stretch():
    """The stretch map F = (h0(ξ0 + κξ0²), h1 ξ1): the GPU E_proj against the closed form of
    tests/test_oracle_projection.py (divided differences of 1/(1+cx))."""
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_oracle_projection import stretch_closed_form, stretch_problem
    from paper_2107_09568_b200 import projection_error
    for kappa, q, n_s in ((0.2, (1, 0), 5), (0.4, (2, 1), 8), (0.3, (4, 2), 6), (0.25, (0, 0), 5)):
        prob = stretch_problem(kappa)
        e = projection_error(prob.macro, q, prob.nu, n_samples=n_s)
        ref = stretch_closed_form(kappa, q[0], n_s, prob.nu)
        assert abs(e - ref) <= 1e-9 * ref + 1e-14, (q, e, ref)


def test_select_degree_parity():
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_oracle_projection import stretch_closed_form, stretch_problem
    from paper_2107_09568_b200 import select_degree, IgaError
    from oracle import projection as PE
    from synth import make_config
    prob = make_config(1, n_el=(2, 2))
    for tol in (1e-3, 0.5, 1e-4):
        q, e = select_degree(prob.macro, prob.nu, tol, n_samples=6)
        q_ref, e_ref = PE.select_degree(prob, tol, n_s=6)
        assert q == q_ref and abs(e - e_ref) < 1e-12, (tol, q, q_ref)
    sp = stretch_problem(0.45)
    E = {q0: stretch_closed_form(0.45, q0, 8, sp.nu) for q0 in range(0, 6)}
    for q0 in (1, 2, 4):
        tol = float(np.sqrt(E[q0] * E[q0 - 1]))
        q, e = select_degree(sp.macro, sp.nu, tol, n_samples=8)
        assert q == (q0, max(q0 - 1, 0)) and abs(e - E[q0]) <= 1e-9 * E[q0]
    with pytest.raises(IgaError, match="ELIMIT"):
        select_degree(prob.macro, prob.nu, 1e-14, n_samples=6)      # unreachable below q_max = 4
    with pytest.raises(IgaError, match="EINVAL"):
        select_degree(prob.macro, prob.nu, 1e-3, n_samples=1)


def test_projection_error_rejects_bad_arguments():
    from paper_2107_09568_b200 import projection_error, IgaError
    from synth import make_config
    prob = make_config(2, n_el=(2, 1, 1))
    with pytest.raises(IgaError, match="EINVAL"):
        projection_error(prob.macro, (1, 5, 1), prob.nu)              # q > 4
    with pytest.raises(IgaError, match="EINVAL"):
        projection_error(prob.macro, 2, 0.5)                           # ν outside (-1, 0.5)
    with pytest.raises(IgaError, match="EINVAL"):
        projection_error(prob.macro, 2, prob.nu, n_samples=9)
