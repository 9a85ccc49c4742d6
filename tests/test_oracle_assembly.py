"""Pins for oracle/assemble.py: lookup K^π (Eqs. 50, 58) vs the standard
full-Gauss K^• (Eq. 49) and the global-matrix invariants."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import assemble as As
from oracle import macro as M
from oracle.dofmap import DofMap, Pattern
from synth import Problem, Spline, make_config


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def csr(ob, vals):
    pt, n = ob["pattern"], ob["dm"].n_dof
    return sp.csr_matrix((vals, pt.col_idx(), pt.row_ptr), shape=(n, n))


def standard_all(ob, **kw):
    prob, tabs = ob["prob"], ob["tabs"]
    pts = As._tile_points(prob, kw.pop("n_g", prob.n_gauss))
    return np.stack([As.local_standard(prob, t, tabs.pairs, pts=pts, **kw) for t in range(prob.n_tiles)])


@pytest.mark.parametrize("c,kw", [(1, dict(macro_amp=0.0)), (2, dict(macro_amp=0.0, n_el=(2, 2, 1)))])
def test_affine_macro_lookup_equals_standard(c, kw, oracle_problem):
    """F affine per element -> Ā constant -> Π_qĀ = Ā -> K^π = K^• to round-off (SPEC.md:654 A3)."""
    ob = oracle_problem(c, **kw)
    vals, local = As.assemble_lookup(ob["prob"], ob["tabs"], ob["pattern"])
    std = standard_all(ob)
    assert rel(local, std) < 1e-13
    assert rel(vals, As.scatter(ob["prob"], ob["pattern"], std)) < 1e-13


@pytest.mark.parametrize("c,kw", [(1, dict(macro_kind="shear")), (2, dict(macro_kind="shear", n_el=(2, 2, 1)))])
def test_shear_macro_exact_at_q2_not_q1(c, kw, oracle_problem):
    """F = (a ξ0 + κ ξ1², b ξ1, c ξ2): det J constant, Ā ∈ Q_2 -> exact at q = 2 (reading R2)."""
    ob = oracle_problem(c, **kw)
    _, local = As.assemble_lookup(ob["prob"], ob["tabs"], ob["pattern"])
    std = standard_all(ob)
    assert rel(local, std) < 1e-13
    ob1 = oracle_problem(c, q=1, **kw)
    _, local1 = As.assemble_lookup(ob1["prob"], ob1["tabs"], ob1["pattern"])
    std1 = standard_all(ob1)
    assert rel(local1, std1) > 1e-8


@pytest.mark.parametrize("c,kw", [(1, dict(macro_kind="shear", q=(0, 2))),
                                  (2, dict(macro_kind="shear", n_el=(2, 2, 1), q=(0, 2, 0)))])
def test_shear_macro_exact_at_anisotropic_q(c, kw, oracle_problem):
    """The shear Ā depends on ξ1 only, quadratically: exact in the anisotropic space
    Q_{0,2(,0)} (n_π = 3) and not in Q_{2,1(,2)}."""
    ob = oracle_problem(c, **kw)
    _, local = As.assemble_lookup(ob["prob"], ob["tabs"], ob["pattern"])
    assert rel(local, standard_all(ob)) < 1e-13
    q_bad = (2, 1) if c == 1 else (2, 1, 2)
    ob1 = oracle_problem(c, **dict(kw, q=q_bad))
    _, local1 = As.assemble_lookup(ob1["prob"], ob1["tabs"], ob1["pattern"])
    assert rel(local1, standard_all(ob1)) > 1e-8


@pytest.mark.parametrize("c,t,q", [(1, 5, None), (3, 0, None), (1, 6, (3, 1)), (2, 3, (1, 2, 3))])
def test_lookup_equals_quadrature_with_interpolated_field(c, t, q, oracle_problem):
    """For ANY F, K^π equals the tile quadrature of Eq. 49 with Π_qĀ in place of Ā
    (also for anisotropic projection spaces)."""
    kw = dict(n_el=(2, 1, 1)) if c == 3 else (dict(n_el=(2, 2, 1)) if c == 2 else {})
    if q is not None:
        kw["q"] = q
    ob = oracle_problem(c, **kw)
    prob, tabs = ob["prob"], ob["tabs"]
    local = As.local_lookup(prob, tabs, prob.macro.ctrl, [t])[0]
    ref = As.local_quadrature_Aform(prob, t, tabs.pairs, As.interpolated_field(prob, t))
    assert rel(local, ref) < 1e-13
    # and the Ā-form with the exact field equals the physical (λ, μ) form of K^•
    ex = As.local_quadrature_Aform(prob, t, tabs.pairs, As.exact_field(prob, t))
    assert rel(ex, As.local_standard(prob, t, tabs.pairs)) < 1e-13


def test_global_invariants_cfg1(oracle_problem):
    ob = oracle_problem(1)
    prob, dm = ob["prob"], ob["dm"]
    vals, _ = As.assemble_lookup(prob, ob["tabs"], ob["pattern"])
    K = csr(ob, vals)
    assert (K != K.T).nnz == 0                         # bitwise symmetric
    n = dm.n_nodes
    scale = abs(K).max()
    for a in range(prob.d):
        tr = np.zeros((n, prob.d))
        tr[:, a] = 1
        assert np.abs(K @ tr.ravel()).max() < 1e-13 * scale * 10
    r = np.random.default_rng(0).standard_normal(dm.n_dof)
    assert r @ (K @ r) > 0


def _node_positions(ob, ctrl=None):
    """Physical image F(t_A) of each node (affine F: linear fields are in the space)."""
    prob, dm = ob["prob"], ob["dm"]
    ctrl = prob.macro.ctrl if ctrl is None else ctrl
    X = np.zeros((dm.n_nodes, prob.d))
    for t in range(prob.n_tiles):
        for p, s in enumerate(prob.tile):
            X[dm.node[t, dm.offsets[p]:dm.offsets[p + 1]]] = M.macro_position(prob.macro, ctrl, t, s.ctrl)
    return X


def test_rotation_kernel_only_for_affine(oracle_problem):
    """D3: rotations are annihilated iff F is affine per element (non-isoparametric space)."""
    for amp, expect_zero in [(0.0, True), (None, False)]:
        ob = oracle_problem(1, macro_amp=amp)
        vals, _ = As.assemble_lookup(ob["prob"], ob["tabs"], ob["pattern"])
        K = csr(ob, vals)
        X = _node_positions(ob)
        rot = np.stack([-X[:, 1], X[:, 0]], axis=1).ravel()
        r = np.abs(K @ rot).max() / (abs(K).max() * np.abs(rot).max())
        assert (r < 1e-13) == expect_zero, r


def test_linear_field_energy_identity(oracle_problem):
    """Affine F: u(x) = G x is exactly representable; uᵀK^•u = (λ tr(ε)² + 2μ ε:ε)·|Ω|
    with |Ω| = Σ_t Σ_g w det J_T det J_F computed by the same tile quadrature."""
    ob = oracle_problem(1, macro_amp=0.0)
    prob, tabs = ob["prob"], ob["tabs"]
    std = standard_all(ob)
    K = csr(ob, As.scatter(prob, ob["pattern"], std))
    X = _node_positions(ob)
    G = np.array([[0.3, -0.7], [0.2, 0.5]])
    u = (X @ G.T).ravel()
    eps = 0.5 * (G + G.T)
    lam, mu = M.lame(1.0, prob.nu)
    dens = lam * np.trace(eps) ** 2 + 2 * mu * np.sum(eps * eps)
    vol = 0.0
    pts = As._tile_points(prob, prob.n_gauss)
    for t in range(prob.n_tiles):
        for xi, DT, _, w, _ in pts[0]:
            vol += np.sum(w * DT * np.linalg.det(M.macro_jacobian(prob.macro, prob.macro.ctrl, t, xi)))
    assert abs(u @ (K @ u) - dens * vol) < 1e-12 * dens * vol


def test_young_scaling_and_homogeneity(oracle_problem):
    ob = oracle_problem(2, n_el=(2, 1, 1))
    prob, tabs = ob["prob"], ob["tabs"]
    l1 = As.local_lookup(prob, tabs, prob.macro.ctrl, [1])
    l2 = As.local_lookup(prob, tabs, 2.0 * prob.macro.ctrl, [1])
    assert np.allclose(l2, 2.0 * l1, rtol=1e-13, atol=1e-15)        # K(2P) = 2^{d-2} K(P), d = 3
    prob.young = prob.young * 3.0
    l3 = As.local_lookup(prob, tabs, prob.macro.ctrl, [1])
    prob.young = prob.young / 3.0
    assert np.allclose(l3, 3.0 * l1, rtol=1e-13, atol=1e-15)


def test_Emat_decreases_with_q():
    """Fig. 7 trend: E_mat (Eq. 62) decreases as the degree grows."""
    errs = []
    for q in range(0, 5):
        prob = make_config(1, q=q)
        dm = DofMap(prob)
        tabs = As.Tables(prob)
        pt = Pattern(prob, dm, tabs.pairs)
        ob = dict(prob=prob, dm=dm, pattern=pt, tabs=tabs)
        vals, _ = As.assemble_lookup(prob, tabs, pt)
        std = As.scatter(prob, pt, standard_all(ob))
        errs.append(rel(vals, std))
    assert all(b < a for a, b in zip(errs, errs[1:])), errs


def _tiny_problem(q, n_g_tile=None):
    """One curved macro element (degree 2, interior control point moved) and a
    one-element degree-2 tile with its interior control point moved."""
    U = np.array([0, 0, 0, 1, 1, 1.0])
    g = np.array([0, 0.5, 1.0])
    mesh = np.meshgrid(g, g, indexing="ij")
    base = np.stack([m.T.reshape(-1) for m in mesh], axis=1)
    mac = base * np.array([2.0, 1.0])
    mac[4] += np.array([0.25, -0.15])
    til = base.copy()
    til[4] += np.array([0.08, 0.05])
    return Problem("tiny", 2, 2, q, 0.3, Spline([2, 2], [U, U], mac), [Spline([2, 2], [U, U], til)],
                   [], np.ones(1), (1, 1), 0)


def test_brute_force_single_tiny_tile():
    """K^•(n_g) self-converges as n_g -> 30; K^π(q) -> K^•(converged) as q grows."""
    from oracle.tables import icoo
    prob = _tiny_problem(2)
    pairs = [icoo(prob.tile[0])]
    Ks = {n: As.local_standard(prob, 0, pairs, n_g=n) for n in (16, 24, 30)}
    assert rel(Ks[24], Ks[30]) < 1e-12 and rel(Ks[16], Ks[30]) < 1e-9
    errs = []
    for q in range(0, 9):
        pq = _tiny_problem(q)
        tabs = As.Tables(pq)
        errs.append(rel(As.local_lookup(pq, tabs, pq.macro.ctrl, [0])[0], Ks[30]))
    assert errs[-1] < 1e-6 and errs[-1] < errs[0] * 1e-3, errs
