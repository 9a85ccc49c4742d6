"""Pins of the oracle's volume / volume-gradient / load-vector lookup (§3.1
Eqs. 14-19, Eq. 53, Eqs. 66-67) against closed forms, the standard
composed-map quadrature, partition-of-unity identities and homogeneity."""
import numpy as np
import pytest

from oracle import volume as V
from oracle.dofmap import DofMap
from synth import make_config


def _identity_tile_problem(d, q):
    """cfg1/cfg2 with the tile replaced by the identity map (control points at the
    Greville abscissae, zero perturbation)."""
    import dataclasses
    p = make_config(1 if d == 2 else 2, q=q)
    sp = p.tile[0]
    from synth.configs import greville
    g = [greville(sp.knots[k], sp.degree[k]) for k in range(d)]
    n = [len(x) for x in g]
    ctrl = np.zeros((int(np.prod(n)), d))
    for A in range(len(ctrl)):
        idx, r = [], A
        for k in range(d):
            idx.append(r % n[k])
            r //= n[k]
        ctrl[A] = [g[k][idx[k]] for k in range(d)]
    tile = [dataclasses.replace(sp, ctrl=ctrl)]
    return dataclasses.replace(p, tile=tile)


@pytest.mark.parametrize("d,q", [(2, 2), (2, 3), (3, 2)])
def test_volume_table_identity_tile_closed_form(d, q):
    """Identity tile: det J_T = 1, t^h_C = ∫ N_C = (q+1)^{-d} exactly (Bernstein)."""
    p = _identity_tile_problem(d, q)
    th = V.volume_table(p)
    assert np.allclose(th, (q + 1.0) ** -d, rtol=0, atol=1e-15)


@pytest.mark.parametrize("c", [1, 2, 3])
def test_load_table_partition_of_unity(c):
    """Σ_A 𝔉[A][C] = t^h_C (the B-spline basis of each patch sums to one)."""
    p = make_config(c, n_el=(2, 2) if c == 1 else (2, 1, 1))
    F = V.load_tables(p)
    th = V.volume_table(p)
    assert np.allclose(F.sum(axis=0), th, rtol=1e-13, atol=0)
    assert np.all(F >= -1e-15)                      # R_A, N_C, det J_T >= 0


@pytest.mark.parametrize("kw", [dict(c=1, macro_amp=0.0), dict(c=2, macro_amp=0.0, n_el=(2, 1, 1)),
                                dict(c=1, q=3)])
def test_volume_lookup_equals_standard_when_det_in_Qq(kw):
    """det J_ℳ ∈ Q_q (affine elements; or 2D with q >= d·p_M - 1 = 3, Eq. 22): the lookup
    volume equals the composed-map quadrature (same rule) to round-off."""
    kw = dict(kw)
    p = make_config(kw.pop("c"), **kw)
    assert abs(V.volume_lookup(p) - V.volume_standard(p)) < 1e-13 * V.volume_standard(p)


@pytest.mark.parametrize("c", [1, 2])
def test_volume_gradient_invariants(c):
    """Σ_k ∂V/∂P_k = 0 (translation), Σ P·∂V/∂P = d·V (V(sP) = s^d V), and a central
    difference agrees."""
    p = make_config(c, n_el=(2, 2) if c == 1 else (2, 1, 1))
    g = V.volume_gradient(p)
    vol = V.volume_lookup(p)
    assert np.abs(g.sum(0)).max() < 1e-12 * np.abs(g).max()
    assert abs(np.sum(p.macro.ctrl * g) - p.d * vol) < 1e-12 * vol
    k, a, h = 4, 1, 1e-6
    cp, cm = p.macro.ctrl.copy(), p.macro.ctrl.copy()
    cp[k, a] += h
    cm[k, a] -= h
    fd = (V.volume_lookup(p, cp) - V.volume_lookup(p, cm)) / (2 * h)
    assert abs(fd - g[k, a]) < 1e-7 * np.abs(g).max()


@pytest.mark.parametrize("kw", [dict(c=1), dict(c=2, n_el=(2, 1, 1)), dict(c=3, n_el=(1, 1, 2))])
def test_load_vector_total_force(kw):
    """Σ_I f_I = b·V^π (partition of unity of the tile bases)."""
    kw = dict(kw)
    p = make_config(kw.pop("c"), **kw)
    dm = DofMap(p)
    b = np.array([0.3, -1.0, 2.0][:p.d])
    f = V.load_vector(p, dm.node, dm.n_nodes, b)
    assert np.allclose(f.sum(0), b * V.volume_lookup(p), rtol=1e-13, atol=0)


@pytest.mark.parametrize("kw", [dict(c=1, macro_amp=0.0), dict(c=1, q=3), dict(c=2, macro_amp=0.0, n_el=(2, 1, 1))])
def test_load_vector_equals_standard_when_det_in_Qq(kw):
    kw = dict(kw)
    p = make_config(kw.pop("c"), **kw)
    dm = DofMap(p)
    b = np.array([1.0, -0.5, 0.25][:p.d])
    f = V.load_vector(p, dm.node, dm.n_nodes, b)
    fs = V.load_standard(p, dm.node, dm.n_nodes, b)
    assert np.abs(f - fs).max() < 1e-13 * np.abs(fs).max()
