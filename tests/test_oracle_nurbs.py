"""Pins of the oracle's NURBS macro map (Eq. 4 with rational
basis, §3.3.4): the exact quarter annulus of synth.macro_annulus_nurbs."""
import math

import numpy as np
import pytest

from oracle import macro as M
from oracle import volume as V
from synth import make_config


def _nurbs(n_el=(2, 2, 2)):
    return make_config(3, macro_kind="nurbs", n_el=n_el)


def test_nurbs_annulus_is_exact():
    """F maps the radial faces onto circles: |F_xy| = R_i on u1 = 0, R_o on u1 = 1 (to
    round-off), and z = H u2."""
    p = _nurbs((3, 2, 2))
    mac = p.macro
    rng = np.random.default_rng(0)
    for t in range(p.n_tiles):
        e1 = (t // p.n_el[0]) % p.n_el[1]
        xi = rng.random((16, 3))
        if e1 == 0:
            xi[:, 1] = 0.0
            X = M.macro_position(mac, mac.ctrl, t, xi)
            assert np.abs(np.hypot(X[:, 0], X[:, 1]) - 1.0).max() < 1e-14
        if e1 == p.n_el[1] - 1:
            xi[:, 1] = 1.0
            X = M.macro_position(mac, mac.ctrl, t, xi)
            assert np.abs(np.hypot(X[:, 0], X[:, 1]) - 2.0).max() < 1e-14


def test_nurbs_jacobian_matches_finite_differences():
    p = _nurbs()
    mac = p.macro
    xi = np.random.default_rng(1).uniform(0.1, 0.9, (5, 3))
    for t in (0, 3, 7):
        J = M.macro_jacobian(mac, mac.ctrl, t, xi)
        h = 1e-6
        for k in range(3):
            e = np.zeros(3)
            e[k] = h
            fd = (M.macro_position(mac, mac.ctrl, t, xi + e) - M.macro_position(mac, mac.ctrl, t, xi - e)) / (2 * h)
            assert np.abs(J[:, :, k] - fd).max() < 1e-8


def test_unit_weights_reduce_to_bspline():
    import dataclasses
    p = _nurbs()
    mac = p.macro
    ones = dataclasses.replace(mac, weights=np.ones(mac.ctrl.shape[0]))
    plain = dataclasses.replace(mac, weights=None)
    xi = np.random.default_rng(2).random((7, 3))
    for t in (0, 5):
        assert np.abs(M.macro_jacobian(ones, mac.ctrl, t, xi) - M.macro_jacobian(plain, mac.ctrl, t, xi)).max() < 1e-14


def test_nurbs_annulus_volume():
    """Identity tile: the composed-map quadrature converges to the exact quarter-annulus
    volume (π/4)(R_o² - R_i²)H = 3π/4, and the lookup volume converges with q."""
    import dataclasses
    from synth.configs import greville, tile_single
    p = _nurbs((2, 2, 2))
    tile = tile_single(2, (1, 1, 1), np.random.default_rng(0), 0.0)
    pi = dataclasses.replace(p, tile=tile, interfaces=[])
    exact = 0.75 * math.pi
    assert abs(V.volume_standard(pi, n_g=10) - exact) < 1e-12 * exact
    err = [abs(V.volume_lookup(dataclasses.replace(pi, q=q)) - exact) for q in (1, 2, 3, 4)]
    assert err[3] < err[1] and err[3] < 1e-6 * exact
