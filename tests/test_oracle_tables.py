"""Pins for oracle/tables.py: I_coo (Eq. 56) and 𝔎 (Eqs. 51-52, 57)."""
from fractions import Fraction as Fr
from math import comb

import numpy as np
import pytest

from oracle.tables import icoo, lookup_table
from synth import Spline, open_uniform_knots


# ---- exact polynomial arithmetic (power basis, Fractions) -------------------
def pmul(a, b):
    out = [Fr(0)] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            out[i + j] += x * y
    return out


def ppow(a, n):
    out = [Fr(1)]
    for _ in range(n):
        out = pmul(out, a)
    return out


def pder(a):
    return [i * a[i] for i in range(1, len(a))] or [Fr(0)]


def pint01(a):
    return sum(c / (i + 1) for i, c in enumerate(a))


def bern(q, c, o=Fr(0), s=Fr(1)):
    """B_c^q(o + s θ) as a polynomial in θ."""
    x = [o, s]
    omx = [1 - o, -s]
    return [comb(q, c) * v for v in pmul(ppow(x, c), ppow(omx, q - c))]


def exact_affine_table(p, q, o, s):
    """𝔎 for the single-element degree-p tile 𝒯(θ) = o + s⊙θ, exactly (Eq. 52 by
    change of variables: ∂_ξk = (1/s_k) ∂_θk, dξ = Π s_k dθ)."""
    d = len(o)
    qv = (q,) * d if np.ndim(q) == 0 else tuple(q)   # per-direction degrees
    n1 = p + 1
    nT, npi = n1 ** d, int(np.prod([x + 1 for x in qv]))
    pairs = [(A, B) for A in range(nT) for B in range(A, nT)]
    T = np.zeros((len(pairs), d, d, npi))
    for r, (A, B) in enumerate(pairs):
        a = [(A // n1 ** k) % n1 for k in range(d)]
        b = [(B // n1 ** k) % n1 for k in range(d)]
        for i in range(d):
            for j in range(d):
                for C in range(npi):
                    c, rem = [], C
                    for k in range(d):
                        c.append(rem % (qv[k] + 1))
                        rem //= qv[k] + 1
                    val = Fr(1)
                    for k in range(d):
                        fa = bern(p, a[k])
                        fb = bern(p, b[k])
                        if k == i:
                            fa = [x / s[k] for x in pder(fa)]
                        if k == j:
                            fb = [x / s[k] for x in pder(fb)]
                        val *= s[k] * pint01(pmul(pmul(fa, fb), bern(qv[k], c[k], o[k], s[k])))
                    T[r, i, j, C] = float(val)
    return T.reshape(len(pairs), -1)


@pytest.mark.parametrize("p,q,o,s", [
    (2, 2, (Fr(1, 4), Fr(1, 10)), (Fr(1, 2), Fr(3, 5))),
    (2, 1, (Fr(0), Fr(1, 5)), (Fr(1), Fr(2, 5))),
    (1, 1, (Fr(1, 8), Fr(0), Fr(1, 4)), (Fr(3, 4), Fr(1), Fr(1, 2))),
    # anisotropic projection spaces (the twist's p_π = 3, 3, 4)
    (2, (1, 3), (Fr(1, 4), Fr(1, 10)), (Fr(1, 2), Fr(3, 5))),
    (1, (0, 2, 1), (Fr(1, 8), Fr(0), Fr(1, 4)), (Fr(3, 4), Fr(1), Fr(1, 2))),
])
def test_table_exact_rational_affine_tile(p, q, o, s):
    d = len(o)
    U = np.array([0.0] * (p + 1) + [1.0] * (p + 1))
    g = [np.array([float(oo + ss * Fr(i, p)) for i in range(p + 1)]) for oo, ss in zip(o, s)]
    mesh = np.meshgrid(*g, indexing="ij")
    ctrl = np.stack([m.transpose(*reversed(range(d))).reshape(-1) for m in mesh], axis=1)
    spline = Spline([p] * d, [U] * d, ctrl)
    n_g = p + (max(np.atleast_1d(q)) + 2) // 2
    T, pairs = lookup_table(spline, q, n_g)
    ref = exact_affine_table(p, q, o, s)
    assert np.allclose(T, ref, rtol=0, atol=2e-15 * np.abs(ref).max())


def perturbed_tile(d, p, n_el, amp, seed):
    r = np.random.default_rng(seed)
    from synth.configs import tile_single
    return tile_single(p, n_el, r, amp)[0]


def _check_row_sums_and_symmetry(spline, q, d):
    T, pairs = lookup_table(spline, q, spline.degree[0] + (max(np.atleast_1d(q)) + 2) // 2)
    npi = int(np.prod([x + 1 for x in ((q,) * d if np.ndim(q) == 0 else q)]))
    T4 = T.reshape(len(pairs), d, d, npi)
    scale = np.abs(T).max()
    nT = spline.n_ctrl
    # Σ_B over ordered pairs of 𝔎(A,B,C,i,j) = 0 (Σ_B R_B ≡ 1)
    acc = np.zeros((nT, d, d, npi))
    for r, (A, B) in enumerate(pairs):
        acc[A] += T4[r]
        if A != B:
            acc[B] += np.transpose(T4[r], (1, 0, 2))
    assert np.abs(acc).max() < 1e-13 * scale * 10
    # diagonal pairs symmetric in (i, j)
    diag = pairs[:, 0] == pairs[:, 1]
    assert np.allclose(T4[diag], np.transpose(T4[diag], (0, 2, 1, 3)), atol=1e-15 * scale * 10)
    return T4, pairs


def test_row_sums_and_symmetry_perturbed_tiles():
    _check_row_sums_and_symmetry(perturbed_tile(2, 2, (4, 4), 0.10, 3), 2, 2)
    _check_row_sums_and_symmetry(perturbed_tile(3, 2, (2, 2, 2), 0.08, 4), 2, 3)
    _check_row_sums_and_symmetry(perturbed_tile(3, 2, (2, 2, 2), 0.08, 4), (1, 3, 2), 3)


def test_row_sums_lattice_patch():
    from synth.configs import tile_lattice
    patches, _ = tile_lattice(2, 6)
    _check_row_sums_and_symmetry(patches[3], 2, 3)


def test_sum_over_C_equals_q0_table():
    """Σ_C N_C ≡ 1 at the same points: Σ_C 𝔎_q[.., C] == 𝔎_0 (micro stiffness kernel)."""
    tile = perturbed_tile(2, 2, (3, 3), 0.10, 5)
    n_g = 4   # same quadrature for both
    Tq, pairs = lookup_table(tile, 2, n_g)
    T0, pairs0 = lookup_table(tile, 0, n_g)
    assert np.array_equal(pairs, pairs0)
    Tq4 = Tq.reshape(len(pairs), 4, 9)
    assert np.allclose(Tq4.sum(-1), T0, rtol=0, atol=1e-14 * np.abs(T0).max())
    Ta, _ = lookup_table(tile, (3, 1), n_g)            # anisotropic Q_{3,1}: still Σ_C N_C ≡ 1
    assert np.allclose(Ta.reshape(len(pairs), 4, 8).sum(-1), T0, rtol=0, atol=1e-14 * np.abs(T0).max())


@pytest.mark.parametrize("n,p,expect", [(6, 2, 15), (4, 2, 9), (7, 3, 22)])
def test_icoo_counts_1d_closed_form(n, p, expect):
    """1D I_coo size: #{A<=B, |A-B|<=p} (n=6, p=2 -> 15)."""
    U = open_uniform_knots(p, n - p)
    sp = Spline([p], [U], np.linspace(0, 1, n)[:, None])
    pr = icoo(sp)
    assert len(pr) == expect
    assert np.all(np.abs(pr[:, 0] - pr[:, 1]) <= p)
    assert np.all(pr[:, 0] <= pr[:, 1])
    assert np.all(np.diff(pr[:, 0] * 1000 + pr[:, 1]) > 0)


def test_icoo_size_tensor():
    from synth import make_config
    for c, n_nz in [(1, 306), (2, 3492), (3, 3396), (4, 9874)]:
        prob = make_config(c)
        assert len(icoo(prob.tile[0])) == n_nz
