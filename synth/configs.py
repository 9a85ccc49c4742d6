"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no basis evaluation, no
quadrature, no macro field, no assembly).  It only places control points
(Greville abscissae, i.e. the Schoenberg variation-diminishing placement),
applies seeded perturbations, and draws seeded E / u / v.  Both `oracle/` and
the CUDA path read the same arrays from here.

Configs follow /root/repo/BASELINE.json `configs[0..4]` (cfg1..cfg5), with
the geometry choices of SURVEY.md §8(d) (D5: cfg5 uses the lattice tile of
0-based config 2 = cfg3; D6: generator choices documented in DESIGN.md §3).

Seed recipe: `np.random.default_rng([210709568, c])` for
config c; draw order: macro interior perturbation, tile perturbation per
patch, E per tile, then u and v (drawn by `draw_uv` once n_dof is known).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

SEED_BASE = 210709568


@dataclass
class Spline:
    """Tensor-product B-spline patch (Eq. 2).

    degree[k], knots[k] (open, normalised to [0,1]), ctrl (n_ctrl, d) with
    control-point index A = i0 + n0*(i1 + n1*i2) (direction-0 fastest)."""
    degree: List[int]
    knots: List[np.ndarray]
    ctrl: np.ndarray
    weights: Optional[np.ndarray] = None   # NURBS weights (n_ctrl,); None = B-spline

    @property
    def dim(self) -> int:
        return len(self.degree)

    @property
    def n_per_dir(self) -> List[int]:
        return [len(U) - p - 1 for U, p in zip(self.knots, self.degree)]

    @property
    def n_ctrl(self) -> int:
        return int(np.prod(self.n_per_dir))


@dataclass
class Interface:
    """Declared intra-tile patch interface: face (dir_a, side_a) of patch_a is
    glued to face (dir_b, side_b) of patch_b (side 0 = parameter 0, 1 = 1)."""
    patch_a: int
    dir_a: int
    side_a: int
    patch_b: int
    dir_b: int
    side_b: int


@dataclass
class Problem:
    name: str
    d: int
    p: int                      # analysis (tile) degree
    q: "int | Tuple[int, ...]"  # projection degree p_pi: isotropic, or per direction
    nu: float
    macro: Spline               # macro map F (Eq. 4)
    tile: List[Spline]          # reference tile patches (Eq. 3)
    interfaces: List[Interface] = field(default_factory=list)
    young: Optional[np.ndarray] = None   # per-tile E (len n_tiles)
    n_el: Tuple[int, ...] = ()
    config_index: int = 0
    n_proj: int = 0             # L2-projection Gauss points per direction (0: q+1 = interpolation)

    @property
    def n_tiles(self) -> int:
        return int(np.prod(self.n_el))

    @property
    def n_gauss(self) -> int:
        """DESIGN.md reading R3: n_g = p + ceil((q+1)/2) per direction per span (q = the
        largest per-direction degree when anisotropic)."""
        q = self.q if np.ndim(self.q) == 0 else max(self.q)
        return self.p + (q + 2) // 2


# --------------------------------------------------------------------------
# knot vectors and Greville abscissae (placement only)
# --------------------------------------------------------------------------
def open_uniform_knots(p: int, n_el: int) -> np.ndarray:
    inner = [i / n_el for i in range(1, n_el)]
    return np.array([0.0] * (p + 1) + inner + [1.0] * (p + 1))


def greville(U: np.ndarray, p: int) -> np.ndarray:
    n = len(U) - p - 1
    if p == 0:
        return np.array([(U[i] + U[i + 1]) / 2 for i in range(n)])
    return np.array([sum(U[i + 1:i + p + 1]) / p for i in range(n)])


def _grid(arrays):
    """Direction-0-fastest tensor grid of 1D arrays -> (n, d)."""
    mesh = np.meshgrid(*arrays, indexing="ij")
    return np.stack([m.transpose(*reversed(range(len(arrays)))).reshape(-1) for m in mesh], axis=1)


def _index_grid(ns):
    return _grid([np.arange(n) for n in ns]).astype(np.int64)


def _interior_mask(ns):
    idx = _index_grid(ns)
    m = np.ones(len(idx), dtype=bool)
    for k, n in enumerate(ns):
        m &= (idx[:, k] > 0) & (idx[:, k] < n - 1)
    return m


# --------------------------------------------------------------------------
# macro maps
# --------------------------------------------------------------------------
def macro_box(p, n_el, lengths, rng, amp):
    """Box [0,L0]x..., control points at Greville, interior perturbed by
    U(-amp, amp)*h_k (h_k = L_k/n_el_k), SURVEY.md §8(c) reading 15."""
    U = [open_uniform_knots(p, n) for n in n_el]
    g = [greville(u, p) * L for u, L in zip(U, lengths)]
    ctrl = _grid(g)
    pert = rng.uniform(-1.0, 1.0, size=ctrl.shape) * np.array([L / n for L, n in zip(lengths, n_el)])
    mask = _interior_mask([len(x) for x in g])
    ctrl = ctrl + amp * pert * mask[:, None]
    return Spline([p] * len(n_el), U, ctrl)


def macro_shear(p, n_el, a=4.0, b=1.0, c=1.0, kappa=0.3):
    """F(xi) = (a xi0 + kappa xi1^2, b xi1[, c xi2]) exactly, via blossoms:
    for degree p=2 the control value of x^2 at index i is U[i+1]*U[i+2] and of
    x is the Greville abscissa (polynomial reproduction; no basis evaluation)."""
    assert p == 2
    U = [open_uniform_knots(p, n) for n in n_el]
    g = [greville(u, p) for u in U]
    sq1 = np.array([U[1][i + 1] * U[1][i + 2] for i in range(len(g[1]))])
    d = len(n_el)
    idx = _index_grid([len(x) for x in g])
    ctrl = np.zeros((len(idx), d))
    ctrl[:, 0] = a * g[0][idx[:, 0]] + kappa * sq1[idx[:, 1]]
    ctrl[:, 1] = b * g[1][idx[:, 1]]
    if d == 3:
        ctrl[:, 2] = c * g[2][idx[:, 2]]
    return Spline([p] * d, U, ctrl)


def macro_annulus(p, n_el, Ri=1.0, Ro=2.0, H=1.0):
    """Quarter annulus swept along z, control
    points = F(Greville) (variation-diminishing placement)."""
    U = [open_uniform_knots(p, n) for n in n_el]
    g = [greville(u, p) for u in U]
    X = _grid(g)
    r = Ri + (Ro - Ri) * X[:, 1]
    ang = 0.5 * math.pi * (1.0 - X[:, 0])     # xi0 runs along the arc, orientation det J > 0
    ctrl = np.stack([r * np.cos(ang), r * np.sin(ang), H * X[:, 2]], axis=1)
    return Spline([p] * 3, U, ctrl)


def _insert_knots_1d(U, p, Pw, new):
    """Boehm knot insertion of the knots `new` into a 1D curve with homogeneous control
    points Pw (n, dim+1): geometry is unchanged (placement only)."""
    U = list(U)
    Pw = [np.asarray(x, dtype=float) for x in Pw]
    for u in new:
        k = max(i for i in range(len(U) - 1) if U[i] <= u < U[i + 1])
        Q = []
        for i in range(len(Pw) + 1):
            if i <= k - p:
                Q.append(Pw[i])
            elif i > k:
                Q.append(Pw[i - 1])
            else:
                a = (u - U[i]) / (U[i + p] - U[i])
                Q.append(a * Pw[i] + (1.0 - a) * Pw[i - 1])
        Pw = Q
        U.insert(k + 1, u)
    return np.array(U), np.array(Pw)


def macro_annulus_nurbs(n_el, Ri=1.0, Ro=2.0, H=1.0):
    """EXACT quarter annulus swept along z as a NURBS (NEXT N4; the paper's torus of
    §3.3.4 in miniature): angular direction = the rational quadratic 90° arc (weights
    1, √2/2, 1) refined by knot insertion to n_el[0] elements; radial and z directions
    polynomial (linear functions placed at the Greville abscissae, exact).  Same
    orientation as macro_annulus (ξ0 along the arc from angle π/2 to 0)."""
    p = 2
    w = math.sqrt(0.5)
    arc = np.array([[0.0, 1.0, 1.0], [w, w, w], [1.0, 0.0, 1.0]])   # homogeneous (w x, w y, w)
    U0, arcw = _insert_knots_1d([0, 0, 0, 1, 1, 1], p, arc, [i / n_el[0] for i in range(1, n_el[0])])
    U1 = open_uniform_knots(p, n_el[1])
    U2 = open_uniform_knots(p, n_el[2])
    r = Ri + (Ro - Ri) * greville(U1, p)
    z = H * greville(U2, p)
    idx = _index_grid([len(arcw), len(r), len(z)])
    wts = arcw[idx[:, 0], 2]
    xy = arcw[idx[:, 0], :2] / wts[:, None]
    ctrl = np.stack([r[idx[:, 1]] * xy[:, 0], r[idx[:, 1]] * xy[:, 1], z[idx[:, 2]]], axis=1)
    return Spline([p] * 3, [np.asarray(U0, float), U1, U2], ctrl, weights=wts)


def macro_twist(p, n_el, length=4.0, twist=0.5 * math.pi):
    """Square 1x1 section extruded along x over `length`, rotated by twist*xi0
    (SURVEY.md §8(d), cfg4), control points = F(Greville)."""
    U = [open_uniform_knots(p, n) for n in n_el]
    g = [greville(u, p) for u in U]
    X = _grid(g)
    th = twist * X[:, 0]
    y0, z0 = X[:, 1] - 0.5, X[:, 2] - 0.5
    ctrl = np.stack([length * X[:, 0],
                     0.5 + np.cos(th) * y0 - np.sin(th) * z0,
                     0.5 + np.sin(th) * y0 + np.cos(th) * z0], axis=1)
    return Spline([p] * 3, U, ctrl)


# --------------------------------------------------------------------------
# tiles
# --------------------------------------------------------------------------
def tile_single(p, n_el, rng, amp):
    """One patch on [0,1]^d: identity (Greville) plus U(-amp,amp)*h on interior
    control points, boundary fixed (BASELINE.json configs[0], configs[1])."""
    U = [open_uniform_knots(p, n) for n in n_el]
    g = [greville(u, p) for u in U]
    ctrl = _grid(g)
    pert = rng.uniform(-1.0, 1.0, size=ctrl.shape) * np.array([1.0 / n for n in n_el])
    mask = _interior_mask([len(x) for x in g])
    ctrl = ctrl + amp * pert * mask[:, None]
    return [Spline([p] * len(n_el), U, ctrl)]


def _square_to_disk(s, t):
    """Elliptical square->disk placement of section control points."""
    return s * np.sqrt(1.0 - 0.5 * t * t), t * np.sqrt(1.0 - 0.5 * s * s)


def tile_lattice(p, n_len, radius=0.15, n_sec=2):
    """6-strut cubic-cross lattice (BASELINE.json configs[2], configs[3]).

    Three axis-aligned bars through the tile centre; bar a is split at the
    centre into half-struts h=0 (x_a in [0,.5]) and h=1 (x_a in [.5,1]);
    patch index = 2a+h.  Parameter directions: theta0 -> axis (a+1)%3,
    theta1 -> axis (a+2)%3 (disk section of radius `radius`), theta2 -> axis a
    (cyclic, orientation preserving).  Half-struts of one bar are glued at the
    centre (declared interface); bars are NOT coupled at the hub (DESIGN.md
    reading R10).  Tile faces are conforming, so tiles glue to neighbours."""
    Usec = open_uniform_knots(p, n_sec)
    Ulen = open_uniform_knots(p, n_len)
    gs = 2.0 * greville(Usec, p) - 1.0
    gl = greville(Ulen, p)
    idx = _index_grid([len(gs), len(gs), len(gl)])
    s, t, L = gs[idx[:, 0]], gs[idx[:, 1]], gl[idx[:, 2]]
    dx, dy = _square_to_disk(s, t)
    patches, ifaces = [], []
    for a in range(3):
        c1, c2 = (a + 1) % 3, (a + 2) % 3
        for h in range(2):
            ctrl = np.zeros((len(idx), 3))
            ctrl[:, c1] = 0.5 + radius * dx
            ctrl[:, c2] = 0.5 + radius * dy
            ctrl[:, a] = 0.5 * L + 0.5 * h
            patches.append(Spline([p] * 3, [Usec.copy(), Usec.copy(), Ulen.copy()], ctrl))
        ifaces.append(Interface(2 * a, 2, 1, 2 * a + 1, 2, 0))
    return patches, ifaces


# --------------------------------------------------------------------------
# configs
# --------------------------------------------------------------------------
def make_config(c: int, *, macro_amp: Optional[float] = None, macro_kind: Optional[str] = None,
                n_el: Optional[Tuple[int, ...]] = None, q=None) -> Problem:
    """Config c in 1..5 (1-based, BASELINE.json configs[c-1]).

    Optional overrides build the exact-regime variants and small cases used by
    tests: macro_amp=0 (affine elements for box macros), macro_kind='shear',
    macro_kind='nurbs' (cfg3/5: the exact rational quarter annulus), a smaller n_el,
    or another q (an int, or per-direction degrees as in the twist's p_pi = 3, 3, 4)."""
    rng = np.random.default_rng([SEED_BASE, c])
    nu = 0.3
    if c == 1:
        n_el = n_el or (4, 4)
        amp = 0.05 if macro_amp is None else macro_amp
        macro = macro_box(2, n_el, (4.0, 1.0), rng, amp)   # always consumes the draw
        if macro_kind == "shear":
            macro = macro_shear(2, n_el)
        tile = tile_single(2, (4, 4), rng, 0.10)
        prob = Problem("cfg1", 2, 2, 2 if q is None else q, nu, macro, tile, [], None, tuple(n_el), c)
    elif c == 2:
        n_el = n_el or (4, 4, 4)
        amp = 0.05 if macro_amp is None else macro_amp
        macro = macro_box(2, n_el, (4.0, 1.0, 1.0), rng, amp)   # always consumes the draw
        if macro_kind == "shear":
            macro = macro_shear(2, n_el)
        tile = tile_single(2, (3, 3, 3), rng, 0.08)
        prob = Problem("cfg2", 3, 2, 2 if q is None else q, nu, macro, tile, [], None, tuple(n_el), c)
    elif c in (3, 5):
        n_el = n_el or ((8, 8, 8) if c == 3 else (32, 16, 16))
        if macro_kind == "box":
            amp = 0.0 if macro_amp is None else macro_amp
            macro = macro_box(2, n_el, (4.0, 1.0, 1.0), rng, amp)
        elif macro_kind == "nurbs":   # exact rational quarter annulus (NEXT N4)
            macro = macro_annulus_nurbs(n_el)
        else:
            macro = macro_annulus(2, n_el)
        tile, ifaces = tile_lattice(2, 6)
        prob = Problem(f"cfg{c}", 3, 2, 2 if q is None else q, nu, macro, tile, ifaces, None, tuple(n_el), c)
    elif c == 4:
        n_el = n_el or (16, 8, 8)
        macro = macro_twist(3, n_el)
        tile, ifaces = tile_lattice(3, 4)
        prob = Problem("cfg4", 3, 3, 3 if q is None else q, nu, macro, tile, ifaces, None, tuple(n_el), c)
    else:
        raise ValueError(f"unknown config {c}")
    n_tiles = int(np.prod(prob.n_el))
    if c == 4:
        prob.young = rng.uniform(0.5, 2.0, size=n_tiles)
    else:
        prob.young = np.ones(n_tiles)
    prob._uv_state = rng.bit_generator.state  # u, v continue this stream
    return prob


def draw_uv(prob: Problem, n_dof: int) -> Tuple[np.ndarray, np.ndarray]:
    """u, v ~ N(0,1) (BASELINE.json configs[4]), drawn after E in the config's stream."""
    rng = np.random.default_rng()
    rng.bit_generator.state = prob._uv_state
    u = rng.standard_normal(n_dof)
    v = rng.standard_normal(n_dof)
    return u, v


def draw_uv_seeded(seed: int, n_dof: int) -> Tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng([SEED_BASE, 99, seed])
    return rng.standard_normal(n_dof), rng.standard_normal(n_dof)
