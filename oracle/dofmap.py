"""ORACLE (test infrastructure): DofMap, CSR pattern and block map.

The paper's solution space is identical on every tile (Eq. 13)
and is silent on how tile-local control points become global unknowns
(readings R9, R10 in DESIGN.md):

R10 (merging).  Tile-local control points (t, p, A) and (t', p', A') denote the
same global node iff they are linked by a chain of elementary identifications:
  (i)  intra-tile: the tile declares an interface (p, face f) <-> (p', face f');
       A lies on face f of patch p, A' on face f' of p', t = t', and the two
       control points coincide (|Δ| <= 1e-10);
  (ii) inter-tile: t' = t + e_k in the macro element grid; A lies on the tile
       face ξ_k = 1, A' on the tile face ξ_k = 0, and pos(A) - e_k == pos(A').
Global ids are assigned in order of first appearance over t (direction-0
fastest), then p, then A.  Two control points of one (t, p) merging is an error.

R9 (pattern).  DOF = node*d + a (interleaved).  Block (I, J) is structural iff
some (t, p, k=(A,B)) maps to {I, J}; all d×d entries of a structural block are
stored, both triangles, columns ascending; row_ptr int64, col_idx int32.
block_map[t*n_rows_tile + row] = (pos(I*d, J*d), pos(J*d, I*d)), row =
Σ_{p'<p} n_nz,p' + k.
"""
from __future__ import annotations

import numpy as np
from scipy.sparse import coo_matrix
from scipy.sparse.csgraph import connected_components

from .bspline import multi_index
from .tables import icoo

TOL = 1e-10


def face_members(spline, direction, side):
    n = spline.n_per_dir
    want = 0 if side == 0 else n[direction] - 1
    return [A for A in range(spline.n_ctrl) if multi_index(n, A)[direction] == want]


def _match(pos_a, pos_b, shift):
    """Pairs (ia, ib) with pos_a[ia] - shift == pos_b[ib]; every point must match."""
    out = []
    for ia, x in enumerate(pos_a):
        dist = np.abs(pos_b - (x - shift)).max(axis=1)
        hits = np.nonzero(dist <= TOL)[0]
        if len(hits) != 1:
            raise ValueError("non-conforming tile: unmatched control point")
        out.append((ia, int(hits[0])))
    return out


def reference_identifications(prob):
    """Identifications on the reference tile: intra-tile pairs ((p,A),(p',A')) and,
    per direction k, inter-tile pairs ((p,A) on ξ_k=1, (p',A') on ξ_k=0)."""
    d = prob.d
    intra = []
    for f in prob.interfaces:
        ma = face_members(prob.tile[f.patch_a], f.dir_a, f.side_a)
        mb = face_members(prob.tile[f.patch_b], f.dir_b, f.side_b)
        pa = prob.tile[f.patch_a].ctrl[ma]
        pb = prob.tile[f.patch_b].ctrl[mb]
        for ia, ib in _match(pa, pb, np.zeros(d)):
            intra.append(((f.patch_a, ma[ia]), (f.patch_b, mb[ib])))
    inter = []
    allpos = [(p, A, prob.tile[p].ctrl[A]) for p in range(len(prob.tile)) for A in range(prob.tile[p].n_ctrl)]
    for k in range(d):
        hi = [(p, A, x) for (p, A, x) in allpos if abs(x[k] - 1.0) <= TOL]
        lo = [(p, A, x) for (p, A, x) in allpos if abs(x[k]) <= TOL]
        if len(hi) != len(lo):
            raise ValueError("non-conforming tile faces")
        if hi:
            e = np.zeros(d)
            e[k] = 1.0
            m = _match(np.array([x for _, _, x in hi]), np.array([x for _, _, x in lo]), e)
            inter.append([((hi[a][0], hi[a][1]), (lo[b][0], lo[b][1])) for a, b in m])
        else:
            inter.append([])
    return intra, inter


class DofMap:
    """node[t, off_p + A] -> global node id; n_nodes."""

    def __init__(self, prob):
        self.prob = prob
        d = prob.d
        self.offsets = np.cumsum([0] + [s.n_ctrl for s in prob.tile])
        nloc = int(self.offsets[-1])
        nt = prob.n_tiles
        self.n_local_ctrl = nloc
        intra, inter = reference_identifications(prob)
        rows, cols = [], []
        tiles = np.arange(nt)
        for (pa, A), (pb, B) in intra:
            rows.append(tiles * nloc + self.offsets[pa] + A)
            cols.append(tiles * nloc + self.offsets[pb] + B)
        n_el = list(prob.n_el)
        tidx = np.stack([(tiles // int(np.prod(n_el[:k]))) % n_el[k] for k in range(d)], axis=1)
        for k in range(d):
            has_next = tidx[:, k] < n_el[k] - 1
            t0 = tiles[has_next]
            t1 = t0 + int(np.prod(n_el[:k]))
            for (pa, A), (pb, B) in inter[k]:
                rows.append(t0 * nloc + self.offsets[pa] + A)
                cols.append(t1 * nloc + self.offsets[pb] + B)
        nv = nt * nloc
        if rows:
            r = np.concatenate(rows)
            c = np.concatenate(cols)
        else:
            r = c = np.zeros(0, dtype=np.int64)
        g = coo_matrix((np.ones(len(r)), (r, c)), shape=(nv, nv))
        ncomp, label = connected_components(g, directed=False)
        first = np.full(ncomp, nv, dtype=np.int64)
        np.minimum.at(first, label, np.arange(nv))
        order = np.argsort(first, kind="stable")
        rank = np.empty(ncomp, dtype=np.int64)
        rank[order] = np.arange(ncomp)
        self.node = rank[label].reshape(nt, nloc)
        self.n_nodes = ncomp
        # same-patch merge check
        for p in range(len(prob.tile)):
            blk = self.node[:, self.offsets[p]:self.offsets[p + 1]]
            s = np.sort(blk, axis=1)
            if np.any(s[:, 1:] == s[:, :-1]):
                raise ValueError("two control points of one patch merged")

    @property
    def n_dof(self):
        return self.n_nodes * self.prob.d


class Pattern:
    """Full symmetric CSR pattern + block map (reading R9)."""

    def __init__(self, prob, dm: DofMap, pairs_per_patch=None):
        d = prob.d
        self.prob, self.dm = prob, dm
        self.pairs = pairs_per_patch or [icoo(s) for s in prob.tile]
        self.row_off = np.cumsum([0] + [len(p) for p in self.pairs])
        self.n_rows_tile = int(self.row_off[-1])
        I_all, J_all = [], []
        for p, pr in enumerate(self.pairs):
            I_all.append(dm.node[:, dm.offsets[p] + pr[:, 0]])   # (nt, n_nz_p)
            J_all.append(dm.node[:, dm.offsets[p] + pr[:, 1]])
        self.I = np.concatenate(I_all, axis=1)                   # (nt, n_rows_tile)
        self.J = np.concatenate(J_all, axis=1)
        nn = dm.n_nodes
        keys = np.concatenate([(self.I * nn + self.J).ravel(), (self.J * nn + self.I).ravel()])
        keys.sort()                                              # unique by sort + adjacent compare
        blocks = keys[np.concatenate([[True], keys[1:] != keys[:-1]])]
        bI, bJ = blocks // nn, blocks % nn
        self.nnzb = np.bincount(bI, minlength=nn).astype(np.int64)
        self.brow_ptr = np.concatenate([[0], np.cumsum(self.nnzb)])
        self.bcol = bJ
        self.blocks = blocks
        # scalar CSR
        rowlen = np.repeat(d * self.nnzb, d)
        self.row_ptr = np.concatenate([[0], np.cumsum(rowlen)]).astype(np.int64)
        self.nnz = int(self.row_ptr[-1])

    def col_idx(self):
        d = self.prob.d
        out = np.empty(self.nnz, dtype=np.int32)
        for I in range(self.dm.n_nodes):
            cols = self.bcol[self.brow_ptr[I]:self.brow_ptr[I + 1]]
            sc = (cols[:, None] * d + np.arange(d)[None, :]).ravel()
            for a in range(d):
                r = I * d + a
                out[self.row_ptr[r]:self.row_ptr[r + 1]] = sc
        return out

    def pos(self, I, J):
        """CSR position of scalar entry (I*d, J*d) for node-block arrays I, J."""
        d = self.prob.d
        nn = self.dm.n_nodes
        key = I * nn + J
        order = np.argsort(key, kind="stable")                  # sorted queries: a faster binary search
        b = np.empty(len(key), dtype=np.int64)
        b[order] = np.searchsorted(self.blocks, key[order])
        assert np.all(self.blocks[b] == key)
        jpos = b - self.brow_ptr[I]
        return self.row_ptr[I * d] + d * jpos

    def block_map(self, tiles=None):
        """(len(tiles) * n_rows_tile, 2) int64: (pos(I*d, J*d), pos(J*d, I*d)); all tiles
        by default, else the given tiles in the given order."""
        I = self.I if tiles is None else self.I[np.asarray(tiles)]
        J = self.J if tiles is None else self.J[np.asarray(tiles)]
        fwd = self.pos(I.ravel(), J.ravel())
        bwd = self.pos(J.ravel(), I.ravel())
        return np.stack([fwd, bwd], axis=1)
