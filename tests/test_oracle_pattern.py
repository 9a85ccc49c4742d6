"""Pins for oracle/dofmap.py: DofMap merging (reading R10) and the CSR pattern /
block map (reading R9), checked against closed-form pair counts."""
import json
import os

import numpy as np
import pytest

from oracle.dofmap import DofMap, Pattern
from synth import make_config

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pattern_counts.json")))


def pairs_1d(n, p):
    return n + 2 * sum(n - k for k in range(1, p + 1))


def closed_form_single_patch(n_el_tile, p, n_tiles_dir, d):
    """Single-patch tile: block (I,J) structural iff per direction both indices lie in
    one tile's index range and |i-j| <= p; 1D count = m*pairs(tile) - (m-1) shared self-pairs."""
    nodes, cnt = 1, 1
    for k in range(d):
        n = n_el_tile[k] + p
        m = n_tiles_dir[k]
        nodes *= m * n - (m - 1)
        cnt *= m * pairs_1d(n, p) - (m - 1)
    return nodes * d, cnt * d * d


def closed_form_lattice(p, n_sec, n_len, n_tiles_dir):
    """Lattice (3 uncoupled bar families, half-struts glued at faces): per bar chain of
    2n half-strut patches, pairs = 2n*full - (2n-1)*face."""
    ns, nl = n_sec + p, n_len + p
    full = pairs_1d(ns, p) ** 2 * pairs_1d(nl, p)
    face = pairs_1d(ns, p) ** 2
    nodes_chain = lambda n: ns * ns * (2 * n * nl - (2 * n - 1))
    blocks, nodes = 0, 0
    for a in range(3):
        n = n_tiles_dir[a]
        chains = int(np.prod([n_tiles_dir[b] for b in range(3) if b != a]))
        blocks += chains * (2 * n * full - (2 * n - 1) * face)
        nodes += chains * nodes_chain(n)
    return nodes * 3, blocks * 9


@pytest.mark.parametrize("c", [1, 2, 3])
def test_pattern_counts(c, oracle_problem):
    ob = oracle_problem(c)
    prob, dm, pt = ob["prob"], ob["dm"], ob["pattern"]
    if c in (1, 2):
        ndof, nnz = closed_form_single_patch([4, 4] if c == 1 else [3, 3, 3], 2, prob.n_el, prob.d)
    else:
        ndof, nnz = closed_form_lattice(2, 2, 6, prob.n_el)
    assert (dm.n_dof, pt.nnz) == (ndof, nnz)
    assert (ndof, nnz) == (GOLD[prob.name]["n_dof"], GOLD[prob.name]["nnz"])


def test_closed_forms_cfg4_cfg5_match_golden():
    assert closed_form_lattice(3, 2, 4, (16, 8, 8)) == (GOLD["cfg4"]["n_dof"], GOLD["cfg4"]["nnz"])
    assert closed_form_lattice(2, 2, 6, (32, 16, 16)) == (GOLD["cfg5"]["n_dof"], GOLD["cfg5"]["nnz"])


@pytest.mark.parametrize("c", [1, 2])
def test_csr_structure_and_block_map(c, oracle_problem):
    ob = oracle_problem(c)
    prob, dm, pt = ob["prob"], ob["dm"], ob["pattern"]
    d = prob.d
    col = pt.col_idx()
    rp = pt.row_ptr
    assert rp.dtype == np.int64 and col.dtype == np.int32
    for r in range(dm.n_dof):
        seg = col[rp[r]:rp[r + 1]]
        assert np.all(np.diff(seg) > 0)
    bm = pt.block_map()
    I, J = pt.I.ravel(), pt.J.ravel()
    assert np.array_equal(col[bm[:, 0]], J * d)
    assert np.array_equal(col[bm[:, 1]], I * d)
    rows = np.searchsorted(rp, bm[:, 0], side="right") - 1
    assert np.array_equal(rows, I * d)
    # symmetric structure: (r, c) present iff (c, r) present
    import scipy.sparse as sp
    S = sp.csr_matrix((np.ones(len(col)), col, rp), shape=(dm.n_dof,) * 2)
    assert (S != S.T).nnz == 0


def test_node_numbering_first_appearance(oracle_problem):
    ob = oracle_problem(1)
    node = ob["dm"].node
    seen = -1
    for x in node.ravel():
        if x > seen:
            assert x == seen + 1
            seen = x
    # tile 0 numbers its 36 control points 0..35 in order
    assert np.array_equal(node[0], np.arange(36))
    # tile 1 (to the right) shares its left face (i0 = 0) with tile 0's right face (i0 = 5)
    assert np.array_equal(node[1][0::6], node[0][5::6])


def test_nonconforming_tile_raises():
    prob = make_config(1)
    prob.tile[0].ctrl[6, 1] += 1e-3       # a point of the face ξ0 = 0 (index (0,1))
    with pytest.raises(ValueError):
        DofMap(prob)


def test_lattice_interfaces_and_no_hub_coupling():
    prob = make_config(3, n_el=(2, 1, 1))
    dm = DofMap(prob)
    off = dm.offsets
    # half-struts of bar 0 share their centre face (16 points): patch 0 face θ2=1 == patch 1 face θ2=0
    n0 = dm.node[0, off[0]:off[1]].reshape(8, 4, 4)
    n1 = dm.node[0, off[1]:off[2]].reshape(8, 4, 4)
    assert np.array_equal(n0[-1], n1[0])
    # different bars never share nodes inside a tile (reading R10: no hub coupling)
    bars = [set(dm.node[0, off[2 * a]:off[2 * a + 2]]) for a in range(3)]
    assert not (bars[0] & bars[1]) and not (bars[0] & bars[2]) and not (bars[1] & bars[2])
    # bar 0 continues into tile 1 across ξ0 = 1
    assert np.array_equal(dm.node[0, off[1]:off[2]].reshape(8, 4, 4)[-1],
                          dm.node[1, off[0]:off[1]].reshape(8, 4, 4)[0])
    # cubic lattice: 5x5 sections put a control point on every bar axis; the hub point
    # (0.5, 0.5, 0.5) belongs to all three bars but is NOT merged across bars
    prob4 = make_config(4, n_el=(1, 1, 1))
    dm4 = DofMap(prob4)
    hub = [[(p, A) for A in range(prob4.tile[p].n_ctrl)
            if np.allclose(prob4.tile[p].ctrl[A], 0.5)] for p in range(6)]
    hub_nodes = {dm4.node[0, dm4.offsets[p] + A] for p in range(6) for (_, A) in hub[p]}
    assert len(hub_nodes) == 3


def test_block_map_and_scatter_by_tile_ranges(oracle_problem):
    """block_map(tiles) is block_map()'s rows of those tiles; scatter over consecutive tile
    ranges into one array (out=, bmap=) equals the single scatter bit for bit (the
    accumulation order t, row is kept) — the chunked form the full-size tests use."""
    from oracle import assemble as As
    ob = oracle_problem(2)
    prob, pt, tabs = ob["prob"], ob["pattern"], ob["tabs"]
    nr = pt.n_rows_tile
    bm = pt.block_map()
    assert np.array_equal(pt.block_map(range(10, 17)), bm[10 * nr:17 * nr])
    local = As.local_lookup(prob, tabs, prob.macro.ctrl, range(prob.n_tiles))
    whole = As.scatter(prob, pt, local)
    acc = np.zeros(pt.nnz)
    for t0 in range(0, prob.n_tiles, 24):
        ts = np.arange(t0, min(prob.n_tiles, t0 + 24))
        As.scatter(prob, pt, local[ts], tiles=ts, out=acc, bmap=pt.block_map(ts))
    assert np.array_equal(acc, whole)
    # disjoint node ranges filled apart add up to the same array, bit for bit
    parts = np.zeros(pt.nnz)
    for n0, n1 in [(0, 1000), (1000, 3001), (3001, ob["dm"].n_nodes)]:
        As.scatter(prob, pt, local, out=parts, nodes=(n0, n1))
    assert np.array_equal(parts, whole)
