"""GPU parity at BASELINE.json's full sizes (cfg4: 1024 tiles, p = q = 3, per-tile E;
cfg5: 8192 tiles, the bench workload), in the launch configuration bench.py times,
against the oracle computed in full (north star: pattern and index maps bit-exact,
≤ 1e-12 per element matrix, ≤ 1e-11 on K's values; gradient ≤ 1e-11 relative 2-norm):

  * sizes against the closed forms of tests/golden/pattern_counts.json and the oracle;
  * row_ptr, col_idx (every entry), the node map and the block map of every tile against
    the oracle's DofMap / Pattern (oracle/dofmap.py, readings R9, R10);
  * the tables of all 6 tile patches (Eq. 52);
  * the element matrices of every tile (Eq. 58; oracle local_lookup);
  * all of K's values (oracle scatter of every tile, reading R9);
  * the sensitivity (Eq. 73): the complete gradient at cfg4, ≥ 256 entries at cfg5 incl.
    the corners and other boundary control points (oracle complex step);
  * the matrix-free apply (Eq. 74) against the oracle's K times u;
  * properties: bitwise K(I,J) = K(J,I)ᵀ and translations in the kernel on sampled rows,
    Σ_k g[k] = 0 and Σ P·g = (d-2)·uᵀKv.
Oracle work runs in a fork pool of host processes (tests/parity_tools.py).
"""
import gc
import json
import os

import numpy as np
import pytest

import parity_tools as PT

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOL_TABLE = 1e-13
TOL_ELEM = 1e-12
TOL_K = 1e-11
TOL_SENS = 1e-11
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pattern_counts.json")))


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module", params=[4, 5], ids=["cfg4", "cfg5"])
def F(request):
    """GPU K (+ element matrices) and the oracle's DofMap / Pattern / tables of one config."""
    from oracle.assemble import Tables
    from oracle.dofmap import DofMap, Pattern
    from paper_2107_09568_b200 import Assembler
    from synth import make_config
    gc.collect()
    torch.cuda.empty_cache()
    c = request.param
    prob = make_config(c)
    A = Assembler(prob)
    s = A.sizes
    d = prob.d
    dev = torch.device("cuda:0")
    g = dict(c=c, prob=prob, A=A, s=s, d=d)
    g["ctrl"] = torch.tensor(prob.macro.ctrl, dtype=torch.float64, device=dev)
    g["young"] = torch.tensor(prob.young, dtype=torch.float64, device=dev)
    g["vals"] = torch.empty(s.nnz, dtype=torch.float64, device=dev)
    g["local"] = torch.empty(s.n_local_rows * s.n_tiles * d * d, dtype=torch.float64, device=dev)
    A.assemble(g["ctrl"], g["young"], prob.nu, g["vals"], g["local"])
    g["rp"] = torch.empty(s.n_dof + 1, dtype=torch.int64, device=dev)
    g["ci"] = torch.empty(s.nnz, dtype=torch.int32, device=dev)
    A.pattern(g["rp"], g["ci"])
    torch.cuda.synchronize()
    g["dm"] = DofMap(prob)
    g["tabs"] = Tables(prob)
    g["pt"] = Pattern(prob, g["dm"], g["tabs"].pairs)
    yield g
    g.clear()
    gc.collect()
    torch.cuda.empty_cache()


def oracle_block_map(F):
    if "bm" not in F:
        pt, nt = F["pt"], F["prob"].n_tiles
        F["bm"] = PT.shared_array((nt * pt.n_rows_tile, 2), np.int64)
        PT.run(PT.w_block_map, PT.tile_chunks(nt, 64), pattern=pt, bm=F["bm"])
    return F["bm"]


def oracle_local(F):
    if "olocal" not in F:
        prob, pt = F["prob"], F["pt"]
        d = prob.d
        F["olocal"] = PT.shared_array((prob.n_tiles, pt.n_rows_tile, d, d), np.float64)
        PT.run(PT.w_local, PT.tile_chunks(prob.n_tiles, 16), prob=prob, tabs=F["tabs"], local=F["olocal"])
    return F["olocal"]


def oracle_vals(F):
    if "ovals" not in F:
        prob, pt = F["prob"], F["pt"]
        F["ovals"] = PT.shared_array((pt.nnz,), np.float64)
        PT.run(PT.w_scatter, PT.node_ranges(pt, prob.d, 4 * PT.n_workers()), prob=prob, pattern=pt,
               local=oracle_local(F), bm=oracle_block_map(F), vals=F["ovals"])
    return F["ovals"]


# ---------------------------------------------------------------------------------------
def test_fullsize_sizes_match_golden_and_oracle(F):
    s, prob = F["s"], F["prob"]
    gold = GOLD[f"cfg{F['c']}"]
    assert (s.n_dof, s.nnz) == (gold["n_dof"], gold["nnz"])
    assert (F["dm"].n_dof, F["pt"].nnz) == (gold["n_dof"], gold["nnz"])
    assert s.n_nodes == F["dm"].n_nodes and s.n_tiles == prob.n_tiles
    assert s.n_local_rows == F["pt"].n_rows_tile


def test_fullsize_row_ptr_and_col_idx_bit_exact(F):
    assert np.array_equal(F["rp"].cpu().numpy(), F["pt"].row_ptr)
    PT.check_col_idx(F["ci"], F["pt"], F["d"])


def test_fullsize_node_map_bit_exact(F):
    nl = F["dm"].n_local_ctrl
    assert np.array_equal(F["A"].node_map_for(nl), F["dm"].node)


def test_fullsize_block_map_bit_exact(F):
    """Every tile's block map (pos(I·d, J·d), pos(J·d, I·d)) against the oracle's."""
    bm = oracle_block_map(F)
    nr, nt = F["pt"].n_rows_tile, F["prob"].n_tiles
    for t0 in range(0, nt, 512):
        t1 = min(nt, t0 + 512)
        assert np.array_equal(F["A"].block_map(t0, t1), bm[t0 * nr:t1 * nr]), (t0, t1)


def test_fullsize_tables_all_patches(F):
    """The lookup tables of all 6 strut patches (Eq. 52; ≤ 1e-13 per patch)."""
    Tg = F["A"].tables()
    assert np.array_equal(F["A"].pairs(), np.concatenate(F["tabs"].pairs))
    off = 0
    for Tp, _ in F["tabs"].per_patch:
        assert rel(Tg[off:off + len(Tp)], Tp) < TOL_TABLE
        off += len(Tp)


def test_fullsize_element_matrices_every_tile(F):
    ref = oracle_local(F)
    s, d = F["s"], F["d"]
    Lg = F["local"].view(s.n_local_rows, s.n_tiles, d, d)
    worst = 0.0
    for t0 in range(0, s.n_tiles, 256):
        t1 = min(s.n_tiles, t0 + 256)
        got = Lg[:, t0:t1].permute(1, 0, 2, 3).cpu().numpy()
        r = ref[t0:t1]
        err = np.linalg.norm((got - r).reshape(t1 - t0, -1), axis=1) / np.linalg.norm(r.reshape(t1 - t0, -1), axis=1)
        worst = max(worst, float(err.max()))
        assert err.max() < TOL_ELEM, (t0 + int(err.argmax()), float(err.max()))
    print(f"cfg{F['c']}: worst element-matrix rel. error {worst:.2e} over {s.n_tiles} tiles")


def test_fullsize_K_values(F):
    """All of K (nnz values) against the oracle's scatter of every tile's element matrices."""
    ref = oracle_vals(F)
    nnz = F["s"].nnz
    num = den = 0.0
    step = 1 << 28
    for e0 in range(0, nnz, step):
        e1 = min(nnz, e0 + step)
        got = F["vals"][e0:e1].cpu().numpy()
        num += float(np.sum((got - ref[e0:e1]) ** 2))
        den += float(np.sum(ref[e0:e1] ** 2))
    err = (num / den) ** 0.5
    print(f"cfg{F['c']}: K rel. Frobenius error {err:.2e} over {nnz} values")
    assert err < TOL_K


def test_fullsize_matrix_free_apply(F):
    """iga_apply (Eq. 74) against the oracle's K times u (all rows)."""
    from synth import draw_uv_seeded
    prob, s, d = F["prob"], F["s"], F["d"]
    u, _ = draw_uv_seeded(F["c"], s.n_dof)
    y = torch.empty(s.n_dof, dtype=torch.float64, device="cuda")
    F["A"].apply(F["ctrl"], F["young"], prob.nu, torch.tensor(u, device="cuda"), y)
    yref = PT.shared_array((s.n_dof,), np.float64)
    PT.run(PT.w_spmv, PT.node_ranges(F["pt"], d, 2 * PT.n_workers()), prob=prob, pattern=F["pt"],
           vals=oracle_vals(F), u=u, y=yref)
    err = rel(y.cpu().numpy(), yref)
    print(f"cfg{F['c']}: apply rel. error {err:.2e}")
    assert err < TOL_K


def sens_entries(prob, n_cp_target):
    """Macro control points: the 2^d corners, points on every face and edge, and interior
    ones; all d coordinates of each."""
    n = prob.macro.n_per_dir
    d = prob.d
    rng = np.random.default_rng(400 + prob.d)
    idx = set()
    for corner in range(2 ** d):
        idx.add(tuple((n[k] - 1) * ((corner >> k) & 1) for k in range(d)))
    while len(idx) < n_cp_target:
        ii = [int(rng.integers(0, n[k])) for k in range(d)]
        if len(idx) % 2 == 0:                     # half of them on the boundary
            k = int(rng.integers(0, d))
            ii[k] = 0 if rng.random() < 0.5 else n[k] - 1
        idx.add(tuple(ii))
    cps = sorted(int(sum(ii[k] * int(np.prod(n[:k])) for k in range(d))) for ii in idx)
    return [(k, a) for k in cps for a in range(d)]


def test_fullsize_sensitivity(F):
    from synth import draw_uv_seeded
    prob, A, s, d = F["prob"], F["A"], F["s"], F["d"]
    u, v = draw_uv_seeded(F["c"], s.n_dof)
    ut, vt = torch.tensor(u, device="cuda"), torch.tensor(v, device="cuda")
    grad = torch.empty(s.n_macro_cp * d, dtype=torch.float64, device="cuda")
    A.sensitivity(F["ctrl"], F["young"], prob.nu, ut, vt, grad)
    got = grad.cpu().numpy().reshape(-1, d)
    entries = None if F["c"] == 4 else sens_entries(prob, 90)           # cfg4: complete gradient
    parts = PT.run(PT.w_sensitivity, PT.tile_chunks(prob.n_tiles, 8), prob=prob, tabs=F["tabs"],
                   pattern=F["pt"], u=u, v=v, entries=entries)
    ref = np.sum(parts, axis=0)
    if entries is None:
        err = rel(got, ref)
        n_checked = got.size
    else:
        assert len(entries) >= 256
        k, a = np.array(entries).T
        err = rel(got[k, a], ref[k, a])
        n_checked = len(entries)
    print(f"cfg{F['c']}: gradient rel. 2-norm error {err:.2e} over {n_checked} entries")
    assert err < TOL_SENS
    # properties over the whole GPU gradient
    scale = np.abs(got).max()
    assert np.abs(got.sum(0)).max() < 1e-10 * scale                      # translation invariance
    uKv = float(np.dot(u, PT_spmv_gpu(F, vt).cpu().numpy()))
    euler = float(np.sum(prob.macro.ctrl * got))
    assert abs(euler - (d - 2) * uKv) < 1e-9 * max(abs(uKv), scale)      # Σ P·g = (d-2) uᵀKv


def PT_spmv_gpu(F, v, max_nnz=1 << 30):
    """K v with the GPU's CSR K (row slices of < 2^30 non-zeros: torch's sparse mv)."""
    rp = F["pt"].row_ptr
    n = len(rp) - 1
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    r0 = 0
    while r0 < n:
        r1 = max(int(np.searchsorted(rp, rp[r0] + max_nnz, side="right")) - 1, r0 + 1)
        a, b = int(rp[r0]), int(rp[r1])
        sub = torch.sparse_csr_tensor(F["rp"][r0:r1 + 1] - a, F["ci"][a:b].to(torch.int64), F["vals"][a:b],
                                      size=(r1 - r0, n))
        out[r0:r1] = torch.mv(sub, v)
        r0 = r1
    return out


def test_fullsize_symmetry_and_rigid_translations(F):
    """Bitwise K(I,J) = K(J,I)ᵀ on sampled node rows; K·(translation) = 0 row-wise."""
    d, pt = F["d"], F["pt"]
    rp = pt.row_ptr
    rng = np.random.default_rng(300 + F["c"])

    def row(I):
        cols = pt.bcol[pt.brow_ptr[I]:pt.brow_ptr[I + 1]]
        blk = np.stack([F["vals"][rp[I * d + a]:rp[I * d + a + 1]].cpu().numpy().reshape(-1, d) for a in range(d)], 1)
        return cols, blk                                                  # blk[m] = K(I, cols[m])
    for I in rng.choice(F["dm"].n_nodes, 16, replace=False):
        cols, blk = row(int(I))
        for a in range(d):
            assert abs(blk[:, a, :].sum(axis=0)).max() < 1e-11 * abs(blk).max()
        for m, J in enumerate(cols[:6]):
            cj, bj = row(int(J))
            k = int(np.searchsorted(cj, I))
            assert cj[k] == I and np.array_equal(bj[k], blk[m].T)
