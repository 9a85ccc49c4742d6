"""The full-size parity machinery (tests/parity_tools.py) on a small config, on the CPU:
the pooled oracle calls reproduce the plain serial oracle bit for bit, and the chunked
column-index check accepts the oracle's own col_idx and rejects a perturbed one."""
import numpy as np
import pytest

import parity_tools as PT


def test_pool_reproduces_serial_oracle(oracle_problem, monkeypatch):
    import scipy.sparse as sp
    from oracle import assemble as As, sensitivity as S
    from synth import draw_uv_seeded
    monkeypatch.setenv("IGA_TEST_WORKERS", "3")
    ob = oracle_problem(2)
    prob, pt, tabs = ob["prob"], ob["pattern"], ob["tabs"]
    d = prob.d
    local = PT.shared_array((prob.n_tiles, pt.n_rows_tile, d, d), np.float64)
    PT.run(PT.w_local, PT.tile_chunks(prob.n_tiles, 7), prob=prob, tabs=tabs, local=local)
    ref_local = As.local_lookup(prob, tabs, prob.macro.ctrl, range(prob.n_tiles))
    assert np.array_equal(local, ref_local)
    bm = PT.shared_array((prob.n_tiles * pt.n_rows_tile, 2), np.int64)
    PT.run(PT.w_block_map, PT.tile_chunks(prob.n_tiles, 5), pattern=pt, bm=bm)
    assert np.array_equal(bm, pt.block_map())
    vals = PT.shared_array((pt.nnz,), np.float64)
    ranges = PT.node_ranges(pt, d, 5)
    assert ranges[0][0] == 0 and ranges[-1][1] == ob["dm"].n_nodes
    assert all(r0[1] == r1[0] for r0, r1 in zip(ranges, ranges[1:]))
    PT.run(PT.w_scatter, ranges, prob=prob, pattern=pt, local=local, bm=bm, vals=vals, chunk=9)
    whole = As.scatter(prob, pt, ref_local)
    assert np.array_equal(vals, whole)
    u, v = draw_uv_seeded(2, pt.row_ptr.size - 1)
    y = PT.shared_array((len(u),), np.float64)
    PT.run(PT.w_spmv, ranges, prob=prob, pattern=pt, vals=vals, u=u, y=y)
    K = sp.csr_matrix((whole, pt.col_idx(), pt.row_ptr), shape=(len(u), len(u)))
    assert np.abs(y - K @ u).max() < 1e-13 * np.abs(K @ u).max()
    ent = [(5, 0), (17, 2), (100, 1)]
    parts = PT.run(PT.w_sensitivity, PT.tile_chunks(prob.n_tiles, 11), prob=prob, tabs=tabs, pattern=pt,
                   u=u, v=v, entries=ent)
    g = S.sensitivity(prob, tabs, pt, u, v, entries=ent)
    assert np.abs(np.sum(parts, axis=0) - g).max() <= 1e-14 * np.abs(g).max()


def test_check_col_idx(oracle_problem):
    torch = pytest.importorskip("torch")
    ob = oracle_problem(1)
    pt = ob["pattern"]
    ci = torch.from_numpy(pt.col_idx())
    PT.check_col_idx(ci, pt, 2, max_entries=4000)          # several chunks
    bad = ci.clone()
    bad[12345] += 2
    with pytest.raises(AssertionError):
        PT.check_col_idx(bad, pt, 2, max_entries=4000)
