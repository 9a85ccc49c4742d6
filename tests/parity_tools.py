"""Test infrastructure for parity at BASELINE.json's full sizes.

* `run(fn, chunks, **state)`: calls `fn(state, chunk)` for every chunk in a fork pool of
  host processes (one BLAS thread each) and returns the results in chunk order.  The
  workers below only call `oracle/` functions on tile or node ranges; outputs that are
  large go to `shared_array`s, which forked workers write in place.
* `check_col_idx`: compares the library's CSR column indices with the oracle's block
  pattern, expanded entry by entry on the device in chunks (cfg5: 2.9e9 entries).

Nothing here computes a reference value itself: every reference number comes from
`oracle/` (local_lookup, block_map, scatter, sensitivity) on the seeded inputs.
"""
from __future__ import annotations

import mmap
import multiprocessing as mp
import os

import numpy as np

_STATE: dict = {}


def n_workers():
    return max(1, min(int(os.environ.get("IGA_TEST_WORKERS", os.cpu_count() or 1)), 48))


def shared_array(shape, dtype):
    """Zero-filled array in anonymous shared memory (visible to forked workers)."""
    count = int(np.prod(shape))
    buf = mmap.mmap(-1, max(count * np.dtype(dtype).itemsize, 1))
    return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)


def _init():
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)


def _call(args):
    fn, chunk = args
    return fn(_STATE, chunk)


def run(fn, chunks, **state):
    _STATE.clear()
    _STATE.update(state)
    chunks = list(chunks)
    if len(chunks) == 1 or n_workers() == 1:
        return [fn(_STATE, c) for c in chunks]
    with mp.get_context("fork").Pool(min(n_workers(), len(chunks)), initializer=_init) as pool:
        return pool.map(_call, [(fn, c) for c in chunks], chunksize=1)


def tile_chunks(n_tiles, size):
    return [np.arange(t, min(n_tiles, t + size)) for t in range(0, n_tiles, size)]


def node_ranges(pattern, d, parts):
    """`parts` node ranges [n0, n1) with about equal numbers of CSR entries."""
    rp = pattern.row_ptr[::d]                       # first row of each node (+ the end)
    nn = len(rp) - 1
    cuts = np.searchsorted(rp, np.linspace(0, rp[-1], parts + 1)[1:-1])
    b = np.unique(np.concatenate([[0], np.clip(cuts, 0, nn), [nn]]))
    return [(int(b[k]), int(b[k + 1])) for k in range(len(b) - 1)]


# --- workers (oracle calls only) ---------------------------------------------------
def w_local(S, tiles):
    """oracle K^π element matrices of `tiles` -> S['local'][tiles]."""
    from oracle import assemble as As
    S["local"][tiles] = As.local_lookup(S["prob"], S["tabs"], S["prob"].macro.ctrl, tiles)


def w_block_map(S, tiles):
    """oracle block map rows of `tiles` (consecutive) -> S['bm']."""
    nr = S["pattern"].n_rows_tile
    S["bm"][tiles[0] * nr:(tiles[-1] + 1) * nr] = S["pattern"].block_map(tiles)


def w_scatter(S, nodes):
    """oracle scatter (reading R9) of every tile, restricted to the CSR rows of `nodes`,
    into S['vals'] (tiles in order, so every entry sums its contributions in (t, row) order)."""
    from oracle import assemble as As
    prob, pt, nr = S["prob"], S["pattern"], S["pattern"].n_rows_tile
    for ts in tile_chunks(prob.n_tiles, S.get("chunk", 128)):
        As.scatter(prob, pt, S["local"][ts], tiles=ts, out=S["vals"],
                   bmap=S["bm"][ts[0] * nr:(ts[-1] + 1) * nr], nodes=nodes)


def w_sensitivity(S, tiles):
    """the oracle's complex-step terms of Eq. 73's sum over `tiles` (entries or all)."""
    from oracle import sensitivity as Se
    return Se.sensitivity(S["prob"], S["tabs"], S["pattern"], S["u"], S["v"], entries=S.get("entries"), tiles=tiles)


def w_spmv(S, nodes):
    """y = K u on the rows of `nodes` with the oracle's K values and block pattern."""
    pt, d, vals, u = S["pattern"], S["prob"].d, S["vals"], S["u"]
    n0, n1 = nodes
    for I in range(n0, n1, 8192):
        I1 = min(n1, I + 8192)
        L = pt.nnzb[I:I1] * d                                     # entries per row of each node
        u_node = u.reshape(-1, d)[pt.bcol[pt.brow_ptr[I]:pt.brow_ptr[I1]]].ravel()
        node_start = np.cumsum(L) - L
        row_len = np.repeat(L, d)
        row_start = np.cumsum(row_len) - row_len
        entry_row = np.repeat(np.arange(len(row_len)), row_len)
        pos = np.arange(int(row_len.sum())) - row_start[entry_row]
        ug = u_node[node_start[entry_row // d] + pos]
        seg = vals[pt.row_ptr[I * d]:pt.row_ptr[I1 * d]]
        S["y"][I * d:I1 * d] = np.add.reduceat(seg * ug, row_start)


# --- device-side comparison of the column indices ------------------------------------
def check_col_idx(ci, pattern, d, max_entries=1 << 28):
    """ci (device int32, nnz): ci[row_ptr[I*d+a] + m*d + b] == bcol[brow_ptr[I] + m]*d + b
    for every node I, a, m, b (the oracle's block pattern, reading R9)."""
    import torch
    dev = ci.device
    bcol = torch.from_numpy(pattern.bcol.astype(np.int64)).to(dev)
    brow = torch.from_numpy(pattern.brow_ptr.astype(np.int64)).to(dev)
    rp = pattern.row_ptr
    nn = len(pattern.nnzb)
    nodes_rp = rp[::d]
    I0 = 0
    while I0 < nn:
        I1 = int(np.searchsorted(nodes_rp, nodes_rp[I0] + max_entries, side="right")) - 1
        I1 = min(nn, max(I1, I0 + 1))
        e0, e1 = int(rp[I0 * d]), int(rp[I1 * d])
        nb = torch.from_numpy(pattern.nnzb[I0:I1].astype(np.int64)).to(dev)
        node_of_row = torch.arange(I0, I1, device=dev).repeat_interleave(d)
        rowlen = nb.repeat_interleave(d) * d
        rowstart = torch.cumsum(rowlen, 0) - rowlen
        entry_row = torch.repeat_interleave(torch.arange(len(rowlen), device=dev), rowlen)
        pos = torch.arange(e1 - e0, device=dev) - rowstart[entry_row]
        expect = bcol[brow[node_of_row[entry_row]] + pos // d] * d + pos % d
        if not torch.equal(ci[e0:e1].to(torch.int64), expect):
            bad = torch.nonzero(ci[e0:e1].to(torch.int64) != expect)[0].item()
            raise AssertionError(f"col_idx differs at entry {e0 + bad}")
        del node_of_row, rowlen, rowstart, entry_row, pos, expect
        I0 = I1
