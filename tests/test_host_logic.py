"""CPU tests of the host-side logic: the C ABI library loads and exports every symbol
declared in include/iga.h; the host topology builder (iga_build_topology) matches the
oracle bit-exactly; bench.py's multi-rank timing reduction (gloo, world_size 2) and its
reference arm."""
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "iga.h")).read()
    return sorted(set(re.findall(r"^(?:iga_status|void|const char \*)\s*(iga_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2107_09568_b200 import _binding as B
    lib = B.load()
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(B.EXPORTS)
    assert b"sm_100a" in lib.iga_version()


def test_library_has_sm100a_code():
    from paper_2107_09568_b200 import _binding as B
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", B.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", B.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass


@pytest.mark.parametrize("c", [1, 2, 3])
def test_host_topology_bit_exact_vs_oracle(c, oracle_problem):
    from paper_2107_09568_b200 import Assembler
    ob = oracle_problem(c)
    prob, dm, pt = ob["prob"], ob["dm"], ob["pattern"]
    A = Assembler(prob, topology_only=True)
    s = A.sizes
    assert (s.n_dof, s.nnz, s.n_local_rows) == (dm.n_dof, pt.nnz, pt.n_rows_tile)
    rp = np.empty(s.n_dof + 1, np.int64)
    ci = np.empty(s.nnz, np.int32) if c < 3 else None
    A.pattern(rp, ci)
    assert np.array_equal(rp, pt.row_ptr)
    if ci is not None:
        assert np.array_equal(ci, pt.col_idx())
    nl = dm.n_local_ctrl
    assert s.n_local_ctrl == nl
    assert np.array_equal(A.node_map_for(nl), dm.node)
    assert np.array_equal(A.node_map_for(), dm.node)
    with pytest.raises(ValueError):   # a wrong row length is refused (the library writes n_tiles * n_local_ctrl)
        A.node_map_for(nl - 1)
    nt = min(prob.n_tiles, 6)
    assert np.array_equal(A.block_map(0, nt), pt.block_map()[:nt * s.n_local_rows])
    assert np.array_equal(A.pairs(), np.concatenate(ob["tabs"].pairs))


def test_binding_validates_buffers():
    """The binding checks dtype, length and contiguity of every [any] buffer before the C
    ABI reads or writes through it (ValueError; no compute call is reached)."""
    from paper_2107_09568_b200 import Assembler
    from synth import make_config
    prob = make_config(1)
    A = Assembler(prob, topology_only=True)
    s = A.sizes
    ctrl = np.ascontiguousarray(prob.macro.ctrl)
    young = np.ones(1)
    good = np.empty(s.nnz)
    with pytest.raises(ValueError, match="dtype"):
        A.assemble(ctrl.astype(np.float32), young, 0.3, good)
    with pytest.raises(ValueError, match="elements"):
        A.assemble(ctrl[:-1], young, 0.3, good)
    with pytest.raises(ValueError, match="elements"):
        A.assemble(ctrl, young, 0.3, np.empty(s.nnz - 1))
    with pytest.raises(ValueError, match="young"):
        A.assemble(ctrl, np.ones(3), 0.3, good)
    with pytest.raises(ValueError, match="contiguous"):
        A.sensitivity(ctrl, young, 0.3, np.empty(2 * s.n_dof)[::2], np.empty(s.n_dof), np.empty(ctrl.size))
    with pytest.raises(ValueError, match="grad"):
        A.sensitivity(ctrl, young, 0.3, np.empty(s.n_dof), np.empty(s.n_dof), np.empty(ctrl.size - 2))
    with pytest.raises(ValueError, match="col_idx"):
        A.pattern(np.empty(s.n_dof + 1, dtype=np.int64), np.empty(s.nnz, dtype=np.int64))
    torch = pytest.importorskip("torch")
    with pytest.raises(ValueError, match="dtype"):
        A.apply(ctrl, young, 0.3, torch.zeros(s.n_dof, dtype=torch.float32), np.empty(s.n_dof))


def test_topology_errors():
    from paper_2107_09568_b200 import Assembler, IgaError
    from synth import make_config
    p = make_config(1)
    p.tile[0].ctrl[6, 1] += 1e-3
    with pytest.raises(IgaError, match="ENONCONFORMING"):
        Assembler(p, topology_only=True)
    p = make_config(1)
    p.tile[0].knots[0] = np.array([0, 0, 0.5, 0.5, 0.5, 1, 1, 1.0])   # interior multiplicity 3 > p
    with pytest.raises(IgaError, match="EINVAL"):
        Assembler(p, topology_only=True)
    p = make_config(1)
    p.tile[0].ctrl[7] = [1.2, 0.5]                                    # outside [0,1]^d
    with pytest.raises(IgaError, match="EINVAL"):
        Assembler(p, topology_only=True)
    p = make_config(1, q=7)
    with pytest.raises(IgaError, match="EINVAL"):
        Assembler(p, topology_only=True)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    v = bench.reduce_max(10.0 + rank, world)
    bench.barrier(world)
    q.put((rank, v))
    dist.destroy_process_group()


def test_reduce_max_over_ranks_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: 11.0, 1: 11.0}


def test_reference_arm_json():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "tiles/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["e2e"]["h2d_bytes_per_step"] == 0


# ---------------------------------------------------------------------------
# sharding one problem (include/iga.h iga_shard): host topology

@pytest.mark.parametrize("c,n", [(2, 2), (3, 3)])
def test_shard_topology_partitions_rows_and_tiles(c, n):
    """Each shard's CSR rows are exactly the corresponding rows of the whole problem's
    pattern; row ranges and owned tiles partition the problem."""
    from paper_2107_09568_b200 import Assembler
    from synth import make_config
    prob = make_config(c)
    full = Assembler(prob, topology_only=True)
    fs = full.sizes
    rp = np.empty(fs.n_dof + 1, np.int64)
    ci = np.empty(fs.nnz, np.int32)
    full.pattern(rp, ci)
    nl = sum(p.n_ctrl for p in prob.tile)
    nm_full = full.node_map_for(nl)
    row, tile = 0, 0
    for s in range(n):
        A = Assembler(prob, topology_only=True, shard=(n, s))
        z = A.sizes
        assert (z.n_dof, z.n_tiles, z.n_nodes) == (fs.n_dof, fs.n_tiles, fs.n_nodes)
        assert z.row_begin == row and z.tile_begin == tile
        r1 = row + z.n_rows
        srp = np.empty(z.n_rows + 1, np.int64)
        sci = np.empty(z.nnz, np.int32)
        A.pattern(srp, sci)
        assert np.array_equal(srp, rp[row:r1 + 1] - rp[row])
        assert np.array_equal(sci, ci[rp[row]:rp[r1]])
        assert np.array_equal(A.node_map_for(nl), nm_full[tile:tile + z.n_tiles_local])
        assert z.n_tiles_local - z.n_tiles_owned in (0, prob.n_tiles // prob.n_el[-1])   # one halo layer
        # block map: positions of owned rows shifted by the shard's first value, -1 elsewhere
        bm = A.block_map(0, 2)
        bf = full.block_map(tile, tile + 2)
        shift = rp[row]
        ok = bm >= 0
        assert np.array_equal(bm[ok], bf[ok] - shift)
        assert np.all((bf[~ok] < shift) | (bf[~ok] >= rp[r1]))
        row, tile = r1, tile + z.n_tiles_owned
    assert row == fs.n_dof and tile == fs.n_tiles


def _shard_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    from paper_2107_09568_b200 import Assembler
    from paper_2107_09568_b200.shard import allreduce_grad, shard_of
    from synth import make_config, draw_uv_seeded
    from oracle.assemble import Tables
    from oracle.dofmap import DofMap, Pattern
    from oracle import sensitivity as S
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prob = make_config(2, n_el=(2, 2, 2))
    z = Assembler(prob, topology_only=True, shard=shard_of(rank, world)).sizes
    ranges = [None] * world
    dist.all_gather_object(ranges, (z.row_begin, z.n_rows, z.tile_begin, z.n_tiles_owned, z.nnz))
    # the data-path collective of the sharded step: partial gradients over owned tiles
    dm = DofMap(prob)
    tabs = Tables(prob)
    pt = Pattern(prob, dm, tabs.pairs)
    u, v = draw_uv_seeded(2, dm.n_dof)
    own = range(z.tile_begin, z.tile_begin + z.n_tiles_owned)
    g = torch.tensor(S.sensitivity(prob, tabs, pt, u, v, tiles=own))
    allreduce_grad(g, world)
    full = S.sensitivity(prob, tabs, pt, u, v) if rank == 0 else None
    q.put((rank, ranges, g.numpy(), full))
    dist.destroy_process_group()


def test_shard_gradient_allreduce_gloo():
    """world_size 2 (gloo, CPU): shards partition rows and tiles, and the all-reduce of the
    per-shard partial gradients (oracle arithmetic over each rank's owned tiles) equals
    the whole problem's gradient."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r, ranges, g, full = q.get(timeout=600)
        res[r] = (ranges, g, full)
    for p in ps:
        p.join(60)
    ranges = res[0][0]
    assert ranges == res[1][0]
    (rb0, nr0, tb0, nt0, _), (rb1, nr1, tb1, nt1, _) = ranges
    assert rb0 == 0 and rb1 == nr0 and tb0 == 0 and tb1 == nt0 and nt0 + nt1 == 8
    full = res[0][2]
    for r in range(2):
        assert np.abs(res[r][1] - full).max() < 1e-13 * np.abs(full).max()


# ---------------------------------------------------------------------------
# The Eq. 38-reduced contraction the GPU evaluates, checked on the host
# against the oracle's plain Eq. 58 product: L = L⁺ ± L⁻ with L⁺ from [𝔎_ii | 𝔎_ij + 𝔎_ji]
# and the symmetric coefficient halves, L⁻ from 𝔎_ij − 𝔎_ji and the antisymmetric halves;
# and uᵀK^πv = Σ (X̃⁺ L⁺ + X̃⁻ L⁻).  (Design identity, numpy; no CUDA.)

def _sym_pairs(d):
    p1 = [(a, a) for a in range(d)] + [(a, b) for a in range(d) for b in range(a + 1, d)]
    p2 = [(a, b) for a in range(d) for b in range(a + 1, d)]
    return p1, p2


@pytest.mark.parametrize("c,kw", [(1, {}), (2, dict(n_el=(2, 1, 1))), (2, dict(n_el=(2, 1, 1), q=(1, 2, 3)))])
def test_eq38_reduced_contraction_identity(c, kw):
    from oracle import assemble as As, macro as M, sensitivity as S
    from oracle.dofmap import DofMap, Pattern
    from synth import make_config, draw_uv_seeded
    prob = make_config(c, **kw)
    d = prob.d
    tabs = As.Tables(prob)
    dm = DofMap(prob)
    pt = Pattern(prob, dm, tabs.pairs)
    npi = tabs.T.shape[1] // (d * d)
    T = tabs.T.reshape(-1, d, d, npi)                       # [r][i][j][C]
    p1, p2 = _sym_pairs(d)
    A1 = np.concatenate([T[:, i, i] if i == j else T[:, i, j] + T[:, j, i] for i, j in p1], axis=1)
    A2 = np.concatenate([T[:, i, j] - T[:, j, i] for i, j in p2], axis=1)
    # multiply-adds per row and tile: n_π(n_p1² + n_p2²) (45 n_π in 3D, 10 n_π in 2D) < d⁴ n_π
    assert A1.shape[1] * len(p1) + A2.shape[1] * len(p2) == (len(p1) ** 2 + len(p2) ** 2) * npi < d ** 4 * npi
    u, v = draw_uv_seeded(c + 70, dm.n_dof)
    utkv = 0.0
    for t in range(prob.n_tiles):
        coef = M.tile_coefficients(prob, prob.macro.ctrl, t)   # [C][i][j][a][b]
        B1 = np.stack([np.concatenate([0.5 * (coef[:, i, j, a, b] + coef[:, i, j, b, a]) for i, j in p1])
                       for a, b in p1], axis=1)
        B2 = np.stack([np.concatenate([0.5 * (coef[:, i, j, a, b] - coef[:, i, j, b, a]) for i, j in p2])
                       for a, b in p2], axis=1)
        Lp, Lm = A1 @ B1, A2 @ B2                           # L⁺/2 and L⁻/2 per output pair
        L = np.zeros((T.shape[0], d, d))
        for o, (a, b) in enumerate(p1):
            L[:, a, b] += Lp[:, o]
            if a != b:
                L[:, b, a] += Lp[:, o]
        for o, (a, b) in enumerate(p2):
            L[:, a, b] += Lm[:, o]
            L[:, b, a] -= Lm[:, o]
        ref = As.local_lookup(prob, tabs, prob.macro.ctrl, [t])[0]
        assert np.linalg.norm(L - ref) <= 1e-13 * np.linalg.norm(ref)
        X = S.adjoint_X(prob, pt, u, v, t)                  # [r][a][b]
        Xp = np.stack([X[:, a, b] if a == b else X[:, a, b] + X[:, b, a] for a, b in p1], axis=1)
        Xm = np.stack([X[:, a, b] - X[:, b, a] for a, b in p2], axis=1)
        utkv += np.sum(Xp * Lp) + np.sum(Xm * Lm)
    K = As.assemble_lookup(prob, tabs, pt)[0]
    import scipy.sparse as sp
    Kc = sp.csr_matrix((K, pt.col_idx(), pt.row_ptr), shape=(dm.n_dof, dm.n_dof))
    ref = u @ (Kc @ v)
    assert abs(utkv - ref) <= 1e-12 * abs(ref)
