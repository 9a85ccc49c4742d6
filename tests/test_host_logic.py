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
    assert np.array_equal(A.node_map_for(nl), dm.node)
    nt = min(prob.n_tiles, 6)
    assert np.array_equal(A.block_map(0, nt), pt.block_map()[:nt * s.n_local_rows])
    assert np.array_equal(A.pairs(), np.concatenate(ob["tabs"].pairs))


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
