"""The sharded step (include/iga.h iga_shard, paper_2107_09568_b200/shard.py) in two
processes on cuda:0 with libiga: every rank forms its slab's CSR rows and its partial
gradient, one gloo all-reduce (through host copies) sums the gradients.  The concatenated
shard rows must equal the one-process K bit for bit, and the all-reduced gradient the
one-process gradient.  The ranks never wait on each other inside a kernel."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rank_main(rank, world, port, q, c, n_el):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2107_09568_b200.shard import ShardedStep
        from synth import make_config, draw_uv_seeded
        torch.cuda.set_device(0)
        prob = make_config(c, n_el=n_el)
        st = ShardedStep(prob, rank, world)
        s = st.sizes
        dev = torch.device("cuda:0")
        ctrl = torch.tensor(prob.macro.ctrl, device=dev)
        young = torch.tensor(prob.young, device=dev)
        vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
        st.assemble(ctrl, young, prob.nu, vals)
        u, v = draw_uv_seeded(c + 50, s.n_dof)
        grad = torch.empty(s.n_macro_cp * prob.d, dtype=torch.float64, device=dev)
        st.sensitivity(ctrl, young, prob.nu, torch.tensor(u, device=dev), torch.tensor(v, device=dev), grad)
        torch.cuda.synchronize()
        q.put((rank, int(s.row_begin), int(s.n_rows), vals.cpu().numpy(), grad.cpu().numpy(), None))
    except Exception as e:   # report, do not hang the parent
        q.put((rank, 0, 0, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("c,n_el", [(2, (2, 2, 4)), (3, (4, 2, 4))])
def test_sharded_step_two_processes(c, n_el):
    import torch.multiprocessing as mp
    from paper_2107_09568_b200 import Assembler
    from synth import make_config, draw_uv_seeded
    world = 2
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = 31500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_rank_main, args=(r, world, port, qu, c, n_el)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r = qu.get(timeout=900)
        assert r[5] is None, r[5]
        res[r[0]] = r[1:5]
    for p in ps:
        p.join(120)
    # the one-process reference on the same GPU
    prob = make_config(c, n_el=n_el)
    A = Assembler(prob)
    s = A.sizes
    dev = torch.device("cuda:0")
    ctrl = torch.tensor(prob.macro.ctrl, device=dev)
    young = torch.tensor(prob.young, device=dev)
    vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
    A.assemble(ctrl, young, prob.nu, vals)
    rp = torch.empty(s.n_dof + 1, dtype=torch.int64, device=dev)
    A.pattern(rp, None)
    u, v = draw_uv_seeded(c + 50, s.n_dof)
    grad = torch.empty(s.n_macro_cp * prob.d, dtype=torch.float64, device=dev)
    A.sensitivity(ctrl, young, prob.nu, torch.tensor(u, device=dev), torch.tensor(v, device=dev), grad)
    full_vals, full_g, rp = vals.cpu().numpy(), grad.cpu().numpy(), rp.cpu().numpy()
    assert res[0][0] == 0 and res[1][0] == res[0][1] and res[0][1] + res[1][1] == s.n_dof   # row ranges partition
    for r in range(world):
        rb, nr, vr, gr = res[r]
        assert np.array_equal(vr, full_vals[rp[rb]:rp[rb + nr]]), r                     # bit-identical rows
        assert np.array_equal(gr, res[0][3])                                            # the same all-reduced g
    g = res[0][3]
    assert np.linalg.norm(g - full_g) <= 1e-13 * np.linalg.norm(full_g)
