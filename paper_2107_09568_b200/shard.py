"""One problem sharded over torch.distributed ranks (include/iga.h
`iga_shard`): rank r forms the slab r of macro-element layers (plus one halo layer) —
its own CSR rows of K, no communication — and its partial gradient, which one
all-reduce sums.  Plumbing only: every arithmetic step runs in libiga's kernels."""
from __future__ import annotations

from ._binding import Assembler


def shard_of(rank: int, world: int):
    return (world, rank) if world > 1 else None


def allreduce_grad(grad, world: int):
    """Σ over ranks of the per-shard partial gradients (n_macro_cp*d doubles): the one
    data-path collective of the sharded step (NCCL on GPUs, gloo on CPU tensors)."""
    if world > 1:
        import torch.distributed as dist
        if grad.is_cuda and dist.get_backend() == "gloo":   # gloo: through a host copy
            h = grad.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM)
            grad.copy_(h)
        else:
            dist.all_reduce(grad, op=dist.ReduceOp.SUM)
    return grad


class ShardedStep:
    """K rows [row_begin, row_begin + n_rows) of this rank and the full gradient."""

    def __init__(self, prob, rank: int, world: int, stream=None):
        self.world = world
        self.A = Assembler(prob, stream=stream, shard=shard_of(rank, world))
        self.sizes = self.A.sizes

    def assemble(self, ctrl, young, nu, values, stream=None):
        self.A.assemble(ctrl, young, nu, values, stream=stream)

    def sensitivity(self, ctrl, young, nu, u, v, grad, stream=None):
        self.A.sensitivity(ctrl, young, nu, u, v, grad, stream=stream)
        return allreduce_grad(grad, self.world)
