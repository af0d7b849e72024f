"""Batch sharding across GPUs (one process per GPU).

Knot points are independent: rank r of W evaluates the
contiguous slice `shard_bounds(N, W, r)` of the batch on its own device; no
data crosses GPUs on the hot path.  `gather` optionally assembles the full
result on every rank with one all-gather per output (NCCL over NVLink when
the tensors are on the GPU) for a device-resident consumer.
"""

import numpy as np


def shard_bounds(N, world, rank):
    """[start, stop) of rank's contiguous slice; sizes differ by at most one."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    base, extra = divmod(int(N), int(world))
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard(arrays, world, rank):
    N = arrays[0].shape[0]
    a, b = shard_bounds(N, world, rank)
    return [x[a:b] for x in arrays], (a, b)


def gather(local, N, group=None):
    """All-gather equal-padded slices of a (n_local, ...) torch tensor into (N, ...)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    size = -(-N // world)
    pad = torch.zeros((size,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    out = torch.empty((size * world,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    parts = []
    for r in range(world):
        a, b = shard_bounds(N, world, r)
        parts.append(out[r * size:r * size + (b - a)])
    return torch.cat(parts, 0)


def run_sharded(evaluate, arrays, group=None, gather_result=False):
    """Evaluate this rank's slice with `evaluate(list_of_arrays) -> list of outputs`;
    optionally all-gather every output to the full batch."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    N = arrays[0].shape[0]
    mine, bounds = shard(arrays, world, rank)
    outs = evaluate(mine)
    if gather_result:
        outs = [gather(o, N, group) for o in outs]
    return outs, bounds


def evaluate_sharded(fn, model, *arrays, group=None, gather_result=False, **kw):
    """This rank's contiguous slice of a batch through a drop-in dynamics
    entry (`fn` = dynamics.fd_grad, rnea, ...) on this rank's device -- the
    generated kernels, one process per GPU, no collective on the hot path;
    with gather_result, the outputs are all-gathered to the full batch (NCCL
    over NVLink for CUDA tensors, gloo for host tensors)."""
    def evaluate(parts):
        out = fn(model, *parts, **kw)
        if hasattr(out, "dq"):
            out = [out.dq, out.dqd] + ([out.qdd] if out.qdd is not None else [])
        elif not isinstance(out, (list, tuple)):
            out = [out]
        return list(out)
    return run_sharded(evaluate, list(arrays), group=group, gather_result=gather_result)


def split_even(N, parts):
    return [shard_bounds(N, parts, r) for r in range(parts)]


__all__ = ["shard_bounds", "shard", "gather", "run_sharded", "evaluate_sharded", "split_even", "np"]
