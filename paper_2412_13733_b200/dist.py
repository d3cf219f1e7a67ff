"""Multi-process plumbing for `bench.py --gpus N` (one process per GPU).

The psi side of the path is element-local (Psi is cellwise discontinuous,
``spaces.py:89-108``), so cells shard across ranks with no data-path
collective: each rank owns a slab of cell columns ``cx in [x0, x1)``.  The
only cross-rank operations are the barrier bracketing the timed region and
the max-over-ranks of the elapsed time (weak scaling: fixed cells per rank).
"""

import os

import torch
import torch.distributed as dist


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend):
    """Initialise the default process group from the torchrun environment."""
    rank, world, local = env_rank()
    if world > 1 and not dist.is_initialized():
        kw = {}
        if backend == "nccl":
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend, **kw)
    return rank, world, local


def slab(ncx, world, rank):
    """Contiguous cell-column range [x0, x1) of a rank (balanced to one column)."""
    base, extra = divmod(ncx, world)
    x0 = rank * base + min(rank, extra)
    return x0, x0 + base + (1 if rank < extra else 0)


def barrier(device=None):
    if dist.is_initialized() and dist.get_world_size() > 1:
        if device is not None and device.type == "cuda":
            dist.barrier(device_ids=[device.index])
        else:
            dist.barrier()


def max_over_ranks(value, device=None):
    """Max of a float over all ranks (the timing rule: slowest rank wins)."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(units_per_rank, steps, world, max_seconds):
    """Whole-job throughput: units all ranks processed / slowest rank's time."""
    return units_per_rank * steps * world / max_seconds
