"""One process per GPU: clique-sharded HSDE-ADMM over NCCL.

    torchrun --nproc-per-node N ...  ->  in every rank:
        comm = multigpu.init_comm()          # NCCL id from rank 0 via torch.distributed
        report = solve_decomposed(cp, settings, comm=comm)

Each rank keeps the cliques of its contiguous range (shard.make_shards) and
meets the others at three ncclAllReduce calls per iteration, captured in the
iteration's CUDA graph (separator pull-scatter partials, partial A t, partial
c.ua).  torch.distributed is used only to broadcast the NCCL unique id and to
gather the final state for the report.
"""

from __future__ import annotations

import os

from . import _lib


def init_comm(backend: str | None = None):
    """Initialise torch.distributed (if needed) and return (world, rank, nccl_id)."""
    import torch.distributed as dist

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend or "gloo")
    world, rank = dist.get_world_size(), dist.get_rank()
    obj = [_lib.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return (world, rank, obj[0])
