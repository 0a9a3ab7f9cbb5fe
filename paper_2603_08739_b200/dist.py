"""Multi-GPU plumbing (row e): one process per GPU under torchrun; torch.distributed is used
only to broadcast the NCCL unique id from rank 0, after which libkareto's own NCCL
communicator carries the objective-vector allgather inside kareto_eval_grid."""
from __future__ import annotations

import os

import paper_2603_08739_b200 as K


def env_world() -> tuple[int, int, int]:
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def broadcast_unique_id(rank: int, world: int, make_id=K.Context.nccl_unique_id) -> bytes | None:
    """Rank 0 creates the 128-byte NCCL unique id; every rank receives it (any backend)."""
    if world <= 1:
        return None
    import torch.distributed as dist
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def create_context(device: int, stream: int | None = None) -> K.Context:
    rank, world, _ = env_world()
    nid = broadcast_unique_id(rank, world)
    return K.Context(device, stream, nid, rank, world)


def slot_size(bounds) -> int:
    """Per-rank padded slot of the allgather (the largest shard), as in kareto_eval_grid."""
    return max(1, max(int(bounds[r + 1] - bounds[r]) for r in range(len(bounds) - 1)))


def assemble(gathered_slots, bounds):
    """Reassemble rank slots into configuration order: rank r's shard [bounds[r], bounds[r+1])
    sits at the start of slot r (the layout libkareto compacts after ncclAllGather)."""
    import numpy as np
    parts = [gathered_slots[r][: int(bounds[r + 1] - bounds[r])] for r in range(len(bounds) - 1)]
    return np.concatenate(parts) if parts else gathered_slots[0][:0]
