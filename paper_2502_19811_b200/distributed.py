"""Multi-GPU bootstrap: one process per GPU, torch.distributed for plumbing.

NCCL (or gloo on CPU test hosts) is used only here, at initialisation:
every rank exports the CUDA IPC handle of its symmetric heap
(``comet_symm_export``), the handles are all-gathered, and each rank maps
all peers (``comet_symm_import``) so the fused kernels reach peer memory
directly over NVLink/NVSwitch.  After that, forwards never call NCCL: the
dispatch pulls and combine pushes are loads/stores on peer pointers issued by
the kernels' communication CTAs, synchronised by epoch flags in the heap.
"""

from __future__ import annotations

import os
from typing import List, Optional, Sequence

import numpy as np

from .config import ConfigurationError, ModelConfig, ParallelSpec


def local_device() -> int:
    """This process's GPU: LOCAL_RANK, or 0 for every rank when
    COMET_SAME_DEVICE=1 (all ranks of a group sharing one GPU -- the
    multi-process IPC path exercised on a single-GPU box, with the layer grid
    split by COMET_GRID so the ranks' persistent kernels are co-resident)."""
    if os.environ.get("COMET_SAME_DEVICE", "0") != "0":
        return 0
    return int(os.environ.get("LOCAL_RANK", 0))


def world_info():
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1, local_device()
    return dist.get_rank(), dist.get_world_size(), local_device()


def exchange_handles(handle: bytes, group=None) -> bytes:
    """All-gather every rank's 64-byte IPC handle, ordered by rank."""
    import torch.distributed as dist
    if len(handle) != 64:
        raise ConfigurationError(f"IPC handle must be 64 bytes, got {len(handle)}")
    if not dist.is_initialized():
        return bytes(handle)
    out: List[Optional[bytes]] = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(handle), group=group)
    return b"".join(out)


def check_world(parallel: ParallelSpec, world: int) -> None:
    if parallel.world_size != world:
        raise ConfigurationError(
            f"ParallelSpec(tp={parallel.tp}, ep={parallel.ep}) needs {parallel.world_size} ranks, "
            f"torch.distributed has {world}")


def token_slice(M: int, rank: int, world: int):
    """This rank's contiguous token range (routing.py:97-104)."""
    base = M // world
    lo = rank * base
    return lo, (M if rank == world - 1 else lo + base)


def broadcast_array(arr: Optional[np.ndarray], src: int = 0, group=None) -> np.ndarray:
    """Broadcast a host array from ``src`` (routing tables for synthetic runs)."""
    import torch.distributed as dist
    if not dist.is_initialized():
        return arr
    box = [arr]
    dist.broadcast_object_list(box, src=src, group=group)
    return box[0]


def init_layer(model: ModelConfig, parallel: ParallelSpec, m_cap: int, rank_weights,
               activation=None, knobs=None, group=None):
    """Create this rank's ``MoELayer`` and map every peer's symmetric heap."""
    import torch
    import torch.distributed as dist
    from .executor import MoELayer
    rank, world, local = world_info()
    check_world(parallel, world)
    torch.cuda.set_device(local)
    layer = MoELayer(model, parallel, rank, m_cap, rank_weights, device=local, activation=activation,
                     knobs=knobs)
    handles = exchange_handles(layer.ctx.export_handle(), group=group)
    if world > 1:
        layer.ctx.import_handles(handles)
        dist.barrier(group=group)
    return layer
