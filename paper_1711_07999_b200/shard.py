"""Multi-GPU plumbing for the path: independent sequences sharded over one
process per GPU (frames of one sequence are serial,
tracker.cpp:79-82, so the path shards only across sequences -- weak scaling,
no collective inside the per-frame loop).

torch.distributed carries only the out-of-loop steps: the barrier around a
timed region, the max-over-ranks of device time, and gathering per-sequence
results at rank 0. NCCL on GPU boxes, gloo for the CPU tests.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Rank:
    rank: int = 0
    world: int = 1
    local_rank: int = 0

    @property
    def is_root(self) -> bool:
        return self.rank == 0


def from_env() -> Rank:
    """RANK / WORLD_SIZE / LOCAL_RANK as torchrun exports them."""
    def geti(k, d):
        try:
            return int(os.environ.get(k, d))
        except ValueError:
            return d
    return Rank(geti("RANK", 0), geti("WORLD_SIZE", 1), geti("LOCAL_RANK", 0))


def init(r: Rank, backend: str = "nccl"):
    """Initialises the process group when world > 1 (127.0.0.1 rendezvous
    comes from torchrun's MASTER_ADDR)."""
    if r.world <= 1:
        return None
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(r.local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", r.local_rank))
        else:
            dist.init_process_group(backend)
    return dist


def shard(n_items: int, r: Rank) -> range:
    """Contiguous balanced block of [0, n_items) owned by rank r: the first
    n_items % world ranks take one extra item."""
    base, extra = divmod(n_items, r.world)
    lo = r.rank * base + min(r.rank, extra)
    return range(lo, lo + base + (1 if r.rank < extra else 0))


def _tensor(vals, device):
    import torch
    return torch.tensor(np.asarray(vals, dtype=np.float64), dtype=torch.float64, device=device)


def max_over_ranks(vals, r: Rank, device="cpu") -> np.ndarray:
    """Element-wise max over ranks (device time of a timed region)."""
    if r.world <= 1:
        return np.asarray(vals, dtype=np.float64)
    import torch.distributed as dist
    t = _tensor(vals, device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().numpy()


def sum_over_ranks(vals, r: Rank, device="cpu") -> np.ndarray:
    if r.world <= 1:
        return np.asarray(vals, dtype=np.float64)
    import torch.distributed as dist
    t = _tensor(vals, device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()


def gather_to_root(obj, r: Rank):
    """Per-rank results -> list ordered by rank at rank 0 (None elsewhere)."""
    if r.world <= 1:
        return [obj]
    import torch.distributed as dist
    out = [None] * r.world if r.is_root else None
    dist.gather_object(obj, out, dst=0)
    return out


def barrier(r: Rank) -> None:
    if r.world > 1:
        import torch.distributed as dist
        dist.barrier()


def track_sequences(bundle, sequence_paths, r: Rank | None = None, **kwargs) -> list | None:
    """api.track_sequence over many .wts files, sharded across ranks (one GPU
    each). Returns the results in input order at rank 0, None on other ranks."""
    from .api import track_sequence
    r = r or from_env()
    mine = shard(len(sequence_paths), r)
    local = [(i, track_sequence(bundle, sequence_paths[i], device=r.local_rank, **kwargs)) for i in mine]
    parts = gather_to_root(local, r)
    if not r.is_root:
        return None
    out = [None] * len(sequence_paths)
    for part in parts:
        for i, res in part:
            out[i] = res
    return out
