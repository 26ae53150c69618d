"""Host-side multi-GPU plumbing (one process per GPU; torch.distributed only moves control data).

Two ways the path shards:
* independent problems (C4 dimension pairs, and the bench's weak-scaling tiles): pair j runs on
  rank j mod world, no data-path collective;
* bank shards (C5): rank r owns integrands [t0, t1) of the bank; the only data exchange is the
  int32 all-reduce of the partial window distances inside libbn (NCCL over NVLink), set up by
  `make_bank_sharded`, which broadcasts the NCCL unique id through torch.distributed.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(T: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced bank shard [t0, t1) of rank `rank` (sizes differ by at most 1)."""
    if not (0 <= rank < world) or T < world:
        raise ValueError(f"cannot split T={T} over world={world} (rank {rank})")
    return T * rank // world, T * (rank + 1) // world


def pairs_of_rank(n_pairs: int, rank: int, world: int) -> list[int]:
    """Independent dimension pairs handled by `rank` (round robin)."""
    return [j for j in range(n_pairs) if j % world == rank]


def _device():
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")


def broadcast_unique_id(uid: bytes | None) -> bytes:
    """Rank 0's 128-byte NCCL unique id, on every rank."""
    obj = [uid if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    if not isinstance(obj[0], (bytes, bytearray)) or len(obj[0]) != 128:
        raise RuntimeError("bad NCCL unique id broadcast")
    return bytes(obj[0])


def max_over_ranks(x: float) -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: int) -> int:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return int(x)
    t = torch.tensor([int(x)], dtype=torch.int64, device=_device())
    dist.all_reduce(t)
    return int(t.item())


def make_bank_sharded(sampler, a, b, px, py, rank: int, world: int):
    """Give `sampler` (a bn.Sampler) this rank's bank shard and join the NCCL communicator."""
    from . import bn

    t0, t1 = shard_range(len(a), rank, world)
    sampler.set_bank(a, b, px, py, t0, t1)
    if world > 1:
        uid = broadcast_unique_id(bn.comm_unique_id() if rank == 0 else None)
        sampler.comm_init(uid, rank, world)
    return t0, t1
