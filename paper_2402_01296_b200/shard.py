"""Multi-GPU sharding of independent slot-set groups.

BHW groups are independent units of work: rank r of W processes a contiguous
range of groups with no data-path collective; every rank regenerates the
same keys from the shared seed (no key broadcast).  The only exchange is the
final gather of the output (logits) ciphertexts to rank 0, which decrypts.
One process per GPU; torch.distributed with NCCL on GPUs (gloo in the CPU
tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_items: int, rank: int, world: int) -> range:
    """Contiguous, balanced split: the first n % world ranks get one extra."""
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def gather_to_root(local: torch.Tensor, n_items: int, root: int = 0) -> torch.Tensor | None:
    """Gather per-rank (n_local, ...) tensors into (n_items, ...) on `root`
    (rank order == item order); other ranks get None.  Shards are padded to
    the largest one so a single collective moves everything."""
    world = dist.get_world_size()
    rank = dist.get_rank()
    cap = len(shard_range(n_items, 0, world))
    buf = local
    if local.shape[0] < cap:
        pad = torch.zeros((cap - local.shape[0], *local.shape[1:]), dtype=local.dtype, device=local.device)
        buf = torch.cat([local, pad])
    buf = buf.contiguous()
    if rank == root:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, gather_list=parts, dst=root)
        return torch.cat([p[:len(shard_range(n_items, r, world))] for r, p in enumerate(parts)])
    dist.gather(buf, dst=root)
    return None
