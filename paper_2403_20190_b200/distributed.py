"""Multi-GPU sharding (one process per GPU, torch.distributed).

PBS items are independent and keys are replicated, so bootstrapping shards
with no data-path collective.  Encrypted training shards images across ranks
exactly like the reference's threaded striping (`hw/hewnn.py:216-229`): each
rank trains a partial model and the partials are summed -- ciphertext
addition mod 2^32, so the result is bit-identical to sequential training.

The sum runs as an int64 all-reduce of the uint32 words (no reliance on
signed-overflow wrap in the backend), reduced mod 2^32 afterwards.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) of `total` items for `rank`."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def stripe(items: list, rank: int, world: int) -> list:
    """The reference's stripes: samples[rank::world] (hw/hewnn.py:223)."""
    return items[rank::world]


def allreduce_u32_(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place exact sum mod 2^32 of int32-stored uint32 words across ranks."""
    wide = t.to(torch.int64) & 0xFFFFFFFF
    dist.all_reduce(wide, op=dist.ReduceOp.SUM, group=group)
    wide &= 0xFFFFFFFF
    t.copy_(torch.where(wide >= 2 ** 31, wide - 2 ** 32, wide).to(torch.int32))
    return t


def merge_models_(rams: torch.Tensor, counts_ct: torch.Tensor, group=None):
    """Federated/sharded merge of partial encrypted models (hw/hewnn.py:226-229, 264-271)."""
    allreduce_u32_(rams, group)
    allreduce_u32_(counts_ct, group)
    return rams, counts_ct
