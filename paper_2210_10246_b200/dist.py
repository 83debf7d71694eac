"""Row sharding across ranks + the one collective of the path.

Every Tempo operator is row-independent except LayerNorm's parameter
gradients dgamma_j = sum_i g*xhat, dbeta_j = sum_i g (ops_tempo.cpp:150-151),
so the path shards by contiguous batch rows:

* rank r of G owns rows [r*R/G, (r+1)*R/G) of every activation (tokens for
  GELU / LayerNorm / hidden dropout, (b, head, query) rows for attention);
* dropout masks are generated from the GLOBAL element index (Philox counter
  offset = first global element of the shard), so G shards reproduce the
  single-GPU masks bit for bit;
* after the backward, each rank's dgamma/dbeta (one bucket: every LN of the
  layer, 2*H floats each) is summed with ONE all-reduce (NCCL over NVLink on
  B200; gloo in the CPU tests).  Only the summation order differs from one GPU.
"""
from __future__ import annotations

from typing import Tuple


def shard_rows(rows: int, rank: int, world: int) -> Tuple[int, int]:
    """[begin, end) rows owned by `rank` (balanced contiguous blocks)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(rows, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def mask_offset(row_begin: int, cols: int) -> int:
    """Philox counter offset of a shard: its first global element index.
    The vector kernels need it to be a multiple of 4 (cols % 4 == 0)."""
    return row_begin * cols


def allreduce_ln_params(bucket, group=None) -> None:
    """Sum the bucketed LayerNorm dgamma/dbeta over all ranks, in place."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(bucket, op=dist.ReduceOp.SUM, group=group)
