"""Multi-GPU row-sharded GEMM: one process per GPU over torch.distributed.

The reference parallelises matmul_block_parallel_into over threads that own
disjoint contiguous spans of row blocks and never exchange data
(linalg.hpp:399-433).  Here each rank (GPU) owns a contiguous span of rows of
A and C; the only exchange is the replication of B from the root rank to every
GPU (NCCL broadcast over NVLink/NVSwitch), then each rank runs the sm_100a
GEMM on its shard.  No reduction follows: rows of C are independent and every
element's accumulation order is the reference's, so the result is
bit-identical for any world size.  An optional all-gather assembles a
replicated C when a caller needs one.
"""
from __future__ import annotations

from typing import Callable, Optional


def shard_rows(m: int, world: int, rank: int, align: int = 64):
    """Contiguous row span [r0, r1) of `rank`: ceil-divided blocks of `align`
    rows, like the reference's `per = ceil(nblocks / nt)` spans
    (linalg.hpp:413-421).  Trailing ranks may get an empty span."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_rows: bad rank/world")
    nblocks = (m + align - 1) // align
    per = (nblocks + world - 1) // world
    r0 = min(m, rank * per * align)
    r1 = min(m, (rank + 1) * per * align)
    return r0, r1


def replicate_b(dB, src: int = 0, group=None):
    """B from the root rank to all ranks (NCCL broadcast on GPU tensors)."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(dB, src=src, group=group)
    return dB


def sharded_gemm_step(W: int, dA, dB, dC, rows: int, n: int, k: int, ld: int, *, stream=None,
                      gemm: Optional[Callable] = None, group=None) -> int:
    """One step of the sharded GEMM on this rank: replicate B, then
    C_shard = A_shard * B.  dA (W, rows, ld), dB (W, k, ld), dC (W, rows, ld)
    float64 tensors.  `gemm` defaults to libmpfk's device entry point;
    returns the number of GEMM kernel launches."""
    replicate_b(dB, group=group)
    if rows == 0:
        return 0
    if gemm is None:
        from . import linalg as L
        s = stream.cuda_stream if stream is not None else 0
        return L.gemm_device(W, rows, n, k, dA.data_ptr(), ld, rows * ld, dB.data_ptr(), ld, k * ld,
                             dC.data_ptr(), ld, rows * ld, s)
    return gemm(W, dA, dB, dC, rows, n, k, ld)


def gather_c(dC_shard, m: int, world: int, group=None, align: int = 64):
    """Assemble the replicated (W, m, ld) C from the row shards
    (all-gather); shards are padded to the common span length.  `align`
    must be the one the shards were cut with (shard_rows)."""
    import torch
    import torch.distributed as dist
    W, rows, ld = dC_shard.shape
    per = max(1, shard_rows(m, world, 0, align)[1])
    buf = torch.zeros((W, per, ld), dtype=dC_shard.dtype, device=dC_shard.device)
    buf[:, :rows] = dC_shard[:, :rows]
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf.contiguous(), group=group)
    spans = [shard_rows(m, world, r, align) for r in range(world)]
    out = torch.cat([p[:, : r1 - r0] for p, (r0, r1) in zip(parts, spans)], dim=1)
    return out.contiguous()
