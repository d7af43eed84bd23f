"""Multi-GPU plumbing for batched evaluation.

Candidates are independent units: rank r of G evaluates the contiguous shard
``shard_range(B, r, G)`` against its own replica of the graph, then the fixed
432-byte ``pdnn_eval_result`` structs are gathered once (NCCL
``all_gather_into_tensor`` over NVLink on the GPU box; ``all_gather`` for
gloo).  There is no per-level exchange: a single graph is never split.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

RESULT_BYTES = 432


def shard_range(B: int, rank: int, world: int):
    """Contiguous, near-equal shard [b0, b1) of B candidates; shards of all
    ranks are padded to the same length ``per`` for the gather."""
    per = (B + world - 1) // world if world > 0 else B
    b0 = min(B, rank * per)
    b1 = min(B, b0 + per)
    return b0, b1, per


def gather_results(local: torch.Tensor, B: int, world: int, group=None) -> torch.Tensor:
    """local: uint8 [per * 432] (this rank's results, zero-padded); returns
    uint8 [B * 432] on every rank, in candidate order."""
    per = local.numel() // RESULT_BYTES
    if world == 1:
        return local[: B * RESULT_BYTES]
    backend = dist.get_backend(group)
    if backend == "nccl":
        out = torch.empty(world * per * RESULT_BYTES, dtype=torch.uint8, device=local.device)
        dist.all_gather_into_tensor(out, local, group=group)
    else:
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local, group=group)
        out = torch.cat(parts)
    return out[: B * RESULT_BYTES]
