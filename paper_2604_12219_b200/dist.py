"""Multi-GPU plumbing for PASA: head partitioning and, only for
sequence-sharded input, a Ulysses all-to-all.

Every (batch, head) is an independent unit of the method (its own pooled
statistics, groups, route and output), so the hot path needs no collective:
rank r owns global heads [r H/P, (r+1) H/P) and passes ``head_offset`` /
``H_total`` to the route so Philox is keyed on the global head (reading R-20)
and results are bitwise identical for any P.

When the caller's activations arrive sequence-sharded ([B, S/P, H, D] per rank,
the HunyuanVideo config), ``ulysses_attention`` moves them to head-sharded
layout with one NCCL ``all_to_all_single`` per tensor over NVLink, runs PASA on
the local heads and moves the output back with one more all-to-all.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def head_range(H: int, world: int, rank: int, even: bool = False):
    """Contiguous head partition: rank r owns global heads [floor(r H / P),
    floor((r+1) H / P)); returns (head_offset, local_heads).  Uneven splits are
    allowed (Wan-1.3B's 12 heads over 8 ranks: 1, 2, 1, 2, ...) unless
    ``even`` (the Ulysses all-to-all needs equal head chunks)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} of world {world}")
    if even and H % world:
        raise ValueError(f"{H} heads do not split evenly over {world} ranks")
    if H < world:
        raise ValueError(f"{H} heads cannot give each of {world} ranks a head")
    off = H * rank // world
    return off, H * (rank + 1) // world - off


def seq_to_head(x: torch.Tensor, group=None) -> torch.Tensor:
    """[B, S/P, H, D] (this rank's sequence shard) -> [B, S, H/P, D] (this rank's heads)."""
    P = dist.get_world_size(group)
    B, Sl, H, D = x.shape
    if H % P:
        raise ValueError("heads must divide the world size")
    Hl = H // P
    # send buffer: chunk p = my sequence shard of rank p's heads
    send = x.reshape(B, Sl, P, Hl, D).permute(2, 0, 1, 3, 4).contiguous()
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    # recv chunk p = rank p's sequence shard of my heads
    return recv.permute(1, 0, 2, 3, 4).reshape(B, P * Sl, Hl, D).contiguous()


def head_to_seq(y: torch.Tensor, group=None) -> torch.Tensor:
    """Inverse of seq_to_head: [B, S, H/P, D] -> [B, S/P, H, D]."""
    P = dist.get_world_size(group)
    B, S, Hl, D = y.shape
    if S % P:
        raise ValueError("sequence must divide the world size")
    Sl = S // P
    send = y.reshape(B, P, Sl, Hl, D).permute(1, 0, 2, 3, 4).contiguous()
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    # recv chunk p = my sequence shard of rank p's heads
    return recv.permute(1, 2, 0, 3, 4).reshape(B, Sl, P * Hl, D).contiguous()


def ulysses_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                      local_attn: Callable[[torch.Tensor, torch.Tensor, torch.Tensor, int, int],
                                           torch.Tensor], group=None) -> torch.Tensor:
    """Sequence-sharded q, k, v [B, S/P, H, D] -> output with the same sharding.

    ``local_attn(q, k, v, head_offset, H_total)`` runs PASA (budget/route/attn)
    on full-sequence, head-sharded tensors [B, S, H/P, D]."""
    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    H = q.shape[2]
    off, _ = head_range(H, P, r, even=True)
    qh, kh, vh = (seq_to_head(t, group) for t in (q, k, v))
    oh = local_attn(qh, kh, vh, off, H)
    return head_to_seq(oh, group)
