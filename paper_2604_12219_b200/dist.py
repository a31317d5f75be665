"""Multi-GPU plumbing for PASA: head partitioning (or, when the head
count does not divide the GPU count, a flattened (head, q-block) partition), the
sharded-latent budget and, only for sequence-sharded input, a Ulysses all-to-all
chunked by head group so attention on arrived heads overlaps the transfer of the rest.

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

from typing import Callable, List, Optional, Tuple

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


# ------------------------------------------------- flattened (head, q-block) split --
def flat_partition(H: int, NQ: int, world: int, rank: int) -> List[Tuple[int, int, int, int]]:
    """Rank r owns the flattened work items [floor(r N / P), floor((r+1) N / P)) of the
    N = H * NQ (head, q-block) items, head-major (Wan-1.3B's 12 heads over
    8 ranks is capped at 75% efficiency by the head split; 3,072 items split to 384 each).
    Returns [(head_offset, n_heads, item_begin, item_end)]: one route handle over the
    n_heads heads the range touches, with the item range relative to that handle
    (RouteCfg(qb_begin=item_begin, qb_end=item_end); (0, 0) = all its items)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} of world {world}")
    N = H * NQ
    a, b = N * rank // world, N * (rank + 1) // world
    if a >= b:
        return []
    h0, h1 = a // NQ, (b - 1) // NQ + 1
    lo, hi = a - h0 * NQ, b - h0 * NQ
    return [(h0, h1 - h0, 0, 0) if (lo, hi) == (0, (h1 - h0) * NQ) else (h0, h1 - h0, lo, hi)]


def partition_heads(segs) -> Tuple[int, int]:
    """(first global head, number of heads) a rank's segments touch (its K/V slice)."""
    if not segs:
        return 0, 0
    h0 = segs[0][0]
    h1 = max(h + n for h, n, _, _ in segs)
    return h0, h1 - h0


# ------------------------------------------------------------ collectives -----------
def _backend(group=None) -> str:
    return dist.get_backend(group)


def all_to_all(recv: torch.Tensor, send: torch.Tensor, group=None, async_op: bool = False):
    """all_to_all_single; NCCL asynchronously on its stream (the returned work's wait()
    makes the current stream wait), gloo through host memory (debug mode: ranks that
    share one GPU)."""
    if _backend(group) == "nccl" or not send.is_cuda:
        return dist.all_to_all_single(recv, send, group=group, async_op=async_op)
    r = torch.empty(send.shape, dtype=send.dtype)
    dist.all_to_all_single(r, send.cpu(), group=group)
    recv.copy_(r)
    return None


def all_gather_sums(local: torch.Tensor, group=None) -> torch.Tensor:
    """[P] float64 on local's device: every rank's 1-element local sum, rank order."""
    P = dist.get_world_size(group)
    if _backend(group) == "nccl" or not local.is_cuda:
        out = torch.empty(P, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local, group=group)
        return out
    parts = [torch.empty(1, dtype=local.dtype) for _ in range(P)]
    dist.all_gather(parts, local.cpu(), group=group)
    return torch.cat(parts).to(local.device)


def sharded_budget(budget, x_t, x_tm1, x_tm2, n_total: int, group=None, **schedule):
    """Budget over latents split across ranks: pasa_budget_local_sum on
    this rank's shard, all_gather of the fp64 sums, pasa_budget_from_sums in rank order."""
    local = budget.local_sum(x_t, x_tm1, x_tm2, **schedule)
    sums = all_gather_sums(local, group) if dist.is_initialized() else local
    return budget.from_sums(sums, n_total, **schedule)


# ------------------------------------------------- chunked Ulysses all-to-all ----
class Ulysses:
    """Sequence-sharded attention input [B, S/P, H, D] per rank -> this rank's heads
    [B, S, H/P, D] -> PASA -> output back to [B, S/P, H, D], in `chunks` head groups:
    all chunks' all-to-alls are issued up front (NCCL, asynchronous, on its own stream);
    chunk c's attention starts once chunk c has arrived and its output is sent back at
    once, so transfers overlap attention.  Packing is one strided copy
    per tensor and chunk into a preallocated send buffer; with B = 1 the receive buffer
    [P, 1, S/P, hc, D] is already the [1, S, hc, D] layout PASA reads (no unpack) and the
    attention writes its output straight into the return send buffer."""

    def __init__(self, B: int, S: int, H: int, D: int, dtype, device, group=None,
                 chunks: int = 1):
        self.P = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.group = group
        if H % self.P or S % self.P:
            raise ValueError(f"H={H}, S={S} must split over {self.P} ranks")
        self.B, self.S, self.H, self.D = B, S, H, D
        self.Hl = H // self.P
        if self.Hl % chunks:
            raise ValueError(f"{self.Hl} local heads do not split into {chunks} chunks")
        self.C, self.hc = chunks, self.Hl // chunks
        Sl = S // self.P
        shp = (self.P, B, Sl, self.hc, D)
        mk = lambda: [torch.empty(shp, dtype=dtype, device=device) for _ in range(chunks)]  # noqa: E731
        self.send = {n: mk() for n in "qkvo"} if self.P > 1 else None
        self.recv = {n: mk() for n in "qkvo"} if self.P > 1 else None

    def head_offset(self, c: int) -> int:
        """Global head index of chunk c's first head on this rank."""
        return self.rank * self.Hl + c * self.hc

    def _heads(self, buf: torch.Tensor) -> torch.Tensor:
        """[P, B, S/P, hc, D] (source rank major) -> [B, S, hc, D]."""
        if self.B == 1:
            return buf.view(1, self.S, self.hc, self.D)
        return buf.permute(1, 0, 2, 3, 4).reshape(self.B, self.S, self.hc, self.D)

    def __call__(self, q_s, k_s, v_s, out_s, compute: Callable) -> torch.Tensor:
        """compute(c, q, k, v, out, head_offset) runs PASA on chunk c ([B, S, hc, D]
        tensors; out is written).  Returns out_s ([B, S/P, H, D])."""
        B, Sl, C, hc, Hl, P = self.B, self.S // self.P, self.C, self.hc, self.Hl, self.P
        if P == 1:
            for c in range(C):
                sl = slice(c * hc, (c + 1) * hc)
                compute(c, q_s[:, :, sl], k_s[:, :, sl], v_s[:, :, sl], out_s[:, :, sl],
                        self.head_offset(c))
            return out_s
        works = []
        for c in range(C):
            w = []
            for n, x in (("q", q_s), ("k", k_s), ("v", v_s)):
                # send[p] = my sequence shard of rank p's chunk-c heads
                src = x.view(B, Sl, P, Hl, self.D)[:, :, :, c * hc:(c + 1) * hc]
                self.send[n][c].copy_(src.permute(2, 0, 1, 3, 4))
                w.append(all_to_all(self.recv[n][c], self.send[n][c], self.group, async_op=True))
            works.append(w)
        back = []
        for c in range(C):
            for w in works[c]:
                if w is not None:
                    w.wait()
            qh, kh, vh = (self._heads(self.recv[n][c]) for n in "qkv")
            if B == 1:
                oh = self.send["o"][c].view(1, self.S, hc, self.D)
                compute(c, qh, kh, vh, oh, self.head_offset(c))
            else:
                oh = torch.empty((B, self.S, hc, self.D), dtype=out_s.dtype, device=out_s.device)
                compute(c, qh, kh, vh, oh, self.head_offset(c))
                self.send["o"][c].copy_(oh.view(B, P, Sl, hc, self.D).permute(1, 0, 2, 3, 4))
            back.append(all_to_all(self.recv["o"][c], self.send["o"][c], self.group,
                                   async_op=True))
        for c in range(C):
            if back[c] is not None:
                back[c].wait()
            # recv[p] = my sequence shard of rank p's chunk-c heads
            dst = out_s.view(B, Sl, P, Hl, self.D)[:, :, :, c * hc:(c + 1) * hc]
            dst.copy_(self.recv["o"][c].permute(1, 2, 0, 3, 4))
        return out_s


def share_tensor(x: torch.Tensor, group=None) -> List[torch.Tensor]:
    """Every rank's ``x`` mapped into this process (CUDA IPC through torch's
    multiprocessing reductions; over NVLink P2P between GPUs of one node, or the same
    device memory when ranks share a GPU).  Returns the list indexed by rank (this rank's
    own entry is ``x`` itself).  Collective: every rank calls it with its tensor."""
    from multiprocessing.reduction import ForkingPickler

    import torch.multiprocessing  # noqa: F401  (registers the CUDA IPC reductions)

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return [x]
    rank = dist.get_rank(group)
    blobs: List[Optional[bytes]] = [None] * world
    dist.all_gather_object(blobs, bytes(ForkingPickler.dumps(x)), group=group)
    return [x if r == rank else ForkingPickler.loads(blobs[r]) for r in range(world)]


class ZeroCopyUlysses:
    """Sequence-sharded input without an all-to-all: the Ulysses exchange fused into PASA's
    own kernels over peer memory (include/pasa.h pasa_route_zc /
    pasa_attn_zc).  Rank r owns heads [r H/P, (r+1) H/P).  ``pasa_route_zc`` reads those
    heads of q, k, v from every rank's shard through its peer mapping into local
    [1, S, Hl, D] buffers while pooling q and k in the same pass; ``pasa_attn_zc`` stores
    each output row straight into the shard of the rank that owns its token.  The shards
    are mapped once (``share_tensor``); each call synchronises the ranks before the gather
    (every shard written) and after the attention (every output row delivered): a device
    synchronise plus a process-group barrier, so no kernel ever waits on another rank's.
    B = 1, bf16; shards may be uneven and need not align to blocks."""

    def __init__(self, q_s, k_s, v_s, out_s, H: int, route_cfg, group=None):
        from . import api

        self.group = group
        self.P = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.h0, self.Hl = head_range(H, self.P, self.rank)
        self.maps = {n: share_tensor(t, group) for n, t in
                     (("q", q_s), ("k", k_s), ("v", v_s), ("o", out_s))}
        S = sum(t.shape[1] for t in self.maps["q"])
        D = q_s.shape[3]
        self.S, self.D = S, D
        dev = q_s.device
        self.loc = [torch.empty((1, S, self.Hl, D), dtype=q_s.dtype, device=dev) for _ in range(3)]
        import dataclasses
        cfg = dataclasses.replace(route_cfg, H_total=H, head_offset=self.h0)
        self.route = api.Route(1, S, self.Hl, D, cfg, dev)

    def sync(self):
        """Every rank's work so far complete (device synchronise + barrier)."""
        torch.cuda.current_stream().synchronize()
        if self.P > 1:
            dist.barrier(group=self.group)

    def gather_route(self, budget, seed: int, step: int):
        """pasa_route_zc: this rank's heads gathered from every shard, pooled, routed."""
        from . import api
        api.route_zc(self.route, self.maps["q"], self.maps["k"], self.maps["v"], budget, seed,
                     step, *self.loc)

    def attend(self):
        """pasa_attn_zc: statistics + attention, rows stored into their owners' out shards."""
        from . import api
        api.attn_zc(*self.loc, self.route, self.maps["o"])

    def __call__(self, budget, seed: int, step: int, sync: bool = True):
        """One PASA step of this rank's heads; the output lands in every rank's out shard."""
        if sync:
            self.sync()
        self.gather_route(budget, seed, step)
        self.attend()
        if sync:
            self.sync()
