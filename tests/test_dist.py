"""Multi-process (gloo, world_size 2, CPU) tests of the multi-GPU plumbing:
head partitioning and the Ulysses sequence<->head all-to-all.  The local
attention plugged in here is the fp64 oracle, so the test checks that
Ulysses + per-rank PASA on local heads (Philox keyed on the global head)
reproduces the single-process result exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_12219_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_pasa(q, k, v, head_offset, H_total, *, Bq=64, Bk=16, beta=0.5, seed=7, step=21,
                 kk=3, G=2):
    import oracle
    r = oracle.route(q, k, Bq=Bq, Bk=Bk, beta=beta, seed=seed, step=step, H_total=H_total,
                     head_offset=head_offset, kk=kk)
    o = oracle.attn_with_route(q, k, v, r["idx"], Bq=Bq, Bk=Bk, G=G)
    return torch.from_numpy(o)


def _worker(rank, world, port, q, k, v, ref, errs):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, S, H, D = q.shape
        Sl = S // world
        sl = slice(rank * Sl, (rank + 1) * Sl)
        xs = q[:, sl].contiguous()
        # round trip is the identity
        back = pdist.head_to_seq(pdist.seq_to_head(xs))
        assert torch.equal(back, xs)
        hs = pdist.seq_to_head(xs)
        off, Hl = pdist.head_range(H, world, rank)
        assert torch.equal(hs, q[:, :, off:off + Hl])
        out = pdist.ulysses_attention(q[:, sl].contiguous(), k[:, sl].contiguous(),
                                      v[:, sl].contiguous(), _oracle_pasa)
        errs[rank] = float((out - ref[:, sl]).abs().max())
    finally:
        dist.destroy_process_group()


def test_head_range():
    assert pdist.head_range(40, 8, 3) == (15, 5)
    assert pdist.head_range(24, 4, 0) == (0, 6)
    # uneven (Wan-1.3B: 12 heads over 8 ranks): contiguous, disjoint, covering
    parts = [pdist.head_range(12, 8, r) for r in range(8)]
    assert [n for _, n in parts] == [1, 2, 1, 2, 1, 2, 1, 2]
    assert all(parts[r][0] + parts[r][1] == parts[r + 1][0] for r in range(7))
    assert parts[-1][0] + parts[-1][1] == 12
    with pytest.raises(ValueError):
        pdist.head_range(12, 8, 0, even=True)
    with pytest.raises(ValueError):
        pdist.head_range(4, 8, 0)


def _uneven_worker(rank, world, port, q, k, v, ref, errs):
    """Uneven head partition (3 heads over 2 ranks): each rank runs PASA on its own
    heads with Philox keyed on the global head; the gathered result equals the
    single-process one exactly."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, S, H, D = q.shape
        off, Hl = pdist.head_range(H, world, rank)
        hs = slice(off, off + Hl)
        mine = _oracle_pasa(q[:, :, hs].contiguous(), k[:, :, hs].contiguous(),
                            v[:, :, hs].contiguous(), off, H).reshape(B, S, Hl, D)
        parts = []
        for r in range(world):                    # uneven shards: one broadcast per rank
            n = pdist.head_range(H, world, r)[1]
            buf = mine.contiguous() if r == rank else torch.empty(B, S, n, D, dtype=mine.dtype)
            dist.broadcast(buf, src=r)
            parts.append(buf)
        errs[rank] = float((torch.cat(parts, 2) - ref).abs().max())
    finally:
        dist.destroy_process_group()


def test_uneven_head_partition_gloo_world2():
    g = torch.Generator().manual_seed(1)
    B, S, H, D = 1, 256, 3, 8
    q, k, v = (torch.randn(B, S, H, D, generator=g, dtype=torch.float64) for _ in range(3))
    ref = _oracle_pasa(q, k, v, 0, H)
    errs = mp.Manager().dict()
    mp.spawn(_uneven_worker, args=(2, _free_port(), q, k, v, ref, errs), nprocs=2, join=True)
    assert errs[0] == 0.0 and errs[1] == 0.0


def test_ulysses_gloo_world2_matches_single_process():
    g = torch.Generator().manual_seed(0)
    B, S, H, D = 1, 256, 4, 8
    q, k, v = (torch.randn(B, S, H, D, generator=g, dtype=torch.float64) for _ in range(3))
    ref = _oracle_pasa(q, k, v, 0, H)
    errs = mp.Manager().dict()
    mp.spawn(_worker, args=(2, _free_port(), q, k, v, ref, errs), nprocs=2, join=True)
    assert errs[0] == 0.0 and errs[1] == 0.0


# ---------------------------------------------------------------- round 2 --------
def test_flat_partition_covers_items_once_and_balances():
    """The flattened (head, q-block) split: every item exactly once, in
    head-major order, each rank floor/ceil of N / P items, one handle per rank whose item
    range lies inside its heads."""
    for H, NQ, P in [(12, 256, 8), (40, 591, 8), (3, 5, 2), (12, 256, 1), (5, 7, 3),
                     (24, 929, 8), (1, 3, 4)]:
        items = []
        for r in range(P):
            segs = pdist.flat_partition(H, NQ, P, r)
            assert len(segs) <= 1
            mine = []
            for h, n, a, b in segs:
                a, b = (0, n * NQ) if (a, b) == (0, 0) else (a, b)
                assert 0 <= a < b <= n * NQ
                assert a < NQ and b > (n - 1) * NQ          # touches every one of its heads
                mine += [divmod(h * NQ + it, NQ) for it in range(a, b)]
            assert len(mine) in (H * NQ // P, -(-H * NQ // P))
            items += mine
        assert items == [(h, i) for h in range(H) for i in range(NQ)]
    # Wan-1.3B over 8 ranks: 384 items each (1.5 heads) instead of 1 or 2 heads
    assert [pdist.flat_partition(12, 256, 8, r)[0] for r in range(3)] == [
        (0, 2, 0, 384), (1, 2, 128, 512), (3, 2, 0, 384)]


def _chunked_worker(rank, world, port, q, k, v, ref, chunks, errs):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, S, H, D = q.shape
        Sl = S // world
        sl = slice(rank * Sl, (rank + 1) * Sl)
        uly = pdist.Ulysses(B, S, H, D, q.dtype, "cpu", chunks=chunks)
        seen = []

        def compute(c, qh, kh, vh, oh, off):
            seen.append(off)
            oh.copy_(_oracle_pasa(qh.contiguous(), kh.contiguous(), vh.contiguous(), off, H)
                     .reshape(oh.shape))

        out = torch.empty(B, Sl, H, D, dtype=q.dtype)
        uly(q[:, sl].contiguous(), k[:, sl].contiguous(), v[:, sl].contiguous(), out, compute)
        assert seen == [rank * (H // world) + c * (H // world // chunks) for c in range(chunks)]
        errs[rank] = float((out - ref[:, sl]).abs().max())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B,chunks", [(1, 2), (2, 2), (1, 1)])
def test_ulysses_chunked_gloo_world2(B, chunks):
    """Chunked Ulysses (head groups, per-chunk all-to-alls, B = 1 zero-copy views and the
    B > 1 unpack path) reproduces the single-process result exactly."""
    g = torch.Generator().manual_seed(3)
    S, H, D = 256, 4, 8
    q, k, v = (torch.randn(B, S, H, D, generator=g, dtype=torch.float64) for _ in range(3))
    ref = _oracle_pasa(q, k, v, 0, H).reshape(B, S, H, D)
    errs = mp.Manager().dict()
    mp.spawn(_chunked_worker, args=(2, _free_port(), q, k, v, ref, chunks, errs), nprocs=2,
             join=True)
    assert errs[0] == 0.0 and errs[1] == 0.0


def _gather_worker(rank, world, port, errs):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = pdist.all_gather_sums(torch.tensor([10.0 * rank + 0.5], dtype=torch.float64))
        errs[rank] = got.tolist()
    finally:
        dist.destroy_process_group()


def test_all_gather_sums_rank_order_gloo_world2():
    errs = mp.Manager().dict()
    mp.spawn(_gather_worker, args=(2, _free_port(), errs), nprocs=2, join=True)
    assert errs[0] == errs[1] == [0.5, 10.5]
