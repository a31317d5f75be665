"""Multi-GPU paths of SURVEY.md §8e through the PRODUCT library (libpasa.so):

* q-block ranges (pasa_route_cfg.qb_begin/qb_end), the building block of the flattened
  (head, q-block) partition: rows in range equal the full run bit for bit, rows outside
  are not written;
* the sharded-latent budget (pasa_budget_local_sum / pasa_budget_from_sums) against the
  unsharded call and the fp64 oracle;
* two ranks (torch.multiprocessing, gloo, both on cuda:0 -- the gpurun box has one GPU):
  the chunked Ulysses all-to-all with PASA per chunk, the flattened partition and the
  sharded budget each reproduce the single-process result exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pasa():
    from paper_2604_12219_b200 import build
    build.build()
    import paper_2604_12219_b200 as P
    return P


def _budget(P, rho=0.15, step=25, T=50):
    b = P.Budget()
    x = torch.zeros(64, device="cuda")
    b(x, x, x, T=T, step=step, rho_table=[rho] * T, l1_mean=1.0)
    return b


def _run(P, q, k, v, cfg, budget, seed=42, step=25, out=None):
    B, S, H, D = q.shape
    r = P.Route(B, S, H, D, cfg)
    r.ws.fill_(0xFF)          # poisoned workspace: nothing may rely on a stale value
    r(q, k, budget, seed, step)
    out = P.attn(q, k, v, r, out)
    torch.cuda.synchronize()
    return r, out


@pytest.mark.parametrize("dtype,Bq,rng", [
    (torch.bfloat16, 128, (3, 17)), (torch.bfloat16, 128, (30, 33)),   # head 0, ragged last
    (torch.bfloat16, 128, (30, 40)),                                    # across the heads
    (torch.bfloat16, 256, (2, 9)), (torch.float32, 128, (0, 5)),        # q256 / SIMT kernels
    (torch.bfloat16, 128, (0, 66)),                                     # the full range
])
def test_qblock_range_equals_full_run(pasa, dtype, Bq, rng):
    """Item ranges [a, b) of the handle's (head, q-block) list, item = h * N_Q + i."""
    P = pasa
    B, S, H, D = 1, 4100, 2, 128
    q, k, v = synth.video_qkv(B, (1, 1, S), H, D, seed=11, dtype=dtype, device="cuda")
    budget = _budget(P)
    full_r, full_o = _run(P, q, k, v, P.RouteCfg(Bq=Bq, G=32, beta=0.1), budget)
    a, b = rng
    NQ = full_r.NQ
    b = min(b, H * NQ)
    out = torch.full_like(q, float("nan"))
    part_r, out = _run(P, q, k, v, P.RouteCfg(Bq=Bq, G=32, beta=0.1, qb_begin=a, qb_end=b),
                       budget, out=out)
    got, want = part_r.read(), full_r.read()
    kk = got["k"]
    assert kk == want["k"]
    inside = torch.zeros(B, S, H, dtype=torch.bool)
    for it in range(a, b):
        h, i = divmod(it, NQ)
        assert np.array_equal(got["idx"][h, i, :kk], want["idx"][h, i, :kk])
        for key in ("count", "mask"):
            assert np.array_equal(got[key][h, i], want[key][h, i]), key
        t0, t1 = i * Bq, min((i + 1) * Bq, S)
        assert torch.equal(out[:, t0:t1, h], full_o[:, t0:t1, h])
        inside[:, t0:t1, h] = True
    assert torch.isnan(out.float()[~inside.cuda()]).all(), "rows outside the range were written"


def test_qblock_range_rejects_bad_ranges(pasa):
    P = pasa
    with pytest.raises(P.PasaError):
        P.Route(1, 4100, 1, 128, P.RouteCfg(qb_begin=5, qb_end=5))
    with pytest.raises(P.PasaError):
        P.Route(1, 4100, 1, 128, P.RouteCfg(qb_begin=0, qb_end=34))   # 33 items


def test_sharded_budget_matches_unsharded_and_oracle(pasa):
    P = pasa
    tp = synth.ThreePhase(shape=(3 * 4096 + 12,), T=50, seed=7, device="cuda")
    xs = [x.contiguous() for x in tp.latents(30)]
    n = xs[0].numel()
    kw = dict(T=50, step=30, rho=0.15, l1_mean=tp.expected_l1_mean(), h_t=1 / 50, h_tm1=1 / 50)
    full = P.Budget()
    full(*xs, **kw)
    want = full.read()
    orc = oracle.budget(*xs, **kw)
    cuts = [0, 4096, 8192 + 8, n]                    # 16-byte aligned shard starts
    b = P.Budget()
    sums = torch.cat([b.local_sum(*(x[c0:c1] for x in xs), **kw)
                      for c0, c1 in zip(cuts[:-1], cuts[1:])])
    b.from_sums(sums, n, **kw)
    got = b.read()
    assert abs(got["l1"] - want["l1"]) <= 1e-12 * want["l1"]
    assert abs(got["l1"] - orc["l1"]) <= 1e-12 * orc["l1"]
    assert abs(got["rho_t"] - want["rho_t"]) <= 1e-12 * want["rho_t"]
    assert (got["dense"], got["clipped"]) == (want["dense"], want["clipped"])
    # the rank-order sum is exactly what from_sums divides
    assert got["l1"] == float(sum(sums.cpu().tolist())) / n


# ------------------------------------------------------------- two ranks ----------
def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CFG = dict(B=1, S=4096, H=4, D=128)


def _inputs():
    q, k, v = synth.video_qkv(CFG["B"], (1, 1, CFG["S"]), CFG["H"], CFG["D"], seed=21,
                              dtype=torch.bfloat16, device="cuda")
    tp = synth.ThreePhase(shape=(8192,), T=50, seed=7, device="cuda")
    xs = [x.contiguous() for x in tp.latents(30)]
    kw = dict(T=50, step=30, rho=0.15, l1_mean=tp.expected_l1_mean(), h_t=1 / 50, h_tm1=1 / 50)
    return q, k, v, xs, kw


def _rank_main(rank, world, port, mode, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2604_12219_b200 as P
        from paper_2604_12219_b200 import dist as pdist
        q, k, v, xs, kw = _inputs()
        B, S, H, D = q.shape
        seed, step = P.layer_seed(42, 0), 30
        budget = P.Budget()
        n = xs[0].numel()
        sl = slice(rank * n // world, (rank + 1) * n // world)
        pdist.sharded_budget(budget, *(x[sl] for x in xs), n_total=n, **kw)
        if mode == "budget":
            result[rank] = budget.read()
            return
        if mode == "ulysses":
            Sl = S // world
            ss = slice(rank * Sl, (rank + 1) * Sl)
            uly = pdist.Ulysses(B, S, H, D, q.dtype, q.device, chunks=2)
            routes = {}

            def compute(c, qh, kh, vh, oh, off):
                r = routes.get(c)
                if r is None:
                    cfg = P.RouteCfg(Bq=128, G=32, beta=0.1, H_total=H, head_offset=off)
                    r = routes[c] = P.Route(B, S, qh.shape[2], D, cfg)
                r(qh, kh, budget, seed, step)
                P.attn(qh, kh, vh, r, oh)

            out = torch.empty(B, Sl, H, D, dtype=q.dtype, device=q.device)
            uly(q[:, ss].contiguous(), k[:, ss].contiguous(), v[:, ss].contiguous(), out, compute)
            torch.cuda.synchronize()
            result[rank] = (ss.start, ss.stop, out.cpu())
        elif mode == "zerocopy":
            # uneven, block-misaligned sequence shards; the exchange fused into PASA's kernels
            cut = [0, 1901, S]
            a, b = cut[rank], cut[rank + 1]
            q_s, k_s, v_s = (t[:, a:b].contiguous() for t in (q, k, v))
            out_s = torch.full_like(q_s, float("nan"))
            zc = pdist.ZeroCopyUlysses(q_s, k_s, v_s, out_s, H, P.RouteCfg(Bq=128, G=32, beta=0.1))
            zc(budget, seed, step)
            torch.cuda.synchronize()
            result[rank] = (a, b, out_s.cpu())
        else:   # flattened (head, q-block) partition
            NQ = (S + 127) // 128
            segs = pdist.flat_partition(H, NQ, world, rank)
            out = torch.full_like(q, float("nan"))
            for h, nh, a, b in segs:
                hs = slice(h, h + nh)
                cfg = P.RouteCfg(Bq=128, G=32, beta=0.1, H_total=H, head_offset=h,
                                 qb_begin=a, qb_end=b)
                r = P.Route(B, S, nh, D, cfg)
                r(q[:, :, hs], k[:, :, hs], budget, seed, step)
                P.attn(q[:, :, hs], k[:, :, hs], v[:, :, hs], r, out[:, :, hs])
            torch.cuda.synchronize()
            result[rank] = (segs, out.cpu())
    finally:
        dist.destroy_process_group()


def _single(P):
    q, k, v, xs, kw = _inputs()
    B, S, H, D = q.shape
    budget = P.Budget()
    n = xs[0].numel()
    sums = torch.cat([budget.local_sum(*(x[c * n // 2:(c + 1) * n // 2] for x in xs), **kw)
                      for c in range(2)])
    budget.from_sums(sums, n, **kw)
    r = P.Route(B, S, H, D, P.RouteCfg(Bq=128, G=32, beta=0.1))
    r(q, k, budget, P.layer_seed(42, 0), 30)
    out = P.attn(q, k, v, r)
    torch.cuda.synchronize()
    return budget.read(), out.cpu()


@pytest.mark.parametrize("mode", ["budget", "ulysses", "flat", "zerocopy"])
def test_two_ranks_reproduce_single_process(pasa, mode):
    rec, ref = _single(pasa)
    res = mp.Manager().dict()
    mp.spawn(_rank_main, args=(2, _port(), mode, res), nprocs=2, join=True)
    if mode == "budget":
        assert res[0] == res[1] == rec
    elif mode in ("ulysses", "zerocopy"):
        for r in range(2):
            a, b, o = res[r]
            assert torch.equal(o, ref[:, a:b]), r
    else:
        got = torch.full_like(ref, float("nan"))
        NQ = (ref.shape[1] + 127) // 128
        for r in range(2):
            segs, o = res[r]
            for h, nh, a, b in segs:
                a, b = (0, nh * NQ) if (a, b) == (0, 0) else (a, b)
                for it in range(a, b):
                    hh, i = divmod(h * NQ + it, NQ)
                    t0, t1 = i * 128, min((i + 1) * 128, ref.shape[1])
                    got[:, t0:t1, hh] = o[:, t0:t1, hh]
        assert torch.equal(got, ref)



@pytest.mark.parametrize("cuts,heads_split", [
    ((0, 1901, 4096), 2),                 # two uneven shards, block-misaligned
    ((0, 700, 2049, 2050, 4096), 4),      # a one-token shard; ranks of 1 head each
    ((0, 4096), 1),                       # one shard (P = 1)
])
def test_zero_copy_shards_match_single_tensor(pasa, cuts, heads_split):
    """pasa_route_zc / pasa_attn_zc in one process: the sequence shards are separate
    tensors (boundaries inside blocks, one of a single token), every "rank" routes its
    heads from all shards and writes its output rows into the shards that own them; the
    route of each head range and the assembled output equal the single-tensor path bit
    for bit."""
    P = pasa
    from paper_2604_12219_b200 import dist as pdist
    q, k, v, xs, kw = _inputs()
    B, S, H, D = q.shape
    budget = _budget(P)
    seed, step = P.layer_seed(42, 0), 30
    full = P.Route(B, S, H, D, P.RouteCfg(Bq=128, G=32, beta=0.1))
    full(q, k, budget, seed, step)
    ref = P.attn(q, k, v, full)
    want = full.read()
    shards = {n: [t[:, a:b].contiguous() for a, b in zip(cuts[:-1], cuts[1:])]
              for n, t in (("q", q), ("k", k), ("v", v))}
    outs = [torch.full_like(x, float("nan")) for x in shards["q"]]
    for r in range(heads_split):
        h0, hl = pdist.head_range(H, heads_split, r)
        route = P.Route(1, S, hl, D, P.RouteCfg(Bq=128, G=32, beta=0.1, H_total=H, head_offset=h0))
        route.ws.fill_(0xFF)
        loc = [torch.full((1, S, hl, D), float("nan"), dtype=q.dtype, device=q.device)
               for _ in range(3)]
        P.route_zc(route, shards["q"], shards["k"], shards["v"], budget, seed, step, *loc)
        torch.cuda.synchronize()
        assert torch.equal(loc[0], q[:, :, h0:h0 + hl]) and torch.equal(loc[2], v[:, :, h0:h0 + hl])
        got = route.read()
        kk = got["k"]
        assert kk == want["k"]
        for key in ("count", "mask"):
            assert np.array_equal(got[key], want[key][h0:h0 + hl]), key
        assert np.array_equal(got["idx"][:, :, :kk], want["idx"][h0:h0 + hl, :, :kk])
        P.attn_zc(*loc, route, outs)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs, 1), ref)
