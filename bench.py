#!/usr/bin/env python
"""bench.py -- one PASA denoising-step layer (budget -> route -> attn) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl pasa|reference]
                    [--config wan14b_720p]

A step is one pass of the whole hot path over the BASELINE.json workload
(default: Wan 2.1-14B 720p, 75,600 tokens, 40 heads, d = 128, rho = 0.15):
pasa_budget on the three-phase latents, pasa_route and pasa_attn for all heads of
one layer.  Under torchrun (N > 1) the heads are partitioned across ranks (rank
r owns heads [r H/N, (r+1) H/N), Philox keyed on the global head); there is no
collective on the data path.  Rank 0 prints one JSON line.

Metric: TFLOP/s-equiv = 4 S^2 d (B H) / t_step (counts the skipped dense work).
Inputs are synthetic, seeded, resident in HBM before the timed region, and
larger than L2 (q, k, v = 2.3 GB >> 126 MB), so no flush is needed.
``--impl reference`` times the fp64 CPU oracle (the reference arm of this
tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PASA attn TFLOP/s-equiv & ms/layer at Wan2.1-14B 720p, 1/2/4/8 B200, % of peak"
UNIT = "TFLOP/s-equiv"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pasa", choices=["pasa", "reference"])
    ap.add_argument("--config", default="wan14b_720p")
    ap.add_argument("--step-t", type=int, default=25, help="denoising step index t")
    ap.add_argument("--budget", default="table", choices=["table", "online"],
                    help="table: rho_t = rho (the 85%%-sparsity config, k = 177 at Wan-14B); "
                         "online: rho_t from the three-phase trajectory at step t")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph replay timing")
    ap.add_argument("--seq-sharded", default="auto", choices=["auto", "yes", "no"],
                    help="inputs arrive sequence-sharded [B, S/P, H, D] and go through the "
                         "Ulysses all-to-all (auto: the HunyuanVideo config, per BASELINE.json)")
    ap.add_argument("--no-dense", action="store_true",
                    help="skip the dense torch SDPA context timing (speedup vs dense)")
    ap.add_argument("--schedule", action="store_true",
                    help="also run the 50-step budget schedule (online budget from the "
                         "three-phase synthetic trajectory): per-step k_t, ms and their sum")
    ap.add_argument("--e2e-chunks", type=int, default=0,
                    help="head chunks of the host pipeline for e2e (1 = serial copy/compute; "
                         "0 = auto: about one chunk per 0.12 ms of device step, 4..20)")
    ap.add_argument("--prior", default="none", choices=["none", "global", "group"],
                    help="Eq. 8 heterogeneity prior in routing (SURVEY.md §8f NEXT 1; off in "
                         "the north-star path)")
    ap.add_argument("--cpu-qblocks", type=int, default=256,
                    help="oracle sample size (q-blocks of one head; ~10 s of CPU work)")
    ap.add_argument("--partition", default="auto", choices=["auto", "heads", "flat"],
                    help="work split over ranks: contiguous heads, or the flattened (head, "
                         "q-block) list (SURVEY.md §8e; auto: flat when the heads do not divide "
                         "the rank count, e.g. Wan-1.3B's 12 heads over 8 GPUs)")
    ap.add_argument("--ulysses", default="nccl", choices=["nccl", "zc"],
                    help="sequence-sharded input: head-chunked NCCL all-to-all overlapped with "
                         "PASA per chunk (nccl), or zero-copy: PASA's kernels read every rank's "
                         "shard through peer memory and store output rows into their owners' "
                         "shards (zc; pasa_route_zc / pasa_attn_zc)")
    ap.add_argument("--ulysses-chunks", type=int, default=0,
                    help="head groups of the sequence-sharded Ulysses all-to-all (attention on "
                         "arrived heads overlaps the rest; 0 = auto, up to 4)")
    ap.add_argument("--bq", type=int, default=0, choices=[0, 128, 256],
                    help="query block size of the route (0: the config's, 128); 256 = the "
                         "Bq = 256 throughput variant (reading R-29, not a BASELINE config)")
    ap.add_argument("--cta-pair", action="store_true",
                    help="Bq = 256 attention on the tcgen05 cta_group::2 CTA pair "
                         "(PASA_ATTN_CTA_PAIR) instead of the one-CTA two-tile kernel")
    ap.add_argument("--qk-precision", default="bf16", choices=["bf16", "fp8"],
                    help="fp8: the opt-in FP8 QK^T variant (SURVEY.md §8f NEXT 4; its own "
                         "tolerance; never the headline configuration)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1.  gloo is a debug mode: ranks may "
                         "share one GPU (device = local_rank %% device_count) and every "
                         "collective goes through host memory, so its timings say nothing; "
                         "it exercises the multi-rank bookkeeping on a one-GPU box")
    return ap.parse_args(argv)


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def torchrun_cmd(argv, n: int, port: int):
    """`python bench.py --gpus N ...` outside torchrun re-launches itself as one process
    per GPU (the driver's own form: torch.distributed.run, 127.0.0.1 rendezvous)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", f"--master-port={port}",
            os.path.abspath(__file__), *argv]


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def algorithmic_flops_per_head(S, D, NK, NG, k, Bk=64):
    """4 S k Bk d (exact) + 4 S N_K d (centroid logits + zeroth
    order, as implemented over all N_K) + 2 S d^2 N_G (grouped first order)."""
    return 4.0 * S * k * Bk * D + 4.0 * S * NK * D + 2.0 * S * D * D * NG


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw.instant,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the first sample lands before the timed region starts (right after the
            # warm-up steps), so short regions still report the clocks they ran at
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, watts = [], 0.0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            try:
                watts.append(float(parts[2]))
            except ValueError:
                pass
            for n, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm.sort()
        watts.sort()
        # board power (instant samples): the long configs run at the 1,000 W limit (sw_power_cap), where the
        # step time is the step's energy / power
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w": watts[len(watts) // 2] if watts else None}


# --------------------------------------------------------------- oracle --
def oracle_sample(cfg, nqb, seed=1000):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload:
    budget on the full latents, then for one head: block statistics + route +
    attention for `nqb` query blocks spread over the head.  Returns
    (TFLOP/s-equiv extrapolated to a full head, seconds, sample description)."""
    import numpy as np
    import torch

    import oracle
    import synth

    S, D, H = cfg["S"], cfg["D"], cfg["H"]
    Bq, Bk, G, rho = cfg["Bq"], cfg["Bk"], cfg["G"], cfg["rho"]
    oracle.build()
    g = torch.Generator().manual_seed(seed)
    q = torch.randn((1, S, 1, D), generator=g).to(torch.bfloat16)
    k = torch.randn((1, S, 1, D), generator=g).to(torch.bfloat16)
    v = torch.randn((1, S, 1, D), generator=g).to(torch.bfloat16)
    tp = synth.ThreePhase(shape=(int(np.prod(cfg["latent"])),), T=50, seed=7)
    xs = tp.latents(25)
    qh, kh, vh = oracle.heads(q), oracle.heads(k), oracle.heads(v)
    NQ = (S + Bq - 1) // Bq
    NK = (S + Bk - 1) // Bk
    t0 = time.perf_counter()
    rec = oracle.budget(*xs, T=50, step=25, rho=rho, l1_mean=tp.expected_l1_mean(),
                        h_t=1 / 50, h_tm1=1 / 50)
    t_budget = time.perf_counter() - t0
    kk = oracle.density_to_k(rho, NK)
    t0 = time.perf_counter()
    r = oracle.route(q, k, Bq=Bq, Bk=Bk, beta=0.1, seed=42, step=25, kk=kk)
    t_route = time.perf_counter() - t0
    cnt = np.full((1, NQ), kk, np.int32)
    blocks = sorted(set(np.linspace(0, NQ - 1, nqb).astype(int).tolist()))
    t0 = time.perf_counter()
    oracle.attn_pairs(None, None, None, r["idx"], cnt, [(0, i) for i in blocks], Bq=Bq, Bk=Bk,
                      G=G, qh=qh, kh=kh, vh=vh)
    t_attn = time.perf_counter() - t0
    # attn_pairs recomputes the head's statistics once; the rest scales with q-blocks
    t_head = t_budget / H + t_route + t_attn * NQ / len(blocks)
    value = 4.0 * S * S * D / t_head / 1e12
    desc = (f"1 of {H} heads: budget on full latents (/H), route for the head, stats + "
            f"attention for {len(blocks)} of {NQ} q-blocks, extrapolated to the full head "
            f"({t_budget + t_route + t_attn:.1f} s measured)")
    return value, t_budget + t_route + t_attn, desc, rec["rho_t"]


def run_reference(args):
    import synth
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    cfg = synth.CONFIGS[args.config]
    vals = []
    total_s = 0.0
    for it in range(args.warmup + args.steps):
        nqb = max(2, args.cpu_qblocks // 4)
        v, secs, desc, _ = oracle_sample(cfg, nqb, seed=1000 + it)
        if it >= args.warmup:
            vals.append(v)
            total_s += secs
    value = sum(vals) / len(vals)
    cores = oracle.num_threads()
    S, D, H = cfg["S"], cfg["D"], cfg["H"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 4.0 * S * S * D * H / (value * 1e12) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": args.config, "S": S, "H": H, "D": D},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": desc, "extrapolated": True},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU --
def run_pasa(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2604_12219_b200 import build as pbuild

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    gloo = args.dist_backend == "gloo"
    if world > 1:
        # gloo debug mode: ranks may share the box's one GPU
        torch.cuda.set_device(local % torch.cuda.device_count() if gloo else local)
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    if rank == 0:
        pbuild.build()
    if world > 1:
        dist.barrier()
    import paper_2604_12219_b200 as P

    cfg = dict(synth.CONFIGS[args.config])
    if args.bq:
        cfg["Bq"] = args.bq
    attn_kw = {"cta_pair": True} if args.cta_pair else {}
    B, S, H, D = cfg["B"], cfg["S"], cfg["H"], cfg["D"]
    from paper_2604_12219_b200 import dist as pdist
    seq_sharded = (args.seq_sharded == "yes"
                   or (args.seq_sharded == "auto" and args.config == "hunyuan_720p"))
    NQ = -(-S // cfg["Bq"])
    partition = args.partition
    if partition == "auto":
        partition = "flat" if (not seq_sharded and H % world) else "heads"
    if seq_sharded and partition == "flat":
        raise SystemExit("the Ulysses path splits whole heads (--partition heads)")
    # contiguous head partition (uneven allowed, e.g. 12 heads over 8 ranks) or the
    # flattened (head, q-block) split; the Ulysses all-to-all needs equal head chunks
    try:
        if partition == "flat":
            segs = pdist.flat_partition(H, NQ, world, rank)
            off, Hl = pdist.partition_heads(segs)     # the heads whose K/V this rank reads
        else:
            off, Hl = pdist.head_range(H, world, rank, even=seq_sharded)
            segs = [(off, Hl, 0, 0)]
    except ValueError as exc:
        raise SystemExit(str(exc))
    # head-equivalents of attention work on this rank ((head, q-block) items / N_Q)
    work_heads = sum((b - a) if (a, b) != (0, 0) else n * NQ for _, n, a, b in segs) / NQ
    dev = torch.device("cuda", torch.cuda.current_device())
    cdev = torch.device("cpu") if gloo else dev      # where collective buffers live

    def all_max(vals):
        """MAX over ranks of a list of floats (device timings: max over ranks)."""
        if world == 1:
            return list(vals)
        tt = torch.tensor(list(vals), device=cdev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return tt.cpu().tolist()

    def all_sum(vals):
        if world == 1:
            return list(vals)
        tt = torch.tensor(list(vals), device=cdev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        return tt.cpu().tolist()

    heads_all = [work_heads]
    if world > 1:
        heads_all = [None] * world
        dist.all_gather_object(heads_all, work_heads)
        assert abs(sum(heads_all) - H) < 1e-9, heads_all
    if seq_sharded and S % world:
        raise SystemExit(f"S = {S} does not split over {world} ranks")
    # every global head drawn from its own seed: the same data for any N
    qs, ks, vs = [], [], []
    heads = range(H) if seq_sharded else range(off, off + Hl)
    r0, r1 = (rank * S // world, (rank + 1) * S // world) if seq_sharded else (0, S)
    for h in heads:
        q1, k1, v1 = synth.iid_qkv(B, S, 1, D, seed=1000 + 7919 * h, dtype=torch.bfloat16,
                                   device=dev)
        qs.append(q1[:, r0:r1]); ks.append(k1[:, r0:r1]); vs.append(v1[:, r0:r1])
    q = torch.cat(qs, 2).contiguous(); k = torch.cat(ks, 2).contiguous()
    v = torch.cat(vs, 2).contiguous()
    del qs, ks, vs
    out = torch.empty_like(q)
    tp = synth.ThreePhase(shape=cfg["latent"], T=50, seed=7, device=dev)
    t_step = args.step_t
    x_t, x_tm1, x_tm2 = (x.contiguous() for x in tp.latents(t_step))
    lbar = tp.expected_l1_mean()
    use_v = args.prior != "none"
    budget = P.Budget(dev)
    seed = P.layer_seed(42, 0)
    stream = torch.cuda.current_stream()
    launches = [0]
    table = [cfg["rho"]] * 50 if args.budget == "table" else None
    bkw = dict(T=50, step=t_step, rho=cfg["rho"], l1_mean=lbar, h_t=1 / 50, h_tm1=1 / 50,
               rho_table=table)

    def rcfg_for(h, a=0, b=0):
        return P.RouteCfg(Bq=cfg["Bq"], Bk=cfg["Bk"], G=cfg["G"], comp="grouped", beta=0.1,
                          H_total=H, head_offset=h, prior=args.prior, qb_begin=a, qb_end=b,
                          qk_precision=args.qk_precision)

    rcfg = rcfg_for(off)
    zc = None   # zero-copy sequence parallelism (--ulysses zc)
    if seq_sharded:
        # sequence-sharded input [B, S/P, H, D] and latents: the step is the sharded budget
        # (one fp64 partial per rank, all_gather) and the chunked Ulysses all-to-all with
        # PASA per head chunk
        q_s, k_s, v_s = q, k, v
        out_s = torch.empty_like(q_s)
        n_lat = x_t.numel()
        la = (rank * n_lat // world) // 4 * 4
        lb = n_lat if rank == world - 1 else ((rank + 1) * n_lat // world) // 4 * 4
        xs_sh = [x.reshape(-1)[la:lb] for x in (x_t, x_tm1, x_tm2)]
        # chunks only pay with a transfer to overlap: one at N = 1
        n_chunks_u = args.ulysses_chunks or (
            1 if world == 1 else max(c for c in (1, 2, 3, 4) if (H // world) % c == 0))
        if args.ulysses == "zc":
            if use_v or args.qk_precision != "bf16" or args.cta_pair or cfg["Bq"] != 128:
                raise SystemExit("--ulysses zc: Bq = 128 bf16 path without prior / FP8 / pair")
            n_chunks_u = 1
            # the shards are mapped into every rank (CUDA IPC) once, outside the timed region
            zc = pdist.ZeroCopyUlysses(q_s, k_s, v_s, out_s, H, rcfg_for(0))
        uly = pdist.Ulysses(B, S, H, D, q.dtype, dev, chunks=n_chunks_u)
        chunk_routes = {}
        chunk_ev = []   # per chunk: [before route, after route, after stats, after attn]

        def compute(c, qh, kh, vh, oh, hoff):
            r = chunk_routes.get(c)
            if r is None:
                r = chunk_routes[c] = P.Route(B, S, qh.shape[2], D, rcfg_for(hoff), dev)
            evs = chunk_ev[-1][c] if chunk_ev and chunk_ev[-1] is not None else None
            if evs:
                evs[0].record(stream)
            r(qh, kh, budget, seed, t_step, v=vh if use_v else None)
            launches[0] += P.last_launch_count()
            if evs:
                evs[1].record(stream)
            P.attn(qh, kh, vh, r, oh, stats_only=True)
            launches[0] += P.last_launch_count()
            if evs:
                evs[2].record(stream)
            P.attn(qh, kh, vh, r, oh, reuse_stats=True, **attn_kw)
            launches[0] += P.last_launch_count()
            if evs:
                evs[3].record(stream)
        if zc is not None:
            zc(budget, seed, t_step)
            route = zc.route
            q, k, v = zc.loc    # this rank's heads, gathered (dense-attention context)
        else:
            # the first call builds the chunk handles (outside any timed region)
            chunk_ev.append(None)
            uly(q_s, k_s, v_s, out_s, compute)
            route = chunk_routes[0]
            # this rank's head-sharded tensors (dense-attention context): chunk 0 as received
            q, k, v = ((q_s, k_s, v_s) if world == 1 else
                       tuple(uly._heads(uly.recv[n][0]) for n in "qkv"))
    else:
        units = []
        for h, n, a, b in segs:
            sl = slice(h - off, h - off + n)
            units.append((P.Route(B, S, n, D, rcfg_for(h, a, b), dev),
                          q[:, :, sl], k[:, :, sl], v[:, :, sl], out[:, :, sl]))
        route = units[0][0]

    def do_budget():
        if seq_sharded:
            pdist.sharded_budget(budget, *xs_sh, n_total=x_t.numel(), **bkw)
        else:
            budget(x_t, x_tm1, x_tm2, **bkw)
        launches[0] += P.last_launch_count()

    def step(ev=None):
        do_budget()
        if ev is not None:
            ev[0].record(stream)
        if seq_sharded and zc is not None:
            # zero copy: every shard complete on every rank, gather + pool + route, then
            # statistics + attention storing rows into their owners' shards, all ranks done
            if world > 1:
                zc.sync()
            zc.gather_route(budget, seed, t_step)
            launches[0] += P.last_launch_count()
            if ev is not None:
                ev[1].record(stream)
                ev[2].record(stream)   # the statistics run inside pasa_attn_zc (counted there)
            zc.attend()
            launches[0] += P.last_launch_count()
            if ev is not None:
                ev[3].record(stream)
            if world > 1:
                zc.sync()
            return
        if seq_sharded:
            if ev is not None:
                chunk_ev.append([[torch.cuda.Event(enable_timing=True) for _ in range(4)]
                                 for _ in range(uly.C)])
            else:
                chunk_ev.append(None)
            uly(q_s, k_s, v_s, out_s, compute)
            if ev is not None:
                for j in (1, 2, 3):
                    ev[j].record(stream)
            return
        for r, qu, ku, vu, ou in units:
            r(qu, ku, budget, seed, t_step, v=vu if use_v else None)
            launches[0] += P.last_launch_count()
        if ev is not None:
            ev[1].record(stream)
        for r, qu, ku, vu, ou in units:
            P.attn(qu, ku, vu, r, ou, stats_only=True)
            launches[0] += P.last_launch_count()
        if ev is not None:
            ev[2].record(stream)
        for r, qu, ku, vu, ou in units:
            P.attn(qu, ku, vu, r, ou, reuse_stats=True, **attn_kw)
            launches[0] += P.last_launch_count()
        if ev is not None:
            ev[3].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    rec = budget.read()
    # k from the device record (same arithmetic as the route kernel, R-14)
    kk = int(max(1, min(route.NK, math.floor(rec["rho_t"] * route.NK + 0.5))))

    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    launches[0] = 0
    with ClockSampler(dev.index) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e_start.record(stream)
        for it in range(K):
            step(evs[it])
        e_end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    gpu_launches = launches[0]
    ms_total = e_start.elapsed_time(e_end)
    t_local = ms_total / K
    # per-kernel durations over the timed region (launch-stream events)
    ph = np.zeros(4)
    per_step = []
    for it in range(K):
        prev = e_start if it == 0 else evs[it - 1][3]
        ph[0] += prev.elapsed_time(evs[it][0])
        if seq_sharded and zc is None:   # route / stats / attention summed over the chunks
            for ce in chunk_ev[-K + it]:
                for j in range(1, 4):
                    ph[j] += ce[j - 1].elapsed_time(ce[j])
        else:
            for j in range(1, 4):
                ph[j] += evs[it][j - 1].elapsed_time(evs[it][j])
        per_step.append(prev.elapsed_time(evs[it][3]))
    ph /= K
    step_p50, step_p90 = (float(np.percentile(per_step, q)) for q in (50, 90))
    mx = all_max([t_local] + ph.tolist())
    t_max = float(mx[0])
    ph = np.array(mx[1:])

    # ---------------- the same step captured once in a CUDA graph, replayed K times -----
    graph = None
    if not args.no_graph and not (seq_sharded and world > 1):   # no collective / sync inside a capture
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            g.replay()
            torch.cuda.synchronize()
            ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ga.record()
            for _ in range(K):
                g.replay()
            gb.record()
            torch.cuda.synchronize()
            tg = all_max([ga.elapsed_time(gb) / K])[0]
            graph = {"ms_per_step": tg, "value": 4.0 * S * S * D * B * H / (tg * 1e-3) / 1e12,
                     "unit": UNIT, "note": "budget+route+stats+attn captured once, replayed"}
        except Exception as exc:  # report, do not hide, a capture failure
            graph = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    # ---------------- the budget kernel inside a CUDA graph of repeated calls ---------
    # (a launch-scale kernel, timed without launch gaps)
    budget_graph = None
    if not args.no_graph and not seq_sharded:
        try:
            reps = 50
            gb = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gb):
                for _ in range(reps):
                    budget(x_t, x_tm1, x_tm2, **bkw)
            gb.replay()
            torch.cuda.synchronize()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record()
            for _ in range(5):
                gb.replay()
            b1.record()
            torch.cuda.synchronize()
            us = b0.elapsed_time(b1) * 1e3 / (5 * reps)
            nbytes = 3 * x_t.numel() * x_t.element_size()
            budget_graph = {"us_per_call": us, "bytes": nbytes,
                            "gbs": nbytes / (us * 1e-6) / 1e9,
                            "note": f"{reps} pasa_budget calls captured in one CUDA graph"}
        except Exception as exc:  # report, do not hide, a capture failure
            budget_graph = {"error": f"{type(exc).__name__}: {exc}"[:200]}

    # ---------------- context: dense attention on the same shapes (library SDPA) -----
    dense = None
    if not args.no_dense and rank == 0:
        try:
            import torch.nn.functional as F
            qt, kt, vt = (t.transpose(1, 2) for t in (q, k, v))      # [B, H, S, D] views
            F.scaled_dot_product_attention(qt, kt, vt)
            torch.cuda.synchronize()
            da, db = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            da.record()
            for _ in range(2):
                F.scaled_dot_product_attention(qt, kt, vt)
            db.record()
            torch.cuda.synchronize()
            td = da.elapsed_time(db) / 2
            dense = {"what": "torch scaled_dot_product_attention (dense, bf16) on this rank's q, k, v; "
                             "context only, not a baseline of the method",
                     "ms": td, "tflops": 4.0 * S * S * D * B * q.shape[2] / (td * 1e-3) / 1e12,
                     "speedup_vs_dense_attn": td / float(ph[2] + ph[3])}
        except Exception as exc:  # e.g. out of memory for the dense workspace
            dense = {"error": f"{type(exc).__name__}: {exc}"[:200]}

    # ---------------- 50-step budget schedule (BASELINE config for CogVideoX) -----
    schedule = None
    if args.schedule:
        T = 50
        xs_hist, ks, mss = [], [], []
        for t, x in enumerate(tp.trajectory()):
            if t >= T:
                break
            xs_hist = (xs_hist + [x.contiguous()])[-3:]
            lat = xs_hist if len(xs_hist) == 3 else [xs_hist[-1]] * 3   # t < 2: dense anyway
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if world > 1:
                dist.barrier()
            ea.record(stream)
            budget(lat[2], lat[1], lat[0], T=T, step=t, rho=cfg["rho"], l1_mean=lbar,
                   h_t=1 / T, h_tm1=1 / T)
            route(q, k, budget, seed, t, v=v if use_v else None)
            P.attn(q, k, v, route, out, **attn_kw)
            eb.record(stream)
            torch.cuda.synchronize()
            ms_t = all_max([ea.elapsed_time(eb)])[0]
            ks.append(route.read()["k"])
            mss.append(ms_t)
        schedule = {"T": T, "budget": "online (three-phase synthetic trajectory, R-16)",
                    "k_t": ks, "ms_t": [round(m, 4) for m in mss], "sum_ms": sum(mss),
                    "sum_k": sum(ks[10:]), "dense_steps": sum(1 for kk_ in ks if kk_ == route.NK)}

    # ---------------- e2e through the public API with host buffers --------------
    e2e = None
    if not args.no_e2e:
        src = (q_s, k_s, v_s) if seq_sharded else (q, k, v)
        hq, hk, hv = (t.cpu().pin_memory() for t in src)
        hx = [x.cpu().pin_memory() for x in (x_t, x_tm1, x_tm2)]
        hout = torch.empty(src[0].shape, dtype=out.dtype, pin_memory=True)
        h2d = sum(t.numel() * t.element_size() for t in (hq, hk, hv, *hx))
        d2h = hout.numel() * hout.element_size()
        # head chunks: about one per 0.12 ms of device step (enough work per chunk to fill
        # the GPU and hide the per-chunk launches; Wan-14B 20, CogVideoX / Wan-1.3B 12)
        n_chunks = args.e2e_chunks or max(4, min(20, round(t_max / 0.12)))
        if seq_sharded and zc is not None:
            # host shard -> this rank's (IPC-shared) device shard -> sharded budget -> zero-copy
            # PASA (rows land in their owners' shards) -> host shard
            dx = [torch.empty_like(x) for x in xs_sh]
            hx = [x.cpu().pin_memory() for x in xs_sh]
            h2d = sum(t.numel() * t.element_size() for t in (hq, hk, hv, *hx))

            def e2e_step():
                for d, hsrc in zip((q_s, k_s, v_s, *dx), (hq, hk, hv, *hx)):
                    d.copy_(hsrc, non_blocking=True)
                pdist.sharded_budget(budget, *dx, n_total=x_t.numel(), **bkw)
                zc(budget, seed, t_step, sync=world > 1)
                hout.copy_(out_s, non_blocking=True)
        elif seq_sharded and world > 1:
            # host shards -> device -> sharded budget -> chunked Ulysses + PASA -> host shard
            dsq, dsk, dsv = (torch.empty_like(t) for t in src)
            dx = [torch.empty_like(x) for x in xs_sh]
            hx = [x.cpu().pin_memory() for x in xs_sh]
            h2d = sum(t.numel() * t.element_size() for t in (hq, hk, hv, *hx))
            dout = torch.empty_like(out_s)

            def e2e_step():
                for d, hsrc in zip((dsq, dsk, dsv, *dx), (hq, hk, hv, *hx)):
                    d.copy_(hsrc, non_blocking=True)
                pdist.sharded_budget(budget, *dx, n_total=x_t.numel(), **bkw)
                chunk_ev.append(None)
                uly(dsq, dsk, dsv, dout, compute)
                hout.copy_(dout, non_blocking=True)
        elif partition == "flat":
            # the rank's heads to the device, its (head, q-block) segments, its rows back
            dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
            dx = [torch.empty_like(x) for x in (x_t, x_tm1, x_tm2)]
            dout = torch.empty_like(out)
            dunits = []
            for (r, *_), (h, n, a, b) in zip(units, segs):
                sl = slice(h - off, h - off + n)
                dunits.append((r, dq[:, :, sl], dk[:, :, sl], dv[:, :, sl], dout[:, :, sl]))

            def e2e_step():
                for d, hsrc in zip((dq, dk, dv, *dx), (hq, hk, hv, *hx)):
                    d.copy_(hsrc, non_blocking=True)
                budget(dx[0], dx[1], dx[2], **bkw)
                for r, qu, ku, vu, ou in dunits:
                    r(qu, ku, budget, seed, t_step, v=vu if use_v else None)
                    P.attn(qu, ku, vu, r, ou, **attn_kw)
                hout.copy_(dout, non_blocking=True)
        elif n_chunks > 1:
            # public API for host-resident tensors: head chunks on copy-in / compute /
            # copy-out streams (paper_2604_12219_b200.pipeline)
            from paper_2604_12219_b200.pipeline import HostPipeline
            pipe = HostPipeline(B, S, Hl, D, rcfg, n_chunks=n_chunks, device=dev, attn_kw=attn_kw)

            def e2e_step():
                pipe(hq, hk, hv, hout, hx, seed, t_step, v_for_prior=use_v, T=50,
                     rho=cfg["rho"], l1_mean=lbar, h_t=1 / 50, h_tm1=1 / 50, rho_table=table)
        else:
            dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
            dx = [torch.empty_like(x) for x in (x_t, x_tm1, x_tm2)]

            def e2e_step():
                for d, hsrc in zip((dq, dk, dv, *dx), (hq, hk, hv, *hx)):
                    d.copy_(hsrc, non_blocking=True)
                budget(dx[0], dx[1], dx[2], T=50, step=t_step, rho=cfg["rho"], l1_mean=lbar,
                       h_t=1 / 50, h_tm1=1 / 50, rho_table=table)
                route(dq, dk, budget, seed, t_step, v=dv if use_v else None)
                P.attn(dq, dk, dv, route, out, **attn_kw)
                hout.copy_(out, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        n_e2e = max(2, min(K, 5))
        a, bq = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        a.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        bq.record(stream)
        torch.cuda.synchronize()
        te = all_max([a.elapsed_time(bq) / n_e2e])[0]
        h2d_all, d2h_all = all_sum([h2d, d2h])          # uneven heads: sum over ranks
        # the e2e roofline: this rank's pinned-host -> device copy bandwidth, measured with
        # one contiguous 512 MB copy (best of 3), and the step's H2D bytes at that rate
        hb = torch.empty(1 << 28, dtype=torch.bfloat16, pin_memory=True)
        db = torch.empty(1 << 28, dtype=torch.bfloat16, device=dev)
        bw = 0.0
        for _ in range(3):
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            db.copy_(hb, non_blocking=True)
            c1.record(stream)
            torch.cuda.synchronize()
            bw = max(bw, hb.numel() * 2 / (c0.elapsed_time(c1) * 1e-3) / 1e9)
        del hb, db
        e2e = {"value": 4.0 * S * S * D * B * H / (te * 1e-3) / 1e12, "unit": UNIT,
               "ms_per_step": te, "h2d_bytes_per_step": int(h2d_all),
               "d2h_bytes_per_step": int(d2h_all), "steps": n_e2e,
               "head_chunks": n_chunks,
               "pcie_h2d_gbs": bw, "h2d_bound_ms": h2d / (bw * 1e9) * 1e3,
               "frac_of_h2d_bound": (h2d / (bw * 1e9) * 1e3) / te}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    pk, which = peaks()
    NK, NG = route.NK, route.NG
    flops_head = algorithmic_flops_per_head(S, D, NK, NG, kk)
    attn_flops = flops_head * B * work_heads   # per step, this rank (all its launches)
    t_attn = float(ph[3])
    achieved = attn_flops / (t_attn * 1e-3) / 1e12
    peak = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "attn_traffic.json")) as f:
            tr = json.load(f)
            if (tr.get("config") == args.config and tr.get("heads") == work_heads
                    and cfg["Bq"] == 128):   # the capture is of the default Bq = 128 kernel
                traffic = tr.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    value = 4.0 * S * S * D * B * H / (t_max * 1e-3) / 1e12
    # secondary roofline of the attention kernel: its exponentials on the MUFU pipe
    # (16 ex2 / clk / SM measured, tools/mufu_bench.cu; 128 x 64 per E or C op, the C ops
    # being every 64-block chunk with a dropped block -- all of them at these densities)
    clocks = clk.summary()
    n_c = 0 if kk >= NK else (NK + 63) // 64
    n_exp = int(B * work_heads * route.NQ * (kk + n_c) * 128 * 64)
    f_hz = (clocks.get("sm_mhz") or 1965.0) * 1e6
    mufu = {"bound": "mufu", "achieved": n_exp / (t_attn * 1e-3) / 1e12,
            "peak": 16 * 148 * f_hz / 1e12, "unit": "Tex2/s",
            "peak_kind": "16 ex2/clk/SM x 148 SMs at the sampled median SM clock",
            "exps_per_launch": n_exp}
    mufu["frac"] = mufu["achieved"] / mufu["peak"]
    cpu = None
    if not args.no_cpu and world == 1:   # the oracle baseline: rank 0 at N = 1 only
        cv, secs, desc, _ = oracle_sample(cfg, args.cpu_qblocks)
        import oracle
        cpu = {"value": cv, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
               "sample": desc, "extrapolated": True}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": t_max, "ms_per_step_p50": step_p50,
        "ms_per_step_p90": step_p90, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {
            "workload": args.config, "B": B, "S": S, "H": H, "D": D,
            "heads_per_rank": work_heads, "nranks": world, "heads_per_rank_all": heads_all,
            "partition": partition, "segments": segs if partition == "flat" else None,
            "ulysses_chunks": (("zero-copy" if zc is not None else uly.C) if seq_sharded
                               else None),
            "dist_backend": (args.dist_backend + (" (debug: ranks share GPUs, timings not "
                                                  "meaningful)" if gloo else "")) if world > 1
            else None,
            "Bq": cfg["Bq"], "Bk": cfg["Bk"], "G": cfg["G"], "rho": cfg["rho"],
            "step_t": t_step, "budget": args.budget, "prior": args.prior,
            "qk_precision": args.qk_precision, "attn_kernel": "cta_pair" if args.cta_pair else ("q256_one_cta" if cfg["Bq"] == 256 else "default"), "l1": rec["l1"], "alpha": rec["alpha"],
            "rho_t": rec["rho_t"], "k": kk, "N_K": NK, "N_G": NG,
            "beta": 0.1, "inputs": "iid N(0,1) bf16, seeded per global head",
            "l2": "inputs larger than L2 (q,k,v 2.3 GB vs 126 MB), no flush",
            "parallelism": (f"sequence-sharded input and latents, chunked Ulysses all-to-all "
                            f"x{world} (ms_layer route/kv_stats/attn summed over the chunks)")
                           if seq_sharded else
                           (f"(head, q-block) partition x{world}" if partition == "flat"
                            else f"head-partition x{world}"),
        },
        "ms_layer": {"budget": float(ph[0]), "route": float(ph[1]), "kv_stats": float(ph[2]),
                     "attn": float(ph[3]), "other": float(t_max - ph.sum())},
        "tflops_algorithmic": flops_head * B * H / (t_max * 1e-3) / 1e12,
        "pct_of_peak_algorithmic": flops_head * B * H / (t_max * 1e-3) / 1e12 / peak,
        "roofline": {"kernel": ("attn_sm100_cta2_kernel" if args.cta_pair else
                                "attn_sm100_q256_kernel" if cfg["Bq"] == 256 else
                                "attn_sm100_kernel"), "bound": "tensor", "achieved": achieved,
                     "peak": peak, "peak_kind": f"bf16 dense, sustained ({which})",
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                     "flops_per_launch": attn_flops},
        "roofline_mufu": mufu,
        "clocks": clocks,
        "gpu_launches": gpu_launches,
        "e2e": e2e,
        "graph": graph,
        "budget_graph": budget_graph,
        "schedule": schedule,
        "dense_context": dense,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.cta_pair and args.bq != 256:
        raise SystemExit("bench.py: --cta-pair runs Bq = 256 routes (add --bq 256)")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (rank 0 prints the JSON line)
        return subprocess.call(torchrun_cmd(argv, args.gpus, free_port()))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE = {world}")
    if args.impl == "reference":
        return run_reference(args)
    return run_pasa(args)


if __name__ == "__main__":
    sys.exit(main())
