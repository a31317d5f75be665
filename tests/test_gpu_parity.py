"""GPU <-> oracle parity through the C ABI (libpasa.so).

Comparison protocol:
* budget: l1 relative error <= 1e-12, rho_t relative <= 1e-12, flags equal;
* route: pooled means bitwise equal; k, count, idx, mask bit-exact, except
  documented ties (|rt_a - rt_b| <= 1e-6 max(1,|rt_b|) on the oracle's scores);
* attention: compared with oracle_attn_with_route(GPU route):
  max|O_gpu - O_orc| <= 2e-2 max|O_orc| (bf16 I/O), <= 1e-5 max|O_orc| (fp32).
Inputs are seeded synthetic tensors from ``synth``.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = {torch.bfloat16: 2e-2, torch.float32: 1e-5}
# Regression bound on the achieved error, well inside the 2e-2 contract: SURVEY.md §8c
# emulated the GPU's bf16 storage / rounding choices at 2.7e-3 (max) and round 1's
# smoke measured 3.5e-3, so a bug that multiplies the error several-fold fails here
# even though it would pass the contract.  Every achieved value is logged
# (conftest.parity_log -> profiles/r02_parity_errors.md).
REG = {torch.bfloat16: 8e-3, torch.float32: 1e-5}


@pytest.fixture(scope="module")
def pasa():
    from paper_2604_12219_b200 import build
    build.build()
    import paper_2604_12219_b200 as P
    return P


def make_budget(P, rho, step=25, T=50):
    b = P.Budget()
    x = torch.zeros(64, device="cuda")
    b(x, x, x, T=T, step=step, rho_table=[rho] * T, l1_mean=1.0)
    return b


def check_route(P, q, k, cfg, rho, seed=42, step=25, heads=None):
    """Build the GPU route and compare it with the oracle; returns (route, read)."""
    B, S, H, D = q.shape
    route = P.Route(B, S, H, D, cfg)
    route.ws.fill_(0xFF)      # poisoned workspace (fp64 NaN, int -1): no stale value can pass
    budget = make_budget(P, rho, step)
    route(q, k, budget, seed, step)
    got = route.read()
    NK = route.NK
    kk = oracle.density_to_k(rho, NK)
    assert got["k"] == kk
    assert (got["count"] == kk).all()
    heads = range(B * H) if heads is None else heads
    qbar, kbar = route.pooled()
    ties = 0
    for bh in heads:
        b, h = divmod(bh, H)
        qh = q[b:b + 1, :, h:h + 1]
        kh = k[b:b + 1, :, h:h + 1]
        # R1: pooled means are bitwise equal to the oracle's sequential sums
        assert np.array_equal(qbar[bh], oracle.block_means(oracle.heads(qh)[0], cfg.Bq))
        assert np.array_equal(kbar[bh], oracle.block_means(oracle.heads(kh)[0], cfg.Bk))
        gh = b * (cfg.H_total or H) + cfg.head_offset + h   # global head (R-20)
        want = oracle.route(qh, kh, Bq=cfg.Bq, Bk=cfg.Bk, beta=cfg.beta, seed=seed, step=step,
                            H_total=gh + 1, head_offset=gh, kk=kk, want_scores=True)
        gi = got["idx"][bh, :, :kk]
        wi = want["idx"][0]
        for i in np.nonzero((gi != wi).any(axis=1))[0]:
            a = sorted(set(gi[i]) - set(wi[i]))
            bb = sorted(set(wi[i]) - set(gi[i]))
            sc = want["scores"][0, i]
            for x, y in zip(a, bb):
                assert abs(sc[x] - sc[y]) <= 1e-6 * max(1.0, abs(sc[y])), (bh, i, x, y)
                ties += 1
        if ties == 0:
            assert np.array_equal(got["mask"][bh], want["mask"][0])
    return route, got, ties


def errors(o, ref):
    """(max|o - ref| / max|ref|, ||o - ref||_F / ||ref||_F) in fp64."""
    d = o - ref
    return (float(np.abs(d).max() / np.abs(ref).max()),
            float(np.sqrt((d * d).sum() / (ref * ref).sum())))


def check_attn(P, q, k, v, route, got, cfg, force_simt=False, pairs=None, log=None, label="",
               cta_pair=False):
    out = P.attn(q, k, v, route, force_simt=force_simt, cta_pair=cta_pair)
    torch.cuda.synchronize()
    B, S, H, D = q.shape
    if pairs is None:
        ref = oracle.attn_with_route(q, k, v, got["idx"], got["count"], Bq=cfg.Bq, Bk=cfg.Bk,
                                     G=cfg.G, comp=cfg.comp)
        err, frob = errors(oracle.f64(out), ref)
    else:
        bhs = sorted({bh for bh, _ in pairs})
        sub = {bh: n for n, bh in enumerate(bhs)}
        sel = lambda t: torch.stack([t[bh // H, :, bh % H] for bh in bhs], 0)  # noqa: E731
        qh, kh, vh = (oracle.f64(sel(t)) for t in (q, k, v))
        idx = np.stack([got["idx"][bh] for bh in bhs])
        cnt = np.stack([got["count"][bh] for bh in bhs])
        lp = [(sub[bh], i) for bh, i in pairs]
        ref = oracle.attn_pairs(None, None, None, idx, cnt, lp, Bq=cfg.Bq, Bk=cfg.Bk, G=cfg.G,
                                comp=cfg.comp, qh=qh, kh=kh, vh=vh)
        os_, rs = [], []
        for n, (bh, i) in enumerate(pairs):
            rows = min(cfg.Bq, S - i * cfg.Bq)
            os_.append(oracle.f64(out[bh // H, i * cfg.Bq:i * cfg.Bq + rows, bh % H]))
            rs.append(ref[n, :rows])
        err, frob = errors(np.concatenate(os_), np.concatenate(rs))
    assert np.isfinite(oracle.f64(out)).all()
    if log is not None:
        log(label or f"B{B} S{S} H{H} D{D} Bq{cfg.Bq} G{cfg.G} {cfg.comp} {str(q.dtype)[6:]}"
            + (f" sampled {len(pairs)} (head, q-block)" if pairs else ""), err, frob, REG[q.dtype])
    assert err <= TOL[q.dtype], err
    assert err <= REG[q.dtype], f"achieved error {err:.3e} above the regression bound"
    return out, err


# ----------------------------------------------------------------- budget --
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_budget_parity_three_phase(pasa, dtype):
    tp = synth.ThreePhase(shape=synth.CONFIGS["cogvideox5b"]["latent"], T=50, seed=7,
                          device="cuda")
    lbar = tp.expected_l1_mean()
    b = pasa.Budget()
    for t in (3, 11, 30, 48):
        xs = [x.to(dtype).contiguous() for x in tp.latents(t)]
        b(*xs, T=50, step=t, rho=0.15, dense_frac=0.2, l1_mean=lbar, h_t=1 / 50, h_tm1=1 / 50)
        got = b.read()
        want = oracle.budget(*xs, T=50, step=t, rho=0.15, dense_frac=0.2, l1_mean=lbar,
                             h_t=1 / 50, h_tm1=1 / 50)
        assert got["l1"] == pytest.approx(want["l1"], rel=1e-12)
        assert got["alpha"] == pytest.approx(want["alpha"], rel=1e-12)
        assert got["rho_t"] == pytest.approx(want["rho_t"], rel=1e-12)
        assert got["dense"] == want["dense"] and got["clipped"] == want["clipped"]
    # deterministic fixed-grid reduction: bitwise identical run to run
    b(*xs, T=50, step=48, rho=0.15, l1_mean=lbar, h_t=1 / 50, h_tm1=1 / 50)
    again = b.read()
    assert again["l1"] == got["l1"]


def test_budget_velocity_table_and_clip(pasa):
    g = torch.Generator(device="cuda").manual_seed(3)
    v1 = torch.randn(100_003, device="cuda", generator=g)
    v0 = torch.randn(100_003, device="cuda", generator=g)
    b = pasa.Budget()
    b(v1, v0, None, kind="velocity", T=50, step=20, rho=0.5, l1_mean=0.1)
    got = b.read()
    want = oracle.budget(v1, v0, kind=1, T=50, step=20, rho=0.5, l1_mean=0.1)
    assert got["l1"] == pytest.approx(want["l1"], rel=1e-12)
    assert got["clipped"] and want["clipped"] and got["rho_t"] == 1.0
    tab = np.linspace(0.05, 0.4, 50)
    b(v1, v0, None, kind="velocity", T=50, step=33, rho_table=tab, l1_mean=1.0)
    assert b.read()["rho_t"] == tab[33]
    b(v1, v0, None, kind="velocity", T=50, step=4, rho=0.15, l1_mean=1.0)
    assert b.read()["dense"] and b.read()["rho_t"] == 1.0


# ------------------------------------------------------------------ route --
ROUTE_CASES = [
    # name, B, S, H, D, Bq, beta, rho, gen
    ("tiny", 1, 1024, 1, 64, 64, 0.1, 0.5, "video"),
    ("ragged1000", 1, 1000, 2, 128, 128, 0.1, 0.15, "iid"),
    ("ragged4100", 2, 4100, 2, 64, 128, 0.1, 0.15, "video"),
    ("beta0", 1, 4100, 2, 128, 128, 0.0, 0.15, "iid"),
    ("bigbeta", 1, 2048, 1, 128, 128, 5.0, 0.3, "iid"),
    # N_K = 256: the select kernel's compacted-window search (few keys near the k-th)
    ("iid16k", 1, 16384, 2, 128, 128, 0.1, 0.15, "iid"),
    # every score within one 1/16 binade: the window holds > 64 keys -> full bit search
    ("clustered16k", 1, 16384, 2, 128, 128, 0.1, 0.15, "clustered"),
]


def gen_qkv(gen, B, S, H, D, dtype, seed=1000):
    if gen == "iid":
        return synth.iid_qkv(B, S, H, D, seed=seed, dtype=dtype, device="cuda")
    if gen == "clustered":   # q, k = 1 + small noise: all block scores near s * d
        q, k, v = synth.iid_qkv(B, S, H, D, seed=seed, dtype=torch.float32, device="cuda")
        return ((1 + 0.05 * q).to(dtype), (1 + 0.05 * k).to(dtype), v.to(dtype))
    F = max(1, S // (32 * 32))
    grid = (F, 32, S // (32 * F)) if S % (32 * F) == 0 else (1, 1, S)
    return synth.video_qkv(B, grid, H, D, seed=seed, dtype=dtype, device="cuda")


@pytest.mark.parametrize("case", ROUTE_CASES, ids=[c[0] for c in ROUTE_CASES])
def test_route_bit_exact(pasa, case):
    name, B, S, H, D, Bq, beta, rho, gen = case
    q, k, _ = gen_qkv(gen, B, S, H, D, torch.bfloat16)
    cfg = pasa.RouteCfg(Bq=Bq, G=32, beta=beta)
    _, got, ties = check_route(pasa, q, k, cfg, rho, seed=pasa.layer_seed(42, 3), step=17)
    assert ties <= 2


def test_route_fp32_and_head_partition(pasa):
    """R-20: Philox keyed on the global head -> routing heads [2,4) at offset 2 of 4
    equals rows 2..3 of the full route, bit for bit."""
    q, k, _ = synth.iid_qkv(1, 3000, 4, 64, seed=5, dtype=torch.float32, device="cuda")
    cfg = pasa.RouteCfg(Bq=128, beta=0.3)
    _, full, _ = check_route(pasa, q, k, cfg, 0.2)
    cfgp = pasa.RouteCfg(Bq=128, beta=0.3, H_total=4, head_offset=2)
    qp, kp = q[:, :, 2:].contiguous(), k[:, :, 2:].contiguous()
    _, part, _ = check_route(pasa, qp, kp, cfgp, 0.2)
    kk = full["k"]
    assert part["k"] == kk
    assert np.array_equal(full["idx"][2:, :, :kk], part["idx"][:, :, :kk])
    assert np.array_equal(full["mask"][2:], part["mask"])


# -------------------------------------------------------------- attention --
ATTN_CASES = [
    # name, B, S, H, D, Bq, G, comp, rho, dtype, gen
    ("tiny_simt", 1, 1024, 1, 64, 64, 32, "grouped", 0.5, torch.bfloat16, "video"),
    ("tiny_g4_simt", 1, 1024, 1, 64, 64, 4, "grouped", 0.5, torch.bfloat16, "video"),
    ("tiny_fp32", 1, 1024, 1, 64, 64, 32, "grouped", 0.5, torch.float32, "video"),
    ("tc_d128_1000", 1, 1000, 2, 128, 128, 32, "grouped", 0.15, torch.bfloat16, "iid"),
    ("tc_d128_4100_g32", 1, 4100, 2, 128, 128, 32, "grouped", 0.15, torch.bfloat16, "video"),
    ("tc_d64_4100_g32", 2, 4100, 2, 64, 128, 32, "grouped", 0.15, torch.bfloat16, "video"),
    ("tc_d128_4100_g64", 1, 4100, 2, 128, 128, 64, "grouped", 0.15, torch.bfloat16, "video"),
    ("tc_d128_4100_global", 1, 4100, 2, 128, 128, 4096, "grouped", 0.15, torch.bfloat16, "iid"),
    ("tc_d128_4100_zeroth", 1, 4100, 2, 128, 128, 32, "zeroth", 0.15, torch.bfloat16, "video"),
    ("tc_d64_4100_none", 1, 4100, 2, 64, 128, 32, "none", 0.15, torch.bfloat16, "iid"),
    ("fp32_d128_4100", 1, 4100, 1, 128, 128, 32, "grouped", 0.15, torch.float32, "video"),
    ("tc_d128_g8", 1, 4100, 1, 128, 128, 8, "grouped", 0.15, torch.bfloat16, "video"),
    ("tc_d64_g16", 1, 9000, 2, 64, 128, 16, "grouped", 0.2, torch.bfloat16, "video"),
    ("tc_d128_g16_ragged", 1, 4100, 1, 128, 128, 16, "grouped", 0.3, torch.bfloat16, "iid"),
    ("tc_d128_g4_simt", 1, 4100, 1, 128, 128, 4, "grouped", 0.15, torch.bfloat16, "video"),
    ("tc_d128_g96_simt", 1, 8200, 1, 128, 128, 96, "grouped", 0.15, torch.bfloat16, "video"),
    ("tc_d128_20000_g128", 1, 20000, 1, 128, 128, 128, "grouped", 0.15, torch.bfloat16, "video"),
    ("tc_d64_20000_g64", 1, 20000, 1, 64, 128, 64, "grouped", 0.2, torch.bfloat16, "video"),
    ("tc_d128_odd_k", 1, 4100, 2, 128, 128, 32, "grouped", 0.11, torch.bfloat16, "iid"),
]


@pytest.mark.parametrize("case", ATTN_CASES, ids=[c[0] for c in ATTN_CASES])
def test_attn_parity(pasa, case, parity_log):
    name, B, S, H, D, Bq, G, comp, rho, dtype, gen = case
    q, k, v = gen_qkv(gen, B, S, H, D, dtype, seed=11)
    cfg = pasa.RouteCfg(Bq=Bq, G=G, comp=comp, beta=0.1)
    route, got, _ = check_route(pasa, q, k, cfg, rho)
    out, err = check_attn(pasa, q, k, v, route, got, cfg, log=parity_log, label=name)
    # determinism: no atomics on the output path -> bitwise reproducible
    out2 = pasa.attn(q, k, v, route)
    assert torch.equal(out, out2)


Q256_CASES = [
    # Bq = 256: one route per 256 queries, two 128-row M tiles
    # sharing every K/V / centroid / Hbar tile
    ("q256_d128_1000", 1, 1000, 2, 128, 256, 32, "grouped", 0.15, torch.bfloat16, "iid"),
    ("q256_d128_4100_g32", 1, 4100, 2, 128, 256, 32, "grouped", 0.15, torch.bfloat16, "video"),
    ("q256_d64_4100_g32", 2, 4100, 2, 64, 256, 32, "grouped", 0.15, torch.bfloat16, "video"),
    ("q256_d128_4100_g64", 1, 4100, 2, 128, 256, 64, "grouped", 0.15, torch.bfloat16, "video"),
    ("q256_d128_4100_global", 1, 4100, 2, 128, 256, 4096, "grouped", 0.15, torch.bfloat16, "iid"),
    ("q256_d128_4100_zeroth", 1, 4100, 2, 128, 256, 32, "zeroth", 0.15, torch.bfloat16, "video"),
    ("q256_d64_4100_none", 1, 4100, 2, 64, 256, 32, "none", 0.15, torch.bfloat16, "iid"),
    ("q256_d128_20000_g128", 1, 20000, 1, 128, 256, 128, "grouped", 0.15, torch.bfloat16, "video"),
    ("q256_d64_9000_odd_k", 1, 9000, 2, 64, 256, 32, "grouped", 0.11, torch.bfloat16, "iid"),
]


@pytest.mark.parametrize("case", Q256_CASES, ids=[c[0] for c in Q256_CASES])
def test_attn_parity_q256(pasa, case, parity_log):
    """Bq = 256 routing (bit-exact against the oracle's route at Bq = 256) and the
    two-tile tensor-core kernel against the oracle's attention at Bq = 256."""
    name, B, S, H, D, Bq, G, comp, rho, dtype, gen = case
    q, k, v = gen_qkv(gen, B, S, H, D, dtype, seed=13)
    cfg = pasa.RouteCfg(Bq=Bq, G=G, comp=comp, beta=0.1)
    route, got, _ = check_route(pasa, q, k, cfg, rho)
    out, _ = check_attn(pasa, q, k, v, route, got, cfg, log=parity_log, label=name)
    assert torch.equal(out, pasa.attn(q, k, v, route))


@pytest.mark.parametrize("S", [1, 100, 256, 257, 511, 640])
def test_attn_q256_edges(pasa, S):
    """Bq = 256 around the tile edges: a q-block with only tile 0 live, exactly one
    q-block, one row past it, and k = 1."""
    q, k, v = synth.iid_qkv(1, S, 2, 128, seed=S + 7, dtype=torch.bfloat16, device="cuda")
    cfg = pasa.RouteCfg(Bq=256, G=32, beta=0.1)
    route, got, _ = check_route(pasa, q, k, cfg, 0.3 if S > 64 else 1.0)
    check_attn(pasa, q, k, v, route, got, cfg)


def test_attn_q256_rejects_unsupported(pasa):
    q, k, v = synth.iid_qkv(1, 1000, 1, 64, seed=3, dtype=torch.float32, device="cuda")
    route = pasa.Route(1, 1000, 1, 64, pasa.RouteCfg(Bq=256, G=32))
    route(q, k, make_budget(pasa, 0.3), 1, 25)
    with pytest.raises(pasa.PasaError):
        pasa.attn(q, k, v, route)


CTA2_CASES = [c for c in Q256_CASES if c[4] == 128]


@pytest.mark.parametrize("case", CTA2_CASES, ids=[c[0] + "_cta2" for c in CTA2_CASES])
def test_attn_parity_cta_pair(pasa, case, parity_log):
    """Bq = 256 on the CTA-pair kernel (tcgen05 cta_group::2, M = 256, each SM holding half
    of every operand tile) against the oracle's attention at Bq = 256; bitwise
    reproducible, and equal to the one-CTA two-tile kernel up to fp32 summation order."""
    name, B, S, H, D, Bq, G, comp, rho, dtype, gen = case
    q, k, v = gen_qkv(gen, B, S, H, D, dtype, seed=13)
    cfg = pasa.RouteCfg(Bq=Bq, G=G, comp=comp, beta=0.1)
    route, got, _ = check_route(pasa, q, k, cfg, rho)
    out, _ = check_attn(pasa, q, k, v, route, got, cfg, log=parity_log, label=name + " cta_pair",
                        cta_pair=True)
    assert torch.equal(out, pasa.attn(q, k, v, route, cta_pair=True))
    one = pasa.attn(q, k, v, route).float()
    assert float((out.float() - one).abs().max()) <= 1e-2 * float(one.abs().max())


@pytest.mark.parametrize("S", [1, 100, 256, 257, 511, 640])
def test_attn_cta_pair_edges(pasa, S):
    """CTA pair around the tile edges: the peer CTA's rows entirely past S (S <= 128),
    exactly one q-block, one row past it, and k = 1."""
    q, k, v = synth.iid_qkv(1, S, 2, 128, seed=S + 7, dtype=torch.bfloat16, device="cuda")
    cfg = pasa.RouteCfg(Bq=256, G=32, beta=0.1)
    route, got, _ = check_route(pasa, q, k, cfg, 0.3 if S > 64 else 1.0)
    check_attn(pasa, q, k, v, route, got, cfg, cta_pair=True)


def test_attn_cta_pair_rejects_unsupported(pasa):
    """d = 64 and Bq = 128 routes are outside the pair kernel's domain: EUNSUPPORTED."""
    for D, Bq in ((64, 256), (128, 128)):
        q, k, v = synth.iid_qkv(1, 1000, 1, D, seed=3, dtype=torch.bfloat16, device="cuda")
        route = pasa.Route(1, 1000, 1, D, pasa.RouteCfg(Bq=Bq, G=32))
        route(q, k, make_budget(pasa, 0.3), 1, 25)
        with pytest.raises(pasa.PasaError):
            pasa.attn(q, k, v, route, cta_pair=True)


EDGE_CASES = [
    # name, S, D, Bq, rho, dtype: degenerate lengths around the block sizes, k = 1
    ("S1", 1, 128, 128, 0.15, torch.bfloat16),
    ("S37", 37, 64, 128, 0.5, torch.bfloat16),
    ("S64", 64, 128, 128, 0.5, torch.bfloat16),
    ("S65", 65, 128, 128, 0.5, torch.bfloat16),
    ("S127", 127, 64, 128, 0.5, torch.bfloat16),
    ("S129", 129, 128, 128, 0.5, torch.bfloat16),
    ("S129_bq64", 129, 64, 64, 0.5, torch.bfloat16),
    ("k1", 3000, 128, 128, 0.001, torch.bfloat16),
    ("k1_fp32", 3000, 64, 128, 0.001, torch.float32),
    ("kNK_minus_1", 640, 128, 128, 0.9, torch.bfloat16),
]


@pytest.mark.parametrize("case", EDGE_CASES, ids=[c[0] for c in EDGE_CASES])
def test_attn_edge_cases(pasa, case, parity_log):
    """Single partial blocks (S < Bk, S < Bq), one-token sequences, lengths one past a
    block edge, k = 1 (the floor of R-14) and k = N_K - 1: route bit-exact, output
    within the tolerance of the dtype."""
    name, S, D, Bq, rho, dtype = case
    q, k, v = synth.iid_qkv(1, S, 2, D, seed=S + D, dtype=dtype, device="cuda")
    cfg = pasa.RouteCfg(Bq=Bq, G=32, beta=0.1)
    route, got, _ = check_route(pasa, q, k, cfg, rho)
    check_attn(pasa, q, k, v, route, got, cfg, log=parity_log, label="edge " + name)


def test_tensor_core_matches_simt_kernel(pasa):
    q, k, v = gen_qkv("video", 1, 4100, 2, 128, torch.bfloat16, seed=21)
    cfg = pasa.RouteCfg(Bq=128, G=32)
    route, got, _ = check_route(pasa, q, k, cfg, 0.15)
    a = pasa.attn(q, k, v, route).float()
    b = pasa.attn(q, k, v, route, force_simt=True).float()
    assert (a - b).abs().max().item() <= 2e-2 * b.abs().max().item()


@pytest.mark.parametrize("D", [64, 128])
def test_dense_step_equals_library_sdpa(pasa, D):
    """rho_t = 1 (dense prefix): k = N_K, U empty -> Eq. 1; checked against torch SDPA."""
    q, k, v = synth.iid_qkv(1, 2000, 2, D, seed=4, dtype=torch.bfloat16, device="cuda")
    cfg = pasa.RouteCfg(Bq=128)
    route = pasa.Route(1, 2000, 2, D, cfg)
    b = pasa.Budget()
    x = torch.zeros(64, device="cuda")
    b(x, x, x, T=50, step=3, l1_mean=1.0)          # step 3 < 10: dense prefix
    assert b.read()["dense"]
    route(q, k, b, 1, 3)
    assert route.read()["k"] == route.NK
    out = pasa.attn(q, k, v, route).float()
    ref = torch.nn.functional.scaled_dot_product_attention(
        *(t.float().permute(0, 2, 1, 3) for t in (q, k, v))).permute(0, 2, 1, 3)
    assert (out - ref).abs().max().item() <= 2e-2 * ref.abs().max().item()


def test_head_partition_outputs_bitwise(pasa):
    """Head-parallel sharding: P = 1 and the rank holding heads
    [2, 4) produce bitwise identical outputs for those heads."""
    q, k, v = synth.iid_qkv(1, 3000, 4, 128, seed=8, dtype=torch.bfloat16, device="cuda")
    full_r = pasa.Route(1, 3000, 4, 128, pasa.RouteCfg(Bq=128, beta=0.2))
    b = make_budget(pasa, 0.2)
    full_r(q, k, b, 9, 25)
    full = pasa.attn(q, k, v, full_r)
    part_r = pasa.Route(1, 3000, 2, 128, pasa.RouteCfg(Bq=128, beta=0.2, H_total=4,
                                                         head_offset=2))
    qs, ks, vs = (t[:, :, 2:].contiguous() for t in (q, k, v))
    part_r(qs, ks, b, 9, 25)
    part = pasa.attn(qs, ks, vs, part_r)
    assert torch.equal(full[:, :, 2:], part)


def test_strided_output_and_inputs(pasa):
    """q/k/v as head-slices of a packed qkv projection, out written into a strided view."""
    qkv = torch.randn(1, 1500, 3, 2, 128, device="cuda").to(torch.bfloat16)
    q, k, v = qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2]
    cfg = pasa.RouteCfg(Bq=128)
    route, got, _ = check_route(pasa, q, k, cfg, 0.25)
    big = torch.zeros(1, 1500, 4, 128, device="cuda", dtype=torch.bfloat16)
    out = pasa.attn(q, k, v, route, out=big[:, :, 1:3])
    ref = oracle.attn_with_route(q, k, v, got["idx"], got["count"], Bq=128, Bk=64, G=32)
    err = np.abs(oracle.f64(out) - ref).max() / np.abs(ref).max()
    assert err <= 2e-2
    assert big[:, :, 0].abs().max().item() == 0 and big[:, :, 3].abs().max().item() == 0


# ----------------------------------------------- full BASELINE configs --
def _pairs(heads, NQ, nq=16):
    """nq q-blocks per head, evenly spread, always q-block 0 and the ragged last one."""
    qs = sorted({0, NQ - 1, *np.linspace(0, NQ - 1, nq).astype(int).tolist()})
    return [(h, int(i)) for h in heads for i in qs]


def _attn_heads(H):
    """4 heads spread over the layer, first and last included."""
    return sorted({0, H - 1, *np.linspace(0, H - 1, 4).round().astype(int).tolist()})


def _full_inputs(c, gen, seed):
    B, S, H, D = c["B"], c["S"], c["H"], c["D"]
    if gen == "video":
        return synth.video_qkv(B, c["grid"], H, D, seed=seed, dtype=torch.bfloat16,
                               device="cuda")
    return synth.iid_qkv(B, S, H, D, seed=seed, dtype=torch.bfloat16, device="cuda")


@pytest.mark.parametrize("name,gen", [
    ("wan13b_480p", "video"),
    ("cogvideox5b", "video"),
    ("wan14b_720p", "iid"),
    ("wan14b_720p", "video"),
    ("hunyuan_720p", "iid"),
])
def test_full_config_sampled(pasa, name, gen, parity_log):
    """SURVEY.md §8c coverage at every BASELINE.json config at full size, in the launch
    configuration bench.py times: route (k, count, idx, mask) against the oracle on ALL
    heads, attention on 4 heads x 16 q-blocks always including q-block 0 and the ragged
    last one (Eq. 7 with App. B grouping)."""
    c = synth.CONFIGS[name]
    B, S, H, D = c["B"], c["S"], c["H"], c["D"]
    q, k, v = _full_inputs(c, gen, 1003)
    cfg = pasa.RouteCfg(Bq=c["Bq"], G=c["G"], beta=0.1)
    route, got, ties = check_route(pasa, q, k, cfg, c["rho"], seed=pasa.layer_seed(42, 0),
                                   step=25, heads=None)
    assert ties <= 4
    pairs = _pairs(_attn_heads(B * H), route.NQ, 16)
    assert len(pairs) >= 4 * 16
    check_attn(pasa, q, k, v, route, got, cfg, pairs=pairs, log=parity_log,
               label=f"{name} {gen} full size, 4 heads x 16 q-blocks")


@pytest.mark.parametrize("name", ["wan13b_480p", "cogvideox5b", "wan14b_720p", "hunyuan_720p"])
def test_full_config_constant_key_blocks_equal_dense(pasa, name, parity_log):
    """Oracle-free end-to-end check at full size: with keys constant inside every
    64-token block, every centroid logit is exact and H_j = 0, so PASA equals dense
    softmax attention (Eq. 1) for ANY route -- including the ragged
    last block's true-length weight n_j (R-2, R-7).  Reference: fp32 dense attention
    computed with torch matmuls, chunked over queries, on 4 heads."""
    c = synth.CONFIGS[name]
    B, S, H, D = c["B"], c["S"], c["H"], c["D"]
    q, k, v = synth.iid_qkv(B, S, H, D, seed=1006, dtype=torch.bfloat16, device="cuda")
    NK = (S + 63) // 64
    first = torch.arange(NK, device="cuda").repeat_interleave(64)[:S] * 64
    k = k[:, first].contiguous()                  # K_n = K of the block's first token
    for rho in (c["rho"], 0.4):
        cfg = pasa.RouteCfg(Bq=c["Bq"], G=c["G"], beta=0.1)
        route = pasa.Route(B, S, H, D, cfg)
        route(q, k, make_budget(pasa, rho), pasa.layer_seed(42, 0), 25)
        out = pasa.attn(q, k, v, route)
        torch.cuda.synchronize()
        assert 0 < route.read()["k"] < NK
        err, frob, mx = 0.0, 0.0, 0.0
        num = den = 0.0
        for bh in _attn_heads(B * H):
            b, h = divmod(bh, H)
            qh, kh, vh = (t[b, :, h].float() for t in (q, k, v))
            s = 1.0 / math.sqrt(D)
            for r0 in range(0, S, 8192):
                p = torch.softmax((qh[r0:r0 + 8192] @ kh.T) * s, dim=-1)
                ref = (p @ vh).double()
                o = out[b, r0:r0 + 8192, h].double()
                err = max(err, (o - ref).abs().max().item())
                mx = max(mx, ref.abs().max().item())
                num += ((o - ref) ** 2).sum().item()
                den += (ref ** 2).sum().item()
        err /= mx
        frob = math.sqrt(num / den)
        parity_log(f"{name} constant-key blocks rho={rho} vs dense fp32 (4 heads)", err, frob,
                   REG[torch.bfloat16], ref="dense")
        assert err <= TOL[torch.bfloat16], err
        assert err <= REG[torch.bfloat16], err


@pytest.mark.parametrize("variant", ["default", "q256", "cta_pair"])
@pytest.mark.parametrize("name", ["wan13b_480p", "cogvideox5b", "wan14b_720p", "hunyuan_720p"])
def test_full_config_repeat_finite_bitwise(pasa, name, variant):
    """Every BASELINE config at full size in bench.py's launch configuration, three
    times: the whole output is finite and bitwise identical run to run.  (A barrier
    lapped by a softmax running two ops ahead at d = 64 once let PV read an unloaded
    V tile: a few rows of NaN in some runs, invisible to sampled parity.)"""
    c = synth.CONFIGS[name]
    B, S, H, D = c["B"], c["S"], c["H"], c["D"]
    if variant == "cta_pair" and D != 128:
        pytest.skip("the CTA-pair kernel is d = 128 only")
    q, k, v = synth.iid_qkv(B, S, H, D, seed=1004, dtype=torch.bfloat16, device="cuda")
    cfg = pasa.RouteCfg(Bq=c["Bq"] if variant == "default" else 256, G=c["G"], beta=0.1)
    route = pasa.Route(B, S, H, D, cfg)
    route(q, k, make_budget(pasa, c["rho"]), pasa.layer_seed(42, 0), 25)
    first = None
    for _ in range(3):
        out = torch.full_like(q, float("nan"))
        pasa.attn(q, k, v, route, out, cta_pair=variant == "cta_pair")
        torch.cuda.synchronize()
        assert bool(torch.isfinite(out).all())
        if first is None:
            first = out
        else:
            assert torch.equal(out, first)


def test_full_config_q256_sampled(pasa, parity_log):
    """Wan 2.1-14B 720p at full size with Bq = 256: route bit-exact on all heads,
    attention on 4 heads x 16 q-blocks incl. the ragged last one, whole output finite
    and bitwise reproducible."""
    c = synth.CONFIGS["wan14b_720p"]
    B, S, H, D = c["B"], c["S"], c["H"], c["D"]
    q, k, v = synth.iid_qkv(B, S, H, D, seed=1005, dtype=torch.bfloat16, device="cuda")
    cfg = pasa.RouteCfg(Bq=256, G=c["G"], beta=0.1)
    route, got, ties = check_route(pasa, q, k, cfg, c["rho"], seed=pasa.layer_seed(42, 0),
                                   step=25)
    assert ties <= 4
    out, _ = check_attn(pasa, q, k, v, route, got, cfg, pairs=_pairs(_attn_heads(H), route.NQ),
                        log=parity_log, label="wan14b_720p Bq=256 full size, 4 heads x 16 q-blocks")
    assert bool(torch.isfinite(out).all())
    assert torch.equal(out, pasa.attn(q, k, v, route))


def test_full_config_cta_pair_sampled(pasa, parity_log):
    """Wan 2.1-14B 720p at full size with Bq = 256 on the CTA-pair kernel: attention on
    4 heads x 16 q-blocks incl. the ragged last one against the oracle, whole output
    finite and bitwise reproducible over three launches."""
    c = synth.CONFIGS["wan14b_720p"]
    B, S, H, D = c["B"], c["S"], c["H"], c["D"]
    q, k, v = synth.iid_qkv(B, S, H, D, seed=1006, dtype=torch.bfloat16, device="cuda")
    cfg = pasa.RouteCfg(Bq=256, G=c["G"], beta=0.1)
    route, got, ties = check_route(pasa, q, k, cfg, c["rho"], seed=pasa.layer_seed(42, 0),
                                   step=25, heads=[0, 17, 39])
    out, _ = check_attn(pasa, q, k, v, route, got, cfg, pairs=_pairs(_attn_heads(H), route.NQ),
                        log=parity_log, label="wan14b_720p Bq=256 cta_pair full size, 4 heads x 16 q-blocks",
                        cta_pair=True)
    for _ in range(2):
        again = torch.full_like(q, float("nan"))
        pasa.attn(q, k, v, route, again, cta_pair=True)
        torch.cuda.synchronize()
        assert bool(torch.isfinite(again).all())
        assert torch.equal(out, again)


def test_long_sequence_200k_route_and_attention(pasa, parity_log):
    """S = 200,000 tokens (N_K = 3,125 > the 2,048 of round 1): the fused
    route keeps its score rows in the workspace scratch (they no longer fit on chip) and the
    tensor-core attention walks a 16-bit op list of up to 4,096 kept blocks.  Route against
    the oracle on every q-block, attention on 16 q-blocks incl. the first and ragged last;
    and a dense step (k = N_K = 3,125 kept blocks) on 4 q-blocks."""
    B, S, H, D = 1, 200_000, 1, 128
    q, k, v = synth.iid_qkv(B, S, H, D, seed=1010, dtype=torch.bfloat16, device="cuda")
    cfg = pasa.RouteCfg(Bq=128, G=32, beta=0.1)
    route, got, ties = check_route(pasa, q, k, cfg, 0.15, seed=pasa.layer_seed(42, 0), step=25)
    assert route.NK == 3125 and ties <= 2
    check_attn(pasa, q, k, v, route, got, cfg, pairs=_pairs([0], route.NQ, 16), log=parity_log,
               label="S = 200,000 (N_K = 3,125)")
    route_d, got_d, _ = check_route(pasa, q, k, cfg, 1.0, seed=pasa.layer_seed(42, 0), step=25)
    assert got_d["k"] == 3125
    check_attn(pasa, q, k, v, route_d, got_d, cfg, pairs=_pairs([0], route_d.NQ, 4),
               log=parity_log, label="S = 200,000 dense step (3,125 kept blocks)")
