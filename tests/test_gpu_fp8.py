"""FP8 QK^T variant (opt-in precision flag RouteCfg(qk_precision="fp8"), SURVEY.md §8f
NEXT 4, reading R-30 of DESIGN.md): QK^T of kept blocks and the centroid logits on the
FP8 tensor cores (E4M3 Q with one scale per token row, E4M3 K with one per 64-token
block, E4M3 Kbar with one per head), PV and the first-order term in bf16.

Its own tolerance, derived from the E4M3 rounding alone: a NumPy emulation of exactly
these scalings on dense attention (S = 4096, d = 128) gives max|dO|/max|O| = 5.6e-2 /
3.8e-2 and relative Frobenius 3.9e-2 / 1.6e-2 (iid / video inputs), so the bound is
1e-1 max-relative and 6e-2 Frobenius against the exact fp64 oracle on the same route.
The route does not depend on the precision flag: it must be identical to the bf16 one.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL_MAX, TOL_FROB = 1e-1, 6e-2


@pytest.fixture(scope="module")
def pasa():
    from paper_2604_12219_b200 import build
    build.build()
    import paper_2604_12219_b200 as P
    return P


def _budget(P, rho, step=25, T=50):
    b = P.Budget()
    x = torch.zeros(64, device="cuda")
    b(x, x, x, T=T, step=step, rho_table=[rho] * T, l1_mean=1.0)
    return b


def _errors(got, ref):
    d = got - ref
    return float(np.abs(d).max() / np.abs(ref).max()), float(np.linalg.norm(d) / np.linalg.norm(ref))


def _run(P, q, k, v, prec, rho, G=32, comp="grouped"):
    B, S, H, D = q.shape
    cfg = P.RouteCfg(Bq=128, G=G, beta=0.1, comp=comp, qk_precision=prec)
    r = P.Route(B, S, H, D, cfg)
    r(q, k, _budget(P, rho), P.layer_seed(42, 0), 25)
    out = P.attn(q, k, v, r)
    torch.cuda.synchronize()
    return r, r.read(), out


@pytest.mark.parametrize("gen,S,G,comp,rho", [
    ("video", 4100, 32, "grouped", 0.15), ("iid", 4100, 32, "grouped", 0.15),
    ("video", 4100, 64, "zeroth", 0.3), ("video", 4100, 4096, "grouped", 0.15),
    ("video", 1000, 32, "none", 0.5), ("iid", 4100, 32, "grouped", 1.0),
])
def test_fp8_qk_parity(pasa, gen, S, G, comp, rho, parity_log):
    P = pasa
    B, H, D = 1, 2, 128
    if gen == "video":
        q, k, v = synth.video_qkv(B, (1, 1, S), H, D, seed=31, dtype=torch.bfloat16, device="cuda")
    else:
        q, k, v = synth.iid_qkv(B, S, H, D, seed=31, dtype=torch.bfloat16, device="cuda")
    r8, got8, out8 = _run(P, q, k, v, "fp8", rho, G, comp)
    r16, got16, out16 = _run(P, q, k, v, "bf16", rho, G, comp)
    kk = got8["k"]
    assert kk == got16["k"]
    for key in ("count", "mask"):
        assert np.array_equal(got8[key], got16[key]), key
    assert np.array_equal(got8["idx"][:, :, :kk], got16["idx"][:, :, :kk])
    ref = oracle.attn_with_route(q, k, v, got8["idx"], got8["count"], Bq=128, Bk=64, G=G,
                                 comp=comp)
    err, frob = _errors(oracle.f64(out8), ref)
    parity_log(f"FP8 QK^T {gen} S={S} G={G} {comp} rho={rho}", err, frob, TOL_MAX)
    assert np.isfinite(oracle.f64(out8)).all()
    assert err <= TOL_MAX and frob <= TOL_FROB, (err, frob)


def test_fp8_qk_full_size_wan14b_sampled(pasa, parity_log):
    """Wan-14B 720p at full size (bench.py --qk-precision fp8): 4 heads x 16 q-blocks incl.
    the first and ragged last against the oracle."""
    P = pasa
    c = synth.CONFIGS["wan14b_720p"]
    B, S, H, D = c["B"], c["S"], c["H"], c["D"]
    q, k, v = synth.video_qkv(B, c["grid"], H, D, seed=1003, dtype=torch.bfloat16, device="cuda")
    r, got, out = _run(P, q, k, v, "fp8", c["rho"])
    heads = [0, 13, 26, 39]
    qs = sorted({0, r.NQ - 1, *np.linspace(0, r.NQ - 1, 16).astype(int).tolist()})
    pairs = [(n, i) for n in range(len(heads)) for i in qs]
    sel = lambda t: torch.stack([t[0, :, h] for h in heads], 0)  # noqa: E731
    qh, kh, vh = (oracle.f64(sel(t)) for t in (q, k, v))
    ref = oracle.attn_pairs(None, None, None, np.stack([got["idx"][h] for h in heads]),
                            np.stack([got["count"][h] for h in heads]), pairs, Bq=128, Bk=64,
                            G=32, qh=qh, kh=kh, vh=vh)
    gs, rs = [], []
    for n, (hn, i) in enumerate(pairs):
        rows = min(128, S - i * 128)
        gs.append(oracle.f64(out[0, i * 128:i * 128 + rows, heads[hn]]))
        rs.append(ref[n, :rows])
    err, frob = _errors(np.concatenate(gs), np.concatenate(rs))
    parity_log("FP8 QK^T Wan-14B full size, 4 heads x 16 q-blocks", err, frob, TOL_MAX)
    assert err <= TOL_MAX and frob <= TOL_FROB, (err, frob)


def test_fp8_qk_rejects_unsupported(pasa):
    P = pasa
    for kw in (dict(Bq=256), dict(G=16)):
        with pytest.raises(P.PasaError):
            P.Route(1, 4096, 1, 128, P.RouteCfg(qk_precision="fp8", **kw))
    with pytest.raises(P.PasaError):
        P.Route(1, 4096, 1, 64, P.RouteCfg(qk_precision="fp8"))
    q, k, v = synth.iid_qkv(1, 4096, 1, 128, seed=2, dtype=torch.float32, device="cuda")
    r = P.Route(1, 4096, 1, 128, P.RouteCfg(qk_precision="fp8"))
    with pytest.raises(P.PasaError):
        r(q, k, _budget(P, 0.15), 7, 25)
