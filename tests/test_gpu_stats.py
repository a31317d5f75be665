"""GPU <-> oracle parity of the K/V statistics pass (Kbar, Vsum, grouped Hbar) and
of the attention kernels built on it.  Tolerances: Kbar is the bf16 rounding of
the oracle's fp64 mean (exact comparison after the same rounding); Vsum and Hbar
are fp32-accumulated and stored in bf16 (reading R-21): max abs error <= 1e-2 of
the oracle's max |value| (bf16 storage alone contributes <= 2^-8 relative)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pasa():
    from paper_2604_12219_b200 import build
    build.build()
    import paper_2604_12219_b200 as P
    return P


def _run(P, q, k, v, G, rho=0.15, Bq=128):
    B, S, H, D = q.shape
    route = P.Route(B, S, H, D, P.RouteCfg(Bq=Bq, G=G))
    bud = P.Budget()
    z = torch.zeros(64, device="cuda")
    bud(z, z, z, T=50, step=25, rho_table=[rho] * 50)
    route(q, k, bud, 7, 25)
    out = P.attn(q, k, v, route)
    torch.cuda.synchronize()
    return route, out


@pytest.mark.parametrize("S,D,G", [(4100, 128, 32), (4100, 128, 64), (4100, 128, 4096),
                                   (4100, 64, 32), (1000, 128, 32)])
def test_kv_stats_vs_oracle(pasa, S, D, G):
    q, k, v = synth.video_qkv(1, (1, 1, S), 2, D, seed=3, dtype=torch.bfloat16, device="cuda")
    route, _ = _run(pasa, q, k, v, G)
    kb, vs, ht = route.stats()
    for h in range(2):
        st = oracle.block_stats(k[0, :, h], v[0, :, h], Bk=64, G=G)
        want_kb = torch.from_numpy(st["Kbar"]).float().to(torch.bfloat16).double().numpy()
        assert np.array_equal(kb[h], want_kb)
        assert np.abs(vs[h] - st["Vsum"]).max() <= 1e-2 * np.abs(st["Vsum"]).max()
        want_ht = st["Hbar"].transpose(0, 2, 1)          # Ht[g][n][k] = Hbar[g][k][n]
        err = np.abs(ht[h] - want_ht).max() / np.abs(want_ht).max()
        assert err <= 1e-2, err


@pytest.mark.parametrize("D,G", [(128, 32), (64, 32), (64, 128), (128, 4096)])
def test_kv_stats_kernels_agree(pasa, D, G):
    """The tcgen05 statistics kernel (d = 64 with a zero-padded M = 128 operand; groups
    of more than 64 blocks in reduced chunks) and the mma.sync one (diagnostic flag
    16) agree."""
    from paper_2604_12219_b200 import _C
    q, k, v = synth.iid_qkv(1, 6000, 2, D, seed=5, dtype=torch.bfloat16, device="cuda")
    route, _ = _run(pasa, q, k, v, G)
    a = route.stats()[2]
    old = _C.lib().pasa_debug_flags(16)
    try:
        route2, _ = _run(pasa, q, k, v, G)
        b = route2.stats()[2]
    finally:
        _C.lib().pasa_debug_flags(old)
    assert np.abs(a - b).max() <= 1e-2 * np.abs(b).max()


@pytest.mark.parametrize("variant", ["default"])
@pytest.mark.parametrize("S,H,D,G,rho", [(4100, 2, 128, 32, 0.15), (4100, 2, 64, 64, 0.2),
                                         (20000, 1, 128, 128, 0.15), (1000, 2, 128, 1000, 0.11),
                                         (9000, 2, 128, 32, 0.05), (9000, 1, 64, 4096, 0.3)])
def test_variant_parity(pasa, S, H, D, G, rho, variant):
    q, k, v = synth.video_qkv(1, (1, 1, S), H, D, seed=9, dtype=torch.bfloat16, device="cuda")
    from paper_2604_12219_b200 import _C
    old = _C.lib().pasa_debug_flags(0)
    try:
        route, out = _run(pasa, q, k, v, G, rho=rho)
    finally:
        _C.lib().pasa_debug_flags(old)
    got = route.read()
    ref = oracle.attn_with_route(q, k, v, got["idx"], got["count"], Bq=128, Bk=64, G=G)
    err = np.abs(oracle.f64(out) - ref).max() / np.abs(ref).max()
    assert err <= 2e-2, err
    out2 = pasa.attn(q, k, v, route)          # default variant: same result up to rounding
    assert (out.float() - out2.float()).abs().max().item() <= 2e-2 * np.abs(ref).max()
