"""GPU <-> oracle parity of Eq. 8's heterogeneity prior,
through the C ABI (pasa_route_v, pasa_route_het_read).

Protocol: het_j = ||H_j - C||_F within 1e-10 relative of the
oracle (both fp64; only the summation order and fma contraction differ); the
route with the prior equals the oracle's route computed with the ORACLE's het
(bit-exact idx/count/mask except documented ties: oracle scores within
1e-6 max(1, |rt|)).  Inputs: seeded synthetic tensors from ``synth``."""
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


def _budget(P, rho):
    b = P.Budget()
    z = torch.zeros(64, device="cuda")
    b(z, z, z, T=50, step=25, rho_table=[rho] * 50)
    return b


def _check(P, q, k, v, mode, G=32, rho=0.15, beta=0.1, seed=11, step=25, heads=None):
    B, S, H, D = q.shape
    cfg = P.RouteCfg(Bq=128, G=G, beta=beta, prior=mode)
    route = P.Route(B, S, H, D, cfg)
    route(q, k, _budget(P, rho), seed, step, v=v)
    got = route.read()
    het = route.het()
    kk = got["k"]
    ties = 0
    for bh in (range(B * H) if heads is None else heads):
        b, h = divmod(bh, H)
        want_het = oracle.heterogeneity(k[b, :, h], v[b, :, h], Bk=64, G=G, mode=mode)
        rel = np.abs(het[bh] - want_het).max() / np.abs(want_het).max()
        assert rel <= 1e-10, (bh, rel)
        qh, kh = q[b:b + 1, :, h:h + 1], k[b:b + 1, :, h:h + 1]
        want = oracle.route(qh, kh, Bq=128, Bk=64, beta=beta, seed=seed, step=step,
                            H_total=bh + 1, head_offset=bh, kk=kk, want_scores=True,
                            het=want_het[None, :])
        gi, wi = got["idx"][bh, :, :kk], want["idx"][0]
        for i in np.nonzero((gi != wi).any(axis=1))[0]:
            a, bb = sorted(set(gi[i]) - set(wi[i])), sorted(set(wi[i]) - set(gi[i]))
            sc = want["scores"][0, i]
            for x, y in zip(a, bb):
                assert abs(sc[x] - sc[y]) <= 1e-6 * max(1.0, abs(sc[y])), (bh, i, x, y)
                ties += 1
        if ties == 0:
            assert np.array_equal(got["mask"][bh], want["mask"][0])
    return route, got, het, ties


@pytest.mark.parametrize("S,D,mode,G,dtype", [
    (4100, 128, "global", 32, torch.bfloat16),     # ragged last block (4 tokens), last group 1 block
    (4100, 128, "group", 32, torch.bfloat16),
    (4100, 64, "global", 32, torch.bfloat16),
    (3000, 64, "group", 8, torch.float32),
    (2000, 128, "group", 4096, torch.bfloat16),    # one group: group mode == global mode
])
def test_prior_parity(pasa, S, D, mode, G, dtype):
    q, k, v = synth.video_qkv(2, (1, 1, S), 2, D, seed=5, dtype=dtype, device="cuda")
    _, _, _, ties = _check(pasa, q, k, v, mode, G=G)
    assert ties <= 2


def test_prior_changes_the_route_and_attention_runs(pasa):
    """The prior moves the selection (video data, Eq. 8 matters) and the
    resulting route drives pasa_attn with parity against the oracle."""
    S, D = 4100, 128
    q, k, v = synth.video_qkv(1, (1, 1, S), 2, D, seed=8, dtype=torch.bfloat16, device="cuda")
    route, got, _, _ = _check(pasa, q, k, v, "global", beta=0.0)
    plain = pasa.Route(1, S, 2, D, pasa.RouteCfg(Bq=128, G=32, beta=0.0))
    plain(q, k, _budget(pasa, 0.15), 11, 25)
    assert not np.array_equal(plain.read()["idx"], got["idx"])
    out = pasa.attn(q, k, v, route)
    ref = oracle.attn_with_route(q, k, v, got["idx"], got["count"], Bq=128, Bk=64, G=32)
    err = np.abs(oracle.f64(out) - ref).max() / np.abs(ref).max()
    assert err <= 2e-2, err


def test_prior_entry_points_reject_mismatched_handles(pasa):
    S, D = 1000, 64
    q, k, v = synth.iid_qkv(1, S, 1, D, seed=1, dtype=torch.bfloat16, device="cuda")
    with_prior = pasa.Route(1, S, 1, D, pasa.RouteCfg(Bq=128, prior="global"))
    with pytest.raises(pasa.PasaError):
        with_prior(q, k, _budget(pasa, 0.2), 1, 25)          # pasa_route: no V
    plain = pasa.Route(1, S, 1, D, pasa.RouteCfg(Bq=128))
    with pytest.raises(pasa.PasaError):
        plain(q, k, _budget(pasa, 0.2), 1, 25, v=v)          # pasa_route_v on a plain handle
    with pytest.raises(pasa.PasaError):
        plain.het()


def test_prior_full_size_sampled(pasa):
    """Wan 2.1-14B 720p shape (S = 75,600, d = 128), one head of the 40 checked
    against the oracle (het of all 1,182 blocks and the full route of the head)."""
    c = synth.CONFIGS["wan14b_720p"]
    S, D = c["S"], c["D"]
    H = 2
    q, k, v = synth.video_qkv(1, c["grid"], H, D, seed=3, dtype=torch.bfloat16, device="cuda")
    _, _, _, ties = _check(pasa, q, k, v, "global", rho=0.15, heads=[1])
    assert ties <= 4
