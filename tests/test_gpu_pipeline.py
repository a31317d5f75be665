"""Host-resident inputs through paper_2604_12219_b200.pipeline.HostPipeline (head
chunks, copy-in / compute / copy-out streams, pasa_copy2d): the output equals the
single-shot device call bit for bit (every head is independent and the route is
keyed by the global head, R-11 / R-20), for uneven chunkings too."""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_chunks", [1, 3, 4])
def test_pipeline_matches_device_call_bitwise(n_chunks):
    from paper_2604_12219_b200 import build
    build.build()
    import paper_2604_12219_b200 as P
    from paper_2604_12219_b200.pipeline import HostPipeline
    B, S, H, D = 1, 8200, 6, 128
    q, k, v = synth.video_qkv(B, (2, 50, 82), H, D, seed=4, dtype=torch.bfloat16, device="cuda")
    tp = synth.ThreePhase(shape=(16, 4, 12, 16), T=50, seed=1, device="cuda")
    xs = [x.contiguous() for x in tp.latents(25)]
    kw = dict(T=50, rho=0.15, l1_mean=tp.expected_l1_mean(), h_t=0.02, h_tm1=0.02)
    cfg = P.RouteCfg(Bq=128, G=32)
    # single-shot device reference
    bud = P.Budget()
    bud(*xs, step=25, **kw)
    route = P.Route(B, S, H, D, cfg)
    route(q, k, bud, 99, 25)
    ref = P.attn(q, k, v, route)
    # host pipeline
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    hx = [x.cpu().pin_memory() for x in xs]
    hout = torch.empty(ref.shape, dtype=ref.dtype, pin_memory=True)
    pipe = HostPipeline(B, S, H, D, cfg, n_chunks=n_chunks)
    pipe(hq, hk, hv, hout, hx, 99, 25, **kw)
    torch.cuda.synchronize()
    assert torch.equal(hout, ref.cpu())
    assert pipe.h2d_bytes == 3 * q.numel() * 2 + sum(x.numel() * 4 for x in xs)
    assert pipe.d2h_bytes == ref.numel() * 2


def test_pipeline_d64_with_prior_bitwise():
    """d = 64, the Eq. 8 prior (pasa_route_v per chunk), B = 2, uneven head chunks."""
    from paper_2604_12219_b200 import build
    build.build()
    import paper_2604_12219_b200 as P
    from paper_2604_12219_b200.pipeline import HostPipeline
    B, S, H, D = 2, 4100, 5, 64
    q, k, v = synth.video_qkv(B, (1, 1, S), H, D, seed=6, dtype=torch.bfloat16, device="cuda")
    tp = synth.ThreePhase(shape=(16, 4, 12, 16), T=50, seed=2, device="cuda")
    xs = [x.contiguous() for x in tp.latents(30)]
    kw = dict(T=50, rho=0.15, l1_mean=tp.expected_l1_mean(), h_t=0.02, h_tm1=0.02)
    cfg = P.RouteCfg(Bq=128, G=32, prior="global")
    bud = P.Budget()
    bud(*xs, step=30, **kw)
    route = P.Route(B, S, H, D, cfg)
    route(q, k, bud, 5, 30, v=v)
    ref = P.attn(q, k, v, route)
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    hx = [x.cpu().pin_memory() for x in xs]
    hout = torch.empty(ref.shape, dtype=ref.dtype, pin_memory=True)
    pipe = HostPipeline(B, S, H, D, cfg, n_chunks=2)
    pipe(hq, hk, hv, hout, hx, 5, 30, v_for_prior=True, **kw)
    torch.cuda.synchronize()
    assert torch.equal(hout, ref.cpu())
