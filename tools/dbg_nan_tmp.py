import os, sys, torch
sys.path.insert(0, "/root/repo")
import synth, paper_2604_12219_b200 as P
cfg = synth.CONFIGS["cogvideox5b"]
B, S, H, D = cfg["B"], cfg["S"], int(os.environ.get("HEADS", cfg["H"])), cfg["D"]
q, k, v = synth.iid_qkv(B, S, H, D, seed=1, dtype=torch.bfloat16, device="cuda")
route = P.Route(B, S, H, D, P.RouteCfg(Bq=128, G=32))
bud = P.Budget(); z = torch.zeros(64, device="cuda")
bud(z, z, z, T=50, step=25, rho_table=[cfg["rho"]] * 50)
route(q, k, bud, 1, 25)
for sw in (True, False, True, False):
    out = torch.full_like(q, 7.0)
    P.attn(q, k, v, route, out, single_wg=sw)
    torch.cuda.synchronize()
    o = out.float()
    bad = ~torch.isfinite(o)
    print("single_wg" if sw else "pp", "nonfinite", int(bad.sum()), "unwritten(7.0)", int((o == 7.0).sum()))
    if bad.any():
        idx = bad.nonzero()
        print(" first", idx[:5].tolist(), " rows(t) unique", torch.unique(idx[:,1] // 128)[:20].tolist(), "heads", torch.unique(idx[:,2]).tolist()[:20])
