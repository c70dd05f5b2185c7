"""Per-phase cycle split of the level-synchronous fusion kernel (needs a
-DSSSD_LS_PROBE build: tools/build_ls_variants.sh probe -DSSSD_LS_PROBE, then
SSSD_LIB=paper_2411_05894_b200/libsssd_probe.so): cfg2 at B=64 and B=16384."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload, _lib
ds = G.build(workload.corpus(100_000_000, 32000), vocab_size=32000)
res = {}
for B in (64, 16384):
    ctx = workload.phrase_stream(B * 2048, 32000, 1)
    seq = torch.from_numpy(ctx.view(np.int32)).cuda()
    off = (torch.arange(B, dtype=torch.int64) * 2048).cuda()
    ln = torch.full((B,), 2048, dtype=torch.int32, device="cuda")
    eng = G.DraftEngine(ds, G.FusionConfig(dec_len=64))
    for _ in range(3):
        eng.propose(seq, off, ln, 2048)
    cyc = torch.zeros(B, 8, dtype=torch.int64, device="cuda")
    _lib.lib().sssd_set_cycle_probe(cyc.data_ptr())
    eng.propose(seq, off, ln, 2048)
    torch.cuda.synchronize()
    _lib.lib().sssd_set_cycle_probe(None)
    st = cyc.cpu().numpy().astype(np.float64)
    tot = st[:, 0]
    r = {"mean_kcyc": round(tot.mean() / 1e3, 2), "p50_kcyc": round(float(np.median(tot)) / 1e3, 2),
         "max_kcyc": round(tot.max() / 1e3, 2),
         "share": {k: round(float(st[:, i].sum() / tot.sum()), 3) for k, i in
                   (("gen", 1), ("sort_cls", 2), ("merge_par", 4), ("flatten", 3))},
         "levels_mean": round(float((st[:, 5].astype(np.int64) & 0xffff).mean()), 2),
         "maxlev_mean": round(float((st[:, 5].astype(np.int64) >> 16).mean()), 1),
         "gen_nodes_mean": round(float(st[:, 6].mean()), 1), "gallocs": int(st[:, 7].sum())}
    o = np.argsort(-tot)[:4]
    r["slowest"] = [{"kcyc": round(tot[i] / 1e3, 1), "gen": round(st[i, 1] / 1e3, 1), "sort": round(st[i, 2] / 1e3, 1),
                     "merge": round(st[i, 4] / 1e3, 1), "flat": round(st[i, 3] / 1e3, 1),
                     "levels": int(st[i, 5]) & 0xffff, "maxlev": int(st[i, 5]) >> 16, "gen_nodes": int(st[i, 6])}
                    for i in o]
    res[f"B{B}"] = r
print(json.dumps(res))
