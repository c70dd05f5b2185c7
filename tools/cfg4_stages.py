"""cfg4 stage times (B=8, ctx 32k prompt-heavy, dec_len 16) and per-request
fusion-kernel cycle statistics."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload, _lib
ds = G.build(workload.corpus(20_000_000, 32000), vocab_size=32000)
Bq, L = 8, 32768
for R in (1, 64):
    ctxs = workload.prompt_heavy_contexts(Bq * R, L, 32000)
    seq = torch.from_numpy(np.concatenate(ctxs).astype(np.uint32).view(np.int32)).cuda()
    off = (torch.arange(Bq * R, dtype=torch.int64) * L).cuda()
    ln = torch.full((Bq * R,), L, dtype=torch.int32, device="cuda")
    eng = G.DraftEngine(ds, G.FusionConfig(dec_len=16))
    eng.propose(seq, off, ln, L)
    ms = np.median([eng.propose_profile(seq, off, ln, L) for _ in range(7)], 0)
    print("B", Bq * R, "stage ms (lookup, scan, setup, fusion)", np.round(ms, 4).tolist())
    cyc = torch.zeros(Bq * R, 8, dtype=torch.int64, device="cuda")
    _lib.lib().sssd_set_cycle_probe(cyc.data_ptr())
    eng.propose(seq, off, ln, L)
    torch.cuda.synchronize()
    _lib.lib().sssd_set_cycle_probe(None)
    c = cyc.cpu().numpy()
    print("  fusion us/request mean %.1f max %.1f flatten %.1f levels %.1f maxlevel mean %.0f max %d gen %.0f gallocs %.2f" % (
        c[:, 0].mean() / 1965, c[:, 0].max() / 1965, c[:, 3].mean() / 1965, (c[:, 5] & 0xffff).mean(),
        (c[:, 5] >> 16).mean(), (c[:, 5] >> 16).max(), c[:, 6].mean(), c[:, 7].mean()))
    ctx_np = np.stack(ctxs[:Bq])
    occ = (ctx_np[:, :-1] == ctx_np[:, -1:]).sum(1)
    print("  occurrences of the last token (first 8):", occ.tolist())
