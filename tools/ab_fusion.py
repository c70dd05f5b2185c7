"""A/B of the two fusion kernels on the cfg2 workload (100M phrase datastore,
16,384 x 2048-token contexts, dec_len 64): stage times and per-request cycle
statistics of each (SSSD_FUSION=heap|ls)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload, _lib
n_tok = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
ds = G.build(workload.corpus(n_tok, 32000), vocab_size=32000)
B = 16384
ctx = workload.phrase_stream(B * 2048, 32000, 1)
seq = torch.from_numpy(ctx.view(np.int32)).cuda()
off = (torch.arange(B, dtype=torch.int64) * 2048).cuda()
ln = torch.full((B,), 2048, dtype=torch.int32, device="cuda")
res = {}
for mode in ("heap", "ls"):
    os.environ["SSSD_FUSION"] = mode
    eng = G.DraftEngine(ds, G.FusionConfig(dec_len=64))
    for _ in range(3):
        out = eng.propose(seq, off, ln, 2048)
    torch.cuda.synchronize()
    eng.check_status()
    res[mode] = {k: getattr(out, k).clone() for k in ("size", "tokens", "parents", "depths", "mask")}
    ms = np.array([eng.propose_profile(seq, off, ln, 2048) for _ in range(5)])
    print(mode, "stage ms (lookup, scan, setup, fusion):", np.round(np.median(ms, 0), 4).tolist())
    st = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st[0].record()
    for _ in range(10):
        eng.propose(seq, off, ln, 2048)
    st[1].record()
    torch.cuda.synchronize()
    print(mode, "overlapped propose ms/step %.4f" % (st[0].elapsed_time(st[1]) / 10))
    cyc = torch.zeros(B, 8, dtype=torch.int64, device="cuda")
    _lib.lib().sssd_set_cycle_probe(cyc.data_ptr())
    eng.propose(seq, off, ln, 2048)
    torch.cuda.synchronize()
    _lib.lib().sssd_set_cycle_probe(None)
    c = cyc.cpu().numpy()
    for k, nm in enumerate(["total_us", "seed_us", "loop_us", "flatten_us"]):
        x = c[:, k] / 1.965e3
        print("  %-10s mean %8.2f p50 %8.2f p99 %8.2f max %8.2f" % (nm, x.mean(), *np.percentile(x, [50, 99]), x.max()))
    for k, nm in enumerate(["pops|levels", "scanned|generated", "max_live|max_level", "spill|gallocs"]):
        x = c[:, 4 + k]
        print("  %-20s mean %8.1f p50 %6.0f p99 %6.0f max %6.0f" % (nm, x.mean(), *np.percentile(x, [50, 99]), x.max()))
same = all(torch.equal(res["heap"][k], res["ls"][k]) for k in res["heap"])
print("drafts identical:", same)
