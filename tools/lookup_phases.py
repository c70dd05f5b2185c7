"""Per-phase cycle split of ds_lookup_warp_kernel (measurement build with
-DSSSD_LK_PROBE exporting sssd_set_lookup_probe; SSSD_LIB=that .so):
search / gather / merge-rank / fold+columns, cfg2 at B=64 and B=16384."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload, _lib
ds = G.build(workload.corpus(100_000_000, 32000), vocab_size=32000)
L = _lib.lib()
L.sssd_set_lookup_probe.argtypes = [C.c_void_p]
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
    L.sssd_set_lookup_probe(cyc.data_ptr())
    eng.propose(seq, off, ln, 2048)
    torch.cuda.synchronize()
    L.sssd_set_lookup_probe(None)
    st = cyc.cpu().numpy().astype(np.float64)
    ph = np.diff(np.concatenate([np.zeros((B, 1)), st[:, :4]], axis=1), axis=1)
    tot = st[:, 3]
    res[f"B{B}"] = {"mean_kcyc": round(tot.mean() / 1e3, 2), "max_kcyc": round(tot.max() / 1e3, 2),
                    "share": dict(zip(("search", "gather", "merge_rank", "fold_cols"),
                                      (ph.sum(0) / tot.sum()).round(3).tolist())),
                    "n_all_mean": round(float(st[:, 4].mean()), 1), "runs_mean": round(float(st[:, 5].mean()), 2),
                    "runs_hist": np.bincount(st[:, 5].astype(int).clip(0, 8)).tolist(),
                    "n_out_mean": round(float(st[:, 6].mean()), 1)}
print(json.dumps(res))
