"""N2 at the cfg2 shape: input-scan stage ms stateless vs with the per-request
index (16,384 x 2048-token contexts, 100M datastore)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload
ds = G.build(workload.corpus(100_000_000, 32000), vocab_size=32000)
B, CTX = 16384, 2048
ctx = workload.phrase_stream(B * CTX, 32000, 1)
seq = torch.from_numpy(ctx.view(np.int32)).cuda()
off = (torch.arange(B, dtype=torch.int64) * CTX).cuda()
ln = torch.full((B,), CTX, dtype=torch.int32, device="cuda")
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=64))
ix = G.InputIndex(B, CTX, "cuda", off)
ix.build(seq, off, ln)
a = np.median([eng.propose_profile(seq, off, ln, CTX) for _ in range(5)], axis=0)
b = np.median([eng.propose_profile(seq, off, ln, CTX, index=ix) for _ in range(5)], axis=0)
print(json.dumps({"stateless_ms": a.round(4).tolist(), "indexed_ms": b.round(4).tolist()}))
