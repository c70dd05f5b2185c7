"""One cfg4 propose (B=8, ctx 32k prompt-heavy, dec_len 16) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload
ds = G.build(workload.corpus(20_000_000, 32000), vocab_size=32000)
B, L = 8, 32768
ctxs = workload.prompt_heavy_contexts(B, L, 32000)
seq = torch.from_numpy(np.concatenate(ctxs).astype(np.uint32).view(np.int32)).cuda()
off = (torch.arange(B, dtype=torch.int64) * L).cuda()
ln = torch.full((B,), L, dtype=torch.int32, device="cuda")
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=16))
for _ in range(3):
    eng.propose(seq, off, ln, L)
torch.cuda.synchronize()
