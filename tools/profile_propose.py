"""Run the cfg2 propose a few times (for ncu captures): 100M-token datastore,
R x 64 contexts of 2048 tokens, dec_len 64."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload

R = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ds = G.build(workload.corpus(100_000_000, 32000), vocab_size=32000)
B = R * 64
ctx = workload.phrase_stream(B * 2048, 32000, 1)
seq = torch.from_numpy(ctx.view(np.int32)).cuda()
off = (torch.arange(B, dtype=torch.int64) * 2048).cuda()
ln = torch.full((B,), 2048, dtype=torch.int32, device="cuda")
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=64))
for _ in range(reps):
    eng.propose(seq, off, ln, 2048)
torch.cuda.synchronize()
eng.check_status()
print("ok")
