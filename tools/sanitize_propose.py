"""Small propose + merge + decode workload for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload
corpus = workload.corpus(200_000, 500)
ds = G.build(corpus, vocab_size=500)
rng = np.random.default_rng(0)
for cfg in (G.FusionConfig(dec_len=64), G.FusionConfig(dec_len=16, P=8, input_branch_len=12)):
    eng = G.DraftEngine(ds, cfg)
    ctxs = [rng.integers(0, 500, int(rng.integers(1, 3000))).tolist() for _ in range(40)]
    eng.propose_host(ctxs)
    # throughput path (>= 2048 requests -> warp lookup, LPT order)
    B, L = 2048, 256
    seq = torch.from_numpy(workload.phrase_stream(B * L, 500, 1).view(np.int32)).cuda()
    off = (torch.arange(B, dtype=torch.int64) * L).cuda()
    ln = torch.full((B,), L, dtype=torch.int32, device="cuda")
    eng.propose(seq, off, ln, L)
    eng.check_status()
sep = G.DraftEngine(ds, G.FusionConfig(dec_len=32), separator=7)
sep.propose_host([rng.integers(0, 500, 300).tolist() for _ in range(16)])
recs = workload.records(16, 128, 32, 500)
G.simulate([G.SimRecord(p, r) for p, r in recs], ds, G.FusionConfig(dec_len=16), slots=8)
torch.cuda.synchronize()
print("sanitize workload ok")
