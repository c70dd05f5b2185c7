"""simulate() wall clock on a teacher-forced decode loop (1,024 records, prompt
512, reference 256, 256 slots, 10M-token datastore, dec_len 32)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload
ds = G.build(workload.corpus(10_000_000, 32000), vocab_size=32000)
recs = [G.SimRecord(p, r) for p, r in workload.records(1024, 512, 256, 32000)]
cfg = G.FusionConfig(dec_len=32)
G.simulate(recs[:256], ds, cfg, slots=256)
torch.cuda.synchronize()
t = time.perf_counter()
rep = G.simulate(recs, ds, cfg, slots=256)
torch.cuda.synchronize()
dt = time.perf_counter() - t
tok = sum(r.tokens_emitted for r in rep.records)
print({"wall_s": round(dt, 4), "tokens_per_s": round(tok / dt), "mean_accepted": round(rep.mean_accepted_per_step, 4),
       "digest": hash(tuple(tuple(r.per_step_tokens) for r in rep.records)) & 0xffffffff})
