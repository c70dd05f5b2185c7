"""Host time to enqueue one async propose_pinned (phased, 5 ranges) vs its device time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload
B, CTX, V = 16384, 2048, 32000
ds = G.build(workload.corpus(20_000_000, V), vocab_size=V)
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=64))
ctx16_h = torch.from_numpy(workload.phrase_stream(B * CTX, V, 1).astype(np.uint16).view(np.int16)).pin_memory()
off_h = torch.arange(B, dtype=torch.int64).pin_memory() * CTX
len_h = torch.full((B,), CTX, dtype=torch.int32).pin_memory()
outs = [eng.propose_pinned(ctx16_h, off_h, len_h, CTX, slot=k) for k in range(2)]
torch.cuda.synchronize()
ts = []
for i in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = eng.propose_pinned(ctx16_h, off_h, len_h, CTX, out_h=outs[i & 1], slot=i & 1, sync=False)
    ts.append((time.perf_counter() - t0) * 1e3)
    p.wait()
print("host enqueue ms per call: median %.3f min %.3f" % (np.median(ts), min(ts)), "cpus", os.cpu_count())
