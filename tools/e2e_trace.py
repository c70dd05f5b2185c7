"""Stream timeline of one propose_pinned call (cfg2 e2e workload, u16
uploads): every kernel / copy with start and duration (us), for schedule
A/B:  python tools/e2e_trace.py [phased|ranges] [chunks]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload

schedule = sys.argv[1] if len(sys.argv) > 1 else "phased"
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 5
B, CTX, V = 16384, 2048, 32000
ds = G.build(workload.corpus(20_000_000, V), vocab_size=V)
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=64))
stream = workload.phrase_stream(B * CTX, V, workload.HELDOUT_SEED)
ctx16_h = torch.from_numpy(stream.astype(np.uint16).view(np.int16)).pin_memory()
off_h = torch.arange(B, dtype=torch.int64).pin_memory() * CTX
len_h = torch.full((B,), CTX, dtype=torch.int32).pin_memory()
out_h = eng.propose_pinned(ctx16_h, off_h, len_h, CTX, chunks=chunks, schedule=schedule)
for _ in range(2):
    eng.propose_pinned(ctx16_h, off_h, len_h, CTX, out_h=out_h, chunks=chunks, schedule=schedule)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eng.propose_pinned(ctx16_h, off_h, len_h, CTX, out_h=out_h, chunks=chunks, schedule=schedule)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in ev)
for e in sorted(ev, key=lambda e: e.time_range.start):
    print("%8.1f %7.1f %s" % (e.time_range.start - t0, e.time_range.end - e.time_range.start, e.name[:60]))
