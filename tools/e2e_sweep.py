"""Sweep propose_pinned's request-range schedule (chunks, taper, tail) on the
cfg2 e2e workload (16,384 lookups, ctx 2048, u16 uploads): median device ms."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload

B, CTX, V = 16384, 2048, 32000
ds = G.build(workload.corpus(20_000_000, V), vocab_size=V)
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=64))
stream = workload.phrase_stream(B * CTX, V, workload.HELDOUT_SEED)
ctx16_h = torch.from_numpy(stream.astype(np.uint16).view(np.int16)).pin_memory()
off_h = torch.arange(B, dtype=torch.int64).pin_memory() * CTX
len_h = torch.full((B,), CTX, dtype=torch.int32).pin_memory()
st = torch.cuda.current_stream()
out_h = eng.propose_pinned(ctx16_h, off_h, len_h, CTX)


def timed(**kw):
    eng.propose_pinned(ctx16_h, off_h, len_h, CTX, out_h=out_h, **kw)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(st)
        eng.propose_pinned(ctx16_h, off_h, len_h, CTX, out_h=out_h, **kw)
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return round(float(np.median(ts)), 3)


sweep = [dict(chunks=5), dict(chunks=4), dict(chunks=6), dict(chunks=5, tail=0.6), dict(chunks=5, tail=0.4),
         dict(chunks=6, tail=0.5), dict(chunks=6, tail=0.3), dict(chunks=4, tail=0.5), dict(chunks=7, tail=0.5),
         dict(chunks=5, schedule="ranges")]
for kw in sweep:
    print(kw, timed(**kw), flush=True)
