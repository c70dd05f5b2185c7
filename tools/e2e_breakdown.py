"""Break down the e2e propose_pinned step: pure H2D of the contexts, pure
resident propose, and the pipelined call at several chunk counts (device ms)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload

B, CTX, V = 16384, 2048, 32000
corpus = workload.corpus(20_000_000, V)
ds = G.build(corpus, vocab_size=V)
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=64))
stream = workload.phrase_stream(B * CTX, V, workload.HELDOUT_SEED)
ctx_h = torch.from_numpy(stream.view(np.int32)).pin_memory()
ctx16_h = torch.from_numpy(stream.astype(np.uint16).view(np.int16)).pin_memory()
seq = ctx_h.cuda()
seq16 = ctx16_h.cuda()
off_h = torch.arange(B, dtype=torch.int64) * CTX
len_h = torch.full((B,), CTX, dtype=torch.int32)
off, ln = off_h.cuda(), len_h.cuda()
st = torch.cuda.current_stream()


def timed(fn, n=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        t0 = time.perf_counter()
        a.record(st); fn(); b.record(st); torch.cuda.synchronize()
        ts.append((a.elapsed_time(b), (time.perf_counter() - t0) * 1e3))
    return np.median([t[0] for t in ts]), np.median([t[1] for t in ts])


print("h2d 134MB", timed(lambda: seq.copy_(ctx_h, non_blocking=True)))
print("h2d 67MB u16", timed(lambda: seq16.copy_(ctx16_h, non_blocking=True)))
print("propose resident", timed(lambda: eng.propose(seq, off, ln, CTX)))
out_h = eng.propose_pinned(ctx_h, off_h, len_h, CTX)  # pinned outputs reused below
for c in (6,):
    print("pinned chunks", c, timed(lambda: eng.propose_pinned(ctx_h, off_h, len_h, CTX, out_h=out_h, chunks=c)))
for c in (4, 5, 6):
    for tl in (None, 0.5, 0.3, 0.15):
        print("pinned u16 chunks", c, "tail", tl, timed(lambda: eng.propose_pinned(ctx16_h, off_h, len_h, CTX, out_h=out_h, chunks=c, tail=tl)))

# stream timeline of the pipelined call (chrome trace -> gpurun_out/)
from torch.profiler import ProfilerActivity, profile
out_h = eng.propose_pinned(ctx_h, off_h, len_h, CTX, chunks=4)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for c in (4,):
        eng.propose_pinned(ctx16_h, off_h, len_h, CTX, out_h=out_h, chunks=c)
        torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
