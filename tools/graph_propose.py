"""Eager propose vs the same propose replayed from a CUDA graph (cfg2 step:
16,384 lookups, and one B=64 batch; L2 flushed between steps): device ms per
step.  Usage: python tools/graph_propose.py [B]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload
ds = G.build(workload.corpus(100_000_000, 32000), vocab_size=32000)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
seq = torch.from_numpy(workload.phrase_stream(B * 2048, 32000, 1).view(np.int32)).cuda()
off = (torch.arange(B, dtype=torch.int64) * 2048).cuda()
ln = torch.full((B,), 2048, dtype=torch.int32, device="cuda")
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=64))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = eng.propose(seq, off, ln, 2048)
ref = out.tokens.clone()
st = torch.cuda.current_stream()


def timed(fn, n=20):
    ts = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(st); fn(); b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return round(float(np.median(ts)), 4)


print("eager", timed(lambda: eng.propose(seq, off, ln, 2048, out=out)))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    eng.propose(seq, off, ln, 2048, out=out)
g.replay(); torch.cuda.synchronize()
assert torch.equal(out.tokens, ref)
print("graph", timed(g.replay))
print("eager", timed(lambda: eng.propose(seq, off, ln, 2048, out=out)))
