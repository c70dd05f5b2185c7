"""cfg2 propose step timed after a write flush of L2 (the bench's method) and
after a write flush followed by a read of a second 256 MB buffer (L2 then holds
clean lines): the difference is what the flush's dirty write-backs cost the
timed step."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload
ds = G.build(workload.corpus(100_000_000, 32000), vocab_size=32000)
B = 16384
ctx = workload.phrase_stream(B * 2048, 32000, 1)
seq = torch.from_numpy(ctx.view(np.int32)).cuda()
off = (torch.arange(B, dtype=torch.int64) * 2048).cuda()
ln = torch.full((B,), 2048, dtype=torch.int32, device="cuda")
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=64))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(3):
    eng.propose(seq, off, ln, 2048)
res = {}
for mode in ("write", "write+read", "write", "write+read"):
    ts = []
    for _ in range(20):
        flush.zero_()
        if mode == "write+read":
            clean.sum()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); eng.propose(seq, off, ln, 2048); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    res.setdefault(mode, []).append(round(float(np.median(ts)), 4))
print(json.dumps(res))
