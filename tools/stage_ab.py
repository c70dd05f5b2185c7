"""A/B of library builds (SSSD_LIB=...): cfg2 stage times at B=16384 and B=64."""
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
eng.propose(seq, off, ln, 2048)
full = np.median([eng.propose_profile(seq, off, ln, 2048) for _ in range(7)], axis=0)
b64 = np.median([eng.propose_profile(seq, off[:64], ln[:64], 2048) for _ in range(21)], axis=0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(10):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); eng.propose(seq, off, ln, 2048); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
out = eng.propose(seq, off, ln, 2048)
dig = int((out.tokens.long() * 1000003 + out.parents.long()).sum().item() % (1 << 61))
print(os.path.basename(os.environ.get("SSSD_LIB", "default")), json.dumps({"step_ms": round(float(np.median(ts)), 4),
      "stages16k": full.round(4).tolist(), "stages64": b64.round(4).tolist(), "digest": dig}))
