"""Small-batch propose latency (cfg2 B=64, cfg4 B=8) and the stage split."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload
ds = G.build(workload.corpus(100_000_000, 32000), vocab_size=32000)
res = {}
for name, (B, L, dl, ctxs) in {"cfg2_b64": (64, 2048, 64, None), "cfg4_b8": (8, 32768, 16, "ph")}.items():
    cs = workload.prompt_heavy_contexts(B, L, 32000) if ctxs else workload.contexts(B, L, 32000)
    seq = torch.from_numpy(np.concatenate(cs).view(np.int32)).cuda()
    off = (torch.arange(B, dtype=torch.int64) * L).cuda()
    ln = torch.full((B,), L, dtype=torch.int32, device="cuda")
    eng = G.DraftEngine(ds, G.FusionConfig(dec_len=dl))
    for _ in range(3):
        eng.propose(seq, off, ln, L)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(21):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); eng.propose(seq, off, ln, L); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    st = np.median([eng.propose_profile(seq, off, ln, L) for _ in range(11)], axis=0)
    res[name] = {"latency_ms": round(float(np.median(ts)), 4), "stages_ms": st.round(4).tolist()}
print(json.dumps(res))
