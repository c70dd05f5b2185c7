"""CTA-per-request fusion (form 2) vs one warp per request (form 0): small-batch
propose latency (cfg2 B=64 and B=8..512, cfg4 B=8), fusion stage ms, and
bit-identical drafts.  Usage: python tools/cta_ab.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload
from paper_2411_05894_b200._lib import lib
ds = G.build(workload.corpus(100_000_000, 32000), vocab_size=32000)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def lat(eng, seq, off, ln, L, reps=21):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); eng.propose(seq, off, ln, L); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


res = {}
shapes = [("cfg2_b%d" % B, B, 2048, 64, False) for B in (8, 64, 256, 512, 2048)] + [("cfg4_b8", 8, 32768, 16, True)]
for name, B, L, dl, ph in shapes:
    cs = workload.prompt_heavy_contexts(B, L, 32000) if ph else workload.contexts(B, L, 32000)
    seq = torch.from_numpy(np.concatenate(cs).view(np.int32)).cuda()
    off = (torch.arange(B, dtype=torch.int64) * L).cuda()
    ln = torch.full((B,), L, dtype=torch.int32, device="cuda")
    eng = G.DraftEngine(ds, G.FusionConfig(dec_len=dl))
    row = {}
    outs = {}
    for form in (0, 2):
        lib().sssd_set_fusion_form(form)
        for _ in range(3):
            eng.propose(seq, off, ln, L)
        o = eng.propose(seq, off, ln, L, nodes=True)
        eng.check_status()
        torch.cuda.synchronize()
        outs[form] = {k: v.clone() for k, v in o.__dict__.items() if isinstance(v, torch.Tensor)}
        st = np.median([eng.propose_profile(seq, off, ln, L) for _ in range(11)], axis=0)
        row["form%d" % form] = {"latency_ms": round(lat(eng, seq, off, ln, L), 4), "stages_ms": st.round(4).tolist()}
    same = all(bool(((outs[0][k] == outs[2][k]) | (torch.isnan(outs[0][k]) & torch.isnan(outs[2][k]))).all())
               if outs[0][k].dtype.is_floating_point else torch.equal(outs[0][k], outs[2][k]) for k in outs[0])
    row["equal"] = same
    res[name] = row
    print(name, json.dumps(row), flush=True)
lib().sssd_set_fusion_form(-1)
print(json.dumps(res))
