"""All-nodes vs level-synchronous fusion (sssd_set_fusion_form): bit-exact
draft comparison over the cfg2 step (B=16384) and cfg4, plus fusion-stage
times at B=16384 / 64 / 8 for both forms."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload
from paper_2411_05894_b200._lib import lib as _lib

lib = _lib()

ds = G.build(workload.corpus(100_000_000, 32000), vocab_size=32000)
res = {}


def outputs(eng, seq, off, ln, L):
    o = eng.propose(seq, off, ln, L, nodes=True)
    torch.cuda.synchronize()
    return {k: v.clone() for k, v in o.__dict__.items() if isinstance(v, torch.Tensor)}


for name, (B, L, dl, ph) in {"cfg2": (16384, 2048, 64, False), "cfg4": (64, 32768, 16, True)}.items():
    cs = workload.prompt_heavy_contexts(B, L, 32000) if ph else None
    if cs is None:
        ctx = workload.phrase_stream(B * L, 32000, 1)
    else:
        ctx = np.concatenate(cs)
    seq = torch.from_numpy(ctx.view(np.int32)).cuda()
    off = (torch.arange(B, dtype=torch.int64) * L).cuda()
    ln = torch.full((B,), L, dtype=torch.int32, device="cuda")
    eng = G.DraftEngine(ds, G.FusionConfig(dec_len=dl))
    r = {}
    outs = {}
    for form in (0, 1):
        lib.sssd_set_fusion_form(form)
        outs[form] = outputs(eng, seq, off, ln, L)
        for nb in sorted({B, 64, 8}):
            if nb > B:
                continue
            st = np.median([eng.propose_profile(seq, off[:nb], ln[:nb], L) for _ in range(9)], axis=0)
            r[f"form{form}_B{nb}_stages"] = st.round(4).tolist()
    bad = {}
    for k in outs[0]:
        a, b = outs[0][k], outs[1][k]
        if a.shape != b.shape:
            bad[k] = "shape"
            continue
        if a.dtype.is_floating_point:
            ne = ~((a == b) | (torch.isnan(a) & torch.isnan(b)))
        else:
            ne = a != b
        if ne.any():
            rows = ne.reshape(B, -1).any(1).nonzero().flatten()
            bad[k] = {"rows": int(rows.numel()), "first": rows[:5].tolist()}
    r["mismatch"] = bad
    r["bitexact"] = not bad
    res[name] = r
    lib.sssd_set_fusion_form(-1)
print(json.dumps(res))
