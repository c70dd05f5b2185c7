import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload, _lib
ds = G.build(workload.corpus(100_000_000, 32000), vocab_size=32000)
B = 64
ctx = workload.phrase_stream(B * 2048, 32000, 1)
seq = torch.from_numpy(ctx.view(np.int32)).cuda()
off = (torch.arange(B, dtype=torch.int64) * 2048).cuda()
ln = torch.full((B,), 2048, dtype=torch.int32, device="cuda")
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=64))
for _ in range(3): eng.propose(seq, off, ln, 2048)
cyc = torch.zeros(B, 8, dtype=torch.int64, device="cuda")
_lib.lib().sssd_set_cycle_probe(cyc.data_ptr())
eng.propose(seq, off, ln, 2048); torch.cuda.synchronize()
_lib.lib().sssd_set_cycle_probe(None)
st = cyc.cpu().numpy(); us = st / 1.965e3
tot = us[:, 0]
o = np.argsort(-tot)
print("B64 per-request fusion us: mean %.1f p50 %.1f max %.1f" % (tot.mean(), np.median(tot), tot.max()))
print("phase means us: gen %.1f sort+cls %.1f merge+par %.1f flat %.1f" % (us[:,1].mean(), us[:,2].mean(), us[:,4].mean(), us[:,3].mean()))
for i in o[:6]:
    print("slow req", i, "tot %.1f gen %.1f sort %.1f merge %.1f flat %.1f levels %d maxlev %d gen_nodes %d gallocs %d" % (tot[i], us[i,1], us[i,2], us[i,4], us[i,3], st[i,5] & 0xffff, st[i,5] >> 16, st[i,6], st[i,7]))
print("stage ms", np.median([eng.propose_profile(seq, off, ln, 2048) for _ in range(21)], axis=0).round(4).tolist())
