"""Per-request fusion cycle split (sssd_set_cycle_probe) for one fusion form at
cfg2 B=64 and cfg4 B=8.  Usage: python tools/cta_probe.py [form ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload
from paper_2411_05894_b200._lib import lib
ds = G.build(workload.corpus(100_000_000, 32000), vocab_size=32000)
forms = [int(x) for x in sys.argv[1:]] or [0, 2]
for name, B, L, dl, ph in (("cfg2_b64", 64, 2048, 64, False), ("cfg4_b8", 8, 32768, 16, True)):
    cs = workload.prompt_heavy_contexts(B, L, 32000) if ph else workload.contexts(B, L, 32000)
    seq = torch.from_numpy(np.concatenate(cs).view(np.int32)).cuda()
    off = (torch.arange(B, dtype=torch.int64) * L).cuda()
    ln = torch.full((B,), L, dtype=torch.int32, device="cuda")
    eng = G.DraftEngine(ds, G.FusionConfig(dec_len=dl))
    for form in forms:
        lib().sssd_set_fusion_form(form)
        for _ in range(3):
            eng.propose(seq, off, ln, L)
        cyc = torch.zeros(B, 8, dtype=torch.int64, device="cuda")
        lib().sssd_set_cycle_probe(cyc.data_ptr())
        eng.propose(seq, off, ln, L)
        torch.cuda.synchronize()
        lib().sssd_set_cycle_probe(None)
        st = cyc.cpu().numpy()
        us = st / 1.965e3
        o = np.argsort(-us[:, 0])
        print("%s form %d: fusion us mean %.1f max %.1f | phase means gen %.1f sort+cls %.1f (cls %.1f) merge+par %.1f flat %.1f"
              % (name, form, us[:, 0].mean(), us[:, 0].max(), us[:, 1].mean(), us[:, 2].mean(),
                 us[:, 7].mean() if form == 2 else -1, us[:, 4].mean(), us[:, 3].mean()))
        for i in o[:3]:
            print("   slow req %d: tot %.1f gen %.1f sort+cls %.1f merge+par %.1f flat %.1f levels %d maxlev %d gen_nodes %d"
                  % (i, us[i, 0], us[i, 1], us[i, 2], us[i, 4], us[i, 3], st[i, 5] & 0xffff, st[i, 5] >> 16, st[i, 6]))
lib().sssd_set_fusion_form(-1)
