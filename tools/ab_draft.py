"""A/B of fusion-kernel builds (SSSD_LIB=...): draft-kernel ms at B=16384 and
B=64 (cfg2 workload) plus per-request latency percentiles."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload, _lib
ds = G.build(workload.corpus(100_000_000, 32000), vocab_size=32000)
B = 16384
ctx = workload.phrase_stream(B * 2048, 32000, 1)
seq = torch.from_numpy(ctx.view(np.int32)).cuda()
off = (torch.arange(B, dtype=torch.int64) * 2048).cuda()
ln = torch.full((B,), 2048, dtype=torch.int32, device="cuda")
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=64))
eng.propose(seq, off, ln, 2048)
full = np.median([eng.propose_profile(seq, off, ln, 2048) for _ in range(5)], axis=0)
b64 = np.median([eng.propose_profile(seq, off[:64], ln[:64], 2048) for _ in range(21)], axis=0)
cyc = torch.zeros(B, 8, dtype=torch.int64, device="cuda")
_lib.lib().sssd_set_cycle_probe(cyc.data_ptr())
eng.propose(seq, off, ln, 2048)
torch.cuda.synchronize()
_lib.lib().sssd_set_cycle_probe(None)
st = cyc.cpu().numpy()
c = st[:, 0] / 1.965e3
pp = 0.0
ph = " ".join("%s %.1f" % (nm, (st[:, k] / 1.965e3).mean()) for k, nm in ((1, "gen"), (2, "sort+cls"), (4, "merge+par"), (3, "flat")))
ph += " levels %.2f maxlev %.1f gen %.1f gallocs %.3f" % ((st[:, 5] & 0xffff).mean(), (st[:, 5] >> 16).mean(), st[:, 6].mean(), st[:, 7].mean())
print(os.path.basename(os.environ.get("SSSD_LIB", "default")), "B16384 stage ms", np.round(full, 3).tolist(),
      "B64 stage ms", np.round(b64, 3).tolist(),
      "req us mean %.0f p50 %.0f p99 %.0f max %.0f" % (c.mean(), *np.percentile(c, [50, 99]), c.max()),
      "| LS phases us:", ph)
