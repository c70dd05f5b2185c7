"""Distribution of per-request fusion-kernel cycles (cfg2 workload) and the
time of the same batch at 1x / 2x / 4x wave counts."""
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
cyc = torch.zeros(B, 8, dtype=torch.int64, device="cuda")
eng.propose(seq, off, ln, 2048)
_lib.lib().sssd_set_cycle_probe(cyc.data_ptr())
eng.propose(seq, off, ln, 2048)
torch.cuda.synchronize()
_lib.lib().sssd_set_cycle_probe(None)
st = cyc.cpu().numpy()
c = st[:, 0] / 1.965e3  # us at 1965 MHz
names = ["total_us", "seed_us", "loop_us", "flatten_us", "pops", "scanned", "max_live", "spill"]
conv = [1.965e3] * 4 + [1] * 4
for k, (nm, cv) in enumerate(zip(names, conv)):
    x = st[:, k] / cv
    print("%-10s mean %9.1f p50 %9.1f p99 %9.1f max %9.1f corr(total) %.3f" % (
        nm, x.mean(), *np.percentile(x, [50, 99]), x.max(), np.corrcoef(x, c)[0, 1]))
slow = np.argsort(-c)[:12]
print("slowest requests (total_us seed_us loop_us flat_us pops scanned max_live spill):")
for i in slow:
    print(" ", [round(float(st[i, k] / conv[k]), 1) for k in range(8)])
print("per-pop loop us: mean %.2f" % (st[:, 2] / 1.965e3 / np.maximum(st[:, 4], 1)).mean())
print("per-request us: mean %.1f p50 %.1f p90 %.1f p99 %.1f max %.1f" % (c.mean(), *np.percentile(c, [50, 90, 99]), c.max()))
for n in (4736, 9472, 16384):
    ms = eng.propose_profile(seq, off[:n], ln[:n], 2048)
    print(n, "requests: draft ms %.3f" % ms[3])
# correlation of per-request cycles with element counts (the LPT proxy)
from paper_2411_05894_b200._lib import lib, ptr
out = eng.propose(seq, off, ln, 2048, lookup=True)
torch.cuda.synchronize()
ws = eng._ws
import ctypes
# re-derive per-request counts from the lookup diagnostics and the input scan
nds = out.n_conts.clamp(min=0).sum(1).cpu().numpy()
tl = ctx.reshape(B, 2048)
last = tl[:, -1:]
nin = (tl[:, :-1] == last).sum(1)
cc = c
for name, x in (("n_ds(all p)", nds), ("n_in", nin), ("n_ds+4n_in", nds + 4 * nin)):
    print(name, "corr %.3f" % np.corrcoef(x, cc)[0, 1])
hi = np.argsort(-cc)[:10]
print("slowest: us", np.round(cc[hi], 0).tolist(), "n_in", nin[hi].tolist(), "n_ds", nds[hi].tolist())
