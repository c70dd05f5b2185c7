"""Fusion-kernel occupancy over time at cfg2 (16,384 requests): per-request
%globaltimer start / end stamps from a -DSSSD_LS_TIMELINE build (SSSD_LIB=...):
how long the tail runs with the GPU partly idle, and how well the LPT order
(cost = datastore + 4 x input elements) predicts per-request time."""
import json, os, sys
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
for _ in range(3):
    eng.propose(seq, off, ln, 2048)
cyc = torch.zeros(B, 8, dtype=torch.int64, device="cuda")
_lib.lib().sssd_set_cycle_probe(cyc.data_ptr())
eng.propose(seq, off, ln, 2048)
torch.cuda.synchronize()
_lib.lib().sssd_set_cycle_probe(None)
st = cyc.cpu().numpy()
t0 = st[:, 6].min()
s = (st[:, 6] - t0) / 1e3  # us
e = (st[:, 7] - t0) / 1e3
T = e.max()
grid = np.linspace(0, T, 400)
act = np.array([((s <= g) & (e > g)).sum() for g in grid])
cap = act.max()
res = {"kernel_us": round(float(T), 1), "max_active": int(cap),
       "busy_us_sum": round(float((e - s).sum()), 0),
       "ideal_us_at_max_active": round(float((e - s).sum() / cap), 1),
       "time_below_90pct_active_us": round(float(T * (act < 0.9 * cap).mean()), 1),
       "time_below_50pct_active_us": round(float(T * (act < 0.5 * cap).mean()), 1),
       "last_start_us": round(float(s.max()), 1),
       "per_request_us": {"mean": round(float((e - s).mean()), 1), "p99": round(float(np.percentile(e - s, 99)), 1),
                          "max": round(float((e - s).max()), 1)},
       "active_profile": act[::20].tolist()}
print(json.dumps(res))

# how well does the LPT cost (datastore + 4 x input elements) predict the time?
out = eng.propose(seq, off, ln, 2048, lookup=True)
torch.cuda.synchronize()
nds = out.n_conts.clamp(min=0).sum(1).cpu().numpy().astype(np.float64)  # raw datastore strings
tl = ctx.reshape(B, 2048)
nin = (tl[:, :-1] == tl[:, -1:]).sum(1).astype(np.float64)
dur = e - s
for name, x in (("n_ds", nds), ("n_in", nin), ("n_ds+4n_in", nds + 4 * nin), ("n_ds+2n_in", nds + 2 * nin),
                ("n_ds+n_in", nds + nin), ("sqrt(n_ds)+n_in", np.sqrt(nds) + nin)):
    print("corr(time, %s) = %.3f" % (name, np.corrcoef(x, dur)[0, 1]))
# the requests that start last (LPT's cheapest) and their durations
late = np.argsort(-s)[:200]
print("last 200 starters: mean dur %.1f us, max %.1f us; overall mean %.1f" % (dur[late].mean(), dur[late].max(), dur.mean()))
