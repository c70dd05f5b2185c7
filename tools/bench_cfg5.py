"""cfg5 on one B200 (BASELINE configs[4]: 1B-token datastore, continuous
batching at B=256): GPU datastore build time, sortedness spot check of the
suffix rows, batched propose at B=256 (latency and throughput), and the
teacher-forced continuous-batching decode loop (4,096 records, prompt 512,
reference 256, 256 slots) with accepted tokens/step.  The reference cannot
index 1B tokens in practical time (375.7 s at 100M), so there is
no CPU leg; drafts are checked bit-exact against the oracle at 100M in the
test suite.  Prints one JSON line (also written to gpurun_out/cfg5.json)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload

N = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000_000
V = 128256
out = {"workload": f"cfg5 (one GPU, replicated): {N/1e9:g}B-token phrase-model datastore, V={V}, B=256"}
t0 = time.perf_counter()
corpus = workload.corpus(N, V)
out["host_corpus_gen_s"] = round(time.perf_counter() - t0, 1)
torch.cuda.synchronize()
t0 = time.perf_counter()
ds = G.build(corpus, vocab_size=V)
torch.cuda.synchronize()
out["gpu_build_s"] = round(time.perf_counter() - t0, 2)
out["gpu_mem_gb"] = round(torch.cuda.max_memory_allocated() / 1e9, 1)
# sortedness spot check: adjacent suffix rows compare <= on their 15 inline tokens
rows = ds.rows
r = torch.randint(0, N - 1, (1 << 20,), device="cuda")
a, b = rows[r, 1:].long(), rows[r + 1, 1:].long()
diff = a != b
first = torch.where(diff.any(1), diff.float().argmax(1), torch.full_like(r, 14))
ok = (a.gather(1, first[:, None]) <= b.gather(1, first[:, None])).all().item()
out["sa_sorted_spot_check_1M_pairs"] = bool(ok)
del corpus
cfg = G.FusionConfig(dec_len=32)
eng = G.DraftEngine(ds, cfg)
B, CTX, R = 256, 512, 64
ctx = workload.phrase_stream(B * R * CTX, V, workload.HELDOUT_SEED)
seq = torch.from_numpy(ctx.view(np.int32)).cuda()
off = (torch.arange(B * R, dtype=torch.int64) * CTX).cuda()
ln = torch.full((B * R,), CTX, dtype=torch.int32, device="cuda")
for _ in range(3):
    eng.propose(seq, off, ln, CTX)
    eng.propose(seq, off[:B], ln[:B], CTX)
torch.cuda.synchronize()
eng.check_status()


def timed(fn, n=10):
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


lat = timed(lambda: eng.propose(seq, off[:B], ln[:B], CTX), 20)
thr = timed(lambda: eng.propose(seq, off, ln, CTX))
out["b256_propose_ms"] = round(lat, 4)
out["b256_lookups_per_s"] = round(B / lat * 1e3, 1)
out["throughput_lookups_per_s"] = round(B * R / thr * 1e3, 1)
out["throughput_batch"] = f"{R} x {B} requests per launch, ctx {CTX}, dec_len 32"
recs = workload.records(4096, 512, 256, V)
t0 = time.perf_counter()
sims = [G.SimRecord(p, q) for p, q in recs]
rep = G.simulate(sims, ds, cfg, slots=256)
dt = rep.wall_seconds
from paper_2411_05894_b200 import harness as H
graphed = H.simulate.last_graph
rep2 = G.simulate(sims, ds, cfg, slots=256, use_graph=False)
assert [r.per_step_tokens for r in rep.records] == [r.per_step_tokens for r in rep2.records]
out["decode_loop"] = {"records": 4096, "slots": 256, "prompt": 512, "reference": 256,
                      "mean_accepted_per_step": round(rep.mean_accepted_per_step, 4),
                      "teacher_forced_tokens_per_s": round(4096 * 256 / dt, 1), "wall_s": round(dt, 3),
                      "cuda_graph": graphed, "eager_wall_s": round(rep2.wall_seconds, 3)}
line = json.dumps(out)
print(line)
os.makedirs("gpurun_out", exist_ok=True)
open("gpurun_out/cfg5.json", "w").write(line + "\n")
