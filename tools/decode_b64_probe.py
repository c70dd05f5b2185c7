"""decode_b64 (TINY, 64 slots, 256 requests x 64 new tokens, prompt 512) wall
vs device time, and the host time spent refilling slots (ServeLoop.load:
prompt upload, per-row prefill, index build)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import model as Mo, workload
from paper_2411_05894_b200.serving import ServeLoop

V, B, plen, n_req, max_new, dl = 32000, 64, 512, 256, 64, 4
ds = G.build(workload.corpus(1_000_000, V), vocab_size=V)
prompts = [p.tolist() for p, _ in workload.records(n_req, plen, 0, V)]
dec = Mo.Decoder(Mo.TINY, B, plen + max_new + dl + 8, seed=0)
loop = ServeLoop(G.DraftEngine(ds, G.FusionConfig(dec_len=dl)), dec, plen, max_new)
loop.run(prompts[:B], 8)
t_load = [0.0]
orig = loop.load


def timed_load(*a, **k):
    torch.cuda.synchronize()
    t = time.perf_counter()
    orig(*a, **k)
    torch.cuda.synchronize()
    t_load[0] += time.perf_counter() - t


if not os.environ.get("NO_WRAP"):
    loop.load = timed_load
t_pre = [0.0]
orig_pre = dec.prefill_rows


def timed_pre(*a, **k):
    torch.cuda.synchronize()
    t = time.perf_counter()
    orig_pre(*a, **k)
    torch.cuda.synchronize()
    t_pre[0] += time.perf_counter() - t
    calls.append(round((time.perf_counter() - t) * 1e3, 2))


calls = []


if not os.environ.get("NO_WRAP"):
    dec.prefill_rows = timed_pre
r = loop.run(prompts, max_new)
print({"tokens_per_s": round(r["tokens_per_s"]), "device_tokens_per_s": round(r["device_tokens_per_s"]),
       "wall_s": round(r["seconds"], 4), "device_s": round(r["device_ms"] / 1e3, 4), "load_s": round(t_load[0], 4), "prefill_s": round(t_pre[0], 4),
       "groups": r["step_groups"], "group": r["group"], "prefill_calls_ms": calls})
