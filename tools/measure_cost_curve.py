"""dec_len planning on B200 from measured curves:

1. acceptance curve: GPU teacher-forced ``sweep`` over dec_len on the
   phrase-model workload (cfg1 scale: 1M-token datastore, 64 records,
   prompt 512, reference 256);
2. cost curve: timed verify forwards of the Llama-3-8B-shaped decoder
   (random init, tcgen05 tree attention, fused layer kernels) at b and
   context s_kv for every s_q, plus the propose time of the drafts;
3. ``plan_dec_len`` with the measured cost beside the roofline model's
   (``perf_model.b200_hardware``, GQA / SwiGLU / lm_head accounting).

    python tools/measure_cost_curve.py [--b 32] [--s-kv 4096] > profiles/r1_cost_curve.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import model as Mo
from paper_2411_05894_b200 import perf_model as pm
from paper_2411_05894_b200 import workload

ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=32)
ap.add_argument("--s-kv", type=int, default=4096)
ap.add_argument("--grid", default="1,2,4,8,16,32,64")
args = ap.parse_args()
grid = [int(x) for x in args.grid.split(",")]

# 1. acceptance: teacher-forced decode of held-out phrase-model text (cfg1 scale)
V = 32000
ds = G.build(workload.corpus(1_000_000, V), vocab_size=V)
recs = [G.SimRecord(p, q) for p, q in workload.records(64, 512, 256, V)]
reports = G.sweep(recs, ds, G.FusionConfig(), grid)
accept = {s: reports[s].mean_accepted_per_step for s in grid}

# 2. measured verify cost: one tree forward (all layers, lm_head) per step, graph-replayed
b, s_kv = args.b, args.s_kv
dec = Mo.Decoder(Mo.LLAMA3_8B, b, s_kv + max(grid) + 8, seed=0, init_on_device=True)
ctx = torch.full((b,), s_kv, dtype=torch.int32, device="cuda")
step_s, fwd_ms = {}, {}
for s in grid:
    W = (s + 63) // 64
    bits = torch.tril(torch.ones(s, s, dtype=torch.bool))
    m = torch.zeros(s, W, dtype=torch.int64)
    for w in range(W):
        blk = bits[:, 64 * w: 64 * (w + 1)].to(torch.int64)
        m[:, w] = (blk << torch.arange(blk.shape[1], dtype=torch.int64)).sum(-1)
    mask = m[None].expand(b, s, W).contiguous().cuda()
    toks = torch.randint(0, 128256, (b, s), device="cuda")
    pos = ctx.long()[:, None] + torch.arange(s, device="cuda")[None]
    for _ in range(2):
        dec.forward(toks, pos, mask, ctx)
    torch.cuda.synchronize()
    # replayed as one CUDA graph (as serving.py runs decode steps): the GPU
    # time of the forward, not the host's launch rate
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        dec.forward(toks, pos, mask, ctx)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    fwd_ms[s] = e0.elapsed_time(e1) / reps
    step_s[s] = fwd_ms[s] / 1e3
    del graph
del dec
torch.cuda.empty_cache()

hw = pm.b200_hardware()
measured = pm.measured_cost_curve(step_s)
model = pm.cost_curve(hw, pm.LLAMA3_8B, b, grid, s_kv)
plan_meas = pm.plan_dec_len(accept, hw, pm.LLAMA3_8B, b, s_kv, cost=measured)
plan_model = pm.plan_dec_len(accept, hw, pm.LLAMA3_8B, b, s_kv)
out = {
    "workload": f"acceptance: teacher-forced sweep, 1M-token phrase-model datastore, 64 records (prompt 512, "
                f"ref 256), V={V}; cost: Llama-3-8B-shaped verify forward, b={b}, s_kv={s_kv}",
    "hardware": {"peak_flops": hw.peak_flops, "mem_bandwidth": hw.mem_bandwidth},
    "accept_per_step": accept,
    "forward_ms": {s: round(v, 4) for s, v in fwd_ms.items()},
    "model_forward_ms": {s: round(pm.forward_time(hw, pm.LLAMA3_8B, b, s, s_kv) * 1e3, 4) for s in grid},
    "cost_measured": {s: round(v, 4) for s, v in measured.items()},
    "cost_model": {s: round(v, 4) for s, v in model.items()},
    "free_budget_b_sq": pm.free_budget(hw, pm.LLAMA3_8B),
    "plan_measured": {"dec_len": plan_meas[0], "speedup": round(plan_meas[1], 3)},
    "plan_model": {"dec_len": plan_model[0], "speedup": round(plan_model[1], 3)},
}
print(json.dumps(out))
