"""Kernel-time breakdown of one Llama-3-8B-shaped verify forward (torch
profiler) at b, s_q, s_kv:  python tools/profile_forward.py [b] [s_q] [s_kv]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2411_05894_b200 import model as Mo

b, s, s_kv = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (32, 8, 4096))]
dec = Mo.Decoder(Mo.LLAMA3_8B, b, s_kv + s + 8, seed=0, init_on_device=True)
ctx = torch.full((b,), s_kv, dtype=torch.int32, device="cuda")
W = (s + 63) // 64
mask = torch.full((b, s, W), -1, dtype=torch.int64, device="cuda")
toks = torch.randint(0, 128256, (b, s), device="cuda")
pos = ctx.long()[:, None] + torch.arange(s, device="cuda")[None]
for _ in range(2):
    dec.forward(toks, pos, mask, ctx)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    dec.forward(toks, pos, mask, ctx)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14, max_name_column_width=60))
