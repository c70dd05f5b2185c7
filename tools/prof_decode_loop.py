import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
exec(open('tools/decode_b64_probe.py').read().split("t_load = [0.0]")[0])
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as pr:
    r = loop.run(prompts, max_new)
print(r["tokens_per_s"], r["seconds"])
print(pr.key_averages().table(sort_by="cuda_time_total", row_limit=22))
