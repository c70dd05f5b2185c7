"""Kernel time of one continuous-batching refill wave (TINY, 64 rows x 511
prompt tokens through Decoder.prefill_rows), torch profiler."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_05894_b200 import model as Mo, workload

B, plen = 64, 512
prompts = [p.tolist() for p, _ in workload.records(B, plen, 0, 32000)]
dec = Mo.Decoder(Mo.TINY, B, plen + 80, seed=0)
for _ in range(2):
    dec.prefill_rows(list(range(B)), prompts)
torch.cuda.synchronize()
t = time.perf_counter()
dec.prefill_rows(list(range(B)), prompts)
torch.cuda.synchronize()
print("prefill wall ms %.2f (all rows)" % ((time.perf_counter() - t) * 1e3))
for rows in (list(range(50)), list(range(7, 64, 3)), list(range(64))):
    for _ in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        dec.prefill_rows(rows, prompts[: len(rows)])
        torch.cuda.synchronize()
    print("prefill wall ms %.2f (%d rows, first %d)" % ((time.perf_counter() - t) * 1e3, len(rows), rows[0]))
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as pr:
    dec.prefill_rows(list(range(50)), prompts[:50])
    torch.cuda.synchronize()
print(pr.key_averages().table(sort_by="cuda_time_total", row_limit=12))
