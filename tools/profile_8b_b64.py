"""Kernel-time breakdown of one decode_b64 speculative step of the Llama-3-8B
shape (B = 64 slots, prompt 512, dec_len 4) with the torch profiler."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import model as Mo, workload
from paper_2411_05894_b200.serving import SpecDecoder
from torch.profiler import ProfilerActivity, profile
ds = G.build(workload.corpus(10_000_000, 128256), vocab_size=128256)
prompts = [p.tolist() for p, _ in workload.records(64, 512, 0, 128256)]
dec = Mo.Decoder(Mo.LLAMA3_8B, 64, 512 + 64, seed=0, init_on_device=True)
sd = SpecDecoder(G.DraftEngine(ds, G.FusionConfig(dec_len=4)), dec, prompts, 32)
sd.step(); sd.step()
torch.cuda.synchronize()
ev = [torch.cuda.Event(True) for _ in range(2)]
ev[0].record(); sd.step(); ev[1].record(); torch.cuda.synchronize()
print("step ms %.3f" % ev[0].elapsed_time(ev[1]))
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sd.step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=16, max_name_column_width=60))
