"""Kernel-time breakdown of one cfg3 speculative step (Llama-3-8B shape, B=32,
ctx 4096, dec_len 32) with the torch profiler."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import model as Mo, workload
from paper_2411_05894_b200.serving import SpecDecoder
from torch.profiler import ProfilerActivity, profile
corpus = workload.corpus(2_000_000, 128256)
ds = G.build(corpus, vocab_size=128256)
prompts = [c.tolist() for c in workload.contexts(32, 4096, 128256)]
dec = Mo.Decoder(Mo.LLAMA3_8B, 32, 4096 + 2 * 32 + 5 * 33 + 64, seed=0, init_on_device=True)
sd = SpecDecoder(G.DraftEngine(ds, G.FusionConfig(dec_len=32)), dec, prompts, 5 * 33)
sd.step(); sd.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sd.step()
    torch.cuda.synchronize()
tab = prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70)
print(tab)
