"""Round-2 kernels under compute-sanitizer: the own-radix SA build (its 4-gram
first round) + sssd_sa_check, the k-gram index build and its lookups
(find_ranges + propose), per-node draft outputs (priority / source / pos) from
both fusion forms (one warp / one CTA per request), the N2 index build +
indexed propose, the compact sharded exchange (in-process shards), and the
continuous-batching model loop."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload
from paper_2411_05894_b200 import model as M
from paper_2411_05894_b200.serving import ServeLoop
from paper_2411_05894_b200.sharded import LocalShards

corpus = workload.corpus(1_100_000, 500)  # >= 2^20: the first-slot token table path
ds = G.build(corpus, vocab_size=500)
assert ds.check()["ok"]
small = G.build(workload.corpus(5000, 30))
assert small.check()["ok"]
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=32))
ctxs = [c.tolist() for c in workload.contexts(24, 300, 500)]
seq, off, ln, mx = eng.upload(ctxs)
from paper_2411_05894_b200._lib import lib
for form in (0, 2):  # one warp per request, one CTA per request
    lib().sssd_set_fusion_form(form)
    eng.propose(seq, off, ln, mx, nodes=True)
lib().sssd_set_fusion_form(-1)
ds.find_ranges([c[-k:] for c in ctxs[:8] for k in (1, 2, 3, 4, 6)])
ix = G.InputIndex(24, mx + 8, "cuda", off)
ix.build(seq, off, ln)
eng.propose(seq, off, ln, mx, index=ix)
eng.check_status()
G.merge(G.ContinuationTree(), [], G.FusionConfig(dec_len=4), 0)
shards = LocalShards(ds, 3, G.FusionConfig(dec_len=32))
shards.propose([(seq, off, ln, mx)])
spec = M.ModelSpec(n_layers=1, hidden=256, n_q=2, n_kv=1, mlp=512, vocab=500)
loop = ServeLoop(eng, M.Decoder(spec, 3, 200, seed=1), 60, 8, group=2, use_index=True)
loop.run([c[:60] for c in ctxs[:5]], 8, use_graph=False)
torch.cuda.synchronize()
print("sanitize r2 workload ok")
