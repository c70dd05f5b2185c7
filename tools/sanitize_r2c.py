"""Round-2 final-session kernels under compute-sanitizer: the input scan's
merge-sort path (256- and 1,024-thread launches), run bounds by ballot and
16-byte continuation rows in the lookup (both fusion forms; the CTA form's
rank sort on levels of 65-512 nodes), and the tree attention with P in TMEM."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload
from paper_2411_05894_b200._lib import lib
from paper_2411_05894_b200.input_cache import input_elements_batch
from paper_2411_05894_b200.verify import tree_attention

rng = np.random.default_rng(1)
corpus = workload.corpus(300_000, 40)
ds = G.build(corpus, vocab_size=40)
ctxs = [rng.integers(0, 9, 3000).tolist(), rng.integers(0, 12, 9000).tolist(), rng.integers(0, 40, 500).tolist()]
input_elements_batch(ctxs, 4, 8)
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=128))
seq, off, ln, mx = eng.upload(ctxs)
for form in (0, 2):
    lib().sssd_set_fusion_form(form)
    eng.propose(seq, off, ln, mx, nodes=True)
lib().sssd_set_fusion_form(-1)
eng.check_status()
B, S, Hq, Hkv, ctx = 2, 8, 8, 2, 300
q = torch.randn(B, S, Hq, 128, device="cuda").bfloat16()
k = torch.randn(B, Hkv, ctx + S, 128, device="cuda").bfloat16()
v = torch.randn(B, Hkv, ctx + S, 128, device="cuda").bfloat16()
mask = torch.full((B, S, 1), -1, dtype=torch.int64, device="cuda")
c = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
tree_attention(q, k, v, mask, c)
torch.cuda.synchronize()
print("ok")
