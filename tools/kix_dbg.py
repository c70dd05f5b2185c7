import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2411_05894_b200 as G
from oracle import sssd_oracle as O
rng = np.random.default_rng(11)
corpus = rng.permutation(500).tolist()
ds = G.build(corpus)
kx = ds.kix()
t = kx.view(-1, 4).cpu().numpy()
used = t[(t[:, 0] != 0) | (t[:, 1] != 0)]
print("kix slots", t.shape[0], "used", used.shape[0], "sample", used[:5].tolist())
sa = O.suffix_array(corpus)
tok = np.array(corpus)
for pat in ([corpus[40], corpus[41]], corpus[40:43], corpus[40:44], corpus[100:104]):
    print(pat, "oracle", O.find_range(tok, sa, pat), "gpu", ds.find_ranges([pat]))
eng = G.DraftEngine(ds, G.FusionConfig(P=4, dec_len=16, branch_len=8, input_branch_len=8, T=1))
ctx = [corpus[30:60]]
f = eng.propose_host(ctx)[0]
st = O.Store(tok.astype(np.uint32), sa)
d = O.propose(st, ctx[0], O.Cfg(P=4, dec_len=16, branch_len=8, input_branch_len=8, T=1))
print("gpu", f.tokens, "\noracle", d.tokens)
