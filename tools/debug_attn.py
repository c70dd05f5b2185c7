import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_05894_b200.verify import tree_attention
B, S, Hq, Hkv, ctx, P = 1, 32, 32, 8, 100, 256
q = torch.randn(B, S, Hq, 128, device="cuda").bfloat16()
k = torch.randn(B, Hkv, P, 128, device="cuda").bfloat16()
v = torch.randn(B, Hkv, P, 128, device="cuda").bfloat16()
mask = torch.zeros(B, S, 1, dtype=torch.int64, device="cuda")
for i in range(S): mask[0, i, 0] = (1 << (i + 1)) - 1 if i < 63 else -1
c = torch.tensor([ctx], dtype=torch.int32, device="cuda")
print("launch", flush=True)
o = tree_attention(q, k, v, mask, c)
torch.cuda.synchronize()
print("done", o.float().abs().max().item(), flush=True)
