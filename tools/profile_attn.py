import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_05894_b200.verify import tree_attention
B, S, Hq, Hkv, ctx = 32, 32, 32, 8, 4096
q = torch.randn(B, S, Hq, 128, device="cuda").bfloat16()
k = torch.randn(B, Hkv, ctx + S, 128, device="cuda").bfloat16()
v = torch.randn(B, Hkv, ctx + S, 128, device="cuda").bfloat16()
mask = torch.full((B, S, 1), -1, dtype=torch.int64, device="cuda")
c = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
for _ in range(2):
    tree_attention(q, k, v, mask, c)
torch.cuda.synchronize()
