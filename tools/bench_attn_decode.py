"""Tree attention at decode shapes (the batch-64 serving loop's verify step:
s_q = 5, Llama-3-8B heads 32/8 and TINY heads 8/2) over the context length:
the slope is the per-key-block cost, the intercept the per-CTA fixed cost.
L2 flushed between launches."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_05894_b200.verify import tree_attention

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {}
for name, (B, S, Hq, Hkv) in {"8b": (64, 5, 32, 8), "tiny": (64, 5, 8, 2)}.items():
    for ctx in (123, 251, 571, 1147):
        P = ctx + S
        q = torch.randn(B, S, Hq, 128, device="cuda").bfloat16()
        k = torch.randn(B, Hkv, P, 128, device="cuda").bfloat16()
        v = torch.randn(B, Hkv, P, 128, device="cuda").bfloat16()
        mask = torch.full((B, S, 1), -1, dtype=torch.int64, device="cuda")
        c = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
        for _ in range(3):
            tree_attention(q, k, v, mask, c)
        ts = []
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record(); tree_attention(q, k, v, mask, c); b.record()
            torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        ms = sorted(ts)[len(ts) // 2]
        byt = 2 * B * Hkv * P * 128 * 2
        res[f"{name}_ctx{ctx}"] = {"us": round(ms * 1e3, 1), "TB/s": round(byt / ms / 1e9, 2)}
print(json.dumps(res))
