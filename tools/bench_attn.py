"""Time the tree-attention kernel at the cfg3 / cfg4 shapes (one layer).
HBM roofline bytes per layer: 2*b*n_kv*(s_kv+s_q)*d*2 + 2*b*n_q*s_q*d*2 + 8*b*s_q."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_05894_b200.verify import tree_attention

_pk = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
# B200_PROFILING.md fallbacks when the driver has not written measured peaks
peak = json.load(open(_pk)) if os.path.exists(_pk) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
res = {}
for name, (B, S, Hq, Hkv, ctx) in {"cfg3": (32, 32, 32, 8, 4096), "cfg4": (8, 16, 32, 8, 32768)}.items():
    P = ctx + S
    q = torch.randn(B, S, Hq, 128, device="cuda").bfloat16()
    k = torch.randn(B, Hkv, P, 128, device="cuda").bfloat16()
    v = torch.randn(B, Hkv, P, 128, device="cuda").bfloat16()
    mask = torch.full((B, S, 1), -1, dtype=torch.int64, device="cuda")
    c = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    # ATTN_FLUSH=rw: after the write, read a second 256 MB buffer so L2 holds
    # clean lines (no dirty write-backs from the flush inside the timed region)
    clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda") if os.environ.get("ATTN_FLUSH") == "rw" else None
    for _ in range(3):
        tree_attention(q, k, v, mask, c)
    ts = []
    for _ in range(20):
        flush.zero_()
        if clean is not None:
            clean.sum()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); tree_attention(q, k, v, mask, c); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    byt = 2 * B * Hkv * (ctx + S) * 128 * 2 + 2 * B * Hq * S * 128 * 2 + 8 * B * S
    flops = 4 * B * S * (ctx + S) * Hq * 128
    res[name] = {"ms": ms, "GB/s": byt / ms / 1e6, "hbm_frac": byt / ms / 1e6 / peak["hbm_gbs"],
                 "TFLOP/s": flops / ms / 1e9, "tensor_frac": flops / ms / 1e9 / peak["bf16_tflops"]}
print(json.dumps(res))
