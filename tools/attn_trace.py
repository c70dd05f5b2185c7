"""Per-CTA clock timeline of the persistent tree-attention kernel (diagnostic
build: tools/build_attn_variants.sh trace -DSSSD_ATTN_TRACE, then
SSSD_LIB=.../libsssd_trace.so python tools/attn_trace.py).  For each shape:
cycles from CTA start to the first block's softmax done, per-item durations,
item-boundary gaps (epilogue done -> next item's first block done) and the
CTA end, as medians / maxima over CTAs."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2411_05894_b200 import _lib
from paper_2411_05894_b200.verify import tree_attention

L = _lib.lib()
L.sssd_attn_trace_read.argtypes = [C.c_void_p, C.c_int]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
shapes = {"cfg3": (32, 32, 32, 8, 4096), "cfg4": (8, 16, 32, 8, 32768), "8b_dec571": (64, 5, 32, 8, 571),
          "tiny_dec123": (64, 5, 8, 2, 123)}
out = {}
for name, (B, S, Hq, Hkv, ctx) in shapes.items():
    P = ctx + S
    q = torch.randn(B, S, Hq, 128, device="cuda").bfloat16()
    k = torch.randn(B, Hkv, P, 128, device="cuda").bfloat16()
    v = torch.randn(B, Hkv, P, 128, device="cuda").bfloat16()
    mask = torch.full((B, S, 1), -1, dtype=torch.int64, device="cuda")
    c = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    for _ in range(3):
        tree_attention(q, k, v, mask, c)
    flush.zero_()
    tree_attention(q, k, v, mask, c)
    torch.cuda.synchronize()
    buf = np.zeros((1024, 32), dtype=np.uint64)
    n = L.sssd_attn_trace_read(buf.ctypes.data, 1024)
    t = buf[:n].astype(np.int64)
    t0 = t[:, 0:1]
    rel = np.where(t > 0, t - t0, -1)
    items = []
    for kk in range(10):
        s_, f_, e_ = rel[:, 1 + 3 * kk], rel[:, 2 + 3 * kk], rel[:, 3 + 3 * kk]
        ok = (s_ >= 0) & (e_ >= 0)
        if not ok.any():
            break
        items.append({"item": kk, "ctas": int(ok.sum()),
                      "start_med": int(np.median(s_[ok])), "first_block_med": int(np.median(f_[ok])),
                      "epilogue_done_med": int(np.median(e_[ok])), "epilogue_done_max": int(e_[ok].max())})
    out[name] = {"ctas": int(n), "end_med": int(np.median(rel[:, 31])), "end_max": int(rel[:, 31].max()),
                 "items": items}
print(json.dumps(out, indent=1))
