"""Row argmax of fp32 logits: sssd_argmax_f32 vs torch.argmax(-1).to(int32),
at the TINY (V = 32,000) and Llama-3-8B (V = 128,256) verify shapes (320 rows)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_05894_b200.serving import argmax_rows

for V in (32000, 128256):
    x = torch.randn(320, V, device="cuda")
    for name, fn in (("sssd", lambda: argmax_rows(x)), ("torch", lambda: x.argmax(-1).to(torch.int32))):
        for _ in range(3):
            fn()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(50):
            fn()
        b.record()
        torch.cuda.synchronize()
        print(V, name, "%.2f us" % (a.elapsed_time(b) / 50 * 1e3))
