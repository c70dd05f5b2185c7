"""SA build timing (sssd_sa_build alone, CUDA events) and full verification
(sssd_sa_check) at n tokens of the phrase corpus: python tools/sa_build_bench.py [n]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload, datastore as D
from paper_2411_05894_b200._lib import lib, ptr, stream_ptr, check

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
V = 32000 if n <= 200_000_000 else 128256
tok = D._device_tokens(workload.corpus(n, V), "cuda")
ws = torch.empty(lib().sssd_sa_build_workspace(n), dtype=torch.uint8, device="cuda")
sa = torch.empty(n, dtype=torch.int32, device="cuda")
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    check(lib().sssd_sa_build(ptr(tok), n, ptr(sa), ptr(ws), ws.numel(), stream_ptr()))
    e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
rows = D._rows_from_sa(tok, n, sa)
ds = G.Datastore.on_device(tok, rows, n, V)
print(json.dumps({"n": n, "sa_build_ms": [round(t, 2) for t in ts], "mtok_per_s": round(n / min(ts) / 1e3, 1),
                  "workspace_gb": round(ws.numel() / 1e9, 2), "check": ds.check()}))
