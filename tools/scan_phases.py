"""Per-phase cycle split of input_scan_kernel at cfg4 (B=8, 32k prompt-heavy
contexts; measurement build -DSSSD_LK_PROBE via tools/build_lk_variants.sh,
SSSD_LIB=that .so): occurrence scan, key build, sort, output (cycles from the
kernel start, per request), with the occurrence counts."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload, _lib
ds = G.build(workload.corpus(20_000_000, 32000), vocab_size=32000)
L = _lib.lib()
L.sssd_set_lookup_probe.argtypes = [C.c_void_p]
Bq, n = 8, 32768
ctxs = workload.prompt_heavy_contexts(Bq, n, 32000)
seq = torch.from_numpy(np.concatenate(ctxs).astype(np.uint32).view(np.int32)).cuda()
off = (torch.arange(Bq, dtype=torch.int64) * n).cuda()
ln = torch.full((Bq,), n, dtype=torch.int32, device="cuda")
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=16))
for _ in range(3):
    eng.propose(seq, off, ln, n)
cyc = torch.zeros(Bq, 8, dtype=torch.int64, device="cuda")
L.sssd_set_lookup_probe(cyc.data_ptr())
eng.propose(seq, off, ln, n)
torch.cuda.synchronize()
L.sssd_set_lookup_probe(None)
st = cyc.cpu().numpy()[:, 4:8]
ctx_np = np.stack(ctxs)
occ = (ctx_np[:, :-1] == ctx_np[:, -1:]).sum(1)
print(json.dumps({"occurrences": occ.tolist(), "us_scan_keys_sort_end": (st / 1965.0).round(1).tolist()}))
