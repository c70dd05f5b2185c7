"""Back-to-back cfg2 steps (16,384 lookups each, inputs > L2, no flush): one
stream vs two alternating streams with their own workspace / outputs, so step
i+1's lookup and scan can fill the SMs the fusion of step i releases."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import workload
ds = G.build(workload.corpus(100_000_000, 32000), vocab_size=32000)
B, K = 16384, 30
seq = torch.from_numpy(workload.phrase_stream(B * 2048, 32000, 1).view(np.int32)).cuda()
off = (torch.arange(B, dtype=torch.int64) * 2048).cuda()
ln = torch.full((B,), 2048, dtype=torch.int32, device="cuda")
eng = G.DraftEngine(ds, G.FusionConfig(dec_len=64))
ws = [eng.workspace(B, 2048).clone() for _ in range(2)]
outs = [eng.outputs(B) for _ in range(2)]
streams = [torch.cuda.Stream() for _ in range(2)]
main = torch.cuda.current_stream()


def run(nstreams):
    for s_ in streams:
        s_.wait_stream(main)
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(main)
    for s_ in streams:
        s_.wait_event(a)
    for i in range(K):
        k = i % nstreams
        eng.propose(seq, off, ln, 2048, out=outs[k], ws=ws[k], stream=streams[k])
    for s_ in streams:
        main.wait_stream(s_)
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


for _ in range(2):
    print("1 stream ms/step %.4f" % run(1), "2 streams ms/step %.4f" % run(2))
ref = eng.propose(seq, off, ln, 2048)
assert all(torch.equal(o.tokens, ref.tokens) for o in outs)
