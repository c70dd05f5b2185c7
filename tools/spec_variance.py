"""Repeated cfg1 speculative-decode runs (wall time per run) to check run-to-run variance."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05894_b200 as G
from paper_2411_05894_b200 import model as Mo, workload
from paper_2411_05894_b200.serving import SpecDecoder
ds = G.build(workload.corpus(1_000_000, 32000), vocab_size=32000)
prompts = [p.tolist() for p, _ in workload.records(8, 512, 256, 32000)]
for i in range(4):
    sd = SpecDecoder(G.DraftEngine(ds, G.FusionConfig()), Mo.Decoder(Mo.TINY, 8, 1024, seed=0), prompts, 256)
    r = sd.run()
    print(i, round(r["tokens_per_s"]), round(r["steady_tokens_per_s"]), round(r["seconds"], 3), r["steps"], r["cuda_graph"], getattr(sd, "graph_error", None))
