"""Debug helper: find the first golden case the GPU path gets wrong."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2411_05894_b200 as G
from paper_2411_05894_b200.datastore import ds_paths
from paper_2411_05894_b200.fusion import _cfg_struct

which = sys.argv[1]
if which == "lookup":
    cases = json.load(open(os.path.join(ROOT, "tests/golden/lookup.json")))
    for ci, case in enumerate(cases):
        ds = G.build(case["corpus"])
        c = case["cfg"]
        cs, keep = _cfg_struct(P=c["P"], dec_len=1, branch_len=c["branch_len"], input_branch_len=1, M=c["M"],
                               T=c["T"], separator=c["separator"], device=ds.device)
        for q in case["queries"]:
            try:
                paths = ds_paths(ds, [q["prefix"]], cs)[0]
            except Exception as e:
                print("EXC", ci, e); raise
            if any(len(p) == 0 for p in paths):
                print("case", ci, "cfg", c, "prefix", q["prefix"], "n corpus", len(case["corpus"]))
                print("paths", paths)
                print("corpus", case["corpus"])
                sys.exit(0)
    print("lookup all ok")
else:
    cases = json.load(open(os.path.join(ROOT, "tests/golden/propose.json")))
    for ci, case in enumerate(cases):
        print(ci, case["cfg"], case["sources"], case["separator"], [len(r["seq"]) for r in case["requests"]], flush=True)
        ds = G.build(case["corpus"])
        cfg = G.FusionConfig(**case["cfg"])
        src = case["sources"]
        eng = G.DraftEngine(ds, cfg, case["separator"], src in ("both", "datastore"), src in ("both", "input"))
        eng.propose_host([r["seq"] for r in case["requests"]])
    print("propose all ok")
