"""Golden vectors for the verification-cost planner, made by running the
REFERENCE ``specdraft.perf_model`` (read-only import, build container only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_perf.py

Writes ``tests/golden/perf_model.json``: op-cost rows, forward times, cost
curves, free budgets and slope breakpoints over a grid of models, hardware
and shapes (reference accounting: no GQA, 2 MLP matrices)."""

from __future__ import annotations

import json
import os
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from specdraft import perf_model as rpm  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

MODELS = {
    "m7b": dict(h=4096, n=32, d=128, h_mlp=11008, n_layers=32),
    "llama3_8b": dict(h=4096, n=32, d=128, h_mlp=14336, n_layers=32),
    "tiny": dict(h=1024, n=8, d=128, h_mlp=2816, n_layers=2),
    "odd": dict(h=96, n=3, d=32, h_mlp=250, n_layers=5, bytes_per_param=1),
}
HWS = {
    "paper": dict(peak_flops=280e12, mem_bandwidth=0.8e12),
    "b200_measured": dict(peak_flops=1398.8e12, mem_bandwidth=6543.1e9),
    "b200_burst": dict(peak_flops=1657.9e12, mem_bandwidth=6543.1e9),
    "flat": dict(peak_flops=4000e12, mem_bandwidth=1e12),
}
SHAPES = [(1, 1, 0), (8, 4, 1024), (32, 32, 4096), (8, 16, 32768), (256, 8, 512), (3, 7, 100)]


def main() -> None:
    cases = []
    for mk, md in MODELS.items():
        m = rpm.ModelSpec(**md)
        for hk, hd in HWS.items():
            hw = rpm.HardwareSpec(**hd)
            case = {"model": mk, "hw": hk, "free_budget": rpm.free_budget(hw, m), "shapes": []}
            for b, s_q, s_kv in SHAPES:
                rows = {name: [r.flops, r.bytes_read, r.bytes_written, r.flops_to_io]
                        for name, r in rpm.op_costs(m, b, s_q, s_kv).rows().items()}
                mask_att = rpm.op_costs(m, b, s_q, s_kv, include_mask_io=True).attention
                grid = [1, 2, 4, 8, 16, 32, 64]
                times = [rpm.forward_time(hw, m, b, s, s_kv) for s in grid]
                case["shapes"].append({
                    "b": b, "s_q": s_q, "s_kv": s_kv, "rows": rows,
                    "mask_attention_read": mask_att.bytes_read,
                    "forward_time": rpm.forward_time(hw, m, b, s_q, s_kv),
                    "relative_cost": rpm.relative_cost(hw, m, b, s_q, s_kv),
                    "cost_curve": {str(k): v for k, v in rpm.cost_curve(hw, m, b, grid, s_kv).items()},
                    "slope_breakpoint": rpm.slope_breakpoint(grid, times),
                })
            cases.append(case)
    out = {"models": MODELS, "hardware": HWS, "cases": cases,
           "slope_b8_1024_m7b_paper": rpm.slope_breakpoint(
               list(range(1, 65)),
               [rpm.forward_time(rpm.HardwareSpec(**HWS["paper"]), rpm.ModelSpec(**MODELS["m7b"]), 8, s, 1024)
                for s in range(1, 65)])}
    with open(os.path.join(HERE, "perf_model.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
