"""Verification-cost planner (paper_2411_05894_b200.perf_model, SURVEY §8(f)
N4) against golden vectors from the reference ``specdraft.perf_model``
(tests/golden/make_golden_perf.py) and the reference tests' hand-derived known
answers (ref tests/test_perf_model.py), plus the B200 accounting extensions
(GQA, SwiGLU, lm_head, measured peaks) and the dec_len planner.  CPU only."""

import json
import math
import os

import pytest

from paper_2411_05894_b200 import perf_model as pm

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "perf_model.json")))
M7B = pm.ModelSpec(h=4096, n=32, d=128, h_mlp=11008, n_layers=32)
HW = pm.HardwareSpec(peak_flops=280e12, mem_bandwidth=0.8e12)


def _close(a, b):
    if isinstance(b, float) and math.isinf(b):
        return a == b
    return a == pytest.approx(b, rel=1e-12, abs=0.0)


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"{c['model']}-{c['hw']}")
def test_matches_reference_golden(case):
    m = pm.ModelSpec(**GOLD["models"][case["model"]])
    hw = pm.HardwareSpec(**GOLD["hardware"][case["hw"]])
    assert _close(pm.free_budget(hw, m), case["free_budget"])
    grid = [1, 2, 4, 8, 16, 32, 64]
    for sh in case["shapes"]:
        b, s_q, s_kv = sh["b"], sh["s_q"], sh["s_kv"]
        rows = pm.op_costs(m, b, s_q, s_kv).rows()
        assert tuple(rows) == pm.OP_NAMES and set(rows) == set(sh["rows"])
        for name, want in sh["rows"].items():
            r = rows[name]
            assert [r.flops, r.bytes_read, r.bytes_written] == want[:3]
            assert _close(r.flops_to_io, want[3])
        assert pm.op_costs(m, b, s_q, s_kv, include_mask_io=True).attention.bytes_read == sh["mask_attention_read"]
        assert _close(pm.forward_time(hw, m, b, s_q, s_kv), sh["forward_time"])
        assert _close(pm.relative_cost(hw, m, b, s_q, s_kv), sh["relative_cost"])
        curve = pm.cost_curve(hw, m, b, grid, s_kv)
        assert set(curve) == {int(k) for k in sh["cost_curve"]}
        for k, v in sh["cost_curve"].items():
            assert _close(curve[int(k)], v)
        times = [pm.forward_time(hw, m, b, s, s_kv) for s in grid]
        assert pm.slope_breakpoint(grid, times) == sh["slope_breakpoint"]


def test_reference_known_answers():
    # ref tests/test_perf_model.py frozen points (b=8, s_q=4, s_kv=1024)
    t = pm.op_costs(M7B, 8, 4, 1024)
    assert t.q_proj.flops == 1_073_741_824
    assert t.q_proj.bytes_read == 33_816_576 and t.q_proj.bytes_written == 262_144
    assert t.attention.flops == 538_968_064 and t.attention.bytes_read == 135_004_160
    assert t.mlp.flops == 5_771_362_304 and t.mlp.bytes_read == 180_617_216
    assert t.k_proj == t.q_proj == t.v_proj == t.o_proj
    assert pm.free_budget(HW, M7B) == pytest.approx(2_867_200 / 6_792, rel=1e-12)
    assert pm.slope_breakpoint(list(range(1, 65)), [pm.forward_time(HW, M7B, 8, s, 1024)
                                                   for s in range(1, 65)]) == GOLD["slope_b8_1024_m7b_paper"] == 53
    assert pm.free_budget(pm.HardwareSpec(2048e12, 1e12), M7B) == math.inf
    assert pm.slope_breakpoint(list(range(1, 11)), [0, .1, .2, .3, .4, 1.4, 2.4, 3.4, 4.4, 5.4]) == 5
    assert pm.expected_speedup({1: 1.0, 2: 1.8, 4: 3.0}, {1: 1.0, 2: 1.1, 4: 2.0}) == (2, pytest.approx(1.8 / 1.1))
    assert pm.expected_speedup({1: 1.0, 2: 2.0}, {1: 1.0, 2: 2.0}) == (1, 1.0)


def test_validation_messages():
    with pytest.raises(ValueError, match="h must equal n \\* d"):
        pm.ModelSpec(h=100, n=4, d=16, h_mlp=400, n_layers=2)
    with pytest.raises(ValueError, match="n_layers"):
        pm.ModelSpec(h=64, n=4, d=16, h_mlp=256, n_layers=0)
    with pytest.raises(ValueError, match="peak_flops"):
        pm.HardwareSpec(0, 1e12)
    with pytest.raises(ValueError, match="mem_bandwidth"):
        pm.HardwareSpec(1e12, -1)
    with pytest.raises(ValueError, match="b and s_q"):
        pm.op_costs(M7B, 1, 0.5, 10)
    with pytest.raises(ValueError, match="s_kv"):
        pm.op_costs(M7B, 1, 1, -1)
    with pytest.raises(ValueError, match="align"):
        pm.slope_breakpoint([1, 2], [1.0])
    with pytest.raises(ValueError, match="at least two"):
        pm.slope_breakpoint([1], [1.0])
    with pytest.raises(ValueError, match="domain mismatch"):
        pm.expected_speedup({1: 1.0, 2: 2.0}, {1: 1.0})
    with pytest.raises(ValueError, match="s_q=1"):
        pm.expected_speedup({2: 2.0}, {2: 1.0})
    with pytest.raises(ValueError, match="normalized"):
        pm.expected_speedup({1: 1.5, 2: 2.0}, {1: 1.0, 2: 1.0})
    with pytest.raises(ValueError, match="n_kv must divide n"):
        pm.ModelSpec(h=4096, n=32, d=128, h_mlp=1, n_layers=1, n_kv=5)


def test_spec_files(tmp_path):
    p = tmp_path / "m.txt"
    p.write_text("h = 4096\nn = 32\nd = 128\nh_mlp = 11008\nn_layers = 32\nbytes_per_param = 2\n")
    assert pm.load_model_spec(p) == M7B
    p.write_text("h = 4096\nn = 32\nd = 128\nh_mlp = 14336\nn_layers = 32\nn_kv = 8\nmlp_mats = 3\n"
                 "vocab = 128256\n")
    assert pm.load_model_spec(p) == pm.LLAMA3_8B
    p.write_text("h = 64\nn = 4\nd = 16\nh_mlp = 256\nn_layers = 2\nwidth = 9\n")
    with pytest.raises(ValueError, match="unknown model keys"):
        pm.load_model_spec(p)
    p.write_text("h = 64\nn = 4\n")
    with pytest.raises(ValueError, match="missing model keys"):
        pm.load_model_spec(p)
    h = tmp_path / "hw.txt"
    h.write_text("peak_flops = 280e12\nmem_bandwidth = 0.8e12\n")
    assert pm.load_hardware_spec(h) == HW
    h.write_text("peak_flops = 1e12\n")
    with pytest.raises(ValueError, match="missing hardware keys"):
        pm.load_hardware_spec(h)


def test_gqa_swiglu_accounting_matches_survey_cfg3():
    # cfg3 attention bytes 2 b n_kv (s_kv+s_q) d 2 + 2 b n_q s_q d 2 (+ 8 b s_q mask words)
    m = pm.LLAMA3_8B
    b, s_q, s_kv = 32, 32, 4096
    t = pm.op_costs(m, b, s_q, s_kv)
    att = t.attention.bytes_read + t.attention.bytes_written
    assert att == 2 * b * 8 * (s_kv + s_q) * 128 * 2 + 2 * b * 32 * s_q * 128 * 2
    assert (att + 8 * b * s_q) / 1e6 == pytest.approx(557.9, abs=0.05)
    assert t.attention.flops == 4 * b * s_q * (s_kv + s_q) * 32 * 128
    assert t.k_proj.bytes_read == (b * s_q * 4096 + 4096 * 1024) * 2 and t.k_proj.flops == 2 * b * s_q * 4096 * 1024
    assert t.q_proj.flops == 2 * b * s_q * 4096 ** 2
    assert t.mlp.flops == 6 * b * s_q * 4096 * 14336  # gate, up, down
    assert t.mlp.bytes_read == (b * s_q * 4096 + 3 * 4096 * 14336) * 2
    # the lm_head row is charged once per forward
    no_head = pm.ModelSpec(h=4096, n=32, d=128, h_mlp=14336, n_layers=32, n_kv=8, mlp_mats=3)
    hw = pm.b200_hardware(peaks_path="/nonexistent/MEASURED_PEAKS.json")
    head = pm.forward_time(hw, m, b, s_q, s_kv) - pm.forward_time(hw, no_head, b, s_q, s_kv)
    assert head == pytest.approx(max(2 * b * s_q * 4096 * 128256 / hw.peak_flops,
                                     (b * s_q * 4096 + 4096 * 128256 + b * s_q * 128256) * 2 / hw.mem_bandwidth))


def test_b200_hardware(tmp_path):
    fb = pm.b200_hardware(peaks_path=tmp_path / "absent.json")
    assert fb.mem_bandwidth == 6650e9 and fb.peak_flops == 1400e12
    assert pm.b200_hardware(sustained=False, peaks_path=tmp_path / "absent.json").peak_flops == 1590e12
    f = tmp_path / "peaks.json"
    f.write_text(json.dumps({"hbm_gbs": 6543.1, "bf16_tflops": 1657.9, "bf16_tflops_sustained": 1398.8,
                             "clocks": {"sm": 1965}}))
    hw = pm.b200_hardware(peaks_path=f)
    assert hw.mem_bandwidth == 6543.1e9 and hw.peak_flops == pytest.approx(1398.8e12)
    # the reference model on the measured B200 gives a free budget of 238.7
    assert pm.free_budget(hw, pm.ModelSpec(h=4096, n=32, d=128, h_mlp=14336, n_layers=32)) == pytest.approx(238.7,
                                                                                                           abs=0.05)


def test_plan_dec_len():
    hw = pm.b200_hardware(peaks_path="/nonexistent/MEASURED_PEAKS.json")
    accept = {1: 1.0, 2: 1.7, 4: 2.4, 8: 2.9, 16: 3.2, 32: 3.35, 64: 3.4}
    # decode at b=8: the forward is weight-bound, wide drafts are nearly free
    s8, r8 = pm.plan_dec_len(accept, hw, pm.LLAMA3_8B, 8, 4096)
    # b=256: compute-bound projections make every extra position cost
    s256, r256 = pm.plan_dec_len(accept, hw, pm.LLAMA3_8B, 256, 4096)
    assert s8 >= s256 and r8 > r256 >= 1.0
    cost = pm.cost_curve(hw, pm.LLAMA3_8B, 8, sorted(accept), 4096)
    assert pm.plan_dec_len(accept, hw, pm.LLAMA3_8B, 8, 4096) == pm.expected_speedup(accept, cost)
    # a measured curve (seconds per verify step) replaces the model
    meas = pm.measured_cost_curve({1: 2e-3, 2: 2.1e-3, 4: 2.2e-3, 8: 2.4e-3, 16: 3e-3, 32: 4.4e-3, 64: 8e-3})
    assert meas[1] == 1.0
    s, r = pm.plan_dec_len({k: 2 * v for k, v in accept.items()}, hw, pm.LLAMA3_8B, 8, 4096, cost=meas)
    assert (s, r) == pm.expected_speedup(accept, meas)
    with pytest.raises(ValueError, match="s_q=1"):
        pm.measured_cost_curve({2: 1.0})
    with pytest.raises(ValueError, match="domain mismatch"):
        pm.plan_dec_len(accept, hw, pm.LLAMA3_8B, 8, 4096, cost={1: 1.0, 2: 1.1})
