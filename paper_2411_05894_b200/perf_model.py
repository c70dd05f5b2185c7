"""Verification-cost planner: how much a wider tree forward
costs on B200, and which draft budget (dec_len = s_q) maximises
accepted-tokens-per-step / relative-step-cost.

Drop-in for ref ``perf_model.py`` (same names, argument meaning and error
messages; ref :26-238): a per-layer roofline that charges every operation
max(FLOPs / peak, bytes / bandwidth).  With the reference's own arguments it
reproduces the reference numbers exactly (``tests/test_perf_model.py`` pins
them against the reference's known answers).  B200-first additions, all
opt-in so reference callers see no change:

* ``ModelSpec.n_kv`` (GQA: K/V projections and the KV cache read n_kv heads,
  ref :108-113 charges n), ``ModelSpec.mlp_mats`` (3 for SwiGLU: gate, up,
  down; the reference counts 2) and ``ModelSpec.vocab`` (lm_head row);
* ``b200_hardware()``: the driver-measured B200 peaks
  (``MEASURED_PEAKS.json``: STREAM copy and cuBLAS bf16, burst or sustained)
  or the B200_PROFILING.md fallback;
* ``measured_cost_curve()``: the cost curve from timed verify steps of the
  real kernels (``tools/measure_cost_curve.py``) instead of the model;
* ``plan_dec_len()``: the budget choice per batch / context.
"""

from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass
from typing import Mapping, Optional, Sequence

from . import kvconfig

OP_NAMES = ("q_proj", "k_proj", "v_proj", "attention", "o_proj", "mlp")


@dataclass(frozen=True)
class ModelSpec:
    """Decoder dims (ref :29-45).  ``h == n * d``.  Optional B200-accounting
    fields: ``n_kv`` (KV heads, default n), ``mlp_mats`` (2 as the reference,
    3 for SwiGLU) and ``vocab`` (adds an lm_head row when set)."""

    h: int
    n: int
    d: int
    h_mlp: int
    n_layers: int
    bytes_per_param: int = 2
    n_kv: Optional[int] = None
    mlp_mats: int = 2
    vocab: Optional[int] = None

    def __post_init__(self) -> None:
        for field in ("h", "n", "d", "h_mlp", "n_layers", "bytes_per_param"):
            value = getattr(self, field)
            if value < 1:
                raise ValueError(f"{field} must be >= 1, got {value}")
        if self.h != self.n * self.d:
            raise ValueError(f"h must equal n * d, got h={self.h}, n*d={self.n * self.d}")
        if self.n_kv is not None and (self.n_kv < 1 or self.n % self.n_kv):
            raise ValueError(f"n_kv must divide n, got n={self.n}, n_kv={self.n_kv}")
        if self.mlp_mats not in (2, 3):
            raise ValueError(f"mlp_mats must be 2 or 3, got {self.mlp_mats}")
        if self.vocab is not None and self.vocab < 1:
            raise ValueError(f"vocab must be >= 1, got {self.vocab}")

    @property
    def kv_heads(self) -> int:
        return self.n if self.n_kv is None else self.n_kv


@dataclass(frozen=True)
class HardwareSpec:
    """Peak FLOP/s and memory bandwidth in bytes/s (ref :48-58)."""

    peak_flops: float
    mem_bandwidth: float

    def __post_init__(self) -> None:
        if self.peak_flops <= 0:
            raise ValueError(f"peak_flops must be positive, got {self.peak_flops}")
        if self.mem_bandwidth <= 0:
            raise ValueError(f"mem_bandwidth must be positive, got {self.mem_bandwidth}")


@dataclass(frozen=True)
class CostRow:
    """One operation of one layer: FLOPs, bytes read / written and the
    intensity in FLOPs per moved element (bytes / bytes_per_param) (ref :61-72)."""

    flops: float
    bytes_read: float
    bytes_written: float
    flops_to_io: float


@dataclass(frozen=True)
class CostTable:
    q_proj: CostRow
    k_proj: CostRow
    v_proj: CostRow
    attention: CostRow
    o_proj: CostRow
    mlp: CostRow

    def rows(self) -> dict[str, CostRow]:
        return {name: getattr(self, name) for name in OP_NAMES}


def _cost(width: float, flops: float, elems_in: float, elems_out: float, extra_in_bytes: float = 0.0) -> CostRow:
    bytes_in = elems_in * width + extra_in_bytes
    bytes_out = elems_out * width
    return CostRow(flops, bytes_in, bytes_out, flops / ((bytes_in + bytes_out) / width))


def _matmul(width: float, tokens: float, k: float, n_out: float) -> CostRow:
    """tokens x k activations times a k x n_out weight (read once)."""
    return _cost(width, 2.0 * tokens * k * n_out, tokens * k + k * n_out, tokens * n_out)


def op_costs(m: ModelSpec, b: float, s_q: float, s_kv: float, include_mask_io: bool = False) -> CostTable:
    """Per-layer cost rows for one forward of ``s_q`` positions per sequence
    over ``s_kv`` cached ones (ref :84-118).  ``include_mask_io`` charges the
    packed tree mask (b * s_q^2 bits) to the attention reads."""
    if b < 1 or s_q < 1:
        raise ValueError(f"b and s_q must be >= 1, got b={b}, s_q={s_q}")
    if s_kv < 0:
        raise ValueError(f"s_kv must be >= 0, got {s_kv}")
    w = float(m.bytes_per_param)
    tokens = b * s_q
    kv_width = m.kv_heads * m.d
    q_proj = _matmul(w, tokens, m.h, m.h)
    kv_proj = q_proj if m.n_kv is None else _matmul(w, tokens, m.h, kv_width)
    # attention: Q (s_q rows), K and V of every visible position (cached
    # s_kv + the s_q tree rows), output s_q rows; n heads of flops
    att_flops = 4.0 * b * s_q * (s_q + s_kv) * m.n * m.d
    att_in = b * (m.n * s_q + 2 * m.kv_heads * (s_kv + s_q)) * m.d
    mask_bytes = b * s_q * s_q / 8 if include_mask_io else 0.0
    attention = _cost(w, att_flops, att_in, b * m.n * s_q * m.d, extra_in_bytes=mask_bytes)
    mlp = _cost(w, 2.0 * m.mlp_mats * tokens * m.h * m.h_mlp, tokens * m.h + m.mlp_mats * m.h * m.h_mlp,
                tokens * m.h)
    return CostTable(q_proj, kv_proj, kv_proj, attention, q_proj, mlp)


def _row_time(hw: HardwareSpec, row: CostRow) -> float:
    return max(row.flops / hw.peak_flops, (row.bytes_read + row.bytes_written) / hw.mem_bandwidth)


def forward_time(hw: HardwareSpec, m: ModelSpec, b: float, s_q: float, s_kv: float,
                 include_mask_io: bool = False) -> float:
    """Modelled seconds of one forward over all layers (ref :121-135), plus
    the lm_head when ``m.vocab`` is set."""
    per_layer = 0.0
    for row in op_costs(m, b, s_q, s_kv, include_mask_io=include_mask_io).rows().values():
        per_layer += _row_time(hw, row)
    total = m.n_layers * per_layer
    if m.vocab is not None:
        total += _row_time(hw, _matmul(float(m.bytes_per_param), b * s_q, m.h, m.vocab))
    return total


def relative_cost(hw: HardwareSpec, m: ModelSpec, b: float, s_q: float, s_kv: float) -> float:
    """Forward time relative to the s_q = 1 (plain decode) forward (ref :138-140)."""
    return forward_time(hw, m, b, s_q, s_kv) / forward_time(hw, m, b, 1, s_kv)


def cost_curve(hw: HardwareSpec, m: ModelSpec, b: float, s_q_values: Sequence[int], s_kv: float) -> dict[int, float]:
    """{s_q: relative_cost} over a grid (ref :143-151)."""
    one = forward_time(hw, m, b, 1, s_kv)
    return {int(s): forward_time(hw, m, b, s, s_kv) / one for s in s_q_values}


def free_budget(hw: HardwareSpec, m: ModelSpec) -> float:
    """The b * s_q at which a square projection turns compute-bound (ref
    :154-170): its intensity per element is 1 / (1/h + 1/(2 b s_q)); equal
    to bytes_per_param * peak / bandwidth at
    b s_q = 1 / (2 (1 / (bytes_per_param * ratio) - 1/h)).  +inf when the
    projection stays memory-bound for every finite b * s_q."""
    ridge = m.bytes_per_param * (hw.peak_flops / hw.mem_bandwidth)
    margin = 1.0 / ridge - 1.0 / m.h
    return math.inf if margin <= 0 else 0.5 / margin


def slope_breakpoint(s_q_values: Sequence[float], times: Sequence[float], rel_tol: float = 0.01) -> float:
    """First grid point from which the (convex, piecewise-linear) time curve
    keeps its final slope within ``rel_tol`` (ref :173-196)."""
    if len(s_q_values) != len(times):
        raise ValueError("s_q_values and times must align")
    if len(s_q_values) < 2:
        raise ValueError("need at least two points")
    steps = [(times[i + 1] - times[i]) / (s_q_values[i + 1] - s_q_values[i]) for i in range(len(times) - 1)]
    floor = (1.0 - rel_tol) * steps[-1]
    return next((s_q_values[i] for i, slope in enumerate(steps) if slope >= floor), s_q_values[-1])


def expected_speedup(accept_curve: Mapping[int, float], cost_curve: Mapping[int, float]) -> tuple[int, float]:
    """argmax over s_q of accept(s_q) / cost(s_q) and that ratio (ref
    :199-219).  Both curves cover the same s_q values including 1 and are
    normalised to accept(1) == cost(1) == 1; ties keep the smaller s_q."""
    if set(accept_curve) != set(cost_curve):
        raise ValueError("domain mismatch between acceptance and cost curves")
    if 1 not in accept_curve:
        raise ValueError("curves must include s_q=1")
    if abs(accept_curve[1] - 1.0) > 1e-6 or abs(cost_curve[1] - 1.0) > 1e-6:
        raise ValueError("curves must be normalized to accept(1) == cost(1) == 1")
    best = (1, accept_curve[1] / cost_curve[1])
    for s in sorted(accept_curve):
        ratio = accept_curve[s] / cost_curve[s]
        if ratio > best[1]:
            best = (s, ratio)
    return best


_MODEL_KEYS = ("h", "n", "d", "h_mlp", "n_layers", "bytes_per_param")
_MODEL_OPTIONAL = ("bytes_per_param", "n_kv", "mlp_mats", "vocab")
_HW_KEYS = ("peak_flops", "mem_bandwidth")


def load_model_spec(path: str | os.PathLike) -> ModelSpec:
    """``key = value`` model file (ref :226-235); ``n_kv`` / ``mlp_mats`` /
    ``vocab`` are accepted as optional B200-accounting keys."""
    items = kvconfig.read_kv(path)
    allowed = set(_MODEL_KEYS) | set(_MODEL_OPTIONAL)
    unknown = set(items) - allowed
    if unknown:
        raise ValueError(f"{path}: unknown model keys {sorted(unknown)}")
    missing = set(_MODEL_KEYS) - set(_MODEL_OPTIONAL) - set(items)
    if missing:
        raise ValueError(f"{path}: missing model keys {sorted(missing)}")
    return ModelSpec(**{key: int(value) for key, value in items.items()})


def load_hardware_spec(path: str | os.PathLike) -> HardwareSpec:
    """``key = value`` hardware file with peak_flops and mem_bandwidth (ref :238-247)."""
    items = kvconfig.read_kv(path)
    unknown = set(items) - set(_HW_KEYS)
    if unknown:
        raise ValueError(f"{path}: unknown hardware keys {sorted(unknown)}")
    missing = set(_HW_KEYS) - set(items)
    if missing:
        raise ValueError(f"{path}: missing hardware keys {sorted(missing)}")
    return HardwareSpec(float(items["peak_flops"]), float(items["mem_bandwidth"]))


# ---------------------------------------------------------------------------
# B200 planning
# ---------------------------------------------------------------------------

# B200_PROFILING.md fallbacks (an earlier measurement on this pool)
_B200_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}

LLAMA3_8B = ModelSpec(h=4096, n=32, d=128, h_mlp=14336, n_layers=32, n_kv=8, mlp_mats=3, vocab=128256)
TINY = ModelSpec(h=1024, n=8, d=128, h_mlp=2816, n_layers=2, n_kv=2, mlp_mats=3, vocab=32000)


def b200_hardware(sustained: bool = True, peaks_path: str | os.PathLike | None = None) -> HardwareSpec:
    """B200 roofline denominators: ``MEASURED_PEAKS.json`` (driver-measured
    STREAM copy ``hbm_gbs`` and cuBLAS bf16 ``bf16_tflops`` burst /
    ``bf16_tflops_sustained``) when present, else the profiling guide's
    fallback.  A verify step is a long kernel sequence: sustained by default."""
    if peaks_path is None:
        peaks_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    peaks = dict(_B200_FALLBACK)
    if os.path.exists(peaks_path):
        with open(peaks_path, encoding="utf-8") as fh:
            peaks.update({k: float(v) for k, v in json.load(fh).items() if k in _B200_FALLBACK})
    tflops = peaks["bf16_tflops_sustained"] if sustained else peaks["bf16_tflops"]
    return HardwareSpec(peak_flops=tflops * 1e12, mem_bandwidth=peaks["hbm_gbs"] * 1e9)


def measured_cost_curve(step_seconds: Mapping[int, float]) -> dict[int, float]:
    """Cost curve from timed verify steps {s_q: seconds} (must include s_q = 1)."""
    if 1 not in step_seconds:
        raise ValueError("measured steps must include s_q=1")
    base = step_seconds[1]
    if base <= 0:
        raise ValueError(f"s_q=1 step time must be positive, got {base}")
    return {int(s): t / base for s, t in step_seconds.items()}


def plan_dec_len(accept_curve: Mapping[int, float], hw: HardwareSpec, m: ModelSpec, b: float, s_kv: float,
                 cost: Mapping[int, float] | None = None) -> tuple[int, float]:
    """Draft budget for a batch of ``b`` sequences at context ``s_kv``: the
    s_q maximising accepted tokens per step over relative step cost.
    ``accept_curve`` = {s_q: mean accepted tokens per step} (e.g. from
    ``simulate``/``sweep`` at dec_len = s_q), normalised here by accept(1);
    ``cost`` = a measured curve (``measured_cost_curve``), else the model's."""
    if 1 not in accept_curve:
        raise ValueError("curves must include s_q=1")
    a1 = accept_curve[1]
    if a1 <= 0:
        raise ValueError(f"accept(1) must be positive, got {a1}")
    accept = {int(s): v / a1 for s, v in accept_curve.items()}
    if cost is None:
        cost = cost_curve(hw, m, b, sorted(accept), s_kv)
    else:
        if 1 not in cost:
            raise ValueError("curves must include s_q=1")
        cost = {int(s): v / cost[1] for s, v in cost.items()}
    return expected_speedup(accept, cost)
