"""Verification forward helpers: tree attention over a KV cache (tcgen05 kernel)
and KV-cache compaction after acceptance.

Semantics follow ref draft.py:205-210: draft node i's prediction is the greedy
next token after ``sequence + path(i)``, i.e. node i attends to the committed
prefix and to its ancestors-or-self inside the draft (the u64 ancestor rows
produced by the fusion kernel).  One call scores every node of every draft.
"""

from __future__ import annotations

import math

import torch

from . import _lib
from ._lib import check, lib, ptr, stream_ptr

_WS: dict = {}


def _workspace(nbytes: int, device) -> torch.Tensor:
    t = _WS.get(device)
    if t is None or t.numel() < nbytes:
        t = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _WS[device] = t
    return t


def tree_attention(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, mask: torch.Tensor,
                   ctx_len: torch.Tensor, scale: float | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """q [B, S, Hq, 128] bf16; k/v cache [B, Hkv, max_pos, 128] bf16 holding the
    committed prefix at [0, ctx_len[b]) and the S draft rows at [ctx_len[b], +S);
    mask [B, S, ceil(S/64)] int64 ancestor-or-self rows; returns o [B, S, Hq, 128]."""
    B, S, Hq, D = q.shape
    Hkv, max_pos = k_cache.shape[1], k_cache.shape[2]
    assert q.dtype == torch.bfloat16 and k_cache.dtype == torch.bfloat16 and v_cache.dtype == torch.bfloat16
    assert q.is_contiguous() and k_cache.is_contiguous() and v_cache.is_contiguous() and mask.is_contiguous()
    if scale is None:
        scale = 1.0 / math.sqrt(D)
    if out is None:
        out = torch.empty_like(q)
    dev = q.device
    ws = _workspace(lib().sssd_tree_attention_workspace(B, S, Hq, max_pos), dev)
    check(lib().sssd_tree_attention(ptr(q), ptr(k_cache), ptr(v_cache), ptr(mask), ptr(ctx_len), B, S, Hq, Hkv,
                                    max_pos, D, float(scale), ptr(out), ptr(ws), ws.numel(), stream_ptr(dev)))
    return out


def kv_compact(kv: torch.Tensor, base: torch.Tensor, path: torch.Tensor, n_acc: torch.Tensor) -> None:
    """kv [layers, B, H, max_pos, D] bf16: move rows base+path[b][k] -> base+1+k (in place)."""
    L, B, H, P, D = kv.shape
    S = path.shape[1]
    check(lib().sssd_kv_compact(ptr(kv), L, B, H, P, D, ptr(base), ptr(path), ptr(n_acc), S,
                                stream_ptr(kv.device)))
