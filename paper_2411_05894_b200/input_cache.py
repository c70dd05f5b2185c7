"""Per-request prompt + self-output source (drop-in for ``specdraft.input_cache``).

The reference keeps an incremental windowed trie (ref input_cache.py:18-121).
Here the sequence itself is the state: ``get_conts`` runs the device input
scan (backward-match lengths m[e] + sorted occurrence elements),
which is what the batched engine does every step, and materialises the P
``ContinuationTree`` objects from the device result.  ``count`` and
``node_count`` are host introspection helpers (not on the drafting path).
"""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr, stream_ptr
from .datastore import as_u32
from .trees import ContinuationTree


class InputCache:
    def __init__(self, prompt: Sequence[int] = (), max_prefix_len: int = 4, input_branch_len: int = 8) -> None:
        if max_prefix_len < 1:
            raise ValueError(f"max_prefix_len must be >= 1, got {max_prefix_len}")
        if input_branch_len < 1:
            raise ValueError(f"input_branch_len must be >= 1, got {input_branch_len}")
        self.max_prefix_len = max_prefix_len
        self.input_branch_len = input_branch_len
        self.window = max_prefix_len + input_branch_len
        self.sequence: list[int] = [int(t) for t in prompt]

    def __len__(self) -> int:
        return len(self.sequence)

    def append(self, tokens: Sequence[int]) -> None:
        self.sequence.extend(int(t) for t in tokens)

    def count(self, ngram: Sequence[int]) -> int:
        ngram = [int(t) for t in ngram]
        if not ngram:
            raise ValueError("ngram must be non-empty")
        if len(ngram) > self.window:
            raise ValueError(f"ngram longer than window ({len(ngram)} > {self.window})")
        s = np.asarray(self.sequence, dtype=np.int64)
        k = len(ngram)
        if s.size < k:
            return 0
        win = np.lib.stride_tricks.sliding_window_view(s, k)
        return int(np.all(win == np.asarray(ngram), axis=1).sum())

    def node_count(self) -> int:
        s = self.sequence
        seen = set()
        for i in range(len(s)):
            for k in range(1, self.window + 1):
                if i + k > len(s):
                    break
                seen.add(tuple(s[i:i + k]))
        return len(seen)

    def get_conts(self) -> list[ContinuationTree]:
        """Tree p (index p-1) = continuations of earlier occurrences of the last p
        tokens, to ``input_branch_len`` deep (ref input_cache.py:88-113)."""
        if not self.sequence:
            raise ValueError("empty sequence")
        return input_trees_batch([self.sequence], self.max_prefix_len, self.input_branch_len)[0]


def input_elements_batch(seqs: list[list[int]], P: int, ibl: int, device=None) -> list[np.ndarray]:
    """Device input scan for B sequences: per sequence the [n, 4] u32 element
    rows (continuation start, first position, len | m << 8, 0) in the kernel's
    output order -- sorted by continuation string (a proper prefix first),
    ties by position, as the fusion consumes them."""
    from .fusion import _cfg_struct

    dev = torch.device(device) if device is not None else _lib.require_cuda()
    if ibl > _lib.SSSD_MAX_DEPTH:
        raise ValueError(f"input_branch_len {ibl} exceeds the compiled limit {_lib.SSSD_MAX_DEPTH}")
    B = len(seqs)
    lens = [len(s) for s in seqs]
    flat = np.concatenate([as_u32(s, "sequence token") for s in seqs])
    offs = np.zeros(B, dtype=np.int64)
    np.cumsum(lens[:-1], out=offs[1:])
    d_seq = torch.from_numpy(flat.view(np.int32)).to(dev)
    d_off = torch.from_numpy(offs).to(dev)
    d_len = torch.tensor(lens, dtype=torch.int32, device=dev)
    mx = max(lens)
    seqs_c = _lib.Seqs(ptr(d_seq), ptr(d_off), ptr(d_len), B, mx)
    c, keep = _cfg_struct(min(P, _lib.SSSD_MAX_P), 1, 1, ibl, 1, 1, device=dev)
    if P > _lib.SSSD_MAX_P:
        raise ValueError(f"max_prefix_len {P} exceeds the compiled limit {_lib.SSSD_MAX_P}")
    cap = max(mx, 1)
    el = torch.zeros(B * cap * 4, dtype=torch.int32, device=dev)
    n_el = torch.zeros(B, dtype=torch.int32, device=dev)
    ws = torch.empty(lib().sssd_input_scan_workspace(B, mx), dtype=torch.uint8, device=dev)
    check(lib().sssd_input_scan(seqs_c, c, ptr(el), ptr(n_el), ptr(ws), ws.numel(), stream_ptr(dev)))
    el_h = el.cpu().numpy().view(np.uint32).reshape(B, cap, 4)
    n_h = n_el.cpu().tolist()
    return [el_h[b, : n_h[b]].copy() for b in range(B)]


def input_trees_batch(seqs: list[list[int]], P: int, ibl: int, device=None) -> list[list[ContinuationTree]]:
    """Device input scan for B sequences, materialised as reference trees."""
    rows_all = input_elements_batch(seqs, P, ibl, device)
    out = []
    for b, s in enumerate(seqs):
        rows = rows_all[b]
        rows = rows[np.argsort(rows[:, 1], kind="stable")]  # insertion order = e ascending
        trees = []
        for p in range(1, P + 1):
            t = ContinuationTree()
            for e, _, lm, _ in rows:
                if (int(lm) >> 8) & 0xFF >= p:
                    t.add_path(s[int(e): int(e) + (int(lm) & 0xFF)])
            trees.append(t)
        out.append(trees)
    return out
