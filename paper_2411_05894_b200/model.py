"""Random-init Llama-style decoders for the verification forward.

The reference has no model; its oracle protocol (ref draft.py:29-32,
205-210) asks, for every draft node i, the greedy next token after
``sequence + path(i)``.  ``Decoder.verify`` answers all nodes of a batch of
drafts in ONE forward: the draft tokens are run at positions L-1+depth, their
K/V rows are written to the cache at [ctx, ctx+S), and attention is the
tcgen05 tree kernel (prefix + ancestor-or-self mask).  Dense projections use
cuBLAS through torch (plain library GEMMs; q|k|v and gate|up fused into one
GEMM each, residual adds folded into addmm); RMSNorm, RoPE + the KV-cache
write, and SwiGLU are one-pass kernels of csrc/layers.cu.

Specs:
  TINY       2 layers, h=1024, n_q=8, n_kv=2, d=128, SwiGLU 2816, V=32000
  LLAMA3_8B  32 layers, h=4096, n_q=32, n_kv=8, d=128, SwiGLU 14336, V=128256
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import check, lib, ptr, stream_ptr
from .verify import kv_compact, tree_attention


@dataclass(frozen=True)
class ModelSpec:
    n_layers: int
    hidden: int
    n_q: int
    n_kv: int
    mlp: int
    vocab: int
    head_dim: int = 128
    rope_theta: float = 500000.0
    eps: float = 1e-5


TINY = ModelSpec(2, 1024, 8, 2, 2816, 32000)
LLAMA3_8B = ModelSpec(32, 4096, 32, 8, 14336, 128256)


def _rope(x: torch.Tensor, pos: torch.Tensor, theta: float) -> torch.Tensor:
    """x [..., S, H, D] (any float), pos [..., S] int -> rotated (float32 math)."""
    D = x.shape[-1]
    inv = 1.0 / (theta ** (torch.arange(0, D, 2, device=x.device, dtype=torch.float32) / D))
    ang = pos.to(torch.float32)[..., None] * inv  # [..., S, D/2]
    cos, sin = ang.cos()[..., None, :], ang.sin()[..., None, :]
    xf = x.float()
    x1, x2 = xf[..., : D // 2], xf[..., D // 2:]
    return torch.cat([x1 * cos - x2 * sin, x1 * sin + x2 * cos], dim=-1)


def _rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps) * w.float()).to(x.dtype)


def _h2d(a: np.ndarray, device) -> torch.Tensor:
    """Non-blocking upload through pinned memory (stream-ordered; the host does
    not wait for the work queued before it)."""
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(device, non_blocking=True)


_CHAIN_MASKS: dict = {}


def _chain_mask(S: int, device) -> torch.Tensor:
    """[S, ceil(S/64)] int64 ancestor rows of a causal chain (row i: bits 0..i),
    cached per (S, device)."""
    key = (S, str(device))
    m = _CHAIN_MASKS.get(key)
    if m is None:
        W = (S + 63) // 64
        bits = torch.tril(torch.ones(S, S, dtype=torch.bool))
        m = torch.zeros(S, W, dtype=torch.int64)
        for w in range(W):
            blk = bits[:, 64 * w: 64 * (w + 1)].to(torch.int64)
            m[:, w] = (blk << torch.arange(blk.shape[1], dtype=torch.int64)).sum(-1)
        m = _CHAIN_MASKS[key] = m.to(device)
    return m


class Decoder:
    """bf16 weights (seeded random init), KV cache [layers, B, n_kv, max_pos, d]."""

    def __init__(self, spec: ModelSpec, batch: int, max_pos: int, device="cuda", seed: int = 0,
                 dtype=torch.bfloat16, init_on_device: bool = False) -> None:
        self.spec, self.B, self.max_pos, self.device, self.dtype = spec, batch, max_pos, torch.device(device), dtype
        # seeded init; large models draw on the device (same seed -> same weights on the same torch/GPU)
        gdev = self.device if init_on_device else torch.device("cpu")
        g = torch.Generator(device=gdev).manual_seed(seed)
        h, d = spec.hidden, spec.head_dim

        def w(*shape, scale):
            return (torch.randn(*shape, generator=g, device=gdev, dtype=torch.float32) * scale).to(dtype).to(self.device)

        self.embed = w(spec.vocab, h, scale=1.0)
        self.layers = []
        for _ in range(spec.n_layers):
            wq = w(h, spec.n_q * d, scale=1 / math.sqrt(h))
            wk = w(h, spec.n_kv * d, scale=1 / math.sqrt(h))
            wv = w(h, spec.n_kv * d, scale=1 / math.sqrt(h))
            wo = w(spec.n_q * d, h, scale=1 / math.sqrt(spec.n_q * d))
            wg = w(h, spec.mlp, scale=1 / math.sqrt(h))
            wu = w(h, spec.mlp, scale=1 / math.sqrt(h))
            wd = w(spec.mlp, h, scale=1 / math.sqrt(spec.mlp))
            # fused projections (one GEMM for q|k|v, one for gate|up); the
            # per-projection names stay available as column views
            wqkv = torch.cat([wq, wk, wv], dim=1)
            wgu = torch.cat([wg, wu], dim=1)
            del wq, wk, wv, wg, wu
            nq, nk = spec.n_q * d, spec.n_kv * d
            self.layers.append({
                "n1": torch.ones(h, dtype=dtype, device=self.device),
                "wqkv": wqkv, "wq": wqkv[:, :nq], "wk": wqkv[:, nq:nq + nk], "wv": wqkv[:, nq + nk:],
                "wo": wo,
                "n2": torch.ones(h, dtype=dtype, device=self.device),
                "wgu": wgu, "wg": wgu[:, :spec.mlp], "wu": wgu[:, spec.mlp:],
                "wd": wd,
            })
        self.norm = torch.ones(h, dtype=dtype, device=self.device)
        self.lm_head = w(h, spec.vocab, scale=1 / math.sqrt(h))
        self.k_cache = torch.zeros(spec.n_layers, batch, spec.n_kv, max_pos, d, dtype=dtype, device=self.device)
        self.v_cache = torch.zeros_like(self.k_cache)
        self.scale = 1.0 / math.sqrt(d)

    def forward(self, tokens: torch.Tensor, positions: torch.Tensor, mask: torch.Tensor,
                ctx_len: torch.Tensor, rows: torch.Tensor | None = None, logits: bool = True,
                kv_rows: torch.Tensor | None = None) -> torch.Tensor | None:
        """Tree forward: tokens / positions [b, S] (rows = cache rows of these b
        requests, default all), mask [b, S, W] int64, ctx_len [b] int32 = committed
        tokens already in the cache.  Writes K/V of the S tokens to cache
        positions ctx..ctx+S-1 and returns logits [b, S, V] (fp32); with
        logits=False (prefill) only the K/V writes happen: the last layer stops
        after its K/V and no lm_head is computed.  kv_rows [b]: the K/V of
        request b go to cache row kv_rows[b], -1 = not written (a padding
        request of a bucketed prefill); attention still reads row rows[b] (or b)."""
        sp = self.spec
        b, S = tokens.shape
        d, h = sp.head_dim, sp.hidden
        n = b * S
        st = stream_ptr(self.device)
        x = self.embed[tokens.reshape(-1).long()]  # [b*S, h]
        pos = positions.reshape(-1).long().contiguous()
        ctx = ctx_len.to(torch.int32).contiguous()
        rows_l = rows.long().contiguous() if rows is not None else None
        if kv_rows is not None:  # K/V destinations (-1: padding request, not written)
            assert rows is not None or b == self.B
            rows_l = kv_rows.long().contiguous()
        hN = torch.empty_like(x)
        q = torch.empty(b, S, sp.n_q, d, dtype=self.dtype, device=self.device)
        for li, L in enumerate(self.layers):
            check(lib().sssd_rmsnorm_bf16(ptr(x), ptr(L["n1"]), ptr(hN), n, h, sp.eps, st))
            qkv = hN @ L["wqkv"]
            kc, vc = self.k_cache[li], self.v_cache[li]
            check(lib().sssd_rope_kv_bf16(ptr(qkv), ptr(pos), ptr(ctx), ptr(rows_l) if rows_l is not None else None,
                                          ptr(q), ptr(kc), ptr(vc), b, S, sp.n_q, sp.n_kv, d, self.max_pos,
                                          sp.rope_theta, st))
            if not logits and li == len(self.layers) - 1:
                return None  # (prefill: this layer's K/V are written; nothing reads its output)
            if rows is None:
                o = tree_attention(q, kc, vc, mask, ctx, self.scale)
            else:
                o = tree_attention(q, kc[rows].contiguous(), vc[rows].contiguous(), mask, ctx, self.scale)
            x.addmm_(o.view(n, sp.n_q * d), L["wo"])  # residual in place (C == D, no copy)
            check(lib().sssd_rmsnorm_bf16(ptr(x), ptr(L["n2"]), ptr(hN), n, h, sp.eps, st))
            gu = hN @ L["wgu"]
            a = torch.empty(n, sp.mlp, dtype=self.dtype, device=self.device)
            check(lib().sssd_swiglu_bf16(ptr(gu), ptr(a), n, sp.mlp, st))
            x.addmm_(a, L["wd"])
        check(lib().sssd_rmsnorm_bf16(ptr(x), ptr(self.norm), ptr(hN), n, h, sp.eps, st))
        # fp32 logits straight from the GEMM's fp32 accumulators (no bf16
        # rounding of the logits: greedy ties stay as rare as in fp32)
        return torch.mm(hN, self.lm_head, out_dtype=torch.float32).view(b, S, -1)

    def reference_logits(self, seq: list) -> torch.Tensor:
        """Verification helper (tests, bench): plain fp32 PyTorch causal forward
        of one whole sequence with this decoder's weights (dense attention,
        separate projections); logits of the last position [V]."""
        sp = self.spec
        d = sp.head_dim
        f = lambda t: t.float()  # noqa: E731
        x = f(self.embed)[torch.as_tensor(seq, device=self.device)]
        n = len(seq)
        pos = torch.arange(n, device=self.device)
        G = sp.n_q // sp.n_kv
        causal = torch.triu(torch.ones(n, n, dtype=torch.bool, device=self.device), 1)
        for L in self.layers:
            h = _rmsnorm(x, f(L["n1"]), sp.eps)
            q = _rope((h @ f(L["wq"])).view(n, sp.n_q, d), pos, sp.rope_theta)
            k = _rope((h @ f(L["wk"])).view(n, sp.n_kv, d), pos, sp.rope_theta).repeat_interleave(G, dim=1)
            v = (h @ f(L["wv"])).view(n, sp.n_kv, d).repeat_interleave(G, dim=1)
            s = torch.einsum("qhd,khd->hqk", q, k) / math.sqrt(d)
            o = torch.einsum("hqk,khd->qhd", torch.softmax(s.masked_fill(causal, float("-inf")), -1), v)
            x = x + o.reshape(n, sp.n_q * d) @ f(L["wo"])
            h = _rmsnorm(x, f(L["n2"]), sp.eps)
            x = x + (torch.nn.functional.silu(h @ f(L["wg"])) * (h @ f(L["wu"]))) @ f(L["wd"])
        return (_rmsnorm(x, f(self.norm), sp.eps) @ f(self.lm_head))[-1]

    def prefill(self, prompts: list, chunk: int = 256) -> None:
        """Write the cache for prompts[b][:-1] (the last prompt token is the first
        draft root) through the tree kernel with causal chain masks."""
        B = len(prompts)
        assert B == self.B
        n = [len(p) - 1 for p in prompts]
        done = [0] * B
        while any(done[b] < n[b] for b in range(B)):
            S = min(chunk, max(n[b] - done[b] for b in range(B)))
            S = max(S, 1)
            toks = np.zeros((B, S), dtype=np.int64)
            for b in range(B):
                seg = prompts[b][done[b]: min(n[b], done[b] + S)]
                toks[b, : len(seg)] = np.asarray(seg, dtype=np.int64)
            mask = _chain_mask(S, self.device)
            ctx = torch.tensor(done, dtype=torch.int32, device=self.device)
            pos = ctx.long()[:, None] + torch.arange(S, device=self.device)[None, :]
            self.forward(torch.from_numpy(toks).to(self.device), pos, mask[None].expand(B, S, -1).contiguous(), ctx,
                         logits=False)
            for b in range(B):
                done[b] = min(n[b], done[b] + S)

    def prefill_rows(self, rows: list, prompts: list, chunk: int = 256) -> None:
        """``prefill`` for a subset of cache rows (continuous batching: a freed
        slot's new request), other rows untouched: the KV rows of prompts[i][:-1]
        go to cache row rows[i]."""
        n = [len(p) - 1 for p in prompts]
        if not rows or max(n) <= 0:
            return
        # Bucketed shape: the batch is padded to the next power of two of
        # refilled rows (all B rows at that size: the plain in-order path, no
        # gathered copy of the cache); padding requests write no K/V and their
        # outputs are discarded.  The GEMM shapes then repeat from refill to
        # refill (a new cuBLAS shape costs ~1 ms of host heuristics per call)
        # while a big model never prefills more than 2x the refilled rows.
        B = self.B
        R = len(rows)
        Rp = 1
        while Rp < R:
            Rp <<= 1
        L = max(n)
        if Rp >= B:
            Rp = B
            att = None
            kv = np.full(B, -1, dtype=np.int64)
            host = np.zeros((B, L), dtype=np.int64)  # all prompt tokens, one upload
            for r_, p, k in zip(rows, prompts, n):
                kv[r_] = r_
                host[r_, :k] = np.asarray(p[:k], dtype=np.int64)
        else:
            att = _h2d(np.array(list(rows) + [rows[0]] * (Rp - R), dtype=np.int64), self.device)
            kv = np.array(list(rows) + [-1] * (Rp - R), dtype=np.int64)
            host = np.zeros((Rp, L), dtype=np.int64)
            for i, (p, k) in enumerate(zip(prompts, n)):
                host[i, :k] = np.asarray(p[:k], dtype=np.int64)
        toks_all = _h2d(host, self.device)
        kv_rows = _h2d(kv, self.device)
        done = 0
        while done < L:
            S = min(chunk, L - done)
            mask = _chain_mask(S, self.device)
            ctx = torch.full((Rp,), done, dtype=torch.int32, device=self.device)
            pos = ctx.long()[:, None] + torch.arange(S, device=self.device)[None, :]
            self.forward(toks_all[:, done: done + S].contiguous(), pos, mask[None].expand(Rp, S, -1).contiguous(), ctx,
                         rows=att, logits=False, kv_rows=kv_rows)
            done += S

    def compact(self, ctx_len: torch.Tensor, path: torch.Tensor, n_acc: torch.Tensor) -> None:
        """Move the K/V rows of accepted draft nodes (cache slot ctx + node) to
        ctx + 1 + k, all layers, in one launch each for K and V."""
        kv_compact(self.k_cache, ctx_len, path, n_acc)
        kv_compact(self.v_cache, ctx_len, path, n_acc)
