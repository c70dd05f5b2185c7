"""CPU baseline for the decode leg.

TEST / BASELINE INFRASTRUCTURE ONLY: imported by tests/ and bench.py's CPU
legs, never by the product package.  It is the reference's step loop
(ref draft.py:202-216 GenerationSession.step: propose -> one oracle call per
draft node -> verify_greedy -> append) with the oracle = a tiny decoder in
fp32 PyTorch on the host cores (``torch.set_num_threads``), answering every
draft node of a step in one tree-masked forward over a per-request prefix KV
cache (the "prefix-KV-cached next" of the survey: node i's prediction is the
greedy next token after sequence + path(i)).  Drafts come from the CPU oracle
port (oracle/sssd_oracle.py propose, pinned to the reference's goldens), and
the weights are the GPU decoder's (bf16 values held as fp32), so the two legs
decode the same requests with the same model.
"""

from __future__ import annotations

import math
import time

import torch

from . import sssd_oracle as O


def _rope(x: torch.Tensor, pos: torch.Tensor, theta: float) -> torch.Tensor:
    D = x.shape[-1]
    inv = 1.0 / (theta ** (torch.arange(0, D, 2, dtype=torch.float32) / D))
    ang = pos.to(torch.float32)[..., None] * inv
    cos, sin = ang.cos()[..., None, :], ang.sin()[..., None, :]
    x1, x2 = x[..., : D // 2], x[..., D // 2:]
    return torch.cat([x1 * cos - x2 * sin, x1 * sin + x2 * cos], dim=-1)


def _rms(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


class CpuDecoder:
    """fp32 host copy of a ``paper_2411_05894_b200.model.Decoder`` with its own
    KV cache [layers][B][n_kv][max_pos][d]."""

    def __init__(self, dec, batch: int, max_pos: int) -> None:
        sp = self.spec = dec.spec
        f = lambda t: t.detach().float().cpu().contiguous()  # noqa: E731
        self.embed, self.norm, self.lm_head = f(dec.embed), f(dec.norm), f(dec.lm_head)
        self.layers = [{k: f(L[k]) for k in ("n1", "wq", "wk", "wv", "wo", "n2", "wg", "wu", "wd")} for L in dec.layers]
        self.B, self.max_pos = batch, max_pos
        self.k = torch.zeros(sp.n_layers, batch, sp.n_kv, max_pos, sp.head_dim)
        self.v = torch.zeros_like(self.k)

    def forward(self, rows: list, tokens: torch.Tensor, pos: torch.Tensor, anc: torch.Tensor,
                ctx: list) -> torch.Tensor:
        """Tree forward of S tokens per request (rows = cache rows): token s of
        request i sits at position pos[i, s], attends to cache [0, ctx[i]) and to
        the tree tokens j with anc[i, s, j]; K/V go to slots ctx[i] + s.
        Returns logits [R, S, V]."""
        sp = self.spec
        R, S = tokens.shape
        d, G = sp.head_dim, sp.n_q // sp.n_kv
        x = self.embed[tokens]
        for li, L in enumerate(self.layers):
            h = _rms(x, L["n1"], sp.eps)
            q = _rope((h @ L["wq"]).view(R, S, sp.n_q, d), pos, sp.rope_theta)
            k = _rope((h @ L["wk"]).view(R, S, sp.n_kv, d), pos, sp.rope_theta)
            v = (h @ L["wv"]).view(R, S, sp.n_kv, d)
            o = torch.empty(R, S, sp.n_q, d)
            for i, r in enumerate(rows):
                c = ctx[i]
                self.k[li, r, :, c:c + S] = k[i].transpose(0, 1)
                self.v[li, r, :, c:c + S] = v[i].transpose(0, 1)
                kk = self.k[li, r, :, : c + S].repeat_interleave(G, 0)  # [n_q, c+S, d]
                vv = self.v[li, r, :, : c + S].repeat_interleave(G, 0)
                s_ = torch.einsum("shd,hkd->hsk", q[i], kk) / math.sqrt(d)
                vis = torch.ones(S, c + S, dtype=torch.bool)
                vis[:, c:] = anc[i]
                s_ = s_.masked_fill(~vis[None], float("-inf"))
                o[i] = torch.einsum("hsk,hkd->shd", torch.softmax(s_, -1), vv)
            x = x + o.reshape(R, S, sp.n_q * d) @ L["wo"]
            h = _rms(x, L["n2"], sp.eps)
            x = x + (torch.nn.functional.silu(h @ L["wg"]) * (h @ L["wu"])) @ L["wd"]
        return _rms(x, self.norm, sp.eps) @ self.lm_head

    def prefill(self, rows: list, prompts: list) -> None:
        for r, p in zip(rows, prompts):
            n = len(p) - 1
            if n <= 0:
                continue
            toks = torch.tensor([p[:n]], dtype=torch.int64)
            self.forward([r], toks, torch.arange(n)[None], torch.tril(torch.ones(n, n, dtype=torch.bool))[None], [0])

    def compact(self, r: int, ctx: int, path: list) -> None:
        for k, node in enumerate(path):
            self.k[:, r, :, ctx + 1 + k] = self.k[:, r, :, ctx + node]
            self.v[:, r, :, ctx + 1 + k] = self.v[:, r, :, ctx + node]


def decode(store, prompts: list, cfg, dec, max_new: int, threads: int | None = None,
           budget_s: float | None = None) -> dict:
    """Speculative decode of every prompt (a batch, one step at a time over all
    live requests) on the host: oracle-port drafts, CPU fp32 tree verify,
    greedy accept.  Stops early when ``budget_s`` is exceeded (the tokens
    decoded so far are reported)."""
    if threads:
        torch.set_num_threads(int(threads))
    B = len(prompts)
    S = cfg.dec_len
    cpu = CpuDecoder(dec, B, max(len(p) for p in prompts) + max_new + S + 2)
    seqs = [[int(t) for t in p] for p in prompts]
    cap = [len(p) + max_new for p in prompts]
    disc = cfg.disc()
    cpu.prefill(list(range(B)), seqs)  # (not timed: the rate is of decode steps, like the GPU leg's device time)
    t0 = time.perf_counter()
    tokens, steps, accepted = 0, 0, []
    with torch.inference_mode():
        while any(len(s) < c for s, c in zip(seqs, cap)):
            if budget_s is not None and time.perf_counter() - t0 > budget_s:
                break
            live = [i for i in range(B) if len(seqs[i]) < cap[i]]
            drafts = [O.propose(store, seqs[i], cfg, disc=disc) for i in live]
            Sm = max(d.size for d in drafts)
            toks = torch.zeros(len(live), Sm, dtype=torch.int64)
            pos = torch.zeros(len(live), Sm, dtype=torch.int64)
            anc = torch.zeros(len(live), Sm, Sm, dtype=torch.bool)
            for j, (i, d) in enumerate(zip(live, drafts)):
                toks[j, : d.size] = torch.tensor(d.tokens, dtype=torch.int64)
                pos[j, : d.size] = len(seqs[i]) - 1 + torch.tensor(d.depths, dtype=torch.int64)
                for a in range(d.size):
                    anc[j, a, : d.size] = torch.tensor([(d.masks[a] >> k) & 1 for k in range(d.size)],
                                                       dtype=torch.bool)
                for a in range(d.size, Sm):
                    anc[j, a, a] = True
            logits = cpu.forward(live, toks, pos, anc, [len(seqs[i]) - 1 for i in live])
            pred = logits.argmax(-1)
            for j, (i, d) in enumerate(zip(live, drafts)):
                path, bonus = O.verify(d, pred[j, : d.size].tolist())
                ctx = len(seqs[i]) - 1
                new = [d.tokens[n] for n in path] + [int(bonus)]
                new = new[: cap[i] - len(seqs[i])]
                seqs[i].extend(new)
                cpu.compact(i, ctx, path)
                tokens += len(new)
                accepted.append(len(new))
            steps += 1
    dt = time.perf_counter() - t0
    return {"sequences": seqs, "tokens": tokens, "seconds": dt, "tokens_per_s": tokens / dt, "steps": steps,
            "accepted_per_step": sum(accepted) / max(1, len(accepted)), "threads": torch.get_num_threads(),
            "finished": all(len(s) >= c for s, c in zip(seqs, cap))}
