"""Speculative decoding with a model on the GPU (continuous batch of B slots).

Each step (ref draft.py:202-216 GenerationSession.step, batched):
  1. ``DraftEngine.propose``      drafts for every live sequence (device)
  2. ``Decoder.forward``          one tree forward -> logits of every node
  3. argmax                       node predictions (the oracle of draft.py:205-210)
  4. ``sssd_accept``              greedy walk, bonus, in-place append
  5. ``Decoder.compact``          K/V rows of accepted nodes -> contiguous slots
The root (last committed token) and the bonus token are never cached before
their own forward, exactly the reference's ordering.
"""

from __future__ import annotations

from time import perf_counter

import numpy as np
import torch

from ._lib import check, lib, ptr, stream_ptr
from .engine import DraftEngine
from .model import Decoder


class SpecDecoder:
    def __init__(self, engine: DraftEngine | None, model: Decoder, prompts: list, max_new: int) -> None:
        self.eng, self.model = engine, model
        dev = model.device
        B = model.B
        assert len(prompts) == B
        self.S = engine.S if engine is not None else 1
        self.cap = max(len(p) for p in prompts) + max_new + self.S + 1
        assert self.cap + self.S <= model.max_pos, "model KV cache too short"
        seq = np.zeros((B, self.cap), dtype=np.uint32)
        for b, p in enumerate(prompts):
            seq[b, : len(p)] = np.asarray(p, dtype=np.int64).astype(np.uint32)
        self.seq = torch.from_numpy(seq.view(np.int32).reshape(-1)).to(dev)
        self.off = torch.arange(B, dtype=torch.int64, device=dev) * self.cap
        self.seq_len = torch.tensor([len(p) for p in prompts], dtype=torch.int32, device=dev)
        self.seq_cap = self.seq_len + max_new
        self.path = torch.empty(B, self.S, dtype=torch.int32, device=dev)
        self.n_acc = torch.empty(B, dtype=torch.int32, device=dev)
        self.bonus = torch.empty(B, dtype=torch.int32, device=dev)
        self.emitted = torch.empty(B, dtype=torch.int32, device=dev)
        model.prefill([list(p) for p in prompts])
        self.steps = 0

    def _draft(self):
        B = self.model.B
        if self.eng is not None:
            out = self.eng.propose(self.seq, self.off, self.seq_len, self.cap)
            return out.tokens, out.parents, out.depths, out.mask, out.size
        # autoregressive: the draft is the root alone
        last = self.seq.view(B, self.cap).gather(1, (self.seq_len.long() - 1)[:, None])
        z = torch.zeros(B, 1, dtype=torch.int32, device=self.seq.device)
        return (last.to(torch.int32), z - 1, z, torch.ones(B, 1, 1, dtype=torch.int64, device=self.seq.device),
                torch.ones(B, dtype=torch.int32, device=self.seq.device))

    def step(self) -> torch.Tensor:
        self._step()
        self.steps += 1
        return self.emitted

    def _step(self) -> None:
        tokens, parents, depths, mask, size = self._draft()
        ctx = self.seq_len - 1
        pos = ctx.long()[:, None] + depths.clamp(min=0).long()
        logits = self.model.forward(tokens, pos, mask, ctx)
        pred = logits.argmax(-1).to(torch.int32).contiguous()
        B, S = tokens.shape
        check(lib().sssd_accept(ptr(tokens), ptr(parents), ptr(size), S, ptr(pred), B, ptr(self.seq),
                                ptr(self.off), ptr(self.seq_len), ptr(self.seq_cap), ptr(self.path),
                                ptr(self.n_acc), ptr(self.bonus), ptr(self.emitted), stream_ptr(self.seq.device)))
        self.model.compact(ctx, self.path if S == self.S else self.path[:, :S].contiguous(), self.n_acc)

    def run(self, graph_steps: int = 8) -> dict:
        """Decode every slot to its cap; returns tokens, steps and timing
        (``tokens_per_s`` over the whole call, ``steady_tokens_per_s`` after
        the first eager step and the graph capture).

        The first step runs eagerly (it creates every lazily allocated buffer);
        later steps run in groups of ``graph_steps`` replayed from one CUDA
        graph with the sequence lengths after each step recorded on the device
        and read back once per group (a finished slot's appends are capped, so
        steps past the end change nothing).  graph_steps <= 1: eager steps."""
        torch.cuda.synchronize()
        t0 = perf_counter()
        start = self.seq_len.clone()
        per_step = []
        cap = self.seq_cap.cpu()
        lens = self.seq_len.cpu()
        if bool((lens < cap).any()):
            self.step()
            now = self.seq_len.cpu()
            per_step.append(now - lens)
            lens = now
        graph = None
        if graph_steps > 1 and bool((lens < cap).any()):
            hist = torch.empty((graph_steps, self.model.B), dtype=torch.int32, device=self.seq.device)

            def group() -> None:
                for g in range(graph_steps):
                    self._step()
                    hist[g].copy_(self.seq_len)

            try:
                torch.cuda.synchronize()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, capture_error_mode="thread_local"):
                    group()
            except Exception as exc:  # capture not possible here: eager steps (same results)
                torch.cuda.synchronize()
                graph = None
                self.graph_error = repr(exc)
        torch.cuda.synchronize()
        t1, lens1 = perf_counter(), lens.clone()  # steady state: after the eager first step and the capture
        while bool((lens < cap).any()):
            if graph is None:
                self.step()
                now = self.seq_len.cpu()
                per_step.append(now - lens)
                lens = now
                continue
            graph.replay()
            H = hist.cpu()
            for g in range(graph_steps):
                if not bool((lens < cap).any()):
                    break  # trailing steps after every slot finished are not counted
                per_step.append(H[g] - lens)
                lens = H[g]
                self.steps += 1
        torch.cuda.synchronize()
        t2 = perf_counter()
        dt = t2 - t0
        gen = int((self.seq_len - start).sum())
        steady = int((self.seq_len.cpu() - lens1).sum())
        return {"tokens": gen, "steps": self.steps, "seconds": dt, "tokens_per_s": gen / dt,
                "steady_tokens_per_s": steady / (t2 - t1) if t2 > t1 and steady else 0.0,
                "accepted_per_step": float(torch.stack(per_step).float().mean()) if per_step else 0.0,
                "cuda_graph": graph is not None}

    def sequences(self) -> list[list[int]]:
        s = self.seq.view(self.model.B, self.cap).cpu().numpy().view(np.uint32)
        return [s[b, : int(n)].tolist() for b, n in enumerate(self.seq_len.cpu())]
