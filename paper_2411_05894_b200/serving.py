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
from .engine import DraftEngine, InputIndex
from .model import Decoder


def h2d(a: np.ndarray, dev) -> torch.Tensor:
    """Host array -> device tensor through pinned memory, non-blocking: the
    copy is stream-ordered but the host does not wait for the work queued
    before it (the pipelined decode loop refills slots while a step group runs)."""
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(dev, non_blocking=True)


def argmax_rows(x: torch.Tensor) -> torch.Tensor:
    """int32 argmax of every row of fp32 [rows, cols] (sssd_argmax_f32: torch.argmax
    semantics, one launch, no int64 intermediate)."""
    assert x.dtype == torch.float32 and x.is_contiguous()
    out = torch.empty(x.shape[0], dtype=torch.int32, device=x.device)
    check(lib().sssd_argmax_f32(ptr(x), x.shape[0], x.shape[1], ptr(out), stream_ptr(x.device)))
    return out


def spec_step(st, tokens, parents, depths, mask, size) -> None:
    """One verification step over every slot of ``st`` (a SpecDecoder or
    ServeLoop: model, seq / off / seq_len / seq_cap, path / n_acc / bonus /
    emitted, S): tree forward at positions L-1+depth, argmax, greedy accept +
    in-place append, KV compaction of the accepted nodes."""
    ctx = st.seq_len - 1
    pos = ctx.long()[:, None] + depths.clamp(min=0).long()
    logits = st.model.forward(tokens, pos, mask, ctx)
    B, S = tokens.shape
    pred = argmax_rows(logits.view(B * S, -1)).view(B, S)
    check(lib().sssd_accept(ptr(tokens), ptr(parents), ptr(size), S, ptr(pred), B, ptr(st.seq), ptr(st.off),
                            ptr(st.seq_len), ptr(st.seq_cap), ptr(st.path), ptr(st.n_acc), ptr(st.bonus),
                            ptr(st.emitted), stream_ptr(st.seq.device)))
    st.model.compact(ctx, st.path if S == st.S else st.path[:, :S].contiguous(), st.n_acc)


def draft_all(st):
    """Drafts of every slot of ``st`` (DraftEngine.propose, with its input index
    if any), or the root alone when ``st.eng`` is None (autoregressive)."""
    B = st.model.B
    if st.eng is not None:
        out = st.eng.propose(st.seq, st.off, st.seq_len, st.cap, index=getattr(st, "index", None))
        return out.tokens, out.parents, out.depths, out.mask, out.size
    last = st.seq.view(B, st.cap).gather(1, (st.seq_len.long() - 1)[:, None])
    z = torch.zeros(B, 1, dtype=torch.int32, device=st.seq.device)
    return (last.to(torch.int32), z - 1, z, torch.ones(B, 1, 1, dtype=torch.int64, device=st.seq.device),
            torch.ones(B, dtype=torch.int32, device=st.seq.device))


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
        return draft_all(self)

    def step(self) -> torch.Tensor:
        self._step()
        self.steps += 1
        return self.emitted

    def _step(self) -> None:
        spec_step(self, *self._draft())

    def run(self, graph_steps: int = 8) -> dict:
        """Decode every slot to its cap; returns tokens, steps and timing
        (``tokens_per_s`` over the whole call, ``steady_tokens_per_s`` after
        the first eager step and the graph capture).

        The first step runs eagerly (it creates every lazily allocated buffer);
        later steps run in groups of ``graph_steps`` replayed from CUDA graphs
        (two captures, alternating history buffers, so the next group is queued
        while the host reads the previous one) with the sequence lengths after
        each step recorded on the device and read back once per group (a
        finished slot's appends are capped, so steps past the end change
        nothing).  graph_steps <= 1: eager steps."""
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
        graphs = None
        if graph_steps > 1 and bool((lens < cap).any()):
            B = self.model.B
            hist = [torch.empty((graph_steps, B), dtype=torch.int32, device=self.seq.device) for _ in range(2)]
            pin = [torch.empty((graph_steps, B), dtype=torch.int32, pin_memory=True) for _ in range(2)]
            evs = [torch.cuda.Event() for _ in range(2)]

            def group(h: torch.Tensor) -> None:
                for g in range(graph_steps):
                    self._step()
                    h[g].copy_(self.seq_len)

            try:
                torch.cuda.synchronize()
                graphs = []
                for i in range(2):  # two copies, one per history buffer: group k+1 is queued before k is read
                    gr = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(gr, capture_error_mode="thread_local"):
                        group(hist[i])
                    graphs.append(gr)
            except Exception as exc:  # capture not possible here: eager steps (same results)
                torch.cuda.synchronize()
                graphs = None
                self.graph_error = repr(exc)
        torch.cuda.synchronize()
        t1, lens1 = perf_counter(), lens.clone()  # steady state: after the eager first step and the capture
        if graphs is None:
            while bool((lens < cap).any()):
                self.step()
                now = self.seq_len.cpu()
                per_step.append(now - lens)
                lens = now
        else:
            # pipelined groups: while group k runs, group k+1 is already queued
            # when the progress so far says some slot will still be unfinished
            # after k (a wrong guess costs one capped group or one lost overlap,
            # never a different result)
            launched = read = 0
            gain = int(per_step[-1].max()) * graph_steps if per_step else 0

            def launch() -> None:
                nonlocal launched
                i = launched & 1
                graphs[i].replay()
                pin[i].copy_(hist[i], non_blocking=True)
                evs[i].record()
                launched += 1

            launch()
            while read < launched:
                if launched - read < 2 and int((cap - lens).max()) > gain:
                    launch()
                i = read & 1
                evs[i].synchronize()
                H = pin[i].clone()
                read += 1
                before = lens
                for g in range(graph_steps):
                    if not bool((lens < cap).any()):
                        break  # trailing steps after every slot finished are not counted
                    per_step.append(H[g] - lens)
                    lens = H[g]
                    self.steps += 1
                gain = max(int((lens - before).max()), 1)
                if read == launched and bool((lens < cap).any()):
                    launch()
        torch.cuda.synchronize()
        t2 = perf_counter()
        dt = t2 - t0
        gen = int((self.seq_len - start).sum())
        steady = int((self.seq_len.cpu() - lens1).sum())
        return {"tokens": gen, "steps": self.steps, "seconds": dt, "tokens_per_s": gen / dt,
                "steady_tokens_per_s": steady / (t2 - t1) if t2 > t1 and steady else 0.0,
                "accepted_per_step": float(torch.stack(per_step).float().mean()) if per_step else 0.0,
                "cuda_graph": graphs is not None}

    def sequences(self) -> list[list[int]]:
        s = self.seq.view(self.model.B, self.cap).cpu().numpy().view(np.uint32)
        return [s[b, : int(n)].tolist() for b, n in enumerate(self.seq_len.cpu())]


class ServeLoop:
    """Continuous batching of speculative decode over a record queue (the
    north_star "continuously batched decode loop"; step semantics ref
    draft.py:202-216, loop semantics ref harness.py:171-237 with a model
    instead of the teacher-forced oracle).

    ``model.B`` slots each hold one live request: its token buffer (prompt,
    then the accepted tokens + bonus appended in place by ``sssd_accept``,
    capped at prompt + max_new) and its rows of the model's KV cache.  Steps
    run in groups of ``group`` replayed from one CUDA graph (propose -> tree
    forward -> argmax -> accept -> KV compaction for every slot); between
    groups, finished slots are refilled with the next queued requests: their
    prompts are written into the slot buffers and prefilled into their cache
    rows only (``Decoder.forward(..., rows=...)``).  A slot that finishes
    inside a group idles (appends capped) until the refill."""

    def __init__(self, engine: DraftEngine | None, model: Decoder, max_prompt: int, max_new: int,
                 group: int = 4, use_index: bool | None = None) -> None:
        self.eng, self.model, self.group = engine, model, max(1, int(group))
        dev = model.device
        B = model.B
        self.S = engine.S if engine is not None else 1
        self.cap = max_prompt + max_new + 1
        assert self.cap + self.S <= model.max_pos, "model KV cache too short"
        self.seq = torch.zeros(B * self.cap, dtype=torch.int32, device=dev)
        self.off = torch.arange(B, dtype=torch.int64, device=dev) * self.cap
        self.seq_len = torch.ones(B, dtype=torch.int32, device=dev)
        self.seq_cap = torch.ones(B, dtype=torch.int32, device=dev)
        self.path = torch.empty(B, self.S, dtype=torch.int32, device=dev)
        self.n_acc = torch.empty(B, dtype=torch.int32, device=dev)
        self.bonus = torch.empty(B, dtype=torch.int32, device=dev)
        self.emitted = torch.empty(B, dtype=torch.int32, device=dev)
        self.hist = torch.empty((self.group, B), dtype=torch.int32, device=dev)
        self._graph = None
        self.ahead_below_ms = 4.0  # queue the next step group before reading this one below this group time
        # N2 per-slot input index (rebuilt on refill): each step scans only the appended tokens
        if use_index is None:  # (see DecodeLoop: the index pays past one 8k-position scan pass)
            use_index = self.cap > 8192
        self.index = (InputIndex(B, self.cap, dev, self.off)
                      if (use_index and engine is not None and engine.use_input) else None)

    def _step(self) -> None:
        spec_step(self, *draft_all(self))

    def load(self, slots: list[int], prompts: list, max_new: list[int]) -> None:
        """Start requests in ``slots``: tokens into the slot buffers, KV-cache
        prefill of prompt[:-1] for those rows only (chunked chain masks)."""
        from .datastore import as_u32

        dev = self.seq.device
        # every prompt into its slot buffer with one upload + one scatter
        lens = [len(p) for p in prompts]
        flat = np.concatenate([as_u32(p, "prompt token") for p in prompts]) if prompts else np.zeros(0, "<u4")
        dst = np.concatenate([np.arange(n, dtype=np.int64) + s * self.cap for s, n in zip(slots, lens)]) \
            if prompts else np.zeros(0, np.int64)
        self.seq[h2d(dst, dev)] = h2d(flat.view(np.int32), dev)
        meta = h2d(np.array([[len(p) for p in prompts], [len(p) + int(m) for p, m in zip(prompts, max_new)]],
                            dtype=np.int32), dev)
        idx = h2d(np.array(list(slots), dtype=np.int64), dev)
        self.seq_len.index_copy_(0, idx, meta[0])
        self.seq_cap.index_copy_(0, idx, meta[1])
        self.model.prefill_rows(list(slots), [list(p) for p in prompts])
        if self.index is not None:
            self.index.build(self.seq, self.off, self.seq_len, rows=list(slots))

    def _group(self) -> None:
        for g in range(self.group):
            self._step()
            self.hist[g].copy_(self.seq_len)

    def run(self, prompts: list, max_new: int, use_graph: bool = True) -> dict:
        """Decode every request of ``prompts`` (each to ``max_new`` new tokens)
        through the slots; returns the generated sequences (request order) and
        throughput (wall clock over the whole loop incl. refills, and the
        device time of the step groups alone)."""
        B = self.model.B
        n_req = len(prompts)
        nxt = min(B, n_req)
        slot_req = np.full(B, -1, dtype=np.int64)
        slot_req[:nxt] = np.arange(nxt)
        free = list(range(nxt, B))
        self.seq_len.fill_(1)
        self.seq_cap.fill_(1)  # idle slots: capped (nothing appended)
        self.load(list(range(nxt)), prompts[:nxt], [max_new] * nxt)
        if free:  # idle slots still need a valid one-token context for the kernels
            self.load(free, [[int(prompts[0][-1])]] * len(free), [0] * len(free))
        out: list = [None] * n_req
        steps_of = np.zeros(n_req, dtype=np.int64)
        if use_graph and self._graph is None:
            self._step()  # eager warm-up step creates the lazily allocated buffers (results discarded below)
            # one prefill per refill bucket (1, 2, 4, .. rows: Decoder.prefill_rows pads
            # to these) so no refill meets a GEMM shape for the first time inside the
            # loop; the caches it writes are reloaded below
            plen = max(len(p) for p in prompts)
            r = 1
            while r < B:
                self.model.prefill_rows(list(range(r)), [[0] * plen] * r)
                r <<= 1
            torch.cuda.synchronize()
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, capture_error_mode="thread_local"):
                    self._group()
                self._graph = g
            except Exception as exc:  # capture not possible here: eager groups (same results)
                torch.cuda.synchronize()
                self.graph_error = repr(exc)
            # restart from clean prompts (the warm-up step appended tokens)
            self.seq_len.fill_(1)
            self.seq_cap.fill_(1)
            self.load(list(range(nxt)), prompts[:nxt], [max_new] * nxt)
            if free:
                self.load(free, [[int(prompts[0][-1])]] * len(free), [0] * len(free))
        lens = self.seq_len.cpu().numpy().astype(np.int64)
        caps = self.seq_cap.cpu().numpy().astype(np.int64)
        dev = self.seq.device
        # finished sequences are copied on the device (stream-ordered, before the
        # refill overwrites the slot) and read back once at the end
        out_dev = torch.zeros((n_req, self.cap), dtype=torch.int32, device=dev)
        out_len = np.zeros(n_req, dtype=np.int64)
        torch.cuda.synchronize()
        t0 = perf_counter()
        dev_ms, groups, tokens = 0.0, 0, 0
        accepted = []
        # Pipelined host loop: group k+1 is queued before group k's history is
        # read, so the GPU never waits for the host's bookkeeping; a slot refilled
        # while group k+1 is queued starts with group k+2 (group k+1 saw it capped,
        # its history there is the old request's and is skipped).
        pin = [torch.empty((self.group, B), dtype=torch.int32).pin_memory() for _ in range(2)]
        inflight: list = []  # (group index, ready event, timing events)
        fresh_from = np.zeros(B, dtype=np.int64)  # first group whose history belongs to the slot's request

        def launch(k: int) -> None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if self._graph is not None:
                self._graph.replay()
            else:
                self._group()
            e1.record()
            pin[k % 2].copy_(self.hist, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record()
            inflight.append((k, ready, e0, e1))

        # Queueing ahead pays when the host's bookkeeping is a sizeable part of a
        # group (small models); for long groups it would only keep finished
        # slots idle one group longer: decided from the first group's device time.
        ahead = None
        k_next = 0
        launch(k_next)
        k_next += 1
        while inflight:
            if ahead and (slot_req >= 0).any():  # keep one group queued ahead while any request is live
                launch(k_next)
                k_next += 1
            k, ready, e0, e1 = inflight.pop(0)
            ready.synchronize()
            H = pin[k % 2].numpy().astype(np.int64)
            gms = e0.elapsed_time(e1)
            dev_ms += gms
            if ahead is None:
                ahead = gms < self.ahead_below_ms
            groups += 1
            live = np.nonzero((slot_req >= 0) & (fresh_from <= k))[0]
            for g in range(self.group):
                act = live[lens[live] < caps[live]]
                if not len(act):
                    break
                em = H[g][act] - lens[act]
                accepted.extend(em.tolist())
                tokens += int(em.sum())
                steps_of[slot_req[act]] += 1
                lens[act] = H[g][act]
            done = live[lens[live] >= caps[live]]
            if len(done):
                rows = self.seq.view(B, self.cap)
                for sl in done:
                    out_dev[slot_req[sl]].copy_(rows[sl])
                    out_len[slot_req[sl]] = lens[sl]
                n_fill = min(len(done), n_req - nxt)
                fill = done[:n_fill].tolist()
                if fill:
                    self.load(fill, prompts[nxt:nxt + n_fill], [max_new] * n_fill)
                    slot_req[done[:n_fill]] = np.arange(nxt, nxt + n_fill)
                    lens[done[:n_fill]] = [len(p) for p in prompts[nxt:nxt + n_fill]]
                    caps[done[:n_fill]] = lens[done[:n_fill]] + max_new
                    fresh_from[done[:n_fill]] = k_next  # the first group queued after the refill
                    nxt += n_fill
                slot_req[done[n_fill:]] = -1
            if not inflight and (slot_req >= 0).any():  # (not queued ahead: the next group now)
                launch(k_next)
                k_next += 1
        o = out_dev.cpu().numpy()
        for r in range(n_req):
            out[r] = o[r, : out_len[r]].view(np.uint32).tolist()
        torch.cuda.synchronize()
        wall = perf_counter() - t0
        return {"sequences": out, "tokens": tokens, "requests": n_req, "slots": B, "seconds": wall,
                "tokens_per_s": tokens / wall, "device_ms": dev_ms, "step_groups": groups, "group": self.group,
                "device_tokens_per_s": tokens / (dev_ms / 1e3) if dev_ms else 0.0,
                "accepted_per_step": float(np.mean(accepted)) if accepted else 0.0,
                "steps_per_request": float(steps_of.mean()), "cuda_graph": self._graph is not None}
