"""Batched GPU drafting: the hot path behind ``GenerationSession.propose``.

``DraftEngine.propose`` is one C-ABI call (``sssd_propose``) that runs, on one
stream, the datastore lookup kernel, the input-scan kernel and the fusion /
flatten kernel for a whole batch of live sequences that are already resident
in HBM.  Outputs stay on the device (``DraftBatch``); ``FlattenedDraft``
objects are materialised only for the reference-compatible API and parity.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr, stream_ptr
from .datastore import Datastore
from .fusion import FusionConfig, cfg_struct


@dataclass
class DraftBatch:
    size: torch.Tensor     # [B] int32
    tokens: torch.Tensor   # [B, S] int32 (uint32 bit pattern)
    parents: torch.Tensor  # [B, S] int32
    depths: torch.Tensor   # [B, S] int32
    mask: torch.Tensor     # [B, S, W] int64 (uint64 bit pattern): ancestor-or-self rows
    ranges: torch.Tensor | None = None   # [B, P, 2] int64
    samples: torch.Tensor | None = None  # [B, P, M] int64
    n_conts: torch.Tensor | None = None  # [B, P] int32
    p_cut: torch.Tensor | None = None    # [B] int32
    pos: torch.Tensor | None = None       # [B, S] int32 position ids L-1+depth (-1 padding)
    priority: torch.Tensor | None = None  # [B, S] float64 DraftNode.priority (+inf root)
    source: torch.Tensor | None = None    # [B, S] int32 merge rank (0 datastore, r: input p=P-r+1; -1 root)

    def c_out(self) -> "_lib.DraftOut":
        return _lib.DraftOut(ptr(self.size), ptr(self.tokens), ptr(self.parents), ptr(self.depths),
                             ptr(self.mask), ptr(self.priority), ptr(self.source), ptr(self.pos))

    def rows(self, r0: int, r1: int) -> "DraftBatch":
        """View of requests [r0, r1)."""
        sl = lambda t: None if t is None else t[r0:r1]  # noqa: E731
        return DraftBatch(self.size[r0:r1], self.tokens[r0:r1], self.parents[r0:r1], self.depths[r0:r1],
                          self.mask[r0:r1], sl(self.ranges), sl(self.samples), sl(self.n_conts), sl(self.p_cut),
                          sl(self.pos), sl(self.priority), sl(self.source))

    @property
    def B(self) -> int:
        return int(self.size.shape[0])


class InputIndex:
    """Incremental per-request input index (the stateful
    analogue of ``InputCache._push``, ref input_cache.py:46-63): request b's
    positions [0, L_b - 1) sorted by (token, position) in device memory, so a
    propose finds the last token's occurrences by binary search and scans only
    the tokens appended since (``sssd_input_index_build`` / ``sssd_propose_ex``).
    Drafts are identical to the stateless scan's."""

    def __init__(self, n_requests: int, cap: int, device, offsets: torch.Tensor | None = None) -> None:
        self.cap = int(cap)
        self.pos_bits = max(1, int(self.cap - 1).bit_length())
        if self.pos_bits > 24:
            raise ValueError(f"index capacity {cap} needs more than 24 position bits")
        self.keys = torch.zeros(max(1, n_requests * self.cap), dtype=torch.int32, device=device)
        self.off = offsets if offsets is not None else (
            torch.arange(n_requests, dtype=torch.int64, device=device) * self.cap)
        self.len = torch.zeros(n_requests, dtype=torch.int32, device=device)

    def c_view(self) -> "_lib.InputIndex":
        return _lib.InputIndex(ptr(self.keys), ptr(self.off), ptr(self.len), self.pos_bits)

    def build(self, seq: torch.Tensor, seq_off: torch.Tensor, seq_len: torch.Tensor, rows=None,
              stream: torch.cuda.Stream | None = None) -> None:
        """(Re)index requests ``rows`` (default all) from their current sequences."""
        B = int(seq_len.shape[0])
        r = None if rows is None else torch.as_tensor(list(rows), dtype=torch.int32).to(seq.device)
        n = B if r is None else int(r.numel())
        seqs = _lib.Seqs(ptr(seq), ptr(seq_off), ptr(seq_len), B, self.cap)
        sp = stream.cuda_stream if stream is not None else stream_ptr(seq.device)
        check(lib().sssd_input_index_build(seqs, self.c_view(), ptr(r), n, sp))


class PendingDrafts:
    """An in-flight ``propose_pinned(..., sync=False)``: ``wait()`` blocks until
    the drafts are in the pinned host buffers and checks the fusion arena."""

    def __init__(self, out_h: "DraftBatch", done, err_h) -> None:
        self.out_h, self.done, self.err_h = out_h, done, err_h

    def wait(self) -> "DraftBatch":
        if self.done is not None:
            self.done.synchronize()
            if int(self.err_h[0]) != 0:
                raise _lib.SSSDError("device workspace overflow (fusion arena) in propose_pinned")
        return self.out_h


class DraftEngine:
    """Drafting for one datastore + config on one GPU."""

    def __init__(self, datastore: Datastore | None, cfg: FusionConfig, separator: int | None = None,
                 use_datastore: bool = True, use_input: bool = True, device=None) -> None:
        if use_datastore and datastore is None:
            raise ValueError("use_datastore=True requires a datastore")
        self.device = torch.device(device) if device is not None else (
            datastore.device if datastore is not None else _lib.require_cuda())
        self.store = datastore
        self.cfg = cfg
        self.separator = separator
        self.use_datastore = use_datastore
        self.use_input = use_input
        if cfg.dec_len > _lib.SSSD_MAX_DRAFT:
            raise ValueError(f"dec_len={cfg.dec_len} exceeds the compiled limit {_lib.SSSD_MAX_DRAFT}")
        if cfg.P > _lib.SSSD_MAX_P:
            raise ValueError(f"P={cfg.P} exceeds the compiled limit {_lib.SSSD_MAX_P}")
        self.c, self._disc = cfg_struct(cfg, separator, use_datastore, use_input, cfg.P, self.device)
        self._ws: torch.Tensor | None = None
        self._ws_key = (0, 0)
        self._out: dict[int, DraftBatch] = {}
        self._null_ds = _lib.Ds(None, None, 0, 0, 0, None, 0, None, 0, 0)

    @property
    def S(self) -> int:
        return self.cfg.dec_len

    @property
    def W(self) -> int:
        return (self.cfg.dec_len + 63) // 64

    def workspace(self, B: int, max_len: int) -> torch.Tensor:
        if self._ws is None or B > self._ws_key[0] or max_len > self._ws_key[1]:
            B2, L2 = max(B, self._ws_key[0]), max(max_len, self._ws_key[1])
            nbytes = lib().sssd_propose_workspace(self.c, B2, L2)
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self._ws_key = (B2, L2)
        return self._ws

    def new_outputs(self, B: int, lookup: bool = False, nodes: bool = False) -> DraftBatch:
        """Fresh device output buffers for a batch of B (``nodes``: also position
        ids, per-node priorities and sources)."""
        dev, S, W, P, M = self.device, self.S, self.W, self.cfg.P, self.cfg.M
        out = DraftBatch(
            size=torch.empty(B, dtype=torch.int32, device=dev),
            tokens=torch.empty((B, S), dtype=torch.int32, device=dev),
            parents=torch.empty((B, S), dtype=torch.int32, device=dev),
            depths=torch.empty((B, S), dtype=torch.int32, device=dev),
            mask=torch.empty((B, S, W), dtype=torch.int64, device=dev),
        )
        if lookup:
            out.ranges = torch.full((B, P, 2), -1, dtype=torch.int64, device=dev)
            out.samples = torch.full((B, P, M), -1, dtype=torch.int64, device=dev)
            out.n_conts = torch.full((B, P), -1, dtype=torch.int32, device=dev)
            out.p_cut = torch.zeros(B, dtype=torch.int32, device=dev)
        if nodes:
            out.pos = torch.empty((B, S), dtype=torch.int32, device=dev)
            out.priority = torch.empty((B, S), dtype=torch.float64, device=dev)
            out.source = torch.empty((B, S), dtype=torch.int32, device=dev)
        return out

    def outputs(self, B: int, lookup: bool = False, nodes: bool = False) -> DraftBatch:
        """The engine's cached output buffers for batch size B (shared by every
        call with the same (B, lookup, nodes): one propose in flight at a time)."""
        key = (B, bool(lookup), bool(nodes))
        out = self._out.get(key)
        if out is None:
            out = self._out[key] = self.new_outputs(B, lookup, nodes)
        return out

    def propose(self, seq: torch.Tensor, seq_off: torch.Tensor, seq_len: torch.Tensor, max_len: int,
                lookup: bool = False, out: DraftBatch | None = None, ws: torch.Tensor | None = None,
                stream: torch.cuda.Stream | None = None, nodes: bool = False,
                index: InputIndex | None = None) -> DraftBatch:
        """Draft for B device-resident sequences: seq (int32 view of u32),
        seq_off [B] int64, seq_len [B] int32 (each >= 1).  Runs on ``stream``
        (default: the current stream) with workspace ``ws`` (default: the
        engine's own; concurrent calls on different streams need their own).
        ``nodes``: also write position ids, node priorities and sources.
        ``index``: an ``InputIndex`` over these requests (N2) instead of the
        stateless context scan (same drafts)."""
        B = int(seq_len.shape[0])
        out = out or self.outputs(B, lookup, nodes)
        if B == 0:
            return out
        if ws is None:
            ws = self.workspace(B, max_len)
        seqs = _lib.Seqs(ptr(seq), ptr(seq_off), ptr(seq_len), B, int(max_len))
        d_out = out.c_out()
        lk = _lib.LookupOut(ptr(out.ranges), ptr(out.samples), ptr(out.n_conts), ptr(out.p_cut)) if lookup else None
        ds = self.store.c_view() if (self.use_datastore and self.store is not None) else self._null_ds
        sp = stream.cuda_stream if stream is not None else stream_ptr(self.device)
        if index is not None:
            check(lib().sssd_propose_ex(ds, seqs, index.c_view(), self.c, d_out, lk, ptr(ws), ws.numel(), sp, None))
        else:
            check(lib().sssd_propose(ds, seqs, self.c, d_out, lk, ptr(ws), ws.numel(), sp))
        return out

    def propose_profile(self, seq, seq_off, seq_len, max_len, index: InputIndex | None = None) -> list[float]:
        """Device ms of [ds_lookup, input_scan, setup, draft] for one propose (synchronises)."""
        import ctypes as C

        B = int(seq_len.shape[0])
        out = self.outputs(B)
        ws = self.workspace(B, max_len)
        seqs = _lib.Seqs(ptr(seq), ptr(seq_off), ptr(seq_len), B, int(max_len))
        ds = self.store.c_view() if (self.use_datastore and self.store is not None) else self._null_ds
        ms = (C.c_float * 4)()
        check(lib().sssd_propose_ex(ds, seqs, index.c_view() if index is not None else None, self.c, out.c_out(),
                                    None, ptr(ws), ws.numel(), stream_ptr(self.device), ms))
        return list(ms)

    def propose_pinned(self, seq_h: torch.Tensor, off_h: torch.Tensor, len_h: torch.Tensor, max_len: int,
                       out_h: DraftBatch | None = None, chunks: int = 5, taper: float = 1.0,
                       tail: float | None = None, schedule: str = "phased", slot: int = 0,
                       sync: bool = True):
        """Host-buffer entry point for a large batch: contexts in pinned host
        memory (seq_h int32 = u32 token ids, or int16 = u16 token ids when the
        vocabulary fits 16 bits: half the upload bytes, widened on the device by
        ``sssd_widen_u16``; off_h int64 [B], len_h int32 [B], CPU tensors),
        drafts returned in pinned host tensors (``out_h``, allocated if None —
        pass it back in to reuse the pinned buffers).

        The batch is cut into ``chunks`` request ranges.  Uploads run on an H2D
        copy stream, drafting alternates between two compute streams with one
        workspace each (so the fusion-kernel tail of range c overlaps the lookup
        and drafting of range c+1), downloads run on a D2H copy stream: PCIe
        both ways and the kernels all run concurrently.  Blocks until the drafts
        are on the host; raises if any range overflowed the fusion arena.

        ``schedule="phased"`` (default, pinned ``seq_h``): one workspace for the
        whole batch; the datastore lookup of every request starts at once from
        its context tail (``sssd_gather_tails`` reads the last P tokens from the
        pinned host buffer), so only the input scan and the fusion follow the
        uploads range by range (``sssd_propose_phase``).  ``"ranges"``: every
        range is an independent propose.

        ``sync=False`` (phased schedule): returns a ``PendingDrafts`` at once
        (``.wait()`` -> the DraftBatch); calls on different ``slot`` s (own
        device buffers each) can then be in flight together, so batch i+1's
        uploads overlap batch i's last drafting and downloads.  Reusing a slot
        (or ``out_h``) requires the previous call on it to have been waited."""
        if schedule == "phased" and seq_h.is_pinned() and (self.use_datastore and self.store is not None):
            return self._propose_pinned_phased(seq_h, off_h, len_h, max_len, out_h, chunks, tail, slot, sync)
        if not sync:
            raise ValueError("sync=False needs the phased schedule (pinned seq_h and a datastore)")
        B = int(len_h.shape[0])
        dev = self.device
        S, W = self.S, self.W
        if out_h is None:
            out_h = DraftBatch(
                size=torch.empty(B, dtype=torch.int32).pin_memory(),
                tokens=torch.empty((B, S), dtype=torch.int32).pin_memory(),
                parents=torch.empty((B, S), dtype=torch.int32).pin_memory(),
                depths=torch.empty((B, S), dtype=torch.int32).pin_memory(),
                mask=torch.empty((B, S, W), dtype=torch.int64).pin_memory())
        if B == 0:
            return out_h
        offs, lens = off_h.numpy(), len_h.numpy()
        if (lens < 1).any():
            raise ValueError("empty prompt: the draft root is the last context token")
        chunks = max(1, min(int(chunks), B))
        # request ranges shrink geometrically (ratio `taper`): the last range's
        # drafting + download is the part no upload hides
        wts = np.power(float(taper), np.arange(chunks))
        if tail is not None and chunks > 1:  # a short last range: less drafting after the last upload
            wts[-1] = float(tail)
        cuts = [0] + [int(round(B * x)) for x in np.cumsum(wts)[:-1] / wts.sum()] + [B]
        bc = max(cuts[c + 1] - cuts[c] for c in range(chunks))
        n_tok = int(seq_h.shape[0])
        st = getattr(self, "_pin", None)
        if st is None:
            st = self._pin = {"streams": [torch.cuda.Stream(dev) for _ in range(4)], "key": None, "ws_key": None}
        narrow = seq_h.dtype == torch.int16
        if not narrow and seq_h.dtype != torch.int32:
            raise ValueError("seq_h must be int32 (u32 tokens) or int16 (u16 tokens)")
        if narrow and (st.get("seq16") is None or st["seq16"].numel() < n_tok):
            st["seq16"] = torch.empty(n_tok, dtype=torch.int16, device=dev)
        if st["key"] != (n_tok, B):
            st["seq"] = torch.empty(n_tok, dtype=torch.int32, device=dev)
            st["off"] = torch.empty(B, dtype=torch.int64, device=dev)
            st["len"] = torch.empty(B, dtype=torch.int32, device=dev)
            st["key"] = (n_tok, B)
        if st["ws_key"] is None or st["ws_key"][0] < bc or st["ws_key"][1] < max_len:
            nbytes = lib().sssd_propose_workspace(self.c, bc, int(max_len))
            st["ws"] = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(2)]
            st["ws_key"] = (bc, int(max_len))
        if st.get("status") is None or st["status"].numel() < chunks:
            st["status"] = torch.zeros(chunks, dtype=torch.int32, device=dev)
        up, down, c0, c1 = st["streams"]
        comp = (c0, c1)
        seq_d, off_d, len_d, status = st["seq"], st["off"], st["len"], st["status"]
        err = [w[_lib.SSSD_STATUS_OFFSET:_lib.SSSD_STATUS_OFFSET + 4].view(torch.int32) for w in st["ws"]]
        main = torch.cuda.current_stream(dev)
        out = self.outputs(B)
        for s_ in st["streams"]:
            s_.wait_stream(main)
        if not (off_h.is_pinned() and len_h.is_pinned()):  # pageable copies would serialise the upload
            pin = st.get("offlen")
            if pin is None or pin[0].numel() < B:
                pin = st["offlen"] = (torch.empty(B, dtype=torch.int64).pin_memory(),
                                      torch.empty(B, dtype=torch.int32).pin_memory())
            pin[0][:B].copy_(off_h)
            pin[1][:B].copy_(len_h)
            off_h, len_h = pin[0][:B], pin[1][:B]
        spans = []  # token span of every request range (computed before any copy is queued)
        for c in range(chunks):
            r0, r1 = cuts[c], cuts[c + 1]
            spans.append((int(offs[r0:r1].min()), int((offs[r0:r1] + lens[r0:r1]).max())))
        with torch.cuda.stream(up):
            uploaded = []
            for c in range(chunks):  # every upload enqueued up front: the copy engine runs ahead
                t0, t1 = spans[c]
                if narrow:
                    st["seq16"][t0:t1].copy_(seq_h[t0:t1], non_blocking=True)
                else:
                    seq_d[t0:t1].copy_(seq_h[t0:t1], non_blocking=True)
                if c == 0:  # offsets / lengths right behind the first range's tokens
                    off_d.copy_(off_h, non_blocking=True)
                    len_d.copy_(len_h, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(up)
                uploaded.append((ev, t0, t1))
        for c in range(chunks):
            r0, r1 = cuts[c], cuts[c + 1]
            cs = comp[c & 1]
            ev_up, t0, t1 = uploaded[c]
            cs.wait_event(ev_up)
            if narrow:
                s16 = st["seq16"]
                check(lib().sssd_widen_u16(s16.data_ptr() + 2 * t0, seq_d.data_ptr() + 4 * t0, t1 - t0,
                                           cs.cuda_stream))
            view = out.rows(r0, r1)
            with torch.cuda.stream(cs):
                self.propose(seq_d, off_d[r0:r1], len_d[r0:r1], max_len, out=view, ws=st["ws"][c & 1], stream=cs)
                status[c:c + 1].copy_(err[c & 1])
                ev = torch.cuda.Event()
                ev.record(cs)
            down.wait_event(ev)
            with torch.cuda.stream(down):
                for dst, src in ((out_h.size, out.size), (out_h.tokens, out.tokens), (out_h.parents, out.parents),
                                 (out_h.depths, out.depths), (out_h.mask, out.mask)):
                    dst[r0:r1].copy_(src[r0:r1], non_blocking=True)
        for s_ in (c0, c1, down):
            main.wait_stream(s_)
        if int(status[:chunks].max().item()) != 0:  # synchronises the current stream
            raise _lib.SSSDError("device workspace overflow (fusion arena) in propose_pinned")
        return out_h

    def _propose_pinned_phased(self, seq_h: torch.Tensor, off_h: torch.Tensor, len_h: torch.Tensor, max_len: int,
                               out_h: DraftBatch | None, chunks: int, tail: float | None = None, slot: int = 0,
                               sync: bool = True):
        B = int(len_h.shape[0])
        dev = self.device
        S, W, P = self.S, self.W, int(self.c.P)
        if out_h is None:
            out_h = DraftBatch(
                size=torch.empty(B, dtype=torch.int32).pin_memory(),
                tokens=torch.empty((B, S), dtype=torch.int32).pin_memory(),
                parents=torch.empty((B, S), dtype=torch.int32).pin_memory(),
                depths=torch.empty((B, S), dtype=torch.int32).pin_memory(),
                mask=torch.empty((B, S, W), dtype=torch.int64).pin_memory())
        if B == 0:
            return out_h if sync else PendingDrafts(out_h, None, None)
        offs, lens = off_h.numpy(), len_h.numpy()
        if (lens < 1).any():
            raise ValueError("empty prompt: the draft root is the last context token")
        narrow = seq_h.dtype == torch.int16
        if not narrow and seq_h.dtype != torch.int32:
            raise ValueError("seq_h must be int32 (u32 tokens) or int16 (u16 tokens)")
        chunks = max(1, min(int(chunks), B))
        # equal ranges; optionally a shorter last one (its drafting + download is what no upload hides)
        wts = np.ones(chunks)
        if tail is not None and chunks > 1:
            wts[-1] = float(tail)
        cuts = [0] + [int(round(B * x)) for x in np.cumsum(wts)[:-1] / wts.sum()] + [B]
        n_tok = int(seq_h.shape[0])
        st = getattr(self, "_pinp", None)
        if st is None:
            st = self._pinp = {"streams": [torch.cuda.Stream(dev) for _ in range(5)], "slots": {}}
        # per-slot device buffers: a call may run while the previous slot's call is in flight
        ss = st["slots"].setdefault(int(slot), {"key": None, "ws_key": None})
        if ss["key"] != (n_tok, B, narrow):
            ss["seq"] = torch.empty(n_tok, dtype=torch.int32, device=dev)
            ss["seq16"] = torch.empty(n_tok, dtype=torch.int16, device=dev) if narrow else None
            ss["off"] = torch.empty(B, dtype=torch.int64, device=dev)
            ss["len"] = torch.empty(B, dtype=torch.int32, device=dev)
            ss["tails"] = torch.empty(B * P, dtype=torch.int32, device=dev)
            ss["toff"] = torch.empty(B, dtype=torch.int64, device=dev)
            ss["tlen"] = torch.empty(B, dtype=torch.int32, device=dev)
            ss["out"] = self.new_outputs(B)  # own buffers: another slot's drafts may still be downloading
            ss["err_h"] = torch.zeros(1, dtype=torch.int32).pin_memory()
            ss["key"] = (n_tok, B, narrow)
        if ss["ws_key"] != (B, int(max_len)):
            ss["ws"] = torch.empty(lib().sssd_propose_workspace(self.c, B, int(max_len)), dtype=torch.uint8,
                                   device=dev)
            ss["ws_key"] = (B, int(max_len))
        up, lk, sc, fu, down = st["streams"]
        seq_d, off_d, len_d, ws, out = ss["seq"], ss["off"], ss["len"], ss["ws"], ss["out"]
        main = torch.cuda.current_stream(dev)
        for s_ in st["streams"]:
            s_.wait_stream(main)
        if not (off_h.is_pinned() and len_h.is_pinned()):  # pageable copies would serialise the upload
            pin = ss.get("offlen")
            if pin is None or pin[0].numel() < B:
                pin = ss["offlen"] = (torch.empty(B, dtype=torch.int64).pin_memory(),
                                      torch.empty(B, dtype=torch.int32).pin_memory())
            pin[0][:B].copy_(off_h)
            pin[1][:B].copy_(len_h)
            off_h, len_h = pin[0][:B], pin[1][:B]
        spans = [(int(offs[cuts[c]:cuts[c + 1]].min()), int((offs[cuts[c]:cuts[c + 1]] + lens[cuts[c]:cuts[c + 1]]).max()))
                 for c in range(chunks)]
        d_out = _lib.DraftOut(ptr(out.size), ptr(out.tokens), ptr(out.parents), ptr(out.depths), ptr(out.mask))
        ds = self.store.c_view()
        full = _lib.Seqs(ptr(seq_d), ptr(off_d), ptr(len_d), B, int(max_len))
        with torch.cuda.stream(up):  # offsets / lengths first, then the token ranges
            off_d.copy_(off_h, non_blocking=True)
            len_d.copy_(len_h, non_blocking=True)
            ev_ol = torch.cuda.Event()
            ev_ol.record(up)
            ev_up = []
            for t0, t1 in spans:
                (ss["seq16"] if narrow else seq_d)[t0:t1].copy_(seq_h[t0:t1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(up)
                ev_up.append(ev)
        # every request's datastore lookup, from its last P tokens read zero-copy
        lk.wait_event(ev_ol)
        tails = _lib.Seqs(ptr(ss["tails"]), ptr(ss["toff"]), ptr(ss["tlen"]), B, P)
        check(lib().sssd_gather_tails(seq_h.data_ptr(), 2 if narrow else 4, ptr(off_d), ptr(len_d), B, P,
                                      ptr(ss["tails"]), ptr(ss["toff"]), ptr(ss["tlen"]), lk.cuda_stream))
        check(lib().sssd_propose_phase(ds, tails, self.c, d_out, None, ptr(ws), ws.numel(),
                                       _lib.SSSD_PHASE_BEGIN | _lib.SSSD_PHASE_LOOKUP, B, int(max_len), 0, B, lk.cuda_stream))
        ev_lk = torch.cuda.Event()
        ev_lk.record(lk)
        fu.wait_event(ev_lk)
        for c in range(chunks):
            r0, r1 = cuts[c], cuts[c + 1]
            t0, t1 = spans[c]
            sc.wait_event(ev_up[c])
            if narrow:
                check(lib().sssd_widen_u16(ss["seq16"].data_ptr() + 2 * t0, seq_d.data_ptr() + 4 * t0, t1 - t0,
                                           sc.cuda_stream))
            check(lib().sssd_propose_phase(ds, full, self.c, d_out, None, ptr(ws), ws.numel(), _lib.SSSD_PHASE_SCAN, B,
                                           int(max_len), r0, r1, sc.cuda_stream))
            ev_sc = torch.cuda.Event()
            ev_sc.record(sc)
            fu.wait_event(ev_sc)
            check(lib().sssd_propose_phase(ds, full, self.c, d_out, None, ptr(ws), ws.numel(), _lib.SSSD_PHASE_FUSE, B,
                                           int(max_len), r0, r1, fu.cuda_stream))
            ev_fu = torch.cuda.Event()
            ev_fu.record(fu)
            down.wait_event(ev_fu)
            with torch.cuda.stream(down):
                for dst, src in ((out_h.size, out.size), (out_h.tokens, out.tokens), (out_h.parents, out.parents),
                                 (out_h.depths, out.depths), (out_h.mask, out.mask)):
                    dst[r0:r1].copy_(src[r0:r1], non_blocking=True)
        err = ws[_lib.SSSD_STATUS_OFFSET:_lib.SSSD_STATUS_OFFSET + 4].view(torch.int32)
        if sync:
            for s_ in (fu, down, sc, lk):
                main.wait_stream(s_)
            if int(err.item()) != 0:  # synchronises the current stream
                raise _lib.SSSDError("device workspace overflow (fusion arena) in propose_pinned")
            return out_h
        with torch.cuda.stream(down):  # after the last fusion (down waited for it) and the last download
            ss["err_h"].copy_(err, non_blocking=True)
            done = torch.cuda.Event()
            done.record(down)
        return PendingDrafts(out_h, done, ss["err_h"])

    def check_status(self) -> None:
        """Synchronise and raise if the device fusion arena overflowed."""
        if self._ws is not None:
            check(lib().sssd_workspace_status(self.c, self._ws_key[0], self._ws_key[1], ptr(self._ws), 0, 0,
                                              stream_ptr(self.device)))

    # -- host convenience --------------------------------------------------------------
    def upload(self, seqs: list) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor, int]:
        lens = [len(s) for s in seqs]
        if any(n < 1 for n in lens):
            raise ValueError("empty prompt: the draft root is the last context token")
        from .datastore import as_u32

        flat = np.concatenate([as_u32(s, "context token") for s in seqs])
        offs = np.zeros(len(seqs), dtype=np.int64)
        np.cumsum(lens[:-1], out=offs[1:])
        dev = self.device
        return (torch.from_numpy(flat.view(np.int32)).to(dev), torch.from_numpy(offs).to(dev),
                torch.tensor(lens, dtype=torch.int32, device=dev), max(lens))

    def propose_host(self, seqs: list, lookup: bool = False):
        from .draft import _drafts_from_device

        seq, off, ln, mx = self.upload(seqs)
        out = self.propose(seq, off, ln, mx, lookup=lookup)
        self.check_status()
        drafts = _drafts_from_device(out.size, out.tokens, out.parents, out.depths, out.mask, len(seqs), self.S)
        return (drafts, out) if lookup else drafts
