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

    @property
    def B(self) -> int:
        return int(self.size.shape[0])


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
        self._null_ds = _lib.Ds(None, None, 0, 0, 0)

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

    def outputs(self, B: int, lookup: bool = False) -> DraftBatch:
        key = B * 2 + int(lookup)
        out = self._out.get(key)
        if out is None:
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
            self._out[key] = out
        return out

    def propose(self, seq: torch.Tensor, seq_off: torch.Tensor, seq_len: torch.Tensor, max_len: int,
                lookup: bool = False, out: DraftBatch | None = None) -> DraftBatch:
        """Draft for B device-resident sequences: seq (int32 view of u32),
        seq_off [B] int64, seq_len [B] int32 (each >= 1)."""
        B = int(seq_len.shape[0])
        out = out or self.outputs(B, lookup)
        if B == 0:
            return out
        ws = self.workspace(B, max_len)
        seqs = _lib.Seqs(ptr(seq), ptr(seq_off), ptr(seq_len), B, int(max_len))
        d_out = _lib.DraftOut(ptr(out.size), ptr(out.tokens), ptr(out.parents), ptr(out.depths), ptr(out.mask))
        lk = _lib.LookupOut(ptr(out.ranges), ptr(out.samples), ptr(out.n_conts), ptr(out.p_cut)) if lookup else None
        ds = self.store.c_view() if (self.use_datastore and self.store is not None) else self._null_ds
        check(lib().sssd_propose(ds, seqs, self.c, d_out, lk, ptr(ws), ws.numel(), stream_ptr(self.device)))
        return out

    def propose_profile(self, seq, seq_off, seq_len, max_len) -> list[float]:
        """Device ms of [ds_lookup, input_scan, setup, draft] for one propose (synchronises)."""
        import ctypes as C

        B = int(seq_len.shape[0])
        out = self.outputs(B)
        ws = self.workspace(B, max_len)
        seqs = _lib.Seqs(ptr(seq), ptr(seq_off), ptr(seq_len), B, int(max_len))
        d_out = _lib.DraftOut(ptr(out.size), ptr(out.tokens), ptr(out.parents), ptr(out.depths), ptr(out.mask))
        ds = self.store.c_view() if (self.use_datastore and self.store is not None) else self._null_ds
        ms = (C.c_float * 4)()
        check(lib().sssd_propose_profile(ds, seqs, self.c, d_out, ptr(ws), ws.numel(), stream_ptr(self.device), ms))
        return list(ms)

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
        flat = np.concatenate([np.asarray(s, dtype=np.int64) for s in seqs]).astype(np.uint32)
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
