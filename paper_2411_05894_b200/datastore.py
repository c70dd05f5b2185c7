"""Device-resident suffix-array datastore (drop-in for ``specdraft.datastore``).

Same public surface as the reference (ref datastore.py:38-304): ``Datastore``
with ``find_range`` / ``get_conts`` / ``save``, ``build``, ``load``,
``read_corpus``, ``sample_range``, ``DatastoreQueryConfig``,
``DatastoreFormatError``; same validation messages and SSSD v1 file format.

Differences are in *where* things live: the corpus and its index stay in HBM
as "suffix rows" (row r = {SA[r], tokens[SA[r]..SA[r]+15)}, 64 B) built by the
GPU suffix-array construction; ``tokens`` / ``suffix_index`` numpy views are
materialised on demand for reference compatibility.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr, stream_ptr
from .trees import ContinuationTree

MAGIC = b"SSSD"
VERSION = 1
_HEADER = struct.Struct("<4sIIQ")


class DatastoreFormatError(ValueError):
    """Malformed datastore file; ``field`` names the bad part (ref datastore.py:38-43)."""

    def __init__(self, field: str, message: str) -> None:
        super().__init__(message)
        self.field = field


@dataclass(frozen=True)
class DatastoreQueryConfig:
    """Knobs of ``Datastore.get_conts`` (ref datastore.py:46-78)."""

    max_prefix_len: int = 4
    sample_cap: int = 100
    min_continuations: int = 16
    branch_len: int = 8
    separator: int | None = None

    def __post_init__(self) -> None:
        for name in ("max_prefix_len", "sample_cap", "min_continuations", "branch_len"):
            v = getattr(self, name)
            if v < 1:
                raise ValueError(f"{name} must be >= 1, got {v}")


def sample_range(lo: int, hi: int, cap: int) -> list[int]:
    """Strided sample of at most ``cap`` ranks of ``[lo, hi)`` (ref datastore.py:112-126).
    Host-side formula; the device computes the same ranks inside the lookup kernel."""
    if lo > hi:
        raise ValueError(f"invalid interval: lo={lo} > hi={hi}")
    if cap < 1:
        raise ValueError(f"cap must be >= 1, got {cap}")
    width = hi - lo
    if width <= cap:
        return list(range(lo, hi))
    return [lo + (k * width) // cap for k in range(cap)]


def as_u32(tokens, what: str = "token") -> np.ndarray:
    """Token ids -> <u4, rejecting ids outside [0, 2^32) (they cannot be
    represented on the device; silently wrapping them would make them match
    real corpus tokens, which the reference's exact int compare never does)."""
    a = np.asarray(tokens)
    if a.size == 0:
        return np.zeros(0, dtype="<u4")
    if a.dtype.kind not in "iu":
        a = np.asarray([int(x) for x in np.ravel(a)], dtype=object).reshape(a.shape)
        lo, hi = (int(a.min()), int(a.max()))
    else:
        lo, hi = int(a.min()), int(a.max())
    if lo < 0 or hi > 0xFFFFFFFF:
        bad = lo if lo < 0 else hi
        raise ValueError(f"{what} id {bad} out of range for uint32")
    return np.ascontiguousarray(a.astype(np.int64) if a.dtype == object else a, dtype=np.int64).astype("<u4")


def _u32_device(arr: np.ndarray, device) -> torch.Tensor:
    a = np.ascontiguousarray(arr, dtype="<u4")
    return torch.from_numpy(a.view(np.int32)).to(device, non_blocking=False)


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


class Datastore:
    """Token corpus + suffix rows resident on one GPU.

    ``Datastore(tokens, suffix_index, vocab_size=None)`` is the reference
    constructor (ref datastore.py:144-154): host arrays, uploaded and indexed
    into suffix rows on the current GPU.  ``Datastore.on_device`` wraps rows
    already built on a device (``build``, ``load``, shards)."""

    def __init__(self, tokens, suffix_index, vocab_size: int | None = None, device=None) -> None:
        dev = torch.device(device) if device is not None else _lib.require_cuda()
        toks = np.ascontiguousarray(np.asarray(tokens), dtype="<u4")
        n = int(toks.size)
        tok = _device_tokens(toks, dev)
        sa = torch.from_numpy(np.ascontiguousarray(suffix_index, dtype=np.int64).astype(np.int32)).to(dev)
        self._init(tok, _rows_from_sa(tok, n, sa), n, vocab_size)
        self._np_tokens = toks

    @classmethod
    def on_device(cls, tokens_dev: torch.Tensor, rows_dev: torch.Tensor, n: int, vocab_size: int | None = None,
                  rank_base: int = 0, n_tokens: int | None = None) -> "Datastore":
        self = cls.__new__(cls)
        self._init(tokens_dev, rows_dev, n, vocab_size, rank_base, n_tokens)
        return self

    def _init(self, tokens_dev: torch.Tensor, rows_dev: torch.Tensor, n: int, vocab_size: int | None = None,
              rank_base: int = 0, n_tokens: int | None = None) -> None:
        self._tok = tokens_dev  # int32 view of <u4 tokens (length n_tokens + 16 pad)
        self._rows = rows_dev  # [n_rows, 16] int32
        self.n_rows = int(n)
        self._n_tokens = int(n if n_tokens is None else n_tokens)
        self.rank_base = int(rank_base)
        self.vocab_size = vocab_size
        self._np_tokens: np.ndarray | None = None
        self._np_sa: np.ndarray | None = None
        self._bucket: torch.Tensor | None = None
        self._kix: torch.Tensor | None = None
        self._kix_done = False
        # the index tables are built here, not on first use: a first use can sit
        # inside a CUDA-graph capture (the decode loops), where the k-gram count
        # readback would capture instead of run
        if self.n_rows > 0:
            self.bucket()
            self.kix()

    # -- reference-compatible views -------------------------------------------------
    @property
    def device(self) -> torch.device:
        return self._rows.device

    @property
    def n_tokens(self) -> int:
        return self._n_tokens

    @property
    def tokens(self) -> np.ndarray:
        if self._np_tokens is None:
            self._np_tokens = self._tok[: self._n_tokens].cpu().numpy().view("<u4").copy()
        return self._np_tokens

    @property
    def suffix_index(self) -> np.ndarray:
        if self._np_sa is None:
            self._np_sa = self.sa64_device().cpu().numpy().astype(np.int64)
        return self._np_sa

    def check(self) -> dict:
        """Full-size verification of the index on the device (``sssd_sa_check``):
        adjacent suffix rows strictly increasing and the SA column a permutation
        of [0, n_tokens) -- together, the unique suffix array."""
        dev = self.device
        ws = _workspace(lib().sssd_sa_check_workspace(self._n_tokens), dev)
        cnt = torch.zeros(3, dtype=torch.int64, device=dev)
        check(lib().sssd_sa_check(ptr(self._tok), self._n_tokens, ptr(self._rows), self.n_rows, ptr(ws), ws.numel(),
                                  ptr(cnt), stream_ptr(dev)))
        c = cnt.cpu().tolist()
        return {"adjacent_not_increasing": c[0], "positions_missing": c[1] if self.n_rows == self._n_tokens else None,
                "positions_out_of_range": c[2], "ok": c[0] == 0 and c[2] == 0 and
                (c[1] == 0 or self.n_rows != self._n_tokens)}

    def sa64_device(self) -> torch.Tensor:
        out = torch.empty(self.n_rows, dtype=torch.int64, device=self.device)
        check(lib().sssd_rows_sa64(ptr(self._rows), self.n_rows, ptr(out), stream_ptr(self.device)))
        return out

    # first-token index over the (local) suffix rows: narrows every range search
    # to the rows starting with the pattern's first token (same bounds)
    MAX_BUCKETS = 1 << 22

    def bucket(self) -> torch.Tensor:
        if self._bucket is None:
            nb = min(int(self.vocab_size) if self.vocab_size else 65536, self.MAX_BUCKETS)
            self._bucket = torch.empty(nb + 1, dtype=torch.int32, device=self.device)
            check(lib().sssd_bucket_build(ptr(self._rows), self.n_rows, nb, ptr(self._bucket),
                                          stream_ptr(self.device)))
        return self._bucket

    # k-gram range index (sssd_kix_build): the exact (local) row range of every
    # 2..4-gram that starts a suffix, so lookups of patterns up to 4 tokens need
    # no search.  A shard's table gives exact local ranges of the k-grams it
    # holds; its absent patterns are still searched (the summed bounds need
    # their local insertion points).  SSSD_NO_KIX=1 disables it (A/B switch).
    KIX_KMAX = 4

    def kix(self) -> torch.Tensor | None:
        if not self._kix_done:
            self._kix_done = True
            if self.n_rows > 0 and os.environ.get("SSSD_NO_KIX", "0") in ("", "0"):
                dev = self.device
                cnt = torch.zeros(1, dtype=torch.int64, device=dev)
                check(lib().sssd_kix_count(ptr(self._rows), self.n_rows, self._n_tokens, self.KIX_KMAX, ptr(cnt),
                                           stream_ptr(dev)))
                cap = 1024
                while cap < 2 * int(cnt.item()):
                    cap <<= 1
                self._kix = torch.empty(cap * 4, dtype=torch.int32, device=dev)
                check(lib().sssd_kix_build(ptr(self._rows), self.n_rows, self._n_tokens, self.KIX_KMAX,
                                           ptr(self._kix), cap, stream_ptr(dev)))
        return self._kix

    def c_view(self) -> _lib.Ds:
        bk = self.bucket() if self.n_rows > 0 else None
        kx = self.kix()
        return _lib.Ds(ptr(self._rows), ptr(self._tok), self._n_tokens, self.rank_base, self.n_rows,
                       ptr(bk) if bk is not None else None, (bk.numel() - 1) if bk is not None else 0,
                       ptr(kx) if kx is not None else None, (kx.numel() // 4 - 1) if kx is not None else 0,
                       self.KIX_KMAX if kx is not None else 0)

    @property
    def rows(self) -> torch.Tensor:
        return self._rows

    @property
    def token_tensor(self) -> torch.Tensor:
        return self._tok

    # -- queries ----------------------------------------------------------------------
    def find_ranges(self, prefixes: Sequence[Sequence[int]]) -> list[tuple[int, int]]:
        """Batched ``find_range`` in one launch (one warp per prefix)."""
        pats = [[int(t) for t in p] for p in prefixes]
        if any(not p for p in pats):
            raise ValueError("prefix must be non-empty")
        if not pats:
            return []
        dev = self.device
        flat = as_u32(np.concatenate([as_u32(p, "prefix token") for p in pats]), "prefix token")
        offs = np.zeros(len(pats), dtype=np.int64)
        np.cumsum([len(p) for p in pats[:-1]], out=offs[1:])
        d_pat = _u32_device(flat, dev)
        d_off = torch.from_numpy(offs).to(dev)
        d_len = torch.tensor([len(p) for p in pats], dtype=torch.int32, device=dev)
        out = torch.empty(2 * len(pats), dtype=torch.int64, device=dev)
        view = self.c_view()
        check(lib().sssd_find_ranges(view, ptr(d_pat), ptr(d_off), ptr(d_len), len(pats), ptr(out),
                                     stream_ptr(dev)))
        o = out.cpu().tolist()
        return [(o[2 * i], o[2 * i + 1]) for i in range(len(pats))]

    def find_range(self, prefix: Sequence[int]) -> tuple[int, int]:
        """``[lo, hi)`` of suffix-array ranks starting with ``prefix`` (ref datastore.py:156-183)."""
        return self.find_ranges([prefix])[0]

    def get_conts(self, prefix: Sequence[int], cfg: DatastoreQueryConfig) -> ContinuationTree:
        """Continuation tree of the longest usable suffixes of ``prefix`` (ref datastore.py:185-218)."""
        prefix = [int(t) for t in prefix]
        if not prefix:
            raise ValueError("prefix must be non-empty")
        from .fusion import _cfg_struct  # local: fusion imports datastore

        c, keep = _cfg_struct(P=cfg.max_prefix_len, dec_len=1, branch_len=cfg.branch_len,
                              input_branch_len=1, M=cfg.sample_cap, T=cfg.min_continuations,
                              separator=cfg.separator, device=self.device)
        paths = ds_paths(self, [prefix], c)[0]
        tree = ContinuationTree()
        for p in paths:
            tree.add_path(p)
        return tree

    def save(self, path: str | os.PathLike) -> None:
        """SSSD v1 file (ref datastore.py:11-19,220-226)."""
        with open(path, "wb") as fh:
            fh.write(_HEADER.pack(MAGIC, VERSION, self.vocab_size or 0, self.n_tokens))
            fh.write(np.ascontiguousarray(self.tokens, dtype="<u4").tobytes())
            fh.write(np.ascontiguousarray(self.suffix_index, dtype="<u8").tobytes())


def ds_paths(store: Datastore, prefixes: list[list[int]], c) -> list[list[list[int]]]:
    """Run the device lookup for a batch of prefixes and return, per prefix, the
    evaluated continuation paths in the reference's insertion order."""
    dev = store.device
    B = len(prefixes)
    P, M, BL = c.P, c.M, c.branch_len
    seq = np.concatenate([np.asarray(p, dtype=np.int64) for p in prefixes]).astype("<u4")
    offs = np.zeros(B, dtype=np.int64)
    np.cumsum([len(p) for p in prefixes[:-1]], out=offs[1:])
    d_seq = _u32_device(seq, dev)
    d_off = torch.from_numpy(offs).to(dev)
    d_len = torch.tensor([len(p) for p in prefixes], dtype=torch.int32, device=dev)
    seqs = _lib.Seqs(ptr(d_seq), ptr(d_off), ptr(d_len), B, max(len(p) for p in prefixes))
    tab = torch.zeros(B * P * M * BL, dtype=torch.int32, device=dev)
    lens = torch.zeros(B * P * M, dtype=torch.uint8, device=dev)
    el = torch.zeros(B * P * M * 4, dtype=torch.int32, device=dev)
    n_el = torch.zeros(B, dtype=torch.int32, device=dev)
    view = store.c_view()
    ws = _workspace(lib().sssd_ds_lookup_workspace(c, B), dev)
    check(lib().sssd_ds_lookup(view, seqs, c, ptr(tab), ptr(lens), ptr(el), ptr(n_el), None,
                               ptr(ws), ws.numel(), stream_ptr(dev)))
    tab_h = tab.cpu().numpy().view("<u4")
    el_h = el.cpu().numpy().view("<u4").reshape(B, P * M, 4)
    n_h = n_el.cpu().tolist()
    out = []
    for b in range(B):
        rows = el_h[b, : n_h[b]]
        order = np.argsort(rows[:, 1], kind="stable")
        base = b * P * M * BL
        out.append([tab_h[base + int(r[0]): base + int(r[0]) + int(r[2] & 0xFF)].tolist()
                    for r in rows[order]])
    return out


def _validate_corpus(corpus, vocab_size) -> np.ndarray:
    tokens = np.ascontiguousarray(np.asarray(corpus), dtype="<u4")
    if tokens.ndim != 1:
        raise ValueError(f"corpus must be one-dimensional, got shape {tokens.shape}")
    if tokens.size == 0:
        raise ValueError("empty corpus")
    if vocab_size is not None:
        if vocab_size < 1:
            raise ValueError(f"vocab_size must be >= 1, got {vocab_size}")
        top = int(tokens.max())
        if top >= vocab_size:
            raise ValueError(f"token id {top} out of range for vocab_size {vocab_size}")
    return tokens


def _device_tokens(tokens: np.ndarray, device) -> torch.Tensor:
    pad = np.zeros(tokens.size + 16, dtype="<u4")
    pad[: tokens.size] = tokens
    return _u32_device(pad, device)


def _rows_from_sa(tok_dev: torch.Tensor, n: int, sa_dev: torch.Tensor) -> torch.Tensor:
    rows = torch.empty((n, 16), dtype=torch.int32, device=tok_dev.device)
    assert rows.data_ptr() % 64 == 0
    check(lib().sssd_rows_build(ptr(tok_dev), n, ptr(sa_dev), ptr(rows), stream_ptr(tok_dev.device)))
    return rows


def build_device(tok_dev: torch.Tensor, n: int) -> torch.Tensor:
    """GPU suffix array (u32 as int32) of the first n tokens of tok_dev."""
    dev = tok_dev.device
    sa = torch.empty(n, dtype=torch.int32, device=dev)
    ws = _workspace(lib().sssd_sa_build_workspace(n), dev)
    check(lib().sssd_sa_build(ptr(tok_dev), n, ptr(sa), ptr(ws), ws.numel(), stream_ptr(dev)))
    return sa


def build_suffix_array(tokens: np.ndarray, device=None) -> np.ndarray:
    """Suffix array of a host token array (ref datastore.py:81-109), computed on
    the GPU by radix-sort prefix doubling; int64 like the reference's."""
    toks = np.ascontiguousarray(np.asarray(tokens), dtype="<u4")
    n = int(toks.size)
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    dev = torch.device(device) if device is not None else _lib.require_cuda()
    return build_device(_device_tokens(toks, dev), n).cpu().numpy().view(np.uint32).astype(np.int64)


def build(corpus: Sequence[int] | np.ndarray, vocab_size: int | None = None,
          device: torch.device | str | None = None) -> Datastore:
    """Index ``corpus`` on the GPU (ref datastore.py:229-242): suffix array by
    radix-sort prefix doubling, then the suffix rows."""
    tokens = _validate_corpus(corpus, vocab_size)
    dev = torch.device(device) if device is not None else _lib.require_cuda()
    n = int(tokens.size)
    if n >= 0xFFFFFFFF:
        raise ValueError("corpus longer than 2^32-1 tokens is not supported on one GPU")
    tok = _device_tokens(tokens, dev)
    sa = build_device(tok, n)
    rows = _rows_from_sa(tok, n, sa)
    ds = Datastore.on_device(tok, rows, n, vocab_size)
    ds._np_tokens = tokens
    return ds


def from_arrays(tokens: np.ndarray, suffix_index: np.ndarray, vocab_size: int | None = None,
                device=None) -> Datastore:
    """Datastore over a precomputed suffix array (e.g. one loaded from disk)."""
    return Datastore(tokens, suffix_index, vocab_size, device=device)


def _read_exact(fh, nbytes: int, field: str) -> bytes:
    data = fh.read(nbytes)
    if len(data) != nbytes:
        raise DatastoreFormatError(field, f"truncated {field}: expected {nbytes} bytes, got {len(data)}")
    return data


def load(path: str | os.PathLike, device=None) -> Datastore:
    """Load and validate an SSSD v1 file (ref datastore.py:254-283), then upload."""
    with open(path, "rb") as fh:
        magic, version, vocab, n = _HEADER.unpack(_read_exact(fh, _HEADER.size, "header"))
        if magic != MAGIC:
            raise DatastoreFormatError("magic", f"bad magic: expected {MAGIC!r}, got {magic!r}")
        if version != VERSION:
            raise DatastoreFormatError("version", f"unsupported version {version}, expected {VERSION}")
        if n == 0:
            raise DatastoreFormatError("n_tokens", "n_tokens is zero (empty corpus)")
        tokens = np.frombuffer(_read_exact(fh, 4 * n, "tokens"), dtype="<u4")
        sa = np.frombuffer(_read_exact(fh, 8 * n, "suffix_index"), dtype="<u8")
        if fh.read(1):
            raise DatastoreFormatError("trailer", "trailing bytes after suffix array")
    if sa.size and int(sa.max()) >= n:
        raise DatastoreFormatError("suffix_index",
                                   f"suffix position {int(sa.max())} out of range for {n} tokens")
    vocab = int(vocab) or None
    if vocab is not None and int(tokens.max()) >= vocab:
        raise DatastoreFormatError("tokens", f"token id {int(tokens.max())} out of range for vocab_size {vocab}")
    ds = from_arrays(tokens.copy(), sa.astype(np.int64), vocab, device)
    ds._np_sa = sa.astype(np.int64)
    return ds


def read_corpus(path: str | os.PathLike) -> np.ndarray:
    """Raw little-endian u32 (``.tok``) or whitespace-separated decimal text (ref datastore.py:286-304)."""
    path = os.fspath(path)
    if path.endswith(".tok"):
        return np.fromfile(path, dtype="<u4")
    with open(path, "r", encoding="utf-8") as fh:
        fields = fh.read().split()
    out = np.empty(len(fields), dtype="<u4")
    for i, f in enumerate(fields):
        try:
            v = int(f)
        except ValueError as exc:
            raise ValueError(f"{path}: token #{i + 1}: not a decimal integer: {f!r}") from exc
        if not 0 <= v < 2**32:
            raise ValueError(f"{path}: token #{i + 1}: {v} outside u32 range")
        out[i] = v
    return out
