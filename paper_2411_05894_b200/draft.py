"""Flattened drafts, masks, greedy verification and sessions (drop-in for
``specdraft.draft``, ref draft.py:29-216).

``GenerationSession.propose`` and ``verify_greedy`` run on the GPU
(``sssd_propose`` / ``sssd_accept``); the containers and the bit-packing
helpers are host utilities with the reference's exact byte formats.
"""

from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field
from time import perf_counter
from typing import Protocol, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr, stream_ptr
from .datastore import Datastore, as_u32
from .fusion import DraftTree, FusionConfig


class Oracle(Protocol):
    """Anything that names the greedy next token for a context (ref draft.py:29-32)."""

    def next(self, context: Sequence[int]) -> int: ...


@dataclass
class AcceptResult:
    accepted_path: list[int]
    bonus_token: int

    @property
    def tokens_emitted(self) -> int:
        return len(self.accepted_path) + 1


@dataclass
class FlattenedDraft:
    """DFS arrays of one draft (ref draft.py:48-64); ``mask[i, j]`` = j is i or an ancestor."""

    tokens: list[int]
    parents: list[int]
    depths: list[int]
    mask: np.ndarray

    @property
    def s_q(self) -> int:
        return len(self.tokens)


def _mask_from_words(words: np.ndarray, n: int) -> np.ndarray:
    """u64 ancestor words [n, W] -> bool [n, n]."""
    bits = np.unpackbits(words.astype("<u8").view(np.uint8).reshape(n, -1), axis=1, bitorder="little")
    return bits[:, :n].astype(bool)


def _drafts_from_device(size, toks, par, dep, mask, B: int, S: int) -> list[FlattenedDraft]:
    W = (S + 63) // 64
    size_h = size.cpu().numpy()
    tok_h = toks.reshape(B, S).cpu().numpy().view(np.uint32)
    par_h = par.reshape(B, S).cpu().numpy()
    dep_h = dep.reshape(B, S).cpu().numpy()
    mask_h = mask.reshape(B, S, W).cpu().numpy().view(np.uint64)
    out = []
    for b in range(B):
        n = int(size_h[b])
        out.append(FlattenedDraft([int(x) for x in tok_h[b, :n]], [int(x) for x in par_h[b, :n]],
                                  [int(x) for x in dep_h[b, :n]], _mask_from_words(mask_h[b, :n], n)))
    return out


def flatten(tree: DraftTree) -> FlattenedDraft:
    """DFS pre-order of a caller-built ``DraftTree`` (ref draft.py:67-86).  Host
    traversal of a host object: drafts produced by the engine are flattened on
    the device inside ``draft_kernel``."""
    tokens, parents, depths = [], [], []
    stack = [(tree.root, -1)]
    while stack:
        node, par = stack.pop()
        idx = len(tokens)
        tokens.append(node.token)
        parents.append(par)
        depths.append(0 if par < 0 else depths[par] + 1)
        stack.extend((c, idx) for c in reversed(list(node.children.values())))
    n = len(tokens)
    mask = np.zeros((n, n), dtype=bool)
    for i in range(n):
        j = i
        while j >= 0:
            mask[i, j] = True
            j = parents[j]
    return FlattenedDraft(tokens, parents, depths, mask)


def pack_mask(mask: np.ndarray) -> bytes:
    """u64 row count, then row-major LSB-first bits (ref draft.py:89-93)."""
    n = mask.shape[0]
    return struct.pack("<Q", n) + np.packbits(mask.reshape(-1).astype(np.uint8), bitorder="little").tobytes()


def unpack_mask(data: bytes) -> np.ndarray:
    if len(data) < 8:
        raise ValueError(f"truncated mask: {len(data)} bytes is shorter than the header")
    (n,) = struct.unpack_from("<Q", data)
    need = 8 + (n * n + 7) // 8
    if len(data) != need:
        raise ValueError(f"truncated mask: expected {need} bytes for {n} rows, got {len(data)}")
    bits = np.unpackbits(np.frombuffer(data, dtype=np.uint8, offset=8), count=n * n, bitorder="little")
    return bits.reshape(n, n).astype(bool)


def mask_debug_json(mask: np.ndarray) -> str:
    n = mask.shape[0]
    return json.dumps({"size": n, "ancestors": [sorted(int(j) for j in np.nonzero(mask[i])[0]) for i in range(n)]})


def verify_batch(drafts: Sequence[FlattenedDraft], predictions: Sequence[Sequence[int]], device=None):
    """GPU greedy accept for B drafts (ref draft.py:114-138): one ``sssd_accept`` launch."""
    dev = torch.device(device) if device is not None else _lib.require_cuda()
    B = len(drafts)
    for d, p in zip(drafts, predictions):
        if len(p) != d.s_q:
            raise ValueError(f"length mismatch: {len(p)} predictions for {d.s_q} draft nodes")
    if B == 0:
        return []
    # sssd_accept walks children at indices above their parent (DFS / any
    # topological numbering).  A caller-built draft numbered otherwise is
    # renumbered by (depth, index) -- parents first, siblings in index order, so
    # the first-index-wins rule of ref draft.py:127-128 is unchanged -- and the
    # accepted path mapped back.
    perms: list = [None] * B
    for b, d in enumerate(drafts):
        if all(0 <= d.parents[i] < i for i in range(1, d.s_q)):
            continue
        depth = [0] * d.s_q
        for i in range(1, d.s_q):
            j, k = i, 0
            while j > 0 and k <= d.s_q:
                j, k = d.parents[j], k + 1
            depth[i] = k if j == 0 else d.s_q + 1  # unreachable from the root: never accepted
        perm = sorted(range(d.s_q), key=lambda i: (depth[i], i))
        new = {old_i: n for n, old_i in enumerate(perm)}
        par2 = [-1] + [new.get(d.parents[o], -1) if depth[o] <= d.s_q else -1 for o in perm[1:]]
        drafts = list(drafts)
        predictions = list(predictions)
        drafts[b] = FlattenedDraft([d.tokens[o] for o in perm], par2, [depth[o] for o in perm], d.mask)
        predictions[b] = [predictions[b][o] for o in perm]
        perms[b] = perm
    S = max(d.s_q for d in drafts)
    odd: list[dict] = [{} for _ in range(B)]  # out-of-range predictions by node
    tok = np.zeros((B, S), dtype=np.uint32)
    par = np.full((B, S), -1, dtype=np.int32)
    prd = np.zeros((B, S), dtype=np.uint32)
    for b, (d, p) in enumerate(zip(drafts, predictions)):
        tok[b, : d.s_q] = as_u32(d.tokens, "draft token")
        par[b, : d.s_q] = d.parents
        pv = [int(x) for x in p]
        if any(x < 0 or x > 0xFFFFFFFF for x in pv):
            # a prediction no u32 draft token can equal: stand in a value absent
            # from this draft (the walk stops there, as the reference's exact
            # compare does); the bonus is restored below
            free = next(v for v in range(d.s_q + 1) if v not in set(int(t) for t in d.tokens))
            odd[b] = {i: x for i, x in enumerate(pv) if x < 0 or x > 0xFFFFFFFF}
            pv = [free if i in odd[b] else x for i, x in enumerate(pv)]
        prd[b, : d.s_q] = np.asarray(pv, dtype=np.int64).astype(np.uint32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).to(dev)  # noqa: E731
    d_tok, d_par, d_prd = t(tok), t(par), t(prd)
    d_size = torch.tensor([d.s_q for d in drafts], dtype=torch.int32, device=dev)
    seq = torch.zeros(1, dtype=torch.int32, device=dev)
    zeros64 = torch.zeros(B, dtype=torch.int64, device=dev)
    zeros32 = torch.zeros(B, dtype=torch.int32, device=dev)
    path = torch.full((B, S), -1, dtype=torch.int32, device=dev)
    n_acc = torch.empty(B, dtype=torch.int32, device=dev)
    bonus = torch.empty(B, dtype=torch.int32, device=dev)
    emitted = torch.empty(B, dtype=torch.int32, device=dev)
    seq_len = zeros32.clone()
    check(lib().sssd_accept(ptr(d_tok), ptr(d_par), ptr(d_size), S, ptr(d_prd), B, ptr(seq), ptr(zeros64),
                            ptr(seq_len), ptr(zeros32), ptr(path), ptr(n_acc), ptr(bonus), ptr(emitted),
                            stream_ptr(dev)))
    na = n_acc.cpu().tolist()
    ph = path.cpu().tolist()
    bh = bonus.cpu().numpy().view(np.uint32).tolist()
    res = []
    for b in range(B):
        path = ph[b][: na[b]]
        last = path[-1] if path else 0
        bonus_b = odd[b].get(last, int(bh[b]))
        res.append(AcceptResult(path if perms[b] is None else [perms[b][i] for i in path], bonus_b))
    return res


def verify_greedy(draft: FlattenedDraft, node_predictions: Sequence[int]) -> AcceptResult:
    """Accept the chain of draft tokens matching the predictions (ref draft.py:114-138)."""
    return verify_batch([draft], [list(node_predictions)])[0]


@dataclass
class GenerationSession:
    """One request: sequence + both retrieval sources (ref draft.py:141-216).
    ``propose`` is a B=1 call into the batched GPU engine; ``step`` asks the
    host ``Oracle`` for every node, then verifies on the GPU."""

    datastore: Datastore | None
    cfg: FusionConfig
    sequence: list[int]
    separator: int | None = None
    use_datastore: bool = True
    use_input: bool = True
    retrieval_seconds: float = 0.0
    steps: int = 0
    _engine: object = field(default=None, repr=False)

    @classmethod
    def start(cls, datastore: Datastore | None, prompt: Sequence[int], cfg: FusionConfig,
              separator: int | None = None, use_datastore: bool = True,
              use_input: bool = True) -> "GenerationSession":
        prompt = [int(t) for t in prompt]
        if not prompt:
            raise ValueError("empty prompt: the draft root is the last context token")
        if use_datastore and datastore is None:
            raise ValueError("use_datastore=True requires a datastore")
        from .engine import DraftEngine

        eng = DraftEngine(datastore, cfg, separator, use_datastore, use_input)
        return cls(datastore, cfg, list(prompt), separator, use_datastore, use_input, _engine=eng)

    @property
    def cache(self):
        from .input_cache import InputCache

        return InputCache(self.sequence, self.cfg.P, self.cfg.input_branch_len)

    def propose(self) -> FlattenedDraft:
        t0 = perf_counter()
        flat = self._engine.propose_host([self.sequence])[0]
        self.retrieval_seconds += perf_counter() - t0
        return flat

    def step(self, oracle: Oracle) -> AcceptResult:
        flat = self.propose()
        contexts: list[list[int]] = [self.sequence]
        preds = [int(oracle.next(self.sequence))]
        for i in range(1, flat.s_q):
            ctx = contexts[flat.parents[i]] + [flat.tokens[i]]
            contexts.append(ctx)
            preds.append(int(oracle.next(ctx)))
        res = verify_greedy(flat, preds)
        self.sequence.extend([flat.tokens[i] for i in res.accepted_path] + [res.bonus_token])
        self.steps += 1
        return res
