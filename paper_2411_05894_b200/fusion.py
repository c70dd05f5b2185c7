"""Fusion of source tries into one bounded draft tree (drop-in for ``specdraft.fusion``).

``FusionConfig`` / ``Source`` / ``discount`` / ``DraftNode`` / ``DraftTree``
keep the reference semantics (ref fusion.py:29-206).  ``merge`` runs on the
GPU: the caller's trees are serialised as path multisets, sorted on the
device, and fused by the same best-first kernel the batched propose uses
(``draft_kernel``, ref fusion.py:209-261).
"""

from __future__ import annotations

import functools
import math
import os
from dataclasses import dataclass, fields, replace
from typing import Iterable, Mapping, Sequence

import numpy as np
import torch

from . import _lib, kvconfig
from ._lib import check, lib, ptr, stream_ptr
from .datastore import Datastore, DatastoreQueryConfig
from .trees import ContinuationTree

_INT_KEYS = ("P", "dec_len", "branch_len", "input_branch_len", "M", "T")
_FLOAT_KEYS = ("alpha", "beta", "gamma_ds", "gamma_in")


@dataclass(frozen=True)
class FusionConfig:
    """Drafting knobs (ref fusion.py:29-113)."""

    P: int = 4
    dec_len: int = 30
    branch_len: int | None = None
    input_branch_len: int = 8
    M: int = 100
    T: int = 16
    alpha: float = 0.8
    beta: float = 0.8
    gamma_ds: float = 1.0
    gamma_in: float = 0.95

    def __post_init__(self) -> None:
        if self.branch_len is None:
            object.__setattr__(self, "branch_len", max(1, min(8, self.dec_len - 1)))
        for name in ("P", "dec_len", "branch_len", "input_branch_len", "M", "T"):
            v = getattr(self, name)
            if v < 1:
                raise ValueError(f"{name} must be >= 1, got {v}")
        if not 0.0 <= self.alpha <= 1.0:
            raise ValueError(f"alpha must be in [0, 1], got {self.alpha}")
        for name in ("beta", "gamma_ds", "gamma_in"):
            v = getattr(self, name)
            if not 0.0 < v <= 1.0:
                raise ValueError(f"{name} must be in (0, 1], got {v}")

    def query_config(self, separator: int | None = None) -> DatastoreQueryConfig:
        return DatastoreQueryConfig(max_prefix_len=self.P, sample_cap=self.M,
                                    min_continuations=self.T, branch_len=self.branch_len,
                                    separator=separator)

    def to_kv(self) -> dict[str, object]:
        return {f.name: getattr(self, f.name) for f in fields(self)}

    def to_file(self, path: str | os.PathLike) -> None:
        kvconfig.write_kv(path, self.to_kv())

    @classmethod
    def from_kv(cls, items: Mapping[str, str], base: "FusionConfig | None" = None) -> "FusionConfig":
        values: dict[str, object] = {}
        for key, raw in items.items():
            if key in _INT_KEYS:
                values[key] = int(raw)
            elif key in _FLOAT_KEYS:
                values[key] = float(raw)
            else:
                raise ValueError(f"unknown config key {key!r}")
        return cls(**values) if base is None else replace(base, **values)

    @classmethod
    def from_file(cls, path: str | os.PathLike, base: "FusionConfig | None" = None) -> "FusionConfig":
        return cls.from_kv(kvconfig.read_kv(path), base=base)


@dataclass(frozen=True)
class Source:
    """Provenance of a draft candidate (ref fusion.py:116-138)."""

    kind: str
    prefix_len: int | None = None

    DATASTORE = "datastore"
    INPUT = "input"

    def __post_init__(self) -> None:
        if self.kind == self.DATASTORE:
            if self.prefix_len is not None:
                raise ValueError("datastore source carries no prefix_len")
        elif self.kind == self.INPUT:
            if self.prefix_len is None or self.prefix_len < 1:
                raise ValueError(f"input source needs prefix_len >= 1, got {self.prefix_len}")
        else:
            raise ValueError(f"unknown source kind {self.kind!r}")


DATASTORE_SOURCE = Source(Source.DATASTORE)


def discount(cfg: FusionConfig, source: Source, depth: int) -> float:
    """Per-source multiplier (ref fusion.py:141-155); the device uses a table of
    exactly these Python floats (``discount_table``)."""
    if depth < 1:
        raise ValueError(f"depth must be >= 1, got {depth}")
    if source.kind == Source.DATASTORE:
        return cfg.gamma_ds ** (depth - 1)
    if source.prefix_len > cfg.P:  # type: ignore[operator]
        raise ValueError(f"prefix_len {source.prefix_len} exceeds P={cfg.P}")
    return cfg.alpha * cfg.beta ** (cfg.P - source.prefix_len) * cfg.gamma_in ** (depth - 1)


def discount_table(cfg_P: int, max_depth: int, alpha: float, beta: float, gamma_ds: float,
                   gamma_in: float) -> np.ndarray:
    """[(P+1), max_depth+1] float64: rank 0 = datastore, rank r = input p = P-r+1."""
    tab = np.zeros((cfg_P + 1, max_depth + 1), dtype=np.float64)
    for rank in range(cfg_P + 1):
        for depth in range(1, max_depth + 1):
            if rank == 0:
                tab[rank, depth] = gamma_ds ** (depth - 1)
            else:
                p = cfg_P - rank + 1
                tab[rank, depth] = alpha * beta ** (cfg_P - p) * gamma_in ** (depth - 1)
    return tab


_DISC_CACHE: dict[tuple, torch.Tensor] = {}


def _disc_device(key: tuple, device) -> torch.Tensor:
    k = key + (str(device),)
    t = _DISC_CACHE.get(k)
    if t is None:
        t = torch.from_numpy(discount_table(*key)).to(device)
        _DISC_CACHE[k] = t
    return t


def _cfg_struct(P: int, dec_len: int, branch_len: int, input_branch_len: int, M: int, T: int,
                alpha: float = 0.8, beta: float = 0.8, gamma_ds: float = 1.0, gamma_in: float = 0.95,
                separator: int | None = None, use_datastore: bool = True, use_input: bool = True,
                n_input_trees: int | None = None, device=None):
    md = max(branch_len, input_branch_len)
    key = (P, md, alpha, beta, gamma_ds, gamma_in)
    disc = _disc_device(key, device)
    c = _lib.Cfg(P, dec_len, branch_len, input_branch_len, M, T, int(use_datastore), int(use_input),
                 P if n_input_trees is None else n_input_trees, int(separator is not None),
                 0 if separator is None else int(separator) & 0xFFFFFFFF, md + 1, ptr(disc),
                 fusion_mode(key))
    return c, disc


@functools.lru_cache(maxsize=64)
def _disc_monotone(key: tuple) -> bool:
    tab = discount_table(*key)
    return bool(np.all(tab[:, 2:] <= tab[:, 1:-1])) if tab.shape[1] > 2 else True


def fusion_mode(key: tuple) -> int:
    """Fusion kernel: 0 = level-synchronous (csrc/fusion_ls.cu), 1 = heap order
    (csrc/fusion.cu).  The level-synchronous form relies on priorities never
    growing along a source path, i.e. every discount row non-increasing in
    depth; FusionConfig's ranges (ref fusion.py:74-79) guarantee it, the check
    keeps the heap form for anything else.  SSSD_FUSION=heap|ls overrides."""
    env = os.environ.get("SSSD_FUSION", "").lower()
    if env == "heap":
        return 1
    mono = _disc_monotone(key)
    if env == "ls" and not mono:
        raise ValueError("SSSD_FUSION=ls needs non-increasing discount rows")
    return 0 if mono else 1


def cfg_struct(cfg: FusionConfig, separator=None, use_datastore=True, use_input=True,
               n_input_trees=None, device=None):
    return _cfg_struct(cfg.P, cfg.dec_len, cfg.branch_len, cfg.input_branch_len, cfg.M, cfg.T,
                       cfg.alpha, cfg.beta, cfg.gamma_ds, cfg.gamma_in, separator, use_datastore,
                       use_input, n_input_trees, device)


class DraftNode:
    __slots__ = ("token", "source", "priority", "parent", "children")

    def __init__(self, token: int, source: Source | None, priority: float, parent: "DraftNode | None") -> None:
        self.token = token
        self.source = source
        self.priority = priority
        self.parent = parent
        self.children: dict[int, DraftNode] = {}


class DraftTree:
    """Draft rooted at the last accepted token (ref fusion.py:178-206)."""

    def __init__(self, root_token: int) -> None:
        self.root = DraftNode(int(root_token), None, math.inf, None)
        self.size = 1

    def insert(self, token: int, parent: DraftNode, source: Source, priority: float) -> tuple[DraftNode, bool]:
        existing = parent.children.get(token)
        if existing is not None:
            return existing, False
        node = DraftNode(token, source, priority, parent)
        parent.children[token] = node
        self.size += 1
        return node, True

    def to_shape(self) -> tuple:
        def render(node: DraftNode) -> tuple:
            return (node.token, [render(c) for c in node.children.values()])

        return render(self.root)


def _serialise_sources(trees_per_request: list[list[ContinuationTree | None]], P: int):
    """Path multisets of every (request, source) as one token buffer + elements."""
    tok: list[int] = []
    elems: list[tuple[int, int, int]] = []
    offs, ns = [], []
    for srcs in trees_per_request:
        for s in range(P + 1):
            t = srcs[s] if s < len(srcs) else None
            paths = t.to_paths() if t is not None else []
            offs.append(len(elems))
            ns.append(len(paths))
            for i, path in enumerate(paths):
                elems.append((len(tok), i, len(path)))
                tok.extend(int(x) for x in path)
    return tok, elems, offs, ns


def merge_batch(requests: list[tuple[ContinuationTree, Sequence[ContinuationTree], int]],
                cfg: FusionConfig, device=None, with_nodes: bool = False):
    """GPU fusion of B independent (datastore tree, input trees, root) sets.
    ``with_nodes``: also return, per draft, the per-node (priority, merge rank)
    lists in DFS order (``sssd_draft_out.priority`` / ``.source``)."""
    from .draft import FlattenedDraft, _drafts_from_device

    dev = torch.device(device) if device is not None else _lib.require_cuda()
    for _, ins, _ in requests:
        if len(ins) > cfg.P:
            raise ValueError(f"got {len(ins)} input trees for P={cfg.P}")
    n_trees = max((len(ins) for _, ins, _ in requests), default=0)
    B = len(requests)
    per = [[ds] + list(ins) + [None] * (n_trees - len(ins)) for ds, ins, _ in requests]
    tok, elems, offs, ns = _serialise_sources(per, cfg.P)
    for ds, ins, _ in requests:
        for t in [ds, *ins]:
            for path in t.to_paths():
                if len(path) > _lib.SSSD_MAX_DEPTH:
                    raise ValueError(f"tree depth {len(path)} exceeds the compiled limit {_lib.SSSD_MAX_DEPTH}")
    depth = max([max((len(p) for p in t.to_paths()), default=1)
                 for ds, ins, _ in requests for t in [ds, *ins]] + [1])
    c, keep = _cfg_struct(cfg.P, cfg.dec_len, depth, 1, cfg.M, cfg.T, cfg.alpha, cfg.beta, cfg.gamma_ds,
                          cfg.gamma_in, n_input_trees=n_trees, device=dev)
    # the discount table must reach the deepest path
    d_tok = torch.tensor(np.asarray(tok + [0], dtype=np.int64).astype(np.uint32).view(np.int32), device=dev)
    el = np.zeros((max(len(elems), 1), 4), dtype=np.uint32)
    for i, (o, orig, ln) in enumerate(elems):
        el[i] = (o, orig, ln | (255 << 8), 0)
    d_el = torch.from_numpy(el.view(np.int32)).to(dev)
    d_off = torch.tensor(offs, dtype=torch.int64, device=dev)
    d_n = torch.tensor(ns, dtype=torch.int32, device=dev)
    roots = torch.tensor(np.asarray([int(r) & 0xFFFFFFFF for _, _, r in requests], dtype=np.uint32).view(np.int32),
                         device=dev)
    S = cfg.dec_len
    W = (S + 63) // 64
    size = torch.empty(B, dtype=torch.int32, device=dev)
    toks = torch.empty(B * S, dtype=torch.int32, device=dev)
    par = torch.empty(B * S, dtype=torch.int32, device=dev)
    dep = torch.empty(B * S, dtype=torch.int32, device=dev)
    mask = torch.empty(B * S * W, dtype=torch.int64, device=dev)
    prio = torch.empty(B * S, dtype=torch.float64, device=dev) if with_nodes else None
    src = torch.empty(B * S, dtype=torch.int32, device=dev) if with_nodes else None
    out = _lib.DraftOut(ptr(size), ptr(toks), ptr(par), ptr(dep), ptr(mask), ptr(prio), ptr(src), None)
    total = len(elems)
    ws = torch.empty(lib().sssd_merge_workspace(c, B, total), dtype=torch.uint8, device=dev)
    st = stream_ptr(dev)
    check(lib().sssd_merge(ptr(d_tok), ptr(d_el), ptr(d_off), ptr(d_n), total, ptr(roots), B, c, out,
                           ptr(ws), ws.numel(), st))
    check(lib().sssd_workspace_status(c, B, 0, ptr(ws), 1, total, st))
    flats = _drafts_from_device(size, toks, par, dep, mask, B, S)
    if not with_nodes:
        return flats
    prio_h = prio.reshape(B, S).cpu().numpy()
    src_h = src.reshape(B, S).cpu().numpy()
    return flats, [(prio_h[b, :f.s_q].tolist(), src_h[b, :f.s_q].tolist()) for b, f in enumerate(flats)]


def merge(datastore_tree: ContinuationTree, input_trees: Sequence[ContinuationTree], cfg: FusionConfig,
          root_token: int) -> DraftTree:
    """Best-first fusion (ref fusion.py:209-261), computed on the GPU.  Returns a
    ``DraftTree`` with the reference's child insertion order and, per node, the
    priority and ``Source`` of its first insertion (ref fusion.py:185-198),
    read back from the fusion kernel's per-node outputs."""
    if len(input_trees) > cfg.P:
        raise ValueError(f"got {len(input_trees)} input trees for P={cfg.P}")
    flats, nodes = merge_batch([(datastore_tree, list(input_trees), int(root_token))], cfg, with_nodes=True)
    prio, ranks = nodes[0]
    return draft_tree_from_flat(flats[0], prio, [source_of_rank(r, cfg.P) for r in ranks])


def source_of_rank(rank: int, P: int) -> Source | None:
    """Merge rank -> provenance (ref fusion.py:245-249): 0 = datastore, r >= 1 =
    the input tree of prefix length P - r + 1; -1 = the root (no source)."""
    if rank < 0:
        return None
    return DATASTORE_SOURCE if rank == 0 else Source(Source.INPUT, P - rank + 1)


def draft_tree_from_flat(flat, priorities=None, sources=None) -> DraftTree:
    """Rebuild a ``DraftTree`` from DFS arrays (children in pre-order = insertion
    order).  Without per-node data the nodes carry NaN priority and no source."""
    tree = DraftTree(flat.tokens[0])
    nodes = [tree.root]
    for i in range(1, flat.s_q):
        pr = float(priorities[i]) if priorities is not None else float("nan")
        sc = sources[i] if sources is not None else None
        node, _ = tree.insert(flat.tokens[i], nodes[flat.parents[i]], sc, pr)
        nodes.append(node)
    return tree


def calibrate(dataset: Sequence, datastore: Datastore, grid: Iterable[FusionConfig], sources: str = "both",
              separator: int | None = None) -> FusionConfig:
    """Grid search of mean accepted tokens per step (ref fusion.py:264-289), simulated on the GPU."""
    from .harness import simulate

    records = list(dataset)
    if not records:
        raise ValueError("empty dataset")
    configs = list(grid)
    if not configs:
        raise ValueError("empty grid")
    best, best_score = None, -math.inf
    for cfg in configs:
        score = simulate(records, datastore, cfg, sources=sources, separator=separator).mean_accepted_per_step
        if score > best_score:
            best, best_score = cfg, score
    return best
