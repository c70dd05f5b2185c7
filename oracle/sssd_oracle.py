"""CPU oracle for the SSSD drafting hot path.  TEST INFRASTRUCTURE ONLY.

This module is the *checker*: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.  The
product path (``paper_2411_05894_b200``) never calls into it and fails loudly
when its CUDA library is missing.

It restates the reference algorithm (``/root/reference/pkg/src/specdraft``)
in the *stateless / phase-split* forms of SURVEY.md Appendix A, which are the
forms the CUDA kernels implement:

* suffix array by prefix doubling over packed 64-bit keys
  (ref ``datastore.py:81-109``; any correct SA is identical, A.1);
* ``[lo, hi)`` by lower/upper-bound binary search (ref ``datastore.py:129-183``);
* strided sampling (ref ``datastore.py:112-126``);
* datastore continuation lists per prefix length, then the T cut-off scan
  (ref ``datastore.py:185-218``; phase-split form A.3);
* input-cache trees from one backward-match-length pass ``m[e]``
  (ref ``input_cache.py:88-121``; stateless form A.4);
* best-first fusion driven by a sibling-group frontier instead of a heap
  (ref ``fusion.py:209-261``; A.5), with the discount table evaluated by the
  reference's own float expression (ref ``fusion.py:141-155``);
* DFS flattening, u64 ancestor masks, ``pack_mask`` bytes, greedy verify and the
  ``draft_digest`` fingerprint (ref ``draft.py:67-138``, ``harness.py:316-322``);
* teacher-forced decode loop with final-step truncation (ref ``harness.py:49-67,171-209``).

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by the reference itself (``tests/golden/make_golden.py``)
and against the reference tests' hand-written known answers.
"""

from __future__ import annotations

import hashlib
import heapq
import json
import struct
from dataclasses import dataclass, field

import numpy as np

EXHAUSTED = 0xFFFFFFFF  # ref harness.py:29-32


# ---------------------------------------------------------------------------
# suffix array  (ref datastore.py:81-109)
# ---------------------------------------------------------------------------


def suffix_array(tokens) -> np.ndarray:
    """Prefix doubling: sort positions by (rank[i], rank[i+k]+1) packed into one
    int64 key; a position past the end contributes 0 so shorter suffixes sort
    first (ref datastore.py:94-95)."""
    t = np.asarray(tokens).astype(np.uint32, copy=False)
    n = int(t.size)
    if n == 0:
        raise ValueError("empty corpus")
    if n == 1:
        return np.zeros(1, dtype=np.int64)
    # dense rank of the first token
    order = np.argsort(t, kind="stable")
    st = t[order]
    head = np.empty(n, dtype=np.int64)
    head[0] = 0
    head[1:] = np.cumsum(st[1:] != st[:-1])
    rank = np.empty(n, dtype=np.int64)
    rank[order] = head
    k = 1
    base = np.int64(n + 1)
    while True:
        second = np.zeros(n, dtype=np.int64)
        second[: n - k] = rank[k:] + 1
        key = rank * base + second
        order = np.argsort(key, kind="stable")
        sk = key[order]
        head = np.empty(n, dtype=np.int64)
        head[0] = 0
        head[1:] = np.cumsum(sk[1:] != sk[:-1])
        rank = np.empty(n, dtype=np.int64)
        rank[order] = head
        if head[-1] == n - 1:
            return order.astype(np.int64)
        k *= 2


# ---------------------------------------------------------------------------
# range search + sampling  (ref datastore.py:112-183)
# ---------------------------------------------------------------------------


def _cmp(tokens: np.ndarray, pos: int, pat: list[int]) -> int:
    n = tokens.shape[0]
    for j, want in enumerate(pat):
        if pos + j >= n:
            return -1
        have = int(tokens[pos + j])
        if have != want:
            return -1 if have < want else 1
    return 0


def find_range(tokens: np.ndarray, sa: np.ndarray, pat) -> tuple[int, int]:
    pat = [int(x) for x in pat]
    if not pat:
        raise ValueError("prefix must be non-empty")
    n = int(sa.shape[0])
    a, b = 0, n
    while a < b:  # first rank with suffix >= pat
        mid = (a + b) >> 1
        if _cmp(tokens, int(sa[mid]), pat) < 0:
            a = mid + 1
        else:
            b = mid
    lo = a
    b = n
    while a < b:  # first rank with suffix > pat
        mid = (a + b) >> 1
        if _cmp(tokens, int(sa[mid]), pat) <= 0:
            a = mid + 1
        else:
            b = mid
    return lo, a


def sample_ranks(lo: int, hi: int, cap: int) -> list[int]:
    if lo > hi:
        raise ValueError(f"invalid interval: lo={lo} > hi={hi}")
    if cap < 1:
        raise ValueError(f"cap must be >= 1, got {cap}")
    w = hi - lo
    if w <= cap:
        return list(range(lo, hi))
    return [lo + (k * w) // cap for k in range(cap)]


# ---------------------------------------------------------------------------
# source string lists (the trie is derived from an ordered list of paths)
# ---------------------------------------------------------------------------


@dataclass
class DsLookup:
    """Phase-split datastore lookup for one request."""

    ranges: list  # [(p, lo, hi)] for every evaluated p, descending
    samples: list  # [(p, [sa positions])]
    strings: list  # ordered list of non-empty continuation paths (p desc, SA order)


def ds_lookup(tokens, sa, prefix, P, M, T, branch_len, separator=None) -> DsLookup:
    prefix = [int(x) for x in prefix]
    if not prefix:
        raise ValueError("prefix must be non-empty")
    tokens = np.asarray(tokens)
    n = int(tokens.shape[0])
    ranges, samples, strings = [], [], []
    for p in range(min(P, len(prefix)), 0, -1):
        lo, hi = find_range(tokens, sa, prefix[len(prefix) - p:])
        ranges.append((p, lo, hi))
        pos_list = []
        for r in sample_ranks(lo, hi, M):
            pos = int(sa[r])
            pos_list.append(pos)
            start = pos + p
            cont = [int(x) for x in tokens[start:min(start + branch_len, n)]]
            if separator is not None and separator in cont:
                cont = cont[: cont.index(separator)]
            if cont:
                strings.append(cont)
        samples.append((p, pos_list))
        if len(strings) >= T:
            break
    return DsLookup(ranges, samples, strings)


def match_lengths(seq, P: int) -> np.ndarray:
    """m[e] = longest k <= min(P, e) with seq[e-k:e] == seq[L-k:L] (A.4); m[0] = 0."""
    s = np.asarray(seq, dtype=np.int64)
    L = s.size
    m = np.zeros(L, dtype=np.int64)
    if L < 2:
        return m
    alive = np.ones(L - 1, dtype=bool)  # e = 1..L-1
    e = np.arange(1, L)
    for j in range(min(P, L - 1)):
        ok = alive & (e - 1 - j >= 0)
        idx = np.where(ok, e - 1 - j, 0)
        ok &= s[idx] == s[L - 1 - j]
        m[1:][ok] = j + 1
        alive = ok
    return m


def input_strings(seq, P: int, ibl: int) -> list[list[list[int]]]:
    """Per p = 1..P: ordered continuation paths of earlier occurrences of the
    last p tokens (ref input_cache.py:88-113, trailing occurrence excluded)."""
    seq = [int(x) for x in seq]
    if not seq:
        raise ValueError("empty sequence")
    L = len(seq)
    m = match_lengths(seq, P)
    out = []
    for p in range(1, P + 1):
        out.append([seq[e:e + ibl] for e in range(1, L) if m[e] >= p])
    return out


# ---------------------------------------------------------------------------
# tries built from ordered path lists: children in first-appearance order
# ---------------------------------------------------------------------------


class Trie:
    __slots__ = ("count", "kids")

    def __init__(self) -> None:
        self.count = 0
        self.kids: dict[int, Trie] = {}


def trie_of(paths) -> Trie:
    root = Trie()
    for path in paths:
        root.count += 1
        node = root
        for tok in path:
            nxt = node.kids.get(tok)
            if nxt is None:
                nxt = node.kids[tok] = Trie()
            nxt.count += 1
            node = nxt
    return root


def trie_counts(t: Trie) -> dict:
    """``ContinuationTree.to_counts()`` rendering (ref trees.py:84-96)."""

    def r(x: Trie) -> dict:
        return {"count": x.count, "children": {k: r(v) for k, v in x.kids.items()}}

    return {"root_count": t.count, "children": {k: r(v) for k, v in t.kids.items()}}


def trie_shape(t: Trie) -> list:
    """Order-sensitive rendering: [count, [[token, subtree], ...]]."""
    return [t.count, [[k, trie_shape(v)] for k, v in t.kids.items()]]


# ---------------------------------------------------------------------------
# fusion  (ref fusion.py:141-261) — sibling-group frontier (A.5)
# ---------------------------------------------------------------------------


def discount_table(P: int, max_depth: int, alpha: float, beta: float,
                   gamma_ds: float, gamma_in: float) -> list[list[float]]:
    """disc[rank][depth] with rank 0 = datastore, rank r>=1 = input p=P-r+1;
    the float expression is the reference's (ref fusion.py:152,155)."""
    tab = []
    for rank in range(P + 1):
        row = [0.0]
        for depth in range(1, max_depth + 1):
            if rank == 0:
                row.append(gamma_ds ** (depth - 1))
            else:
                p = P - rank + 1
                row.append(alpha * beta ** (P - p) * gamma_in ** (depth - 1))
        tab.append(row)
    return tab


@dataclass
class Draft:
    tokens: list
    parents: list
    depths: list
    masks: list  # one python int bitmask per row (bit j = ancestor-or-self j)

    @property
    def size(self) -> int:
        return len(self.tokens)


def fuse(ds: Trie | None, inputs: list, P: int, dec_len: int, disc, root_token: int):
    """Best-first fusion; returns the draft as (token, children) shape plus
    the per-node insertion-ordered child lists.

    Every pop of the reference heap (ref fusion.py:252-259) takes the minimum of
    (-priority, depth, rank, ticket).  Children pushed together form one
    sibling group with consecutive tickets, so the heap minimum is the minimum
    over group heads of (-priority, depth, rank, group sequence), where a
    group's head is its best remaining child by (priority desc, child order
    asc).  (Priority is monotone in count inside a group, but not strictly:
    alpha = 0 or underflow makes unequal counts tie, so the exact double
    priority is what orders a group.)
    """
    if len(inputs) > P:
        raise ValueError(f"got {len(inputs)} input trees for P={P}")
    # draft: node id -> token, parent, ordered children (token -> id)
    d_tok = [int(root_token)]
    d_par = [-1]
    d_kids: list[dict] = [{}]
    groups = []  # [neg-key fields..., state]

    def new_group(src: Trie, rank: int, depth: int, pp, dparent: int) -> None:
        kids = list(src.kids.items())
        if not kids:
            return
        dsc = disc[rank][depth]
        cand = []
        for i, (tok, c) in enumerate(kids):
            if pp is None:
                cpp = c.count / src.count  # seed (ref fusion.py:244)
            else:
                cpp = pp * (c.count / src.count)  # ref fusion.py:259
            cand.append((-(cpp * dsc), i, tok, c, cpp))
        cand.sort(key=lambda x: (x[0], x[1]))  # (priority desc, ticket asc)
        groups.append({"cand": cand, "next": 0, "rank": rank, "depth": depth,
                       "dparent": dparent, "seq": len(groups)})

    def head(g):
        negp, _, tok, c, cpp = g["cand"][g["next"]]
        return (negp, g["depth"], g["rank"], g["seq"]), tok, c, cpp

    if ds is not None and ds.count > 0:
        new_group(ds, 0, 1, None, 0)
    for i in range(len(inputs) - 1, -1, -1):
        t = inputs[i]
        if t is not None and t.count > 0:
            new_group(t, P - (i + 1) + 1, 1, None, 0)

    # group heads in a binary heap (the minimum over heads, as the reference's
    # heapq pop over individual candidates, ref fusion.py:252)
    heap: list = []
    pushed = 0

    def push_head(g) -> None:
        if g["next"] < len(g["cand"]):
            heapq.heappush(heap, (head(g)[0], g["seq"]))

    for g in groups:
        push_head(g)
    pushed = len(groups)
    size = 1
    while size < dec_len:
        while pushed < len(groups):  # groups created by the previous pop
            push_head(groups[pushed])
            pushed += 1
        if not heap:
            break
        _, gs = heapq.heappop(heap)
        g = groups[gs]
        key, tok, c, pp = head(g)
        g["next"] += 1
        push_head(g)
        par = g["dparent"]
        nid = d_kids[par].get(tok)
        if nid is None:
            nid = len(d_tok)
            d_tok.append(tok)
            d_par.append(par)
            d_kids.append({})
            d_kids[par][tok] = nid
            size += 1
        new_group(c, g["rank"], g["depth"] + 1, pp, nid)
    return d_tok, d_par, d_kids


def flatten(d_tok, d_par, d_kids) -> Draft:
    """DFS pre-order, children in insertion order (ref draft.py:67-86)."""
    tokens, parents, depths, masks = [], [], [], []
    stack = [(0, -1)]
    while stack:
        nid, par = stack.pop()
        idx = len(tokens)
        tokens.append(d_tok[nid])
        parents.append(par)
        depths.append(0 if par < 0 else depths[par] + 1)
        masks.append((1 << idx) | (masks[par] if par >= 0 else 0))
        for kid in reversed(list(d_kids[nid].values())):
            stack.append((kid, idx))
    return Draft(tokens, parents, depths, masks)


def mask_matrix(draft: Draft) -> np.ndarray:
    n = draft.size
    out = np.zeros((n, n), dtype=bool)
    for i, m in enumerate(draft.masks):
        for j in range(n):
            out[i, j] = (m >> j) & 1
    return out


def pack_mask_rows(masks, n: int) -> bytes:
    """Same bytes as ref draft.py:89-93 (u64 row count, row-major LSB-first)."""
    bits = 0
    for i, m in enumerate(masks):
        bits |= (m & ((1 << n) - 1)) << (i * n)
    nbytes = (n * n + 7) // 8
    return struct.pack("<Q", n) + bits.to_bytes(nbytes, "little")


def digest(drafts) -> str:
    """ref harness.py:316-322."""
    h = hashlib.sha256()
    for d in drafts:
        h.update(json.dumps([d.tokens, d.parents, d.depths]).encode())
        h.update(pack_mask_rows(d.masks, d.size))
    return h.hexdigest()


def verify(draft: Draft, preds) -> tuple[list[int], int]:
    """Greedy accept (ref draft.py:114-138)."""
    preds = [int(x) for x in preds]
    if len(preds) != draft.size:
        raise ValueError(f"length mismatch: {len(preds)} predictions for {draft.size} draft nodes")
    kids: list[dict] = [{} for _ in range(draft.size)]
    for i in range(1, draft.size):
        kids[draft.parents[i]].setdefault(draft.tokens[i], i)
    path, cur = [], 0
    while True:
        nxt = kids[cur].get(preds[cur])
        if nxt is None:
            return path, preds[cur]
        path.append(nxt)
        cur = nxt


# ---------------------------------------------------------------------------
# propose / session / simulate  (ref draft.py:141-216, harness.py:171-237)
# ---------------------------------------------------------------------------


@dataclass
class Cfg:
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
            self.branch_len = max(1, min(8, self.dec_len - 1))

    def disc(self):
        return discount_table(self.P, max(self.branch_len, self.input_branch_len), self.alpha,
                              self.beta, self.gamma_ds, self.gamma_in)


@dataclass
class Store:
    tokens: np.ndarray
    sa: np.ndarray


def session_inputs(seq, cfg: Cfg, use_in=True) -> list:
    """The input tries of a context (what the reference's GenerationSession.start
    builds once per session into its InputCache, ref draft.py:156-181), so that
    ``propose(..., inputs=...)`` times only the per-step work, like the
    reference's bench_retrieval over pre-started sessions (harness.py:325-370)."""
    seq = [int(x) for x in seq]
    return [trie_of(s) for s in input_strings(seq, cfg.P, cfg.input_branch_len)] if use_in else []


def propose(store: Store | None, seq, cfg: Cfg, separator=None, use_ds=True, use_in=True,
            disc=None, inputs=None) -> Draft:
    seq = [int(x) for x in seq]
    if disc is None:
        disc = cfg.disc()
    ds = None
    if use_ds:
        prefix = seq[len(seq) - min(cfg.P, len(seq)):]
        look = ds_lookup(store.tokens, store.sa, prefix, cfg.P, cfg.M, cfg.T, cfg.branch_len,
                         separator)
        ds = trie_of(look.strings)
    if inputs is not None:
        ins = inputs
    else:
        ins = [trie_of(s) for s in input_strings(seq, cfg.P, cfg.input_branch_len)] if use_in else []
    return flatten(*fuse(ds, ins, cfg.P, cfg.dec_len, disc, seq[-1]))


def teacher_predictions(draft: Draft, L: int, prompt_len: int, reference) -> list[int]:
    """Node i's greedy next token = ref[L - plen + depth_i] (ref harness.py:61-67)."""
    out = []
    for d in draft.depths:
        i = L - prompt_len + d
        out.append(int(reference[i]) if i < len(reference) else EXHAUSTED)
    return out


def run_record(store, prompt, reference, cfg: Cfg, separator=None, use_ds=True, use_in=True):
    """Per-step emitted-token counts (ref harness.py:171-209)."""
    seq = [int(x) for x in prompt]
    target = len(prompt) + len(reference)
    disc = cfg.disc()
    per_step = []
    while len(seq) < target:
        d = propose(store, seq, cfg, separator, use_ds, use_in, disc)
        preds = teacher_predictions(d, len(seq), len(prompt), reference)
        path, bonus = verify(d, preds)
        emitted = [d.tokens[i] for i in path] + [bonus]
        seq.extend(emitted)
        n = len(emitted)
        over = len(seq) - target
        if over > 0:
            del seq[target:]
            n -= over
        per_step.append(n)
    if seq != [int(x) for x in prompt] + [int(x) for x in reference]:
        raise AssertionError("speculative output diverged from the reference")
    return per_step


def hash_oracle_next(ctx, alphabet: int, salt: int = 0) -> int:
    """Content-hash oracle (ref tests/oracles.py:245-257)."""
    h = (len(ctx) * 1_000_003 + salt) & 0xFFFFFFFF
    for tok in list(ctx[-3:]):
        h = (h * 31 + int(tok) + 7) & 0xFFFFFFFF
    return h % alphabet


# ---------------------------------------------------------------------------
# C restatement of the SA build (oracle/sa_oracle.c), for host-side baselines
# ---------------------------------------------------------------------------

_HERE = __import__("os").path.dirname(__import__("os").path.abspath(__file__))
_SA_LIB = __import__("os").path.join(_HERE, "_build", "libsa_oracle.so")


def build_c_oracle() -> str:
    """Compile oracle/sa_oracle.c with gcc (called by __graft_entry__.build())."""
    import os
    import subprocess

    src = os.path.join(_HERE, "sa_oracle.c")
    os.makedirs(os.path.dirname(_SA_LIB), exist_ok=True)
    if not os.path.exists(_SA_LIB) or os.path.getmtime(_SA_LIB) < os.path.getmtime(src):
        subprocess.run(["gcc", "-O3", "-shared", "-fPIC", "-o", _SA_LIB, src], check=True)
    return _SA_LIB


def suffix_array_c(tokens) -> np.ndarray:
    """Same result as suffix_array(), via the C oracle (u32 positions)."""
    import ctypes

    t = np.ascontiguousarray(np.asarray(tokens), dtype=np.uint32)
    n = int(t.size)
    if n == 0:
        raise ValueError("empty corpus")
    lib = ctypes.CDLL(build_c_oracle())
    out = np.empty(n, dtype=np.uint32)
    rc = lib.sa_oracle_build(t.ctypes.data_as(ctypes.c_void_p), ctypes.c_uint64(n),
                             out.ctypes.data_as(ctypes.c_void_p))
    if rc != 0:
        raise RuntimeError(f"sa_oracle_build failed ({rc})")
    return out
