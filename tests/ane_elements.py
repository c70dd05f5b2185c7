"""All-nodes fusion over SORTED ELEMENT ARRAYS (test infrastructure): the
data-structure-level plan of the all-nodes fusion kernel (csrc/fusion_ane.cu),
stated in Python so it can be checked against the oracle's heap merge (ref
fusion.py:209-261) before and alongside the CUDA code.  tests/ane_model.py
states the same algorithm over tries; this form works on what the kernel
sees -- per merge rank, the continuation strings sorted by (string, first
appearance) with a backward-match length m and a fold weight -- and uses only
per-element / per-depth steps:

* lcp[i] = common prefix of elements i-1 and i; at depth d, element i starts a
  run (a trie node) iff len[i] >= d and (i == 0 or lcp[i] < d); the run ends at
  the next element with lcp < d; its count is a prefix-sum difference of the
  rank's weights (m >= threshold), its parent is the depth-(d-1) run start at
  or before i, its first appearance the minimum position in the run among
  counted elements;
* path probabilities depth by depth (parent first): seed count / root count,
  then pp(parent) * (count / count(parent)); priority = pp * discount;
* a threshold T on ~bits(priority) (radix select of the C-th smallest), the
  candidates k0 <= T sorted by (k0, depth, rank, ord chain), dedupe by path
  depth by depth, first dec_len-1 distinct paths; C doubles if too few.
"""

from __future__ import annotations

import struct

from oracle import sssd_oracle as O


def _k0(pr: float) -> int:
    return (~struct.unpack("<Q", struct.pack("<d", pr))[0]) & 0xFFFFFFFFFFFFFFFF


def nodes_of_rank(rank: int, elems, thr: int, disc):
    """Live nodes of one rank: dicts with k0, pr, pp, cnt, depth, rank, parent (index
    into the returned list or -1), first, tok, path."""
    n = len(elems)
    w = [e[3] if e[2] >= thr else 0 for e in elems]
    W = [0] * (n + 1)
    for i in range(n):
        W[i + 1] = W[i] + w[i]
    root = W[n]
    if root == 0:
        return []
    lens = [len(e[0]) for e in elems]
    lcp = [0] * n
    for i in range(1, n):
        a, b = elems[i - 1][0], elems[i][0]
        k = 0
        while k < min(len(a), len(b)) and a[k] == b[k]:
            k += 1
        lcp[i] = k
    out = []
    prev_id = {}  # element index of a depth-(d-1) run start -> node id (live only)
    dmax = max(lens) if lens else 0
    for d in range(1, dmax + 1):
        cur_id = {}
        bounds = [i for i in range(n) if i == 0 or lcp[i] < d]
        for bi, i in enumerate(bounds):
            if lens[i] < d:
                continue
            e = bounds[bi + 1] if bi + 1 < len(bounds) else n
            cnt = W[e] - W[i]
            if cnt == 0:
                continue
            if d == 1:
                par, pp = -1, cnt / root
            else:
                j = max(x for x in prev_id if x <= i)  # the depth-(d-1) run start containing i
                par = prev_id[j]
                pn = out[par]
                pp = pn["pp"] * (cnt / pn["cnt"])
            pr = pp * disc[rank][d]
            first = min(elems[x][1] for x in range(i, e) if w[x] > 0)
            node = {"k0": _k0(pr), "pr": pr, "pp": pp, "cnt": cnt, "depth": d, "rank": rank, "parent": par,
                    "first": first, "tok": elems[i][0][d - 1], "path": elems[i][0][:d]}
            cur_id[i] = len(out)
            out.append(node)
        prev_id = {i: v for i, v in cur_id.items()}
    return out


def fuse_elements(sources, P: int, dec_len: int, disc, root_token: int, C0: int | None = None, stats=None):
    """sources: list of (rank, thr, elems) with elems [(string, orig, m, wt)] sorted."""
    K = dec_len - 1
    nodes = []
    for rank, thr, elems in sources:
        base = len(nodes)
        for nd in nodes_of_rank(rank, elems, thr, disc):
            if nd["parent"] >= 0:
                nd["parent"] += base
            nodes.append(nd)
    N = len(nodes)
    if stats is not None:
        stats["nodes"] = N

    def ordkey(i):  # (k0, ord(parent), first) nested, as ane_model's ord
        nd = nodes[i]
        return (nd["k0"], ordkey(nd["parent"]) if nd["parent"] >= 0 else (), nd["first"])

    C = max(K, 1) if C0 is None else C0
    picked = []
    while K > 0 and N:
        ks = sorted(nd["k0"] for nd in nodes)
        T = ks[min(C, N) - 1]
        cand = [i for i in range(N) if nodes[i]["k0"] <= T]
        cand.sort(key=lambda i: (nodes[i]["k0"], nodes[i]["depth"], nodes[i]["rank"], ordkey(i)))
        pos = {i: p for p, i in enumerate(cand)}
        # path ids depth by depth: the first candidate (G order) with the same (parent path, token)
        pid = {}
        for d in range(1, max(nodes[i]["depth"] for i in cand) + 1):
            seen = {}
            for i in cand:  # (G order)
                nd = nodes[i]
                if nd["depth"] != d:
                    continue
                key = (pid[nd["parent"]] if nd["parent"] >= 0 else -1, nd["tok"])
                if key not in seen:
                    seen[key] = pos[i]
                pid[i] = seen[key]
        picked = [i for i in cand if pid[i] == pos[i]][:K]
        if len(picked) == K or len(cand) == N:
            break
        C *= 2
    if stats is not None:
        stats["C"] = C
    d_tok = [int(root_token)]
    d_par = [-1]
    d_kids: list[dict] = [{}]
    nid_of_path = {(): 0}
    for i in picked:
        path = nodes[i]["path"]
        par = nid_of_path[path[:-1]]
        nid = len(d_tok)
        nid_of_path[path] = nid
        d_tok.append(path[-1])
        d_par.append(par)
        d_kids.append({})
        d_kids[par][path[-1]] = nid
    return d_tok, d_par, d_kids


def elements_for(store, seq, cfg, separator=None, use_ds=True, use_in=True):
    """The kernel's element arrays for one request: the datastore's sorted,
    folded continuations (rank 0) and the input array shared by ranks 1..P
    (threshold p = P - rank + 1), as the lookup / scan kernels produce them."""
    seq = [int(x) for x in seq]
    srcs = []
    if use_ds:
        prefix = seq[len(seq) - min(cfg.P, len(seq)):]
        look = O.ds_lookup(store.tokens, store.sa, prefix, cfg.P, cfg.M, cfg.T, cfg.branch_len, separator)
        raw = sorted(((tuple(s), i) for i, s in enumerate(look.strings)), key=lambda x: (x[0], x[1]))
        folded = []
        for s, i in raw:
            if folded and folded[-1][0] == s:
                f = folded[-1]
                folded[-1] = (s, f[1], 255, f[3] + 1)
            else:
                folded.append((s, i, 255, 1))
        srcs.append((0, 0, folded))
    if use_in and len(seq) >= 2:
        m = O.match_lengths(seq, cfg.P)
        L = len(seq)
        els = sorted(((tuple(seq[e:e + cfg.input_branch_len]), e, int(m[e]), 1) for e in range(1, L) if m[e] >= 1),
                     key=lambda x: (x[0], x[1]))
        for rank in range(1, cfg.P + 1):
            srcs.append((rank, cfg.P - rank + 1, els))
    return srcs


def propose_elements(store, seq, cfg, stats=None, C0=None):
    seq = [int(x) for x in seq]
    return O.flatten(*fuse_elements(elements_for(store, seq, cfg), cfg.P, cfg.dec_len, cfg.disc(), seq[-1],
                                    C0=C0, stats=stats))
