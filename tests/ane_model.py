"""All-nodes restatement of best-first fusion (test infrastructure).

The reference heap (ref fusion.py:209-261) pops source-trie nodes in the
order G = (-priority, depth, rank, ticket) and the draft is the first dec_len-1
distinct token paths in that order (tests/ls_model.py).  The
ticket order of two nodes of equal (priority, depth, rank) follows their
parents' pop order, then child order, so inside one (depth, rank) class the
order is the recursive key

    ord(n) = (-priority(n), ord(parent(n)), child index of n)

(ord of a seed's parent = ()): lexicographic over the chain of ancestor
priorities from n upwards, then over the child indices from the top down.

This form needs no levels: enumerate every live node of every source trie
with its priority, depth, rank and ord, take the nodes whose priority is at
least a threshold T (the C-th largest priority, C >= dec_len - 1), sort them
by G and keep the first dec_len - 1 distinct paths.  Whenever those
candidates hold dec_len - 1 distinct paths the result equals the global one
(every node that precedes the last kept path in G has priority >= its
priority >= T, so it is a candidate); otherwise C grows.  This module states
that algorithm over the oracle's tries so it can be checked against the
oracle's heap merge before any CUDA (the plan of an all-nodes fusion kernel).
"""

from __future__ import annotations

from oracle import sssd_oracle as O


def enumerate_nodes(ds, inputs, P: int, disc):
    """Every live source node: (priority, depth, rank, ord, path, trie node)."""
    srcs = []
    if ds is not None and ds.count > 0:
        srcs.append((0, ds))
    for i in range(len(inputs) - 1, -1, -1):
        t = inputs[i]
        if t is not None and t.count > 0:
            srcs.append((P - i, t))
    nodes = []
    for rk, t in srcs:
        stack = [(t, None, (), 0, ())]  # (trie node, pp, ord, depth, path)
        while stack:
            node, pp, od, d, path = stack.pop()
            for ci, (tok, c) in enumerate(node.kids.items()):
                cpp = c.count / node.count if pp is None else pp * (c.count / node.count)
                pr = cpp * disc[rk][d + 1]
                o = (-pr, od, ci)
                nodes.append((pr, d + 1, rk, o, path + (tok,), c))
                stack.append((c, cpp, o, d + 1, path + (tok,)))
    return nodes


def fuse_ane(ds, inputs, P: int, dec_len: int, disc, root_token: int, stats: dict | None = None, C0: int | None = None):
    K = dec_len - 1
    nodes = enumerate_nodes(ds, inputs, P, disc)
    if stats is not None:
        stats["nodes"] = len(nodes)
    C = max(K, 1) if C0 is None else C0
    order = None
    while True:
        if K <= 0 or not nodes:
            cand = []
        else:
            prios = sorted((n[0] for n in nodes), reverse=True)
            T = prios[min(C, len(prios)) - 1]
            cand = [n for n in nodes if n[0] >= T]
        cand.sort(key=lambda n: (-n[0], n[1], n[2], n[3]))
        seen, picked = set(), []
        for n in cand:
            if len(picked) == K:
                break
            if n[4] not in seen:
                seen.add(n[4])
                picked.append(n)
        if len(picked) == K or len(cand) == len(nodes):
            order = picked
            break
        C *= 2
    if stats is not None:
        stats["C"] = C
    d_tok = [int(root_token)]
    d_par = [-1]
    d_kids: list[dict] = [{}]
    nid_of = {(): 0}
    for n in order:
        path = n[4]
        par = nid_of[path[:-1]]
        nid = len(d_tok)
        nid_of[path] = nid
        d_tok.append(path[-1])
        d_par.append(par)
        d_kids.append({})
        d_kids[par][path[-1]] = nid
    return d_tok, d_par, d_kids


def propose_ane(store, seq, cfg, separator=None, use_ds=True, use_in=True, stats=None):
    seq = [int(x) for x in seq]
    disc = cfg.disc()
    ds = None
    if use_ds:
        prefix = seq[len(seq) - min(cfg.P, len(seq)):]
        look = O.ds_lookup(store.tokens, store.sa, prefix, cfg.P, cfg.M, cfg.T, cfg.branch_len, separator)
        ds = O.trie_of(look.strings)
    ins = [O.trie_of(s) for s in O.input_strings(seq, cfg.P, cfg.input_branch_len)] if use_in else []
    return O.flatten(*fuse_ane(ds, ins, cfg.P, cfg.dec_len, disc, seq[-1], stats))
