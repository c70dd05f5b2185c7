"""Level-synchronous restatement of best-first fusion (test infrastructure).

This is the algorithm the GPU ``draft_ls_kernel`` implements, written over the
oracle's tries so it can be checked against the heap-ordered ``oracle.fuse``
(ref fusion.py:209-261) on the golden merges and on random tie-heavy cases.

Why it is equivalent:

* every source node's key (-priority, depth, rank, ticket) is larger than its
  parent's (priorities never grow along a path: count ratios <= 1 and the
  discount table is non-increasing in depth), so the reference heap pops the
  source nodes of all tries in global key order;
* the ticket order of two nodes of equal (priority, depth, rank) is the pop
  order of their parents, then child order: within one (depth, rank) class the
  order is (-priority, parent's position in its class, child index), so one
  sort per level yields every node's position ``tb`` and the global key
  (-priority, depth, rank, tb);
* the draft is the first dec_len-1 distinct token paths in that order, and a
  path's parent path always comes first, so a node whose key exceeds the
  current dec_len-1'th best distinct-path key can never contribute: each level
  only expands nodes at or below that threshold, and a child whose
  (-priority, depth, rank) already exceeds the threshold of the earlier levels
  is not generated (it sorts after every node that can matter, so class
  positions and first path occurrences of those are unchanged).
"""

from __future__ import annotations

from oracle import sssd_oracle as O


def fuse_ls(ds, inputs, P: int, dec_len: int, disc, root_token: int, stats: dict | None = None):
    K = dec_len - 1
    srcs = []
    if ds is not None and ds.count > 0:
        srcs.append((0, ds))
    for i in range(len(inputs) - 1, -1, -1):
        t = inputs[i]
        if t is not None and t.count > 0:
            srcs.append((P - i, t))
    # parent entries: (rank, source node, path prob or None for a root, tb, path id)
    parents = [(rk, t, None, 0, 0) for rk, t in srcs]
    paths = {}  # (parent path id, token) -> path id
    info = {0: (int(root_token), -1)}
    top = []  # (global key, path id) of the best distinct paths, key order
    depth = 1
    levels = []
    tau = None
    while parents and K > 0:
        nodes = []
        for rk, node, pp, tb, pid in parents:
            for i, (tok, c) in enumerate(node.kids.items()):
                dsc = disc[rk][depth]
                r = c.count / node.count
                cpp = r if pp is None else pp * r
                if tau is not None and (-(cpp * dsc), depth, rk) > tau[:3]:
                    continue  # beyond the threshold of the earlier levels
                nodes.append(((-(cpp * dsc), rk, tb, i), rk, c, cpp, pid, tok))
        nodes.sort(key=lambda x: x[0])
        cls = {}
        new = []
        keyed = []
        for sk, rk, c, cpp, pid, tok in nodes:
            tbn = cls.get(rk, 0)
            cls[rk] = tbn + 1
            g = (sk[0], depth, rk, tbn)
            q = paths.get((pid, tok))
            if q is None:
                q = paths[(pid, tok)] = len(info)
                info[q] = (tok, pid)
                new.append((g, q))
            keyed.append((g, rk, c, cpp, tbn, q))
        top = sorted(top + new)[:K]
        tau = top[-1][0] if len(top) == K else None
        parents = [(rk, c, cpp, tbn, q) for g, rk, c, cpp, tbn, q in keyed if tau is None or g <= tau]
        levels.append((len(nodes), len(new), len(parents)))
        depth += 1
    if stats is not None:
        stats["levels"] = levels
    # insertion order = key order of the selected paths
    d_tok = [int(root_token)]
    d_par = [-1]
    d_kids: list[dict] = [{}]
    nid_of = {0: 0}
    for _, q in top:
        tok, pid = info[q]
        par = nid_of[pid]
        nid = len(d_tok)
        nid_of[q] = nid
        d_tok.append(tok)
        d_par.append(par)
        d_kids.append({})
        d_kids[par][tok] = nid
    return d_tok, d_par, d_kids


def propose_ls(store, seq, cfg, separator=None, use_ds=True, use_in=True, stats=None):
    seq = [int(x) for x in seq]
    disc = cfg.disc()
    ds = None
    if use_ds:
        prefix = seq[len(seq) - min(cfg.P, len(seq)):]
        look = O.ds_lookup(store.tokens, store.sa, prefix, cfg.P, cfg.M, cfg.T, cfg.branch_len, separator)
        ds = O.trie_of(look.strings)
    ins = [O.trie_of(s) for s in O.input_strings(seq, cfg.P, cfg.input_branch_len)] if use_in else []
    return O.flatten(*fuse_ls(ds, ins, cfg.P, cfg.dec_len, disc, seq[-1], stats))
