"""GPU: per-node outputs of the fusion kernel (sssd_draft_out.priority /
.source / .pos) against the CPU oracle's heap merge, merge()'s DraftTree node
attributes (ref fusion.py:156-198, pkg/tests/test_fusion.py:171-260), and two
propose_pinned calls with DIFFERENT batches in flight on two slots."""

import math

import numpy as np
import pytest

from oracle import sssd_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2411_05894_b200 as G  # noqa: E402
from paper_2411_05894_b200 import workload  # noqa: E402
from paper_2411_05894_b200.fusion import DATASTORE_SOURCE, Source  # noqa: E402
from paper_2411_05894_b200.trees import tree_from_paths  # noqa: E402


def _ref_nodes(ds_tree, inputs, cfg, root):
    """(token path -> (priority, source)) of the reference merge restated
    with per-node provenance: the heap pop order of ref fusion.py:231-259."""
    import heapq
    import itertools

    tick = itertools.count()
    heap = []
    P = cfg.P

    def push(node, src, rank, depth, pp, parent_path):
        pr = pp * G.discount(cfg, src, depth)
        heapq.heappush(heap, (-pr, depth, rank, next(tick), node, pp, parent_path, src))

    def seed(t, src, rank):
        if t.is_empty:
            return
        for ch in t.children.values():
            push(ch, src, rank, 1, ch.count / t.root_count, ())

    seed(ds_tree, DATASTORE_SOURCE, 0)
    for i in range(len(inputs) - 1, -1, -1):
        seed(inputs[i], Source(Source.INPUT, i + 1), P - i)
    got = {(): (math.inf, None)}
    while heap and len(got) < cfg.dec_len:
        negp, depth, rank, _, node, pp, ppath, src = heapq.heappop(heap)
        path = ppath + (node.token,)
        if path not in got:
            got[path] = (-negp, src)
        for ch in node.children.values():
            push(ch, src, rank, depth + 1, pp * (ch.count / node.count), path)
    return got


def _tree_nodes(tree):
    out = {}
    stack = [(tree.root, ())]
    while stack:
        n, path = stack.pop()
        out[path] = (n.priority, n.source)
        for c in n.children.values():
            stack.append((c, path + (c.token,)))
    return out


def test_merge_carries_priority_and_source():
    rng = np.random.default_rng(5)
    for trial in range(60):
        cfg = G.FusionConfig(P=3, dec_len=int(rng.integers(2, 24)), alpha=float(rng.choice([0.5, 0.8, 1.0])),
                             beta=float(rng.choice([0.5, 1.0])), gamma_ds=float(rng.choice([0.5, 1.0])),
                             gamma_in=float(rng.choice([0.5, 0.95])))
        mk = lambda n, L, A: tree_from_paths([rng.integers(0, A, int(rng.integers(1, L + 1))).tolist()  # noqa: E731
                                              for _ in range(n)])
        ds = mk(int(rng.integers(0, 8)), 5, 4)
        ins = [mk(int(rng.integers(0, 5)), 4, 4) for _ in range(int(rng.integers(0, 4)))]
        tree = G.merge(ds, ins, cfg, root_token=9)
        want = _ref_nodes(ds, ins, cfg, 9)
        got = _tree_nodes(tree)
        assert set(got) == set(want), trial
        for path, (pr, src) in want.items():
            assert got[path][1] == src, (trial, path)
            assert got[path][0] == pr, (trial, path)  # bit-exact doubles


def test_merge_walkthrough_nodes():
    ds = tree_from_paths([[7, 5], [7], [8]])
    tree = G.merge(ds, [], G.FusionConfig(dec_len=4, gamma_ds=1.0), root_token=0)
    assert tree.root.priority == math.inf and tree.root.source is None
    assert tree.root.children[7].priority == 2 / 3 and tree.root.children[8].priority == 1 / 3
    assert tree.root.children[7].children[5].priority == 1 / 3
    ds, inp = tree_from_paths([[7, 5]]), tree_from_paths([[7, 9]])
    cfg = G.FusionConfig(P=1, dec_len=4, alpha=0.9, gamma_ds=1.0, gamma_in=1.0)
    tree = G.merge(ds, [inp], cfg, root_token=0)
    assert tree.root.children[7].source == DATASTORE_SOURCE and tree.root.children[7].priority == 1.0
    assert tree.root.children[7].children[9].source == Source(Source.INPUT, 1)


def test_propose_node_outputs_match_oracle():
    corpus = workload.corpus(200_000, 500)
    ds = G.build(corpus, vocab_size=500)
    store = O.Store(corpus, ds.suffix_index)
    cfg = G.FusionConfig(dec_len=32)
    eng = G.DraftEngine(ds, cfg)
    ctxs = [c.tolist() for c in workload.contexts(24, 96, 500)]
    ctxs += [c[: 1 + i] for i, c in enumerate(ctxs[:8])]  # short contexts: position ids from small L
    seq, off, ln, mx = eng.upload(ctxs)
    out = eng.propose(seq, off, ln, mx, nodes=True)
    eng.check_status()
    size = out.size.cpu().numpy()
    pos, pri, src = out.pos.cpu().numpy(), out.priority.cpu().numpy(), out.source.cpu().numpy()
    dep = out.depths.cpu().numpy()
    oc = O.Cfg(dec_len=32)
    toks = out.tokens.cpu().numpy().view(np.uint32)
    par = out.parents.cpu().numpy()
    for b, c in enumerate(ctxs):
        n = int(size[b])
        assert (pos[b, :n] == len(c) - 1 + dep[b, :n]).all() and (pos[b, n:] == -1).all()
        assert pri[b, 0] == math.inf and src[b, 0] == -1
        d = O.propose(store, c, oc)
        assert d.tokens == toks[b, :n].tolist()
        # expected provenance: the reference heap over the oracle's source tries
        prefix = c[len(c) - min(cfg.P, len(c)):]
        look = O.ds_lookup(store.tokens, store.sa, prefix, cfg.P, cfg.M, cfg.T, cfg.branch_len)
        ds_tree = tree_from_paths(look.strings)
        ins = [tree_from_paths(x) for x in O.input_strings(c, cfg.P, cfg.input_branch_len)]
        want = _ref_nodes(ds_tree, ins, cfg, c[-1])
        paths = [()]
        for i in range(1, n):
            paths.append(paths[par[b, i]] + (int(toks[b, i]),))
        assert set(paths) == set(want)
        for i in range(1, n):
            wp, ws = want[paths[i]]
            assert pri[b, i] == wp, (b, i)
            assert G.fusion.source_of_rank(int(src[b, i]), cfg.P) == ws, (b, i)


def test_two_different_batches_in_flight():
    """slots own their device outputs, so batch A's drafts are
    never overwritten by batch B's fusion while A downloads."""
    corpus = workload.corpus(300_000, 500)
    ds = G.build(corpus, vocab_size=500)
    eng = G.DraftEngine(ds, G.FusionConfig(dec_len=32))
    batches = []
    for seed in (11, 12):
        ctxs = workload.contexts(96, 200, 500, seed=seed)
        flat = np.concatenate(ctxs).astype(np.uint32)
        seq_h = torch.from_numpy(flat.view(np.int32)).pin_memory()
        off_h = torch.arange(96, dtype=torch.int64) * 200
        len_h = torch.full((96,), 200, dtype=torch.int32)
        ref = eng.propose_host([c.tolist() for c in ctxs])
        batches.append((seq_h, off_h, len_h, ref))
    for rep in range(3):
        pend = [eng.propose_pinned(s, o, l_, 200, chunks=3, slot=k, sync=False)
                for k, (s, o, l_, _) in enumerate(batches)]
        for p_, (_, _, _, ref) in zip(pend, batches):
            got = p_.wait()
            for b, f in enumerate(ref):
                n = f.s_q
                assert int(got.size[b]) == n
                assert got.tokens[b, :n].numpy().view(np.uint32).tolist() == f.tokens
                assert got.parents[b, :n].tolist() == f.parents
