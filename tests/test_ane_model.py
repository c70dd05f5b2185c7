"""The all-nodes fusion restatements (tests/ane_model.py over tries,
tests/ane_elements.py over the kernel's sorted element arrays -- the algorithm
of csrc/fusion_ane.cu) are bit-identical to the oracle's heap-order merge (ref
fusion.py:209-261): on every golden merge the reference produced, on random
tie-heavy source tries (with a small initial candidate count, so the
threshold-doubling path runs) and on real proposals."""

import numpy as np

from oracle import sssd_oracle as O
from tests import ane_elements as AE
from tests import ane_model as AM


def _flat(d):
    return d.tokens, d.parents, d.depths


def _elements(paths):
    """Element array of a tree given as its path multiset: (path, first
    appearance, m, weight) sorted by (path, first appearance); thr 0."""
    return sorted(((tuple(p), i, 255, 1) for i, p in enumerate(paths)), key=lambda e: (e[0], e[1]))


def _sources(ds_paths, in_paths, P):
    srcs = [(0, 0, _elements(ds_paths))]
    for i, ps in enumerate(in_paths):  # input tree p = i + 1 merges at rank P - p + 1
        srcs.append((P - i, 0, _elements(ps)))
    return srcs


def test_ane_matches_golden_merges(golden):
    for case in golden("merge.json"):
        c = case["cfg"]
        disc = O.discount_table(c["P"], 8, c["alpha"], c["beta"], c["gamma_ds"], c["gamma_in"])
        ds = O.trie_of(case["ds"])
        ins = [O.trie_of(p) for p in case["inputs"]]
        want = (case["flat"]["tokens"], case["flat"]["parents"], case["flat"]["depths"])
        assert _flat(O.flatten(*AM.fuse_ane(ds, ins, c["P"], c["dec_len"], disc, case["root"]))) == want
        srcs = _sources(case["ds"], case["inputs"], c["P"])
        assert _flat(O.flatten(*AE.fuse_elements(srcs, c["P"], c["dec_len"], disc, case["root"]))) == want


def test_ane_random_tie_heavy():
    rng = np.random.default_rng(11)
    for _ in range(600):
        P = int(rng.integers(1, 5))
        dec = int(rng.integers(1, 70))
        disc = O.discount_table(P, 8, float(rng.choice([0.0, 0.5, 0.8, 1.0])), float(rng.choice([0.5, 0.8, 1.0])),
                                float(rng.choice([0.5, 1.0])), float(rng.choice([0.5, 0.95, 1.0])))
        alph = int(rng.choice([2, 3, 5, 20]))

        def paths(n):
            out = []
            for _ in range(int(rng.integers(0, n))):
                p = rng.integers(0, alph, int(rng.integers(1, 9))).tolist()
                out += [p] * int(rng.integers(1, 4))
            return out

        dsp = paths(40)
        insp = [paths(30) for _ in range(int(rng.integers(0, P + 1)))]
        want = _flat(O.flatten(*O.fuse(O.trie_of(dsp), [O.trie_of(p) for p in insp], P, dec, disc, 0)))
        c0 = int(rng.integers(1, 8))
        got = O.flatten(*AE.fuse_elements(_sources(dsp, insp, P), P, dec, disc, 0, C0=c0))
        assert _flat(got) == want


def test_ane_real_proposals():
    from paper_2411_05894_b200 import workload

    corpus = workload.corpus(200_000, 2000)
    store = O.Store(corpus, O.suffix_array(corpus))
    cfg = O.Cfg(dec_len=64)
    for c in workload.contexts(20, 1024, 2000):
        want = _flat(O.propose(store, c, cfg))
        assert _flat(AM.propose_ane(store, c, cfg)) == want
        assert _flat(AE.propose_elements(store, c, cfg)) == want
