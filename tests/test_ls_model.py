"""The level-synchronous fusion restatement (tests/ls_model.py — the algorithm
of the default GPU fusion kernel, csrc/fusion_ls.cu) is bit-identical to the
oracle's heap-order merge (ref fusion.py:209-261): on every golden merge the
reference produced, on random tie-heavy source tries (tiny alphabets,
duplicated paths, alpha = 0, gamma = 1) and on real proposals."""

import numpy as np

from oracle import sssd_oracle as O
from tests import ls_model as L


def _flat(d):
    return d.tokens, d.parents, d.depths


def test_ls_model_matches_golden_merges(golden):
    for case in golden("merge.json"):
        c = case["cfg"]
        disc = O.discount_table(c["P"], 8, c["alpha"], c["beta"], c["gamma_ds"], c["gamma_in"])
        ds = O.trie_of(case["ds"])
        ins = [O.trie_of(p) for p in case["inputs"]]
        a = O.flatten(*O.fuse(ds, ins, c["P"], c["dec_len"], disc, case["root"]))
        b = O.flatten(*L.fuse_ls(ds, ins, c["P"], c["dec_len"], disc, case["root"]))
        assert _flat(a) == _flat(b)
        assert _flat(b) == (case["flat"]["tokens"], case["flat"]["parents"], case["flat"]["depths"])


def test_ls_model_random_tie_heavy():
    rng = np.random.default_rng(7)
    for _ in range(1500):
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

        ds = O.trie_of(paths(40))
        ins = [O.trie_of(paths(30)) for _ in range(int(rng.integers(0, P + 1)))]
        a = O.flatten(*O.fuse(ds, ins, P, dec, disc, 0))
        b = O.flatten(*L.fuse_ls(ds, ins, P, dec, disc, 0))
        assert _flat(a) == _flat(b)


def test_ls_model_real_proposals():
    from paper_2411_05894_b200 import workload

    corpus = workload.corpus(200_000, 2000)
    store = O.Store(corpus, O.suffix_array(corpus))
    cfg = O.Cfg(dec_len=64)
    for c in workload.contexts(40, 1024, 2000):
        assert _flat(O.propose(store, c, cfg)) == _flat(L.propose_ls(store, c, cfg))
