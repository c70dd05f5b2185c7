"""Generate golden vectors by running the REFERENCE implementation.

Run once in the build container (the reference is not available on GPU boxes):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``specdraft`` read-only from /root/reference/pkg/src and writes
``tests/golden/*.json``.  Those fixtures pin both the CPU oracle
(``oracle/sssd_oracle.py``) and the CUDA path.  Every case records the inputs
and the reference's ordered outputs (``to_shape`` / flattened arrays / packed
mask bytes), never order-insensitive dict views alone.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from specdraft import datastore as rds  # noqa: E402
from specdraft import draft as rdr  # noqa: E402
from specdraft import fusion as rfu  # noqa: E402
from specdraft import harness as rha  # noqa: E402
from specdraft import input_cache as ric  # noqa: E402
from specdraft import trees as rtr  # noqa: E402

from paper_2411_05894_b200 import workload  # noqa: E402


def shape_tree(t) -> list:
    def r(node):
        return [node.count, [[int(k), r(v)] for k, v in node.children.items()]]

    return [t.root_count, [[int(k), r(v)] for k, v in t.children.items()]]


def cfg_dict(cfg) -> dict:
    return {k: v for k, v in cfg.to_kv().items()}


def flat_dict(flat) -> dict:
    return {
        "tokens": [int(x) for x in flat.tokens],
        "parents": [int(x) for x in flat.parents],
        "depths": [int(x) for x in flat.depths],
        "mask": rdr.pack_mask(flat.mask).hex(),
    }


def dump(name: str, obj) -> None:
    path = os.path.join(HERE, name)
    with open(path, "w") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def gen_sa(rng) -> None:
    cases = [[5, 6, 7, 5, 6, 8, 5, 6, 7, 9], [1, 1, 1], [3], [2] * 50, [4000000000, 7, 4000000000, 7]]
    for _ in range(40):
        n = int(rng.integers(1, 120))
        cases.append(rng.integers(0, int(rng.integers(1, 6)), n).tolist())
    cases.append(rng.integers(0, 7, 4000).tolist())
    cases.append(workload.corpus(20000, 500).tolist())
    out = []
    for c in cases:
        sa = rds.build_suffix_array(np.asarray(c, dtype="<u4"))
        out.append({"corpus": [int(x) for x in c], "sa": [int(x) for x in sa]})
    dump("sa.json", out)


def gen_lookup(rng) -> None:
    """find_range + sample_range + get_conts over random corpora and configs."""
    out = []
    for case in range(120):
        alphabet = int(rng.integers(2, 8))
        n = int(rng.integers(1, 300))
        corpus = rng.integers(0, alphabet, n).tolist()
        sep = None
        if rng.random() < 0.3:
            sep = alphabet
            for pos in rng.integers(0, n, max(1, n // 15)):
                corpus[int(pos)] = sep
        store = rds.build(corpus)
        qc = rds.DatastoreQueryConfig(
            max_prefix_len=int(rng.integers(1, 6)),
            sample_cap=int(rng.choice([1, 3, 8, 100])),
            min_continuations=int(rng.choice([1, 4, 16, 64])),
            branch_len=int(rng.integers(1, 9)),
            separator=sep,
        )
        queries = []
        for _ in range(8):
            plen = int(rng.integers(1, 7))
            if rng.random() < 0.6 and n > plen:
                s = int(rng.integers(0, n - plen + 1))
                prefix = corpus[s:s + plen]
            else:
                prefix = rng.integers(0, alphabet + 1, plen).tolist()
            prefix = [int(x) for x in prefix]
            ranges = []
            for p in range(1, len(prefix) + 1):
                lo, hi = store.find_range(prefix[-p:])
                ranges.append([p, int(lo), int(hi), [int(store.suffix_index[r]) for r in
                                                    rds.sample_range(lo, hi, qc.sample_cap)]])
            tree = store.get_conts(prefix, qc)
            queries.append({"prefix": prefix, "ranges": ranges, "tree": shape_tree(tree)})
        out.append({"corpus": corpus, "cfg": {"P": qc.max_prefix_len, "M": qc.sample_cap,
                                              "T": qc.min_continuations, "branch_len": qc.branch_len,
                                              "separator": sep}, "queries": queries})
    dump("lookup.json", out)


def gen_input(rng) -> None:
    out = []
    for case in range(150):
        L = int(rng.integers(1, 200))
        seq = rng.integers(0, int(rng.integers(2, 6)), L).tolist()
        P = int(rng.integers(1, 5))
        ibl = int(rng.integers(1, 9))
        cut = int(rng.integers(0, L + 1))
        cache = ric.InputCache(seq[:cut], P, ibl)
        cache.append(seq[cut:])
        trees = cache.get_conts()
        out.append({"seq": [int(x) for x in seq], "P": P, "ibl": ibl,
                    "trees": [shape_tree(t) for t in trees]})
    dump("input.json", out)


def _random_paths(rng, alphabet, max_paths, max_depth, tie):
    if rng.random() < 0.15:
        return []
    if tie:
        alphabet = min(alphabet, 3)
    paths = []
    for _ in range(int(rng.integers(1, max_paths + 1))):
        path = rng.integers(0, alphabet, int(rng.integers(1, max_depth + 1))).tolist()
        for _ in range(int(rng.integers(1, 4)) if tie else 1):
            paths.append([int(x) for x in path])
    return paths


def gen_merge(rng) -> None:
    out = []
    for trial in range(600):
        P = int(rng.integers(1, 5))
        cfg = rfu.FusionConfig(
            P=P,
            dec_len=int(rng.integers(1, 40)),
            alpha=float(rng.choice([0.0, 0.5, 0.8, 1.0])),
            beta=float(rng.choice([0.5, 0.8, 1.0])),
            gamma_ds=float(rng.choice([0.5, 1.0])),
            gamma_in=float(rng.choice([0.5, 0.95, 1.0])),
        )
        tie = bool(rng.random() < 0.35)
        ds_paths = _random_paths(rng, 5, 10, 5, tie)
        n_in = int(rng.integers(0, P + 1))
        in_paths = [_random_paths(rng, 5, 6, 5, tie) for _ in range(n_in)]
        root = int(rng.integers(0, 5))
        tree = rfu.merge(rtr.tree_from_paths(ds_paths), [rtr.tree_from_paths(p) for p in in_paths],
                         cfg, root_token=root)
        flat = rdr.flatten(tree)
        out.append({"cfg": cfg_dict(cfg), "ds": ds_paths, "inputs": in_paths, "root": root,
                    "shape": json.loads(json.dumps(tree.to_shape())), "flat": flat_dict(flat)})
    dump("merge.json", out)


def gen_propose(rng) -> None:
    """GenerationSession.propose on random small stores (sources / separators / configs)."""
    out = []
    for trial in range(200):
        alphabet = int(rng.integers(3, 9))
        n = int(rng.integers(20, 400))
        corpus = rng.integers(0, alphabet, n).tolist()
        sep = None
        if rng.random() < 0.25:
            sep = alphabet
            for pos in rng.integers(0, n, max(1, n // 20)):
                corpus[int(pos)] = sep
        store = rds.build(corpus)
        cfg = rfu.FusionConfig(
            P=int(rng.integers(1, 6)),
            dec_len=int(rng.choice([1, 2, 5, 8, 16, 30, 64])),
            input_branch_len=int(rng.integers(1, 9)),
            M=int(rng.choice([4, 16, 100])),
            T=int(rng.choice([1, 4, 16])),
            alpha=float(rng.choice([0.0, 0.5, 0.8, 1.0])),
            beta=float(rng.choice([0.5, 0.8, 1.0])),
            gamma_ds=float(rng.choice([0.5, 1.0])),
            gamma_in=float(rng.choice([0.5, 0.95, 1.0])),
        )
        sources = ["both", "both", "both", "datastore", "input"][int(rng.integers(0, 5))]
        use_ds, use_in = sources in ("both", "datastore"), sources in ("both", "input")
        seqs = []
        for _ in range(4):
            L = int(rng.integers(1, 120))
            if rng.random() < 0.5:
                s = int(rng.integers(0, max(1, n - L)))
                seq = [int(x) for x in corpus[s:s + L] if x != sep] or [0]
            else:
                seq = rng.integers(0, alphabet, L).tolist()
            sess = rdr.GenerationSession.start(store, seq, cfg, separator=sep,
                                               use_datastore=use_ds, use_input=use_in)
            seqs.append({"seq": [int(x) for x in seq], "flat": flat_dict(sess.propose())})
        out.append({"corpus": corpus, "cfg": cfg_dict(cfg), "separator": sep, "sources": sources,
                    "requests": seqs})
    dump("propose.json", out)


def gen_simulate(rng) -> None:
    out = []
    for trial in range(60):
        alphabet = int(rng.integers(4, 9))
        n = int(rng.integers(80, 201))
        corpus = rng.integers(0, alphabet, n).tolist()
        prompt = rng.integers(0, alphabet, int(rng.integers(1, 9))).tolist()
        ref = []
        while len(ref) < 24:
            if rng.random() < 0.5:
                k = int(rng.integers(3, 11))
                s = int(rng.integers(0, n - k + 1))
                ref.extend(corpus[s:s + k])
            else:
                ref.extend(rng.integers(0, alphabet, int(rng.integers(1, 6))).tolist())
        ref = [int(x) for x in ref[:24]]
        cfg = rfu.FusionConfig(P=int(rng.integers(1, 5)), dec_len=int(rng.integers(2, 13)),
                               input_branch_len=int(rng.integers(1, 9)),
                               M=int(rng.choice([8, 64])), T=int(rng.choice([1, 4])))
        store = rds.build(corpus)
        stats = rha.run_record(0, rha.SimRecord(prompt, ref), store, cfg)
        out.append({"corpus": [int(x) for x in corpus], "prompt": [int(x) for x in prompt],
                    "reference": ref, "cfg": cfg_dict(cfg), "per_step": stats.per_step_tokens})
    dump("simulate.json", out)


def gen_phrase() -> None:
    """Phrase-model workload at a moderate scale: propose digests and a
    teacher-forced simulation, the CPU-scale stand-ins for cfg1/cfg2."""
    corpus = workload.corpus(300_000, 32000)
    store = rds.build(corpus, vocab_size=32000)
    out = {"n": 300_000, "vocab": 32000, "cases": []}
    ctxs = workload.contexts(32, 512, 32000)
    for dec_len in (16, 64):
        cfg = rfu.FusionConfig(dec_len=dec_len)
        sess = [rdr.GenerationSession.start(store, c, cfg) for c in ctxs]
        drafts = [s.propose() for s in sess]
        out["cases"].append({"kind": "propose", "B": 32, "ctx": 512, "cfg": cfg_dict(cfg),
                             "digest": rha.draft_digest(drafts),
                             "flats": [flat_dict(f) for f in drafts]})
    recs = workload.records(6, 256, 48, 32000)
    cfg = rfu.FusionConfig(dec_len=16)
    sims = [rha.run_record(i, rha.SimRecord(p, r), store, cfg).per_step_tokens
            for i, (p, r) in enumerate(recs)]
    out["cases"].append({"kind": "simulate", "records": 6, "prompt": 256, "ref": 48,
                         "cfg": cfg_dict(cfg), "per_step": sims})
    sa = store.suffix_index
    out["sa_sha256"] = __import__("hashlib").sha256(np.asarray(sa, dtype="<u8").tobytes()).hexdigest()
    dump("phrase.json", out)


def gen_files() -> None:
    """SSSD v1 datastore files written by the reference (ref datastore.py:
    220-226): sha256 of the exact bytes, which the GPU-built file must equal."""
    import hashlib
    import tempfile

    cases = [([5, 6, 7, 5, 6, 8, 5, 6, 7, 9], None), ([1, 1, 1], 4),
             (workload.corpus(50_000, 1000).tolist(), 1000), (workload.corpus(200_000, 32000).tolist(), None)]
    out = []
    with tempfile.TemporaryDirectory() as d:
        for corpus, vocab in cases:
            path = os.path.join(d, "ds.bin")
            rds.build(corpus, vocab_size=vocab).save(path)
            data = open(path, "rb").read()
            rec = {"vocab": vocab, "n": len(corpus), "bytes": len(data), "sha256": hashlib.sha256(data).hexdigest()}
            if len(corpus) <= 16:
                rec["corpus"] = corpus
                rec["hex"] = data.hex()
            else:
                rec["workload"] = "corpus(%d, %d)" % (len(corpus), 1000 if vocab == 1000 else 32000)
            out.append(rec)
    dump("files.json", out)


def main() -> None:
    gen_sa(np.random.default_rng(0xC0FFEE))
    gen_lookup(np.random.default_rng(1))
    gen_input(np.random.default_rng(2))
    gen_merge(np.random.default_rng(3))
    gen_propose(np.random.default_rng(4))
    gen_simulate(np.random.default_rng(5))
    gen_phrase()
    gen_files()


if __name__ == "__main__":
    main()
