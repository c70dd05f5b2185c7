"""GPU parity: the CUDA path (through the C ABI) against golden vectors made by
the reference and against the CPU oracle.  Bit-exact for every integer output
(suffix arrays, [lo, hi) ranges, sampled positions, ordered trees, flattened
drafts, packed masks, per-step token counts)."""

import hashlib

import numpy as np
import pytest

from oracle import sssd_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2411_05894_b200 as G  # noqa: E402
from paper_2411_05894_b200 import workload  # noqa: E402
from paper_2411_05894_b200.draft import pack_mask  # noqa: E402


def shape_of(tree) -> list:
    def r(node):
        return [node.count, [[int(k), r(v)] for k, v in node.children.items()]]

    return [tree.root_count, [[int(k), r(v)] for k, v in tree.children.items()]]


def flat_dict(f) -> dict:
    return {"tokens": [int(x) for x in f.tokens], "parents": list(f.parents), "depths": list(f.depths),
            "mask": pack_mask(f.mask).hex()}


def test_sa_build_golden(golden):
    for case in golden("sa.json"):
        ds = G.build(case["corpus"])
        assert ds.suffix_index.tolist() == case["sa"]


def test_sa_build_phrase_and_random():
    g = __import__("json").load(open(__import__("os").path.join(__import__("os").path.dirname(__file__),
                                                                "golden", "phrase.json")))
    corpus = workload.corpus(g["n"], g["vocab"])
    ds = G.build(corpus, vocab_size=g["vocab"])
    assert hashlib.sha256(ds.suffix_index.astype("<u8").tobytes()).hexdigest() == g["sa_sha256"]
    rng = np.random.default_rng(5)
    for alpha, n in [(2, 20000), (3, 50000), (1000, 200000), (2**32 - 1, 3000)]:
        c = rng.integers(0, alpha, n, dtype=np.int64).astype(np.uint32)
        assert np.array_equal(G.build(c).suffix_index, O.suffix_array(c))


def test_lookup_golden(golden):
    """find_range + sample_range positions + ordered get_conts trees."""
    for case in golden("lookup.json"):
        ds = G.build(case["corpus"])
        c = case["cfg"]
        qc = G.DatastoreQueryConfig(c["P"], c["M"], c["T"], c["branch_len"], c["separator"])
        pats, want = [], []
        for q in case["queries"]:
            for p, lo, hi, pos in q["ranges"]:
                pats.append(q["prefix"][len(q["prefix"]) - p:])
                want.append((lo, hi))
        assert ds.find_ranges(pats) == want
        for q in case["queries"]:
            assert shape_of(ds.get_conts(q["prefix"], qc)) == q["tree"]


def test_lookup_samples_match_oracle():
    """Sampled SA positions and per-p counts from the propose path itself."""
    corpus = workload.corpus(200_000, 500)
    ds = G.build(corpus)
    sa = O.suffix_array(corpus)
    ctxs = workload.contexts(48, 64, 500)
    cfg = G.FusionConfig(dec_len=16, M=20, T=30)
    eng = G.DraftEngine(ds, cfg)
    drafts, out = eng.propose_host([c.tolist() for c in ctxs], lookup=True)
    ranges = out.ranges.cpu().numpy()
    samples = out.samples.cpu().numpy()
    pcut = out.p_cut.cpu().numpy()
    for b, ctx in enumerate(ctxs):
        look = O.ds_lookup(corpus, sa, ctx[-4:].tolist(), cfg.P, cfg.M, cfg.T, cfg.branch_len)
        for p in range(1, 5):
            lo, hi = O.find_range(corpus, sa, ctx[-p:].tolist())
            assert tuple(ranges[b, p - 1]) == (lo, hi)
        assert pcut[b] == look.ranges[-1][0]
        for p, pos in look.samples:
            assert samples[b, p - 1, : len(pos)].tolist() == pos


def test_input_golden(golden):
    from paper_2411_05894_b200.input_cache import input_trees_batch

    cases = golden("input.json")
    for case in cases:
        trees = input_trees_batch([case["seq"]], case["P"], case["ibl"])[0]
        assert [shape_of(t) for t in trees] == case["trees"]


def test_merge_golden(golden):
    cases = golden("merge.json")
    by_cfg: dict = {}
    for case in cases:
        by_cfg.setdefault(tuple(sorted(case["cfg"].items())), []).append(case)
    for key, group in by_cfg.items():
        cfg = G.FusionConfig(**dict(key))
        reqs = [(G.tree_from_paths(cs["ds"]), [G.tree_from_paths(p) for p in cs["inputs"]], cs["root"])
                for cs in group]
        # requests with different numbers of input trees are fused separately
        for n_in in sorted({len(r[1]) for r in reqs}):
            sub = [(r, cs) for r, cs in zip(reqs, group) if len(r[1]) == n_in]
            flats = G.merge_batch([r for r, _ in sub], cfg)
            for f, (_, cs) in zip(flats, sub):
                assert flat_dict(f) == cs["flat"]


def test_propose_golden(golden):
    for case in golden("propose.json"):
        ds = G.build(case["corpus"])
        cfg = G.FusionConfig(**case["cfg"])
        src = case["sources"]
        eng = G.DraftEngine(ds, cfg, case["separator"], src in ("both", "datastore"), src in ("both", "input"))
        flats = eng.propose_host([r["seq"] for r in case["requests"]])
        for f, r in zip(flats, case["requests"]):
            assert flat_dict(f) == r["flat"]


def test_phrase_golden_digests(golden):
    g = golden("phrase.json")
    ds = G.build(workload.corpus(g["n"], g["vocab"]), vocab_size=g["vocab"])
    for case in g["cases"]:
        cfg = G.FusionConfig(**case["cfg"])
        if case["kind"] == "propose":
            ctxs = [c.tolist() for c in workload.contexts(case["B"], case["ctx"], g["vocab"])]
            flats = G.DraftEngine(ds, cfg).propose_host(ctxs)
            assert [flat_dict(f) for f in flats] == case["flats"]
            assert G.draft_digest(flats) == case["digest"]
        else:
            recs = [G.SimRecord(p, r) for p, r in workload.records(case["records"], case["prompt"], case["ref"],
                                                                   g["vocab"])]
            rep = G.simulate(recs, ds, cfg)
            assert [r.per_step_tokens for r in rep.records] == case["per_step"]


def test_simulate_golden(golden):
    for case in golden("simulate.json"):
        ds = G.build(case["corpus"])
        st = G.run_record(0, G.SimRecord(case["prompt"], case["reference"]), ds, G.FusionConfig(**case["cfg"]))
        assert st.per_step_tokens == case["per_step"]


def test_simulate_batch_composition_invariant():
    """Continuous batching: per-record stats independent of slot count."""
    corpus = workload.corpus(100_000, 2000)
    ds = G.build(corpus)
    recs = [G.SimRecord(p, r) for p, r in workload.records(12, 64, 40, 2000)]
    cfg = G.FusionConfig(dec_len=12)
    a = G.simulate(recs, ds, cfg, slots=12).deterministic_dict()
    b = G.simulate(recs, ds, cfg, slots=5).deterministic_dict()
    assert a == b
    store = O.Store(corpus, O.suffix_array(corpus))
    oc = O.Cfg(dec_len=12)
    for i, r in enumerate(recs):
        assert a["records"][i]["per_step_tokens"] == O.run_record(store, r.prompt, r.reference, oc)


def test_propose_vs_oracle_random_shapes():
    """Random stores / configs / long contexts against the oracle (ordered)."""
    rng = np.random.default_rng(11)
    for trial in range(6):
        V = int(rng.choice([3, 8, 50]))
        corpus = rng.integers(0, V, int(rng.integers(500, 20000))).astype(np.uint32)
        sa = O.suffix_array(corpus)
        store = O.Store(corpus, sa)
        ds = G.build(corpus)
        cfg = G.FusionConfig(P=int(rng.integers(1, 6)), dec_len=int(rng.choice([8, 32, 64, 100])),
                             input_branch_len=int(rng.integers(1, 9)), M=int(rng.choice([10, 100])),
                             T=int(rng.choice([1, 16, 50])))
        ctxs = [rng.integers(0, V, int(rng.integers(1, 3000))).tolist() for _ in range(16)]
        flats = G.DraftEngine(ds, cfg).propose_host(ctxs)
        oc = O.Cfg(**{k: getattr(cfg, k) for k in ("P", "dec_len", "branch_len", "input_branch_len", "M", "T",
                                                    "alpha", "beta", "gamma_ds", "gamma_in")})
        for f, ctx in zip(flats, ctxs):
            d = O.propose(store, ctx, oc)
            assert (f.tokens, f.parents, f.depths) == (d.tokens, d.parents, d.depths), trial
            assert pack_mask(f.mask) == O.pack_mask_rows(d.masks, d.size)


def test_long_context_input_sort_path():
    """>4096 occurrences of the last token exercises the global-memory sort."""
    rng = np.random.default_rng(3)
    seq = rng.integers(0, 3, 20000).tolist()
    corpus = rng.integers(0, 3, 5000).astype(np.uint32)
    store = O.Store(corpus, O.suffix_array(corpus))
    cfg = G.FusionConfig(dec_len=16)
    f = G.DraftEngine(G.build(corpus), cfg).propose_host([seq])[0]
    d = O.propose(store, seq, O.Cfg(dec_len=16))
    assert (f.tokens, f.parents, f.depths) == (d.tokens, d.parents, d.depths)


@pytest.mark.parametrize("alphabet,dec_len", [(8, 16), (12, 64), (16, 32)])
def test_long_context_bitonic_input_sort(alphabet, dec_len):
    """1,024 < occurrences <= 4,096 in a > 4,096-token context: the packed keys
    are bitonic-sorted in shared memory (ties by position); drafts bit-exact
    vs the oracle."""
    rng = np.random.default_rng(alphabet)
    seqs = [rng.integers(0, alphabet, int(n)).tolist() for n in (20000, 9000, 30000)]
    corpus = rng.integers(0, alphabet, 50000).astype(np.uint32)
    store = O.Store(corpus, O.suffix_array(corpus))
    cfg = G.FusionConfig(dec_len=dec_len)
    got = G.DraftEngine(G.build(corpus), cfg).propose_host(seqs)
    for seq, f in zip(seqs, got):
        occ = sum(1 for t in seq[:-1] if t == seq[-1])
        assert 1024 < occ <= 4096 or len(seq) < 10000
        d = O.propose(store, seq, O.Cfg(dec_len=dec_len))
        assert (f.tokens, f.parents, f.depths) == (d.tokens, d.parents, d.depths)


@pytest.mark.parametrize("L,alphabet", [(3000, 9), (4000, 12), (9000, 8), (20000, 10), (30000, 14), (2000, 3),
                                        (600, 40), (200, 50)])
def test_input_scan_element_order(L, alphabet):
    """The input scan's element rows, in output order, are sorted by
    continuation string (a proper prefix first) with ties by position, and hold
    exactly the occurrences of the last token with their backward-match
    lengths: checked row by row against numpy for occurrence counts across the
    run-rank (<= 32), merge (33-2,457 at 1,024 threads, 33-409 at 256) and
    bitonic / run-rank fallbacks (larger counts) of both launch widths."""
    from paper_2411_05894_b200.input_cache import input_elements_batch

    rng = np.random.default_rng(L + alphabet)
    P, ibl = 4, 8
    seqs = [rng.integers(0, alphabet, L).tolist() for _ in range(3)]
    seqs.append(workload.prompt_heavy_contexts(1, max(L, 4097), 32000)[0].tolist())
    got = input_elements_batch(seqs, P, ibl)
    for seq, rows in zip(seqs, got):
        s = np.asarray(seq)
        n = len(s)
        last = s[-1]
        occ = [e for e in range(1, n) if s[e - 1] == last]
        m = O.match_lengths(seq, P)
        want = sorted(occ, key=lambda e: (tuple(s[e:e + min(ibl, n - e)].tolist()), e))
        assert rows.shape[0] == len(want)
        assert rows[:, 0].tolist() == want and rows[:, 1].tolist() == want
        assert [int(x) & 0xFF for x in rows[:, 2]] == [min(ibl, n - e) for e in want]
        assert [(int(x) >> 8) & 0xFF for x in rows[:, 2]] == [int(m[e]) for e in want]


def test_verify_matches_oracle():
    rng = np.random.default_rng(9)
    corpus = workload.corpus(50_000, 50)
    ds = G.build(corpus)
    ctxs = [c.tolist() for c in workload.contexts(64, 100, 50)]
    flats = G.DraftEngine(ds, G.FusionConfig(dec_len=24)).propose_host(ctxs)
    preds = []
    for f in flats:
        p = []
        for i in range(f.s_q):
            kids = [f.tokens[j] for j in range(1, f.s_q) if f.parents[j] == i]
            p.append(int(rng.choice(kids)) if kids and rng.random() < 0.7 else int(rng.integers(0, 50)))
        preds.append(p)
    got = G.verify_batch(flats, preds)
    for f, p, r in zip(flats, preds, got):
        d = O.Draft(f.tokens, f.parents, f.depths, [0] * f.s_q)
        assert (r.accepted_path, r.bonus_token) == O.verify(d, p)


def test_save_load_roundtrip(tmp_path):
    corpus = np.random.default_rng(1).integers(0, 1000, 3000)
    ds = G.build(corpus, vocab_size=1000)
    path = tmp_path / "ds.bin"
    ds.save(path)
    back = G.load(path)
    assert np.array_equal(back.suffix_index, ds.suffix_index)
    assert back.vocab_size == 1000
    assert back.find_range([int(corpus[5]), int(corpus[6])]) == ds.find_range([int(corpus[5]), int(corpus[6])])


def test_propose_pinned_equals_resident_propose():
    """The pipelined host-buffer entry point (both schedules: phased — lookup of
    every request from its zero-copy tail, then scan / fusion per uploaded
    range — and independent ranges) returns exactly the drafts of one
    device-resident propose, for
    ragged lengths and offsets in shuffled order; the engine's workspace status
    stays readable after calls of different batch sizes."""
    rng = np.random.default_rng(21)
    corpus = workload.corpus(300_000, 500)
    ds = G.build(corpus, vocab_size=500)
    eng = G.DraftEngine(ds, G.FusionConfig(dec_len=48))
    B = 37
    ctxs = [rng.integers(0, 500, int(rng.integers(1, 900))).astype(np.uint32) for _ in range(B)]
    ctxs[:3] = [rng.integers(0, 500, n).astype(np.uint32) for n in (1, 2, 3)]  # shorter than P (tail views)
    order = rng.permutation(B)  # request r stored at a shuffled position in the flat buffer
    flat, offs, pos = [], np.zeros(B, np.int64), 0
    for r in order:
        offs[r] = pos
        flat.append(ctxs[r])
        pos += len(ctxs[r])
    seq_h = torch.from_numpy(np.concatenate(flat).view(np.int32)).pin_memory()
    off_h = torch.from_numpy(offs)
    len_h = torch.tensor([len(c) for c in ctxs], dtype=torch.int32)
    mx = int(len_h.max())
    want = eng.propose(seq_h.cuda(), off_h.cuda(), len_h.cuda(), mx)
    want = {k: getattr(want, k).cpu().clone() for k in ("size", "tokens", "parents", "depths", "mask")}
    eng.check_status()
    seq16_h = torch.from_numpy(seq_h.numpy().astype(np.uint16).view(np.int16)).pin_memory()  # vocab 500 < 2^16
    for schedule, chunks, src in [(s, c, x) for s in ("phased", "ranges")
                                  for c, x in ((1, seq_h), (3, seq_h), (8, seq_h), (3, seq16_h), (8, seq16_h))]:
        got = eng.propose_pinned(src, off_h, len_h, mx, chunks=chunks, schedule=schedule)
        for k, v in want.items():
            g = getattr(got, k)
            assert not g.is_cuda and g.is_pinned()
            if k == "size":
                assert torch.equal(g, v), (schedule, chunks, k)
            else:  # entries past size are unspecified
                for b in range(B):
                    n = int(want["size"][b])
                    assert torch.equal(g[b, :n], v[b, :n]), (schedule, chunks, k, b)
    # two calls in flight on different slots (async), then waited: both exact
    pend = [eng.propose_pinned(src, off_h, len_h, mx, chunks=3, slot=k, sync=False) for k, src in
            ((0, seq_h), (1, seq16_h))]
    for p_ in pend:
        got = p_.wait()
        assert torch.equal(got.size, want["size"])
        for b in range(B):
            n = int(want["size"][b])
            assert torch.equal(got.tokens[b, :n], want["tokens"][b, :n])
            assert torch.equal(got.mask[b, :n], want["mask"][b, :n])
    eng.propose_host([c.tolist() for c in ctxs[:3]])  # smaller call through a larger workspace
    eng.check_status()


def _engines(monkeypatch, ds, cfg, **kw):
    monkeypatch.setenv("SSSD_FUSION", "heap")
    heap = G.DraftEngine(ds, cfg, **kw)
    monkeypatch.setenv("SSSD_FUSION", "ls")
    ls = G.DraftEngine(ds, cfg, **kw)
    assert heap.c.fusion == 1 and ls.c.fusion == 0
    return heap, ls


def _same_batch(a, b):
    for k in ("size", "tokens", "parents", "depths", "mask"):
        x, y = getattr(a, k), getattr(b, k)
        if k != "size":  # rows past size are padding in both forms
            assert torch.equal(x, y), k
        else:
            assert torch.equal(x, y)


@pytest.mark.parametrize("dec_len,ctx,n_req,alpha", [(64, 2048, 2048, 0.8), (16, 32768, 8, 0.8),
                                                     (100, 1024, 512, 0.0), (256, 512, 256, 1.0)])
def test_level_synchronous_fusion_equals_heap_form(monkeypatch, dec_len, ctx, n_req, alpha):
    """The level-synchronous fusion kernel (fusion_ls.cu, the default) and the
    heap-order kernel (fusion.cu) produce identical drafts over phrase-model
    workloads: cfg2 shape, a prompt-heavy 32k context (big levels in the global
    pool), alpha = 0 (all input priorities tie at 0) and dec_len 256."""
    corpus = workload.corpus(1_000_000, 32000)
    ds = G.build(corpus, vocab_size=32000)
    cfg = G.FusionConfig(dec_len=dec_len, alpha=alpha)
    heap, ls = _engines(monkeypatch, ds, cfg)
    ctxs = workload.prompt_heavy_contexts(n_req, ctx, 32000) if ctx > 4096 else workload.contexts(n_req, ctx, 32000)
    flat = np.concatenate([np.asarray(c, dtype=np.uint32) for c in ctxs])
    seq = torch.from_numpy(flat.view(np.int32)).cuda()
    off = torch.arange(n_req, dtype=torch.int64, device="cuda") * ctx
    ln = torch.full((n_req,), ctx, dtype=torch.int32, device="cuda")
    a = heap.propose(seq, off, ln, ctx)
    heap.check_status()
    b = ls.propose(seq, off, ln, ctx)
    ls.check_status()
    torch.cuda.synchronize()
    _same_batch(a, b)


def test_level_synchronous_fusion_small_alphabets(monkeypatch):
    """Tie-heavy tiny alphabets (many equal counts / priorities, duplicate paths
    across all P+1 sources) through both fusion kernels."""
    rng = np.random.default_rng(5)
    for trial in range(4):
        V = int(rng.choice([2, 3, 5]))
        corpus = rng.integers(0, V, 20000).astype(np.uint32)
        ds = G.build(corpus)
        cfg = G.FusionConfig(P=int(rng.integers(1, 6)), dec_len=int(rng.choice([5, 33, 64, 200])),
                             alpha=float(rng.choice([0.0, 0.5, 1.0])), beta=float(rng.choice([0.5, 1.0])),
                             gamma_ds=float(rng.choice([0.5, 1.0])), gamma_in=float(rng.choice([0.5, 1.0])))
        heap, ls = _engines(monkeypatch, ds, cfg)
        ctxs = [rng.integers(0, V, int(rng.integers(1, 4000))).tolist() for _ in range(64)]
        fa = heap.propose_host(ctxs)
        fb = ls.propose_host(ctxs)
        for x, y in zip(fa, fb):
            assert (x.tokens, x.parents, x.depths) == (y.tokens, y.parents, y.depths), trial


def test_first_token_bucket_index():
    """bucket[t] = first suffix row whose first token >= t (checked against the
    sorted suffixes), and range searches with the index equal the oracle's
    find_range for p = 1..6, including tokens beyond the table."""
    rng = np.random.default_rng(17)
    corpus = rng.integers(0, 40, 30000).astype(np.uint32)
    ds = G.build(corpus, vocab_size=40)
    sa = O.suffix_array(corpus)
    first = corpus[sa]
    bk = ds.bucket().cpu().numpy().astype(np.int64)
    want = np.searchsorted(first, np.arange(bk.size), side="left")
    assert np.array_equal(bk, want)
    pats = [rng.integers(0, 45, int(rng.integers(1, 7))).tolist() for _ in range(300)]
    pats += [corpus[i:i + k].tolist() for i, k in zip(rng.integers(0, 29990, 200), rng.integers(1, 7, 200))]
    got = ds.find_ranges(pats)
    for pt, g in zip(pats, got):
        assert tuple(g) == O.find_range(corpus, sa, pt), pt


@pytest.mark.parametrize("ibl", [4, 12])
def test_propose_large_token_ids(ibl):
    """Token ids >= 65535 (and input_branch_len > 8) take the string-compare
    path of the input-scan sort instead of packed 16-bit keys; drafts stay
    bit-exact against the oracle."""
    rng = np.random.default_rng(23)
    alphabet = np.array([3, 7, 65534, 65535, 70000, 4_000_000_000], dtype=np.uint32)
    corpus = alphabet[rng.integers(0, alphabet.size, 30000)]
    store = O.Store(corpus, O.suffix_array(corpus))
    cfg = G.FusionConfig(dec_len=40, input_branch_len=ibl)
    ctxs = [alphabet[rng.integers(0, alphabet.size, int(rng.integers(50, 600)))].tolist() for _ in range(40)]
    flats = G.DraftEngine(G.build(corpus), cfg).propose_host(ctxs)
    oc = O.Cfg(dec_len=40, input_branch_len=ibl)
    for f, ctx in zip(flats, ctxs):
        d = O.propose(store, ctx, oc)
        assert (f.tokens, f.parents, f.depths) == (d.tokens, d.parents, d.depths)


@pytest.mark.parametrize("dec_len,P,ibl,bl,sep,src", [
    (1, 4, 8, None, None, "both"), (2, 4, 8, None, None, "both"), (3, 8, 8, None, 3, "both"),
    (40, 8, 20, 12, 5, "both"), (64, 3, 32, 6, None, "input"), (64, 6, 4, 16, 2, "datastore"),
    (130, 2, 12, 10, None, "both"), (48, 8, 8, 12, None, "datastore"), (64, 7, 8, 8, None, "both")])
def test_fusion_edge_configs(monkeypatch, dec_len, P, ibl, bl, sep, src):
    """Edge configurations through both fusion kernels and the oracle: tiny
    budgets (dec_len 1-3), P = 8 (the compiled maximum), deep input trees
    (input_branch_len 20/32: levels beyond the 8-level key flatten), datastore
    continuations longer than the 15 inlined row tokens (P + branch_len > 15),
    separators and single-source sessions, 130-node drafts (3 mask words)."""
    rng = np.random.default_rng(dec_len * 7 + P)
    V = 9
    corpus = rng.integers(0, V, 40000).astype(np.uint32)
    ds = G.build(corpus)
    store = O.Store(corpus, O.suffix_array(corpus))
    cfg = G.FusionConfig(P=P, dec_len=dec_len, input_branch_len=ibl,
                         **({"branch_len": bl} if bl is not None else {}))
    use_ds, use_in = src in ("both", "datastore"), src in ("both", "input")
    monkeypatch.setenv("SSSD_FUSION", "heap")
    heap = G.DraftEngine(ds, cfg, sep, use_ds, use_in)
    monkeypatch.setenv("SSSD_FUSION", "ls")
    ls = G.DraftEngine(ds, cfg, sep, use_ds, use_in)
    ctxs = [rng.integers(0, V, int(rng.integers(1, 1500))).tolist() for _ in range(24)]
    fa, fb = heap.propose_host(ctxs), ls.propose_host(ctxs)
    oc = O.Cfg(P=P, dec_len=dec_len, input_branch_len=ibl, branch_len=cfg.branch_len)
    for a, b, ctx in zip(fa, fb, ctxs):
        d = O.propose(store, ctx, oc, separator=sep, use_ds=use_ds, use_in=use_in)
        assert (b.tokens, b.parents, b.depths) == (d.tokens, d.parents, d.depths)
        assert (a.tokens, a.parents, a.depths) == (d.tokens, d.parents, d.depths)
        assert pack_mask(b.mask) == O.pack_mask_rows(d.masks, d.size)
