"""GPU: the incremental per-request input index (N2, engine.InputIndex; the
stateful analogue of InputCache._push, ref input_cache.py:46-63) gives drafts
identical to the stateless scan -- right after a build, after tokens were
appended past the indexed prefix (the decode loop's case), for long prompt-
heavy contexts, and when a token does not fit the key (fallback) -- and the
index-driven decode loop reproduces the reference-pinned simulate goldens."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2411_05894_b200 as G  # noqa: E402
from paper_2411_05894_b200 import workload  # noqa: E402


def _same(a, b, B):
    for k in ("size", "tokens", "parents", "depths", "mask"):
        x, y = getattr(a, k), getattr(b, k)
        if k == "size":
            assert torch.equal(x, y)
        else:
            for i in range(B):
                n = int(a.size[i])
                assert torch.equal(x[i, :n], y[i, :n]), (k, i)


@pytest.mark.parametrize("vocab,L,B,dec_len", [(50, 300, 64, 32), (500, 2048, 32, 64), (32000, 32768, 4, 16)])
def test_index_equals_scan_after_appends(vocab, L, B, dec_len):
    corpus = workload.corpus(300_000, vocab)
    ds = G.build(corpus, vocab_size=vocab)
    eng = G.DraftEngine(ds, G.FusionConfig(dec_len=dec_len))
    ctxs = (workload.prompt_heavy_contexts(B, L, vocab) if L >= 4096 else workload.contexts(B, L, vocab))
    rng = np.random.default_rng(3)
    cap = L + 64
    seq = torch.zeros(B * cap, dtype=torch.int32, device="cuda")
    off = torch.arange(B, dtype=torch.int64, device="cuda") * cap
    for b, c in enumerate(ctxs):
        seq[b * cap: b * cap + L] = torch.from_numpy(c.astype(np.uint32).view(np.int32)).cuda()
    # index built on ragged prefixes, then sequences extended by 0..40 tokens (appends)
    built = torch.tensor(rng.integers(2, L + 1, B), dtype=torch.int32, device="cuda")
    ix = G.InputIndex(B, cap, "cuda", off)
    ix.build(seq, off, built)
    assert int(ix.len.min()) >= 1 and torch.equal(ix.len, built - 1)
    now = torch.clamp(built + torch.tensor(rng.integers(0, 41, B), dtype=torch.int32, device="cuda"), max=L)
    want = eng.propose(seq, off, now, cap)
    want = {k: getattr(want, k).clone() for k in ("size", "tokens", "parents", "depths", "mask")}
    got = eng.propose(seq, off, now, cap, index=ix)
    eng.check_status()
    for k, v in want.items():
        g = getattr(got, k)
        for b in range(B):
            n = int(want["size"][b])
            assert torch.equal(g[b, :n] if k != "size" else g[b], v[b, :n] if k != "size" else v[b]), (k, b)


def test_index_fallback_when_tokens_do_not_fit():
    # tokens >= 2^(32 - pos_bits): the build leaves len 0 and propose scans in full
    corpus = workload.corpus(50_000, 1000)
    ds = G.build(corpus, vocab_size=1 << 24)
    eng = G.DraftEngine(ds, G.FusionConfig(dec_len=16))
    ctxs = [c.tolist() for c in workload.contexts(8, 700, 1000)]
    ctxs[2][100] = (1 << 23) + 5  # inside the indexed prefix: no index for request 2
    ctxs[3][-1] = (1 << 23) + 5   # the last token (not indexed) too wide for a key: full scan
    seq, off, ln, mx = eng.upload(ctxs)
    ix = G.InputIndex(8, 1 << 10, "cuda", off)  # 10 position bits -> tokens must be < 2^22
    ix.build(seq, off, ln)
    assert int(ix.len[2]) == 0 and int(ix.len[0]) == 699 and int(ix.len[3]) == 699
    a = eng.propose(seq, off, ln, mx)
    a = {k: getattr(a, k).clone() for k in ("size", "tokens", "parents", "depths", "mask")}
    b = eng.propose(seq, off, ln, mx, index=ix)
    for k in a:
        for r in range(8):
            n = int(a["size"][r])
            assert torch.equal(getattr(b, k)[r] if k == "size" else getattr(b, k)[r, :n],
                               a[k][r] if k == "size" else a[k][r, :n])


def test_simulate_with_and_without_index(golden):
    for case in golden("simulate.json")[:40]:
        ds = G.build(case["corpus"])
        cfg = G.FusionConfig.from_kv({k: str(v) for k, v in case["cfg"].items()})
        rec = [G.SimRecord(case["prompt"], case["reference"])]
        a = G.simulate(rec, ds, cfg, use_index=True).records[0].per_step_tokens
        b = G.simulate(rec, ds, cfg, use_index=False).records[0].per_step_tokens
        assert a == b == case["per_step"]


# ---------------------------------------------------------------------------
# k-gram range index (sssd_kix_build, the find_range accelerator)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("vocab", [7, 500, 32000])
def test_kgram_index_ranges_and_drafts(monkeypatch, vocab):
    """Patterns of 1..6 tokens (present and absent) get the oracle's exact
    (lo, hi) through the k-gram table, and drafts with the table equal drafts
    without it (SSSD_NO_KIX=1) -- including the lookup kernels' 'absent
    k-gram = empty range' shortcut."""
    from oracle import sssd_oracle as O

    corpus = workload.corpus(200_000, vocab)
    ds = G.build(corpus, vocab_size=vocab)
    assert ds.kix() is not None
    monkeypatch.setenv("SSSD_NO_KIX", "1")
    ds0 = G.Datastore.on_device(ds.token_tensor, ds.rows, ds.n_rows, vocab)
    monkeypatch.delenv("SSSD_NO_KIX")
    assert ds0.kix() is None
    sa = ds.suffix_index
    tok = np.asarray(corpus)
    rng = np.random.default_rng(5)
    pats = []
    for _ in range(300):
        k = int(rng.integers(1, 7))
        s = int(rng.integers(0, len(corpus) - k))
        p = [int(x) for x in corpus[s:s + k]]
        if rng.random() < 0.3:  # perturb: mostly absent k-grams
            p[-1] = int(rng.integers(0, vocab))
        pats.append(p)
    pats.append([int(x) for x in corpus[-2:]])  # suffixes at the corpus end
    pats.append([int(x) for x in corpus[-4:]])
    got = ds.find_ranges(pats)
    for p, g in zip(pats, got):
        assert tuple(g) == O.find_range(tok, sa, p), p
    for B, L in ((64, 2048), (2048, 512)):
        ctxs = workload.contexts(B, L, vocab)
        cfg = G.FusionConfig(dec_len=32)
        a = G.DraftEngine(ds, cfg).propose_host(ctxs)
        b = G.DraftEngine(ds0, cfg).propose_host(ctxs)
        for x, y in zip(a, b):
            assert (x.tokens, x.parents, x.depths) == (y.tokens, y.parents, y.depths)
