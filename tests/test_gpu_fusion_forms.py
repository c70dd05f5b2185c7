"""The all-nodes fusion kernel (csrc/fusion_ane.cu, sssd_set_fusion_form(1))
and the CTA-per-request kernel (csrc/fusion_cta.cu, form 2, the default for
small launches) against the one-warp level-synchronous kernel (form 0):
identical drafts -- tokens, parents,
depths, masks, per-node priority / source / position -- over the cfg2 shape,
a prompt-heavy 32k context (its requests outgrow the shared-memory tables and
take the fallback), tie-heavy tiny alphabets, and the reference's golden
merges.  Two independent algorithms (enumerate-and-select vs level-by-level
expansion) agreeing bit for bit at scale is a cross-check of both."""

import numpy as np
import pytest

from tests.test_gpu_parity import flat_dict

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2411_05894_b200 as G  # noqa: E402
from paper_2411_05894_b200 import workload  # noqa: E402
from paper_2411_05894_b200._lib import lib  # noqa: E402


@pytest.fixture
def form():
    def set_form(f):
        lib().sssd_set_fusion_form(f)

    yield set_form
    lib().sssd_set_fusion_form(-1)


def _batch(eng, seq, off, ln, L):
    o = eng.propose(seq, off, ln, L, nodes=True)
    eng.check_status()
    torch.cuda.synchronize()
    return {k: v.clone() for k, v in o.__dict__.items() if isinstance(v, torch.Tensor)}


def _equal(a, b):
    assert a.keys() == b.keys()
    for k in a:
        x, y = a[k], b[k]
        if x.dtype.is_floating_point:
            assert bool(((x == y) | (torch.isnan(x) & torch.isnan(y))).all()), k
        else:
            assert torch.equal(x, y), k


@pytest.mark.parametrize("other", [1, 2])
@pytest.mark.parametrize("dec_len,ctx,n_req,alpha", [(64, 2048, 2048, 0.8), (16, 32768, 8, 0.8),
                                                     (100, 1024, 512, 0.0), (256, 512, 256, 1.0),
                                                     (64, 2048, 64, 0.8), (16, 32768, 64, 0.5)])
def test_fusion_forms_equal_level_synchronous(form, other, dec_len, ctx, n_req, alpha):
    ds = G.build(workload.corpus(1_000_000, 32000), vocab_size=32000)
    eng = G.DraftEngine(ds, G.FusionConfig(dec_len=dec_len, alpha=alpha))
    ctxs = workload.prompt_heavy_contexts(n_req, ctx, 32000) if ctx > 4096 else workload.contexts(n_req, ctx, 32000)
    flat = np.concatenate([np.asarray(c, dtype=np.uint32) for c in ctxs])
    seq = torch.from_numpy(flat.view(np.int32)).cuda()
    off = torch.arange(n_req, dtype=torch.int64, device="cuda") * ctx
    ln = torch.full((n_req,), ctx, dtype=torch.int32, device="cuda")
    form(0)
    a = _batch(eng, seq, off, ln, ctx)
    form(other)
    b = _batch(eng, seq, off, ln, ctx)
    _equal(a, b)


@pytest.mark.parametrize("other", [1, 2])
def test_fusion_forms_small_alphabets(form, other):
    rng = np.random.default_rng(9)
    for trial in range(4):
        V = int(rng.choice([2, 3, 5]))
        ds = G.build(rng.integers(0, V, 20000).astype(np.uint32))
        cfg = G.FusionConfig(P=int(rng.integers(1, 6)), dec_len=int(rng.choice([5, 33, 64, 200])),
                             alpha=float(rng.choice([0.0, 0.5, 1.0])), beta=float(rng.choice([0.5, 1.0])),
                             gamma_ds=float(rng.choice([0.5, 1.0])), gamma_in=float(rng.choice([0.5, 1.0])))
        eng = G.DraftEngine(ds, cfg)
        ctxs = [rng.integers(0, V, int(rng.integers(1, 4000))).tolist() for _ in range(64)]
        form(0)
        fa = eng.propose_host(ctxs)
        form(other)
        fb = eng.propose_host(ctxs)
        for x, y in zip(fa, fb):
            assert (x.tokens, x.parents, x.depths) == (y.tokens, y.parents, y.depths), trial


@pytest.mark.parametrize("other", [1, 2])
def test_fusion_forms_golden_merges(form, golden, other):
    form(other)
    by_cfg: dict = {}
    for case in golden("merge.json"):
        by_cfg.setdefault(tuple(sorted(case["cfg"].items())), []).append(case)
    for key, group in by_cfg.items():
        cfg = G.FusionConfig(**dict(key))
        reqs = [(G.tree_from_paths(cs["ds"]), [G.tree_from_paths(p) for p in cs["inputs"]], cs["root"])
                for cs in group]
        for n_in in sorted({len(r[1]) for r in reqs}):
            sub = [(r, cs) for r, cs in zip(reqs, group) if len(r[1]) == n_in]
            flats = G.merge_batch([r for r, _ in sub], cfg)
            for f, (_, cs) in zip(flats, sub):
                assert flat_dict(f) == cs["flat"]
