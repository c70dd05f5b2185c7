"""SA-range sharding on one GPU (W in-process ranks): the collective protocol of
paper_2411_05894_b200.sharded must give drafts bit-identical to the unsharded
propose (A.2 sum identity + rank-ordered shards)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2411_05894_b200 as G  # noqa: E402
from paper_2411_05894_b200 import workload  # noqa: E402
from paper_2411_05894_b200.draft import _drafts_from_device  # noqa: E402
from paper_2411_05894_b200.sharded import LocalShards  # noqa: E402


@pytest.mark.parametrize("world,sep", [(2, None), (3, None), (8, None), (4, 7)])
def test_sharded_propose_bit_identical(world, sep):
    corpus = workload.corpus(300_000, 500)
    if sep is not None:
        corpus = corpus.copy()
        corpus[::97] = sep
    ds = G.build(corpus)
    cfg = G.FusionConfig(dec_len=32, M=50, T=20)
    per = 6
    ctxs = [c.tolist() for c in workload.contexts(world * per, 300, 500)]
    full = G.DraftEngine(ds, cfg, sep).propose_host(ctxs)
    ls = LocalShards(ds, world, cfg, sep)
    per_rank = [ls.engines[r].upload(ctxs[r * per:(r + 1) * per]) for r in range(world)]
    outs = ls.propose(per_rank)
    got = []
    for o in outs:
        got += _drafts_from_device(o.size, o.tokens, o.parents, o.depths, o.mask, per, cfg.dec_len)
    for a, b in zip(got, full):
        assert (a.tokens, a.parents, a.depths) == (b.tokens, b.parents, b.depths)
        assert np.array_equal(a.mask, b.mask)
