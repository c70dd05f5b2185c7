"""GPU: the continuously batched model decode loop (serving.ServeLoop).

Slots are refilled from a request queue (prefill of the freed slot's KV rows
only); every request's output must equal greedy autoregressive decoding of
the same model (speculative decoding is lossless, ref test_acceptance.py
criterion 1) -- through the same loop with drafting off, and against an
independent static-batch run for the first requests -- whatever the slot
count (batch composition), up to argmax near-ties of the fp32 reference."""

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2411_05894_b200 as G  # noqa: E402
from paper_2411_05894_b200 import model as M  # noqa: E402
from paper_2411_05894_b200 import workload  # noqa: E402
from paper_2411_05894_b200.serving import ServeLoop, SpecDecoder  # noqa: E402

SMALL = M.ModelSpec(n_layers=2, hidden=512, n_q=8, n_kv=2, mlp=1024, vocab=2000)


def _near_tie_ok(dec, a, b):
    if a == b:
        return True
    j = next(k for k in range(min(len(a), len(b))) if a[k] != b[k])
    top2 = torch.topk(dec.reference_logits(b[:j]), 2).values
    return (top2[0] - top2[1]).item() <= 1e-2 * abs(top2[0].item())


@pytest.mark.parametrize("slots,group", [(4, 3), (7, 1)])
def test_serve_loop_refills_and_is_lossless(slots, group):
    corpus = workload.corpus(300_000, SMALL.vocab)
    ds = G.build(corpus, vocab_size=SMALL.vocab)
    prompts = [c.tolist() for c in workload.contexts(11, 60, SMALL.vocab, seed=7)]
    prompts[3] = prompts[3][:20]  # ragged prompt lengths
    max_new = 24
    spec = ServeLoop(G.DraftEngine(ds, G.FusionConfig(dec_len=12)), M.Decoder(SMALL, slots, 160, seed=2),
                     60, max_new, group=group, use_index=(slots == 4))
    r = spec.run(prompts, max_new)
    ar = ServeLoop(None, M.Decoder(SMALL, slots, 160, seed=2), 60, max_new, group=group).run(prompts, max_new)
    assert r["tokens"] == ar["tokens"] == 11 * max_new
    assert r["requests"] == 11 and all(len(s) == len(p) + max_new for s, p in zip(r["sequences"], prompts))
    ref = M.Decoder(SMALL, 1, 160, seed=2)
    for sa, sb in zip(r["sequences"], ar["sequences"]):
        assert _near_tie_ok(ref, sa, sb)
    # an independent static batch (no refills) of the first `slots` requests
    st = SpecDecoder(None, M.Decoder(SMALL, slots, 160, seed=2), prompts[:slots], max_new)
    st.run()
    for sa, sb in zip(st.sequences(), ar["sequences"][:slots]):
        assert _near_tie_ok(ref, sb, sa)
