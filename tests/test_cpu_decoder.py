"""CPU: the decode leg's host baseline (oracle/cpu_decoder.py, test/bench
infrastructure) reproduces plain greedy autoregressive decoding of the same
fp32 model -- speculative decoding is lossless (ref draft.py:202-216,
test_acceptance.py criterion 1) -- so its tokens/s is a valid CPU reference
for the GPU decode loop."""

from paper_2411_05894_b200 import model as Mo
from paper_2411_05894_b200 import workload

from oracle import cpu_decoder as CD
from oracle import sssd_oracle as O


def test_cpu_speculative_decode_equals_greedy_fp32():
    dec = Mo.Decoder(Mo.ModelSpec(2, 256, 4, 2, 512, 500), batch=2, max_pos=128, device="cpu", seed=0)
    corpus = workload.corpus(20000, 500)
    store = O.Store(corpus, O.suffix_array(corpus))
    prompts = [c.tolist() for c in workload.contexts(3, 40, 500)]
    r = CD.decode(store, prompts, O.Cfg(dec_len=8), dec, 10, threads=2)
    assert r["finished"] and r["tokens"] == 30
    for b, p in enumerate(prompts):
        seq = list(p)
        for _ in range(10):
            seq.append(int(dec.reference_logits(seq).argmax()))
        assert r["sequences"][b] == seq
