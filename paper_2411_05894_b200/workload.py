"""Seeded synthetic token streams (SURVEY.md Appendix B "phrase model").

A dictionary of D phrases (lengths U[4, 32], tokens zipf(1.1) mod V) is
sampled with Zipf-distributed phrase ids and 5 % uniform token noise.  The
corpus uses stream seed 0; request contexts / teacher-forced references use
stream seed 1 of the *same* dictionary, so contexts are held-out text that
shares phrases with the corpus (not corpus spans).  Fully vectorised so 100M
tokens take seconds.  Host-side data generation only — not part of the
measured path.
"""

from __future__ import annotations

import numpy as np

DICT_SEED = 1234
CORPUS_SEED = 0
HELDOUT_SEED = 1


def phrase_dictionary(vocab: int, n_phrases: int = 20000, seed: int = DICT_SEED):
    rng = np.random.default_rng(seed)
    lens = rng.integers(4, 33, n_phrases)
    toks = (rng.zipf(1.1, int(lens.sum())) % vocab).astype(np.uint32)
    offs = np.zeros(n_phrases + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    return toks, offs


# phrases drawn per generator block: a fixed block size (and the block's noise
# drawn right after it) makes every stream PREFIX-STABLE -- phrase_stream(n)
# is the first n tokens of phrase_stream(m) for any m >= n -- so a B=64 batch
# is exactly the first 64 contexts of a 16,384-context step (bench.py's two
# arms draft identical inputs)
BLOCK_PHRASES = 1 << 16


def phrase_stream(n: int, vocab: int, seed: int, n_phrases: int = 20000,
                  noise: float = 0.05, dict_seed: int = DICT_SEED) -> np.ndarray:
    """``n`` tokens (u32) of phrase-model text; prefix-stable in ``n``."""
    toks, offs = phrase_dictionary(vocab, n_phrases, dict_seed)
    lens = offs[1:] - offs[:-1]
    rng = np.random.default_rng(seed)
    out = np.empty(n, dtype=np.uint32)
    filled = 0
    while filled < n:
        ids = (rng.zipf(1.1, BLOCK_PHRASES) - 1) % n_phrases
        ln = lens[ids]
        total = int(ln.sum())
        # position j of the block's concatenation -> offs[phrase] + (j - phrase_begin)
        begin = np.zeros(len(ids), dtype=np.int64)
        np.cumsum(ln[:-1], out=begin[1:])
        seg = toks[np.repeat(offs[ids] - begin, ln) + np.arange(total, dtype=np.int64)]
        mask = rng.random(total) < noise
        seg[mask] = rng.integers(0, vocab, int(mask.sum())).astype(np.uint32)
        take = min(total, n - filled)
        out[filled:filled + take] = seg[:take]
        filled += take
    return out


def corpus(n: int, vocab: int = 32000) -> np.ndarray:
    return phrase_stream(n, vocab, CORPUS_SEED)


def contexts(batch: int, length: int, vocab: int = 32000, seed: int = HELDOUT_SEED) -> list[np.ndarray]:
    """``batch`` held-out request contexts of ``length`` tokens."""
    s = phrase_stream(batch * length, vocab, seed)
    return [s[i * length:(i + 1) * length].copy() for i in range(batch)]


def prompt_heavy_contexts(batch: int, length: int, vocab: int = 32000, spans: int = 40,
                          seed: int = HELDOUT_SEED) -> list[np.ndarray]:
    """Long-context RAG shape (cfg4): copy ``spans`` spans of 8-64 tokens from
    the first half of each context into its second half."""
    base = contexts(batch, length, vocab, seed)
    rng = np.random.default_rng(seed + 100)
    half = length // 2
    for c in base:
        for _ in range(spans):
            k = int(rng.integers(8, 65))
            src = int(rng.integers(0, half - k))
            dst = int(rng.integers(half, length - k))
            c[dst:dst + k] = c[src:src + k]
    return base


def records(count: int, prompt_len: int, ref_len: int, vocab: int = 32000,
            seed: int = HELDOUT_SEED) -> list[tuple[np.ndarray, np.ndarray]]:
    """Teacher-forced (prompt, reference) pairs cut from one held-out stream."""
    per = prompt_len + ref_len
    s = phrase_stream(count * per, vocab, seed)
    return [(s[i * per:i * per + prompt_len].copy(), s[i * per + prompt_len:(i + 1) * per].copy())
            for i in range(count)]
