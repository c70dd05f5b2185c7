"""Tree attention (tcgen05/TMEM kernel) against a plain PyTorch fp32 reference:
dense attention with the draft's ancestor mask (ref draft.py:205-210 semantics).
Tolerance (north_star): max |gpu - ref| <= 1e-2 * max |ref| per output, bf16 I/O."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_05894_b200.verify import tree_attention  # noqa: E402


def ref_tree_attention(q, k, v, mask, ctx, scale):
    B, S, Hq, D = q.shape
    Hkv = k.shape[1]
    G = Hq // Hkv
    out = torch.zeros(B, S, Hq, D, dtype=torch.float32, device=q.device)
    qf, kf, vf = q.float(), k.float(), v.float()
    m = mask.cpu().numpy().view(np.uint64)
    for b in range(B):
        c = int(ctx[b])
        vis = torch.zeros(S, c + S, dtype=torch.bool)
        vis[:, :c] = True
        for i in range(S):
            for j in range(S):
                if (int(m[b, i, j // 64]) >> (j % 64)) & 1:
                    vis[i, c + j] = True
        vis = vis.to(q.device)
        for h in range(Hq):
            kk = kf[b, h // G, : c + S]
            vv = vf[b, h // G, : c + S]
            s = (qf[b, :, h] @ kk.T) * scale
            s = s.masked_fill(~vis, float("-inf"))
            out[b, :, h] = torch.softmax(s, dim=-1) @ vv
    return out


def random_tree_masks(B, S, rng):
    W = (S + 63) // 64
    masks = np.zeros((B, S, W), dtype=np.uint64)
    for b in range(B):
        parents = [-1] + [int(rng.integers(0, i)) for i in range(1, S)]
        rows = []
        for i in range(S):
            r = 1 << i
            if parents[i] >= 0:
                r |= rows[parents[i]]
            rows.append(r)
            for w in range(W):
                masks[b, i, w] = np.uint64((r >> (64 * w)) & 0xFFFFFFFFFFFFFFFF)
    return torch.from_numpy(masks.view(np.int64)).cuda()


@pytest.mark.parametrize("B,S,Hq,Hkv,ctx_max,max_pos", [
    (2, 32, 32, 8, 300, 512),      # cfg3 shape family, GQA 4 -> 128 rows
    (3, 16, 32, 8, 1000, 1200),    # cfg4 family (64 rows, padded tile)
    (1, 8, 8, 2, 5, 64),           # tiny decoder shape, short prefix
    (2, 64, 8, 2, 200, 400),       # two row tiles (G*S = 256), S = 64 masks
    (2, 24, 16, 8, 4000, 4200),    # split-KV path
])
def test_tree_attention_matches_fp32_reference(B, S, Hq, Hkv, ctx_max, max_pos):
    torch.manual_seed(0)
    rng = np.random.default_rng(1)
    D = 128
    q = torch.randn(B, S, Hq, D, device="cuda").to(torch.bfloat16)
    k = torch.randn(B, Hkv, max_pos, D, device="cuda").to(torch.bfloat16)
    v = torch.randn(B, Hkv, max_pos, D, device="cuda").to(torch.bfloat16)
    ctx = torch.tensor([int(rng.integers(max(1, ctx_max // 2), ctx_max + 1)) for _ in range(B)],
                       dtype=torch.int32, device="cuda")
    mask = random_tree_masks(B, S, rng)
    scale = 1.0 / math.sqrt(D)
    got = tree_attention(q, k, v, mask, ctx, scale).float()
    torch.cuda.synchronize()
    want = ref_tree_attention(q, k, v, mask, ctx, scale)
    err = (got - want).abs().max().item()
    assert err <= 1e-2 * want.abs().max().item(), err


@pytest.mark.parametrize("B,S,Hq,Hkv,ctx_max,max_pos", [
    (2, 32, 32, 8, 1500, 1600),   # odd/even block split between the two softmax warpgroups
    (1, 16, 8, 2, 200, 256),      # 2 blocks: one per warpgroup
])
def test_tree_attention_growing_max(B, S, Hq, Hkv, ctx_max, max_pos):
    """Scores that rise along the keys force the running max up block after block
    (the lazy-rescale path: rescale only when the max grows by > 2^8)."""
    torch.manual_seed(3)
    rng = np.random.default_rng(4)
    D = 128
    q = (torch.randn(B, S, Hq, D, device="cuda") * 2).to(torch.bfloat16)
    ramp = torch.linspace(0.2, 3.0, max_pos, device="cuda")[None, None, :, None]
    k = (torch.randn(B, Hkv, max_pos, D, device="cuda") * ramp).to(torch.bfloat16)
    v = torch.randn(B, Hkv, max_pos, D, device="cuda").to(torch.bfloat16)
    ctx = torch.tensor([int(rng.integers(ctx_max // 2, ctx_max + 1)) for _ in range(B)],
                       dtype=torch.int32, device="cuda")
    mask = random_tree_masks(B, S, rng)
    scale = 1.0 / math.sqrt(D)
    got = tree_attention(q, k, v, mask, ctx, scale).float()
    torch.cuda.synchronize()
    want = ref_tree_attention(q, k, v, mask, ctx, scale)
    err = (got - want).abs().max().item()
    assert err <= 1e-2 * want.abs().max().item(), err


@pytest.mark.parametrize("ctxs,S,Hq,Hkv,max_pos", [
    ([20000, 10, 300], 16, 8, 2, 20100),   # skewed contexts: split-KV with near-empty splits
    ([3000] * 40, 32, 32, 8, 3100),        # 320 (b, kv head) units
    ([1, 700, 64, 129], 5, 8, 1, 900),     # G*S = 40 rows (padding warps), block-boundary contexts
    ([900, 50], 64, 8, 2, 1000),           # two row tiles per (b, kv head)
])
def test_tree_attention_ragged_batches(ctxs, S, Hq, Hkv, max_pos):
    """Ragged context lengths and row-tile shapes against the fp32 reference;
    two launches in a row give identical outputs (no state kept between calls)."""
    torch.manual_seed(5)
    rng = np.random.default_rng(6)
    B, D = len(ctxs), 128
    q = torch.randn(B, S, Hq, D, device="cuda").to(torch.bfloat16)
    k = torch.randn(B, Hkv, max_pos, D, device="cuda").to(torch.bfloat16)
    v = torch.randn(B, Hkv, max_pos, D, device="cuda").to(torch.bfloat16)
    ctx = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    mask = random_tree_masks(B, S, rng)
    scale = 1.0 / math.sqrt(D)
    got1 = tree_attention(q, k, v, mask, ctx, scale).float()
    got2 = tree_attention(q, k, v, mask, ctx, scale).float()
    torch.cuda.synchronize()
    assert torch.equal(got1, got2)
    want = ref_tree_attention(q, k, v, mask, ctx, scale)
    assert (got1 - want).abs().max().item() <= 1e-2 * want.abs().max().item()
