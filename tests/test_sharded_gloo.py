"""Multi-process (world 2, gloo, CPU) test of the sharding protocol: the real
``sharded.exchange`` (ShardedDraftEngine.propose's host side: batch-size
exchange + padding, tail all-gather, C1 sum all-reduce of bounds, C2 sum
reduce-scatter of 4-byte sample positions) over ragged per-rank batches, with
the two shard kernels' contracts emulated by the CPU oracle.  Per-shard
lower/upper counts summed equal the global find_range and the
owner-written positions equal the global sample ranks' positions."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sssd_oracle as O


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _local_counts(tokens, sa_slice, pat):
    """(#rows < pat, #rows <= pat) in one sorted shard slice (oracle compare)."""
    def first(pred):
        a, b = 0, len(sa_slice)
        while a < b:
            m = (a + b) // 2
            if pred(O._cmp(tokens, int(sa_slice[m]), pat)):
                a = m + 1
            else:
                b = m
        return a
    return first(lambda c: c < 0), first(lambda c: c <= 0)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2411_05894_b200.sharded import Collective, exchange, shard_bounds, tails_of

    coll = Collective()
    rng = np.random.default_rng(0)
    tokens = rng.integers(0, 5, 3000).astype(np.uint32)
    sa = O.suffix_array(tokens)
    a, b = shard_bounds(len(sa), world, rank)
    P, M = 3, 8
    # ragged per-rank batches (continuous batching): rank r drafts 7 + 5r requests
    B = 7 + 5 * rank
    rs = np.random.default_rng(100 + rank)
    seqs = [rs.integers(0, 5, int(rs.integers(1, 12))).astype(np.int64) for _ in range(B)]
    flat = torch.from_numpy(np.concatenate(seqs).astype(np.uint32).view(np.int32))
    lens = torch.tensor([len(x) for x in seqs], dtype=torch.int32)
    offs = torch.zeros(B, dtype=torch.int64)
    offs[1:] = torch.cumsum(lens.long(), 0)[:-1]
    tails, tlen = tails_of(flat, offs, lens, P)

    def search_fn(all_tails, all_tlen):  # the shard_search kernel's contract, on this rank's SA slice
        out = torch.zeros(all_tails.shape[0], P, 2, dtype=torch.int64)
        for i in range(all_tails.shape[0]):
            n = int(all_tlen[i])
            tail = all_tails[i, P - n:].numpy().view(np.uint32).tolist()
            for p in range(1, n + 1):
                out[i, p - 1] = torch.tensor(_local_counts(tokens, sa[a:b], tail[n - p:]))
        return out

    def gather_fn(gb):  # the shard_gather_pos kernel's contract: owned positions + 1
        out = torch.zeros(gb.shape[0], P, M, dtype=torch.int32)
        for i in range(gb.shape[0]):
            for p in range(P):
                lo, hi = gb[i, p].tolist()
                for k, r in enumerate(O.sample_ranks(lo, hi, M)):
                    if a <= r < b:
                        out[i, p, k] = int(sa[r]) + 1
        return out

    mine, pos = exchange(coll, tails, tlen, P, M, search_fn, gather_fn)
    ok_bounds, ok_pos = mine.shape[0] == B and pos.shape[0] == B, True
    for j, x in enumerate(seqs):
        for p in range(1, min(P, len(x)) + 1):
            lo, hi = O.find_range(tokens, sa, x[-p:].tolist())
            ok_bounds &= tuple(mine[j, p - 1].tolist()) == (lo, hi)
            want = [int(sa[r]) + 1 for r in O.sample_ranks(lo, hi, M)]
            ok_pos &= pos[j, p - 1, :len(want)].tolist() == want and not pos[j, p - 1, len(want):].any()
    allg = coll.all_gather(torch.full((2, P), rank, dtype=torch.int64))
    ok_gather = allg[:, 0].tolist() == [r for r in range(world) for _ in range(2)]
    q.put((rank, bool(ok_bounds), bool(ok_pos), ok_gather))
    dist.destroy_process_group()


def test_sharding_protocol_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert [p.exitcode for p in procs] == [0] * world
    res = [q.get(timeout=10) for _ in range(world)]
    assert all(ok_b and ok_r and ok_g for _, ok_b, ok_r, ok_g in res), res
