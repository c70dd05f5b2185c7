"""Multi-process (world 2, gloo, CPU) test of the sharding protocol's host logic:
per-shard lower/upper counts summed with an all-reduce equal the global
find_range, and the sum-assembled sampled rows equal the rows of
the global sample ranks.  Shard compute is emulated with the CPU oracle; the
collectives are the real torch.distributed gloo ops used by sharded.Collective."""

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
    from paper_2411_05894_b200.sharded import Collective, shard_bounds

    coll = Collective()
    rng = np.random.default_rng(0)
    tokens = rng.integers(0, 5, 3000).astype(np.uint32)
    sa = O.suffix_array(tokens)
    a, b = shard_bounds(len(sa), world, rank)
    P, M = 3, 8
    pats = [rng.integers(0, 5, int(rng.integers(1, P + 1))).tolist() for _ in range(40)]
    local = torch.zeros(len(pats), 2, dtype=torch.int64)
    for i, pat in enumerate(pats):
        local[i] = torch.tensor(_local_counts(tokens, sa[a:b], pat))
    gb = coll.all_reduce_sum(local)
    ok_bounds = all(tuple(gb[i].tolist()) == O.find_range(tokens, sa, pat) for i, pat in enumerate(pats))
    # owner-written rows (pos + 15 tokens), zeros elsewhere, assembled by a sum
    rows = torch.zeros(len(pats), M, 16, dtype=torch.int64)
    for i in range(len(pats)):
        lo, hi = gb[i].tolist()
        for k, r in enumerate(O.sample_ranks(lo, hi, M)):
            if a <= r < b:
                pos = int(sa[r])
                seg = tokens[pos:pos + 15].astype(np.int64)
                rows[i, k, 0] = pos
                rows[i, k, 1:1 + len(seg)] = torch.from_numpy(seg)
    per = len(pats) // world
    mine = coll.reduce_scatter_sum(rows.clone())
    ok_rows = True
    for j in range(per):
        i = rank * per + j
        lo, hi = O.find_range(tokens, sa, pats[i])
        for k, r in enumerate(O.sample_ranks(lo, hi, M)):
            pos = int(sa[r])
            seg = tokens[pos:pos + 15]
            ok_rows &= int(mine[j, k, 0]) == pos and mine[j, k, 1:1 + len(seg)].tolist() == seg.tolist()
    allg = coll.all_gather(torch.full((2, P), rank, dtype=torch.int64))
    ok_gather = allg[:, 0].tolist() == [r for r in range(world) for _ in range(2)]
    q.put((rank, ok_bounds, ok_rows, ok_gather))
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
