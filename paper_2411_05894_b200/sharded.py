"""SA-range sharded drafting across GPUs.

The suffix rows are split into W contiguous global-rank ranges, one per GPU;
decode requests are partitioned (each rank drafts its own B_local).  Per step:

1. all-gather the last P tokens of every request              (u32 [W*B, P])
2. ``sssd_shard_search`` on every request against the local shard -> local
   bounds; SUM all-reduce -> the global ``[lo, hi)`` exactly (A.2: a shard's
   lower/upper bound counts sum to the global ones)            (i64 [W*B, P, 2])
3. ``sssd_shard_gather_pos``: each sampled global rank's corpus position
   (+1) is written by the one shard that owns it, zeros elsewhere; SUM
   reduce-scatter hands each rank the positions of its own requests
                                                               (i32 [B, P, M]: 4 B per sample)
4. ``sssd_rows_from_pos`` rebuilds the 64 B suffix rows from the replicated
   tokens, then ``sssd_propose_pre``: the unchanged lookup-finish / input-scan
   / fusion kernels run locally on them.

Drafts are bit-identical to a single-GPU run because shards are rank-ordered
(A.2/A.3).  Collectives go through ``Collective`` so the same protocol runs on
NCCL (GPUs), gloo (CPU tests) or in-process emulation (one-GPU tests).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr, stream_ptr
from .datastore import Datastore
from .engine import DraftBatch, DraftEngine
from .fusion import FusionConfig


def shard_bounds(n_rows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous global-rank range [a, b) of shard `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n_rows, world)
    a = rank * base + min(rank, extra)
    return a, a + base + (1 if rank < extra else 0)


def shard_view(full: Datastore, world: int, rank: int) -> Datastore:
    """A shard as a Datastore view over rows [a, b) of a full index (global
    n_tokens kept).  On a real multi-GPU run each rank keeps only its slice."""
    a, b = shard_bounds(full.n_rows, world, rank)
    return Datastore.on_device(full.token_tensor, full.rows[a:b], b - a, full.vocab_size, rank_base=a,
                     n_tokens=full.n_tokens)


class Collective:
    """torch.distributed collectives (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None) -> None:
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

        self.gloo = dist.get_backend(group) == "gloo"

    def all_gather(self, x: torch.Tensor) -> torch.Tensor:
        if self.gloo and x.is_cuda:  # (gloo collectives run on host copies)
            return self.all_gather(x.cpu()).to(x.device)
        out = torch.empty((self.world * x.shape[0],) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        self.dist.all_gather_into_tensor(out, x.contiguous(), group=self.group)
        return out

    def all_reduce_sum(self, x: torch.Tensor) -> torch.Tensor:
        if self.gloo and x.is_cuda:
            x.copy_(self.all_reduce_sum(x.cpu()))
            return x
        self.dist.all_reduce(x, op=self.dist.ReduceOp.SUM, group=self.group)
        return x

    def reduce_scatter_sum(self, x: torch.Tensor) -> torch.Tensor:
        n = x.shape[0] // self.world
        if self.gloo:  # gloo has no reduce_scatter
            self.all_reduce_sum(x)
            return x[self.rank * n:(self.rank + 1) * n].clone()
        out = torch.empty((n,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        self.dist.reduce_scatter_tensor(out, x.contiguous(), op=self.dist.ReduceOp.SUM, group=self.group)
        return out


def tails_of(seq: torch.Tensor, off: torch.Tensor, ln: torch.Tensor, P: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Last min(P, L) tokens of each sequence, right-aligned in [B, P] (+ lengths)."""
    B = ln.shape[0]
    idx = (off + ln.long())[:, None] - P + torch.arange(P, device=seq.device)[None, :]
    valid = idx >= off[:, None]
    t = torch.where(valid, seq[idx.clamp(min=0)], torch.zeros((), dtype=seq.dtype, device=seq.device))
    return t.contiguous(), torch.clamp(ln, max=P).to(torch.int32)


def search(shard: Datastore, cfg_c, tails: torch.Tensor, tlen: torch.Tensor) -> torch.Tensor:
    """Local bounds of every tail against one shard: int64 [B, P, 2]."""
    B, P = tails.shape
    dev = tails.device
    off = (torch.arange(B, dtype=torch.int64, device=dev) * P) + (P - tlen.long())
    seqs = _lib.Seqs(ptr(tails), ptr(off), ptr(tlen), B, P)
    out = torch.empty(B, P, 2, dtype=torch.int64, device=dev)
    check(lib().sssd_shard_search(shard.c_view(), seqs, cfg_c, ptr(out), stream_ptr(dev)))
    return out


def gather(shard: Datastore, cfg_c, gbounds: torch.Tensor, M: int) -> torch.Tensor:
    """Owned sample positions: int32 [B, P, M] = corpus position + 1 of every
    sampled global rank this shard owns, 0 elsewhere (4 B per sample: the sum
    over shards is the exchange)."""
    B, P, _ = gbounds.shape
    out = torch.empty(B, P, M, dtype=torch.int32, device=gbounds.device)
    check(lib().sssd_shard_gather_pos(shard.c_view(), cfg_c, B, ptr(gbounds), ptr(out), stream_ptr(gbounds.device)))
    return out


def rows_of(shard: Datastore, pos: torch.Tensor) -> torch.Tensor:
    """Suffix rows [B, P, M, 16] of exchanged positions, read from the
    replicated tokens on this rank (zero rows where pos = 0)."""
    rows = torch.empty(tuple(pos.shape) + (16,), dtype=torch.int32, device=pos.device)
    check(lib().sssd_rows_from_pos(ptr(shard.token_tensor), shard.n_tokens, ptr(pos), pos.numel(), ptr(rows),
                                   stream_ptr(pos.device)))
    return rows


class ShardedDraftEngine(DraftEngine):
    """DraftEngine over one SA-range shard; ``propose`` runs the collective protocol."""

    def __init__(self, shard: Datastore, cfg: FusionConfig, coll: Collective, separator=None,
                 use_input: bool = True, device=None) -> None:
        super().__init__(shard, cfg, separator, True, use_input, device)
        if cfg.P + cfg.branch_len > _lib.SSSD_ROW_TOKENS:
            raise ValueError(f"sharded lookup needs P + branch_len <= {_lib.SSSD_ROW_TOKENS}")
        self.coll = coll

    def propose(self, seq, seq_off, seq_len, max_len, lookup: bool = False, out: DraftBatch | None = None,
                nodes: bool = False):
        """Collective propose: every rank calls it with its own batch (sizes may
        differ under continuous batching, see ``exchange``)."""
        B = int(seq_len.shape[0])
        out = out or self.outputs(B, lookup, nodes)
        tails, tlen = tails_of(seq, seq_off, seq_len, self.cfg.P)
        mine, pos = exchange(self.coll, tails, tlen, self.cfg.P, self.cfg.M,
                             lambda t, n: search(self.store, self.c, t, n),
                             lambda gb: gather(self.store, self.c, gb, self.cfg.M))
        if B == 0:
            return out
        rows = rows_of(self.store, pos)
        ws = self.workspace(B, max_len)
        seqs = _lib.Seqs(ptr(seq), ptr(seq_off), ptr(seq_len), B, int(max_len))
        lk = _lib.LookupOut(ptr(out.ranges), ptr(out.samples), ptr(out.n_conts), ptr(out.p_cut)) if lookup else None
        check(lib().sssd_propose_pre(self.store.c_view(), seqs, self.c, ptr(mine), ptr(rows), out.c_out(), lk,
                                     ptr(ws), ws.numel(), stream_ptr(self.device)))
        return out


    def propose_pinned(self, seq_h, off_h, len_h, max_len, out_h: DraftBatch | None = None, chunks: int = 1,
                       slot: int = 0, sync: bool = True, **_):
        """Host-buffer propose (pinned contexts in, pinned drafts out) through the
        collective protocol: upload, ``propose``, download, on the current stream
        (``chunks`` is accepted for API compatibility; the exchange needs every
        rank's whole batch)."""
        from .engine import PendingDrafts

        B = int(len_h.shape[0])
        dev = self.device
        if out_h is None:
            S, W = self.S, self.W
            out_h = DraftBatch(size=torch.empty(B, dtype=torch.int32).pin_memory(),
                               tokens=torch.empty((B, S), dtype=torch.int32).pin_memory(),
                               parents=torch.empty((B, S), dtype=torch.int32).pin_memory(),
                               depths=torch.empty((B, S), dtype=torch.int32).pin_memory(),
                               mask=torch.empty((B, S, W), dtype=torch.int64).pin_memory())
        st = self.__dict__.setdefault("_pin_slots", {})
        ss = st.get(slot)
        if ss is None or ss[0].numel() < seq_h.numel() or ss[1].numel() < B:
            ss = st[slot] = (torch.empty(seq_h.numel(), dtype=torch.int32, device=dev),
                             torch.empty(B, dtype=torch.int64, device=dev), torch.empty(B, dtype=torch.int32, device=dev),
                             self.new_outputs(B))
        seq_d, off_d, len_d, out = ss
        if seq_h.dtype == torch.int16:
            seq_d[:seq_h.numel()].copy_(seq_h.to(dev, non_blocking=True).to(torch.int32) & 0xFFFF)  # u16 ids
        else:
            seq_d[:seq_h.numel()].copy_(seq_h, non_blocking=True)
        off_d[:B].copy_(off_h, non_blocking=True)
        len_d[:B].copy_(len_h, non_blocking=True)
        self.propose(seq_d, off_d[:B], len_d[:B], max_len, out=out.rows(0, B))
        for dst, src in ((out_h.size, out.size), (out_h.tokens, out.tokens), (out_h.parents, out.parents),
                         (out_h.depths, out.depths), (out_h.mask, out.mask)):
            dst[:B].copy_(src[:B], non_blocking=True)
        done = torch.cuda.Event()
        done.record()
        if sync:
            done.synchronize()
            self.check_status()
            return out_h
        return PendingDrafts(out_h, done, torch.zeros(1, dtype=torch.int32))


def exchange(coll, tails: torch.Tensor, tlen: torch.Tensor, P: int, M: int, search_fn, gather_fn):
    """The host protocol of one sharded propose for
    this rank's B requests (tails [B, P], tlen [B]); ``search_fn(tails, tlen)``
    -> local bounds [W*Bmax, P, 2] and ``gather_fn(global_bounds)`` -> owned
    positions [W*Bmax, P, M] are the shard kernels.  Per-rank batch sizes may
    differ (continuous batching): they are all-gathered first and every rank's
    slice is padded to the largest (padding rows repeat the first request, or
    a length-1 zero tail, and are dropped).  Returns (global bounds of my
    requests [B, P, 2], their sample positions + 1 [B, P, M])."""
    B = int(tlen.shape[0])
    dev = tlen.device
    Bmax = int(coll.all_gather(torch.tensor([B], dtype=torch.int64, device=dev)).max().item())
    if B < Bmax:
        pad_t = tails[:1].expand(Bmax - B, P) if B else torch.zeros((Bmax, P), dtype=tails.dtype, device=dev)
        pad_l = tlen[:1].expand(Bmax - B) if B else torch.ones(Bmax, dtype=tlen.dtype, device=dev)
        tails, tlen = torch.cat([tails, pad_t]), torch.cat([tlen, pad_l])
    if Bmax == 0:
        return (torch.zeros((0, P, 2), dtype=torch.int64, device=dev),
                torch.zeros((0, P, M), dtype=torch.int32, device=dev))
    all_tails = coll.all_gather(tails.contiguous())                        # 1: u32 [W*Bmax, P]
    all_tlen = coll.all_gather(tlen.contiguous())
    gb = coll.all_reduce_sum(search_fn(all_tails, all_tlen))               # 2 (C1): i64 [W*Bmax, P, 2]
    pos = coll.reduce_scatter_sum(gather_fn(gb))                           # 3 (C2): i32 [Bmax, P, M]
    r0 = coll.rank * Bmax
    return gb[r0:r0 + B].contiguous(), pos[:B].contiguous()


class LocalShards:
    """In-process emulation of W ranks for one-GPU tests: the collectives are sums /
    concatenations over per-rank tensors."""

    def __init__(self, full: Datastore, world: int, cfg: FusionConfig, separator=None) -> None:
        self.world = world
        self.shards = [shard_view(full, world, r) for r in range(world)]
        self.engines = [DraftEngine(s, cfg, separator) for s in self.shards]
        self.cfg = cfg

    def propose(self, per_rank: list) -> list:
        """per_rank[r] = (seq, off, len, max_len) device tensors; returns DraftBatch per rank."""
        P, M = self.cfg.P, self.cfg.M
        tails = [tails_of(s, o, l, P) for s, o, l, _ in per_rank]
        all_tails = torch.cat([t for t, _ in tails])
        all_tlen = torch.cat([n for _, n in tails])
        gb = sum(search(s, self.engines[0].c, all_tails, all_tlen) for s in self.shards)
        rows = rows_of(self.shards[0], sum(gather(s, self.engines[0].c, gb, M) for s in self.shards).contiguous())
        outs, b0 = [], 0
        for r, (seq, off, ln, mx) in enumerate(per_rank):
            B = int(ln.shape[0])
            eng = self.engines[r]
            out = eng.outputs(B)
            ws = eng.workspace(B, mx)
            seqs = _lib.Seqs(ptr(seq), ptr(off), ptr(ln), B, int(mx))
            d_out = _lib.DraftOut(ptr(out.size), ptr(out.tokens), ptr(out.parents), ptr(out.depths), ptr(out.mask))
            mine, rr = gb[b0:b0 + B].contiguous(), rows[b0:b0 + B].contiguous()
            check(lib().sssd_propose_pre(self.shards[r].c_view(), seqs, eng.c, ptr(mine), ptr(rr), d_out, None,
                                         ptr(ws), ws.numel(), stream_ptr(seq.device)))
            outs.append(out)
            b0 += B
        return outs
