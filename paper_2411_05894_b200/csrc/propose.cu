// Batched draft construction for SSSD on B200 (sm_100a).
//
//   ds_lookup_kernel   one CTA per request, one warp per prefix length p:
//                      32-ary warp-cooperative lower/upper-bound search over the
//                      suffix rows, strided sampling, continuation gather with
//                      separator / corpus-end cut, T cut-off, and a merge of the
//                      per-p runs (each already lexicographic) into one sorted
//                      element array.  Replaces Datastore.find_range /
//                      sample_range / get_conts (ref datastore.py:112-218).
//   input_scan_kernel  one CTA per request: backward-match lengths m[e] of the
//                      live sequence, occurrence compaction and a
//                      block bitonic sort of the continuation strings.  Replaces
//                      InputCache.get_conts (ref input_cache.py:88-121).
//   (draft_kernel, the fusion + flatten stage, lives in fusion.cu)
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "propose.cuh"

namespace sssd {

// continuation-table compare: vector loads when the rows allow them
__device__ __forceinline__ int cmp_tab(const KCfg& c, const uint32_t* a, uint32_t la, const uint32_t* b, uint32_t lb) {
  return c.tab16 ? cmp_row16(a, la, b, lb) : cmp_str(a, la, b, lb);
}

// --------------------------------------------------------------------------
// suffix-row comparisons (ref datastore.py:129-141)
// --------------------------------------------------------------------------

__device__ __forceinline__ uint32_t row_tok(const uint4& q0, const uint4& q1, const uint4& q2,
                                            const uint4& q3, int j) {
  // row = {pos, t0..t14}; token j lives in word j+1
  switch (j + 1) {
    case 1: return q0.y;
    case 2: return q0.z;
    case 3: return q0.w;
    case 4: return q1.x;
    case 5: return q1.y;
    case 6: return q1.z;
    case 7: return q1.w;
    case 8: return q2.x;
    case 9: return q2.y;
    case 10: return q2.z;
    case 11: return q2.w;
    case 12: return q3.x;
    case 13: return q3.y;
    case 14: return q3.z;
    default: return q3.w;
  }
}

// -1/0/+1: suffix at local row r vs pat[0..p); a suffix that runs out compares below.
__device__ __forceinline__ int cmp_rank(const sssd_ds& ds, uint64_t r, const uint32_t* pat,
                                        int p) {
  const uint4* row = reinterpret_cast<const uint4*>(ds.rows) + r * 4;
  const uint4 q0 = ldg4(row);
  uint4 q1 = make_uint4(0, 0, 0, 0), q2 = q1, q3 = q1;
  if (p > 3) q1 = ldg4(row + 1);
  if (p > 7) q2 = ldg4(row + 2);
  if (p > 11) q3 = ldg4(row + 3);
  const uint64_t avail = ds.n_tokens - q0.x;
#pragma unroll
  for (int j = 0; j < SSSD_ROW_TOKENS; ++j) {
    if (j >= p) return 0;
    if ((uint64_t)j >= avail) return -1;
    const uint32_t have = row_tok(q0, q1, q2, q3, j), want = pat[j];
    if (have != want) return have < want ? -1 : 1;
  }
  for (int j = SSSD_ROW_TOKENS; j < p; ++j) {
    if ((uint64_t)j >= avail) return -1;
    const uint32_t have = __ldg(ds.tokens + q0.x + j), want = pat[j];
    if (have != want) return have < want ? -1 : 1;
  }
  return 0;
}

// Update a monotone-predicate bracket [lo, hi] from one round of 32 sorted probes.
__device__ __forceinline__ void bracket_update(uint32_t bal, uint64_t q, uint64_t& lo,
                                               uint64_t& hi) {
  const int j = bal ? __ffs(bal) - 1 : 32;
  const uint64_t qa = __shfl_sync(SSSD_FULL, q, j > 0 ? j - 1 : 0);
  const uint64_t qb = __shfl_sync(SSSD_FULL, q, j < 32 ? j : 31);
  if (j == 32) {
    lo = max(lo, qb + 1);
  } else {
    hi = min(hi, qb);
    if (j > 0) lo = max(lo, qa + 1);
  }
}

// Warp-cooperative 33-ary search of the first rank in [lo, hi] where pred holds
// (pred(c) = c >= 0 for the lower bound, c > 0 for the upper bound).  Each round
// all 32 lanes probe; the other bound's bracket is tightened from the same probes.
template <bool kUpper>
__device__ uint64_t warp_search(const sssd_ds& ds, const uint32_t* pat, int p, uint64_t lo,
                                uint64_t hi, uint64_t& olo, uint64_t& ohi) {
  const int lane = lane_id();
  while (hi - lo > 32) {
    const uint64_t w = hi - lo;
    const uint64_t q = lo + (w * (uint64_t)(lane + 1)) / 33u;
    const int c = cmp_rank(ds, q, pat, p);
    const uint32_t ge = __ballot_sync(SSSD_FULL, c >= 0);
    const uint32_t gt = __ballot_sync(SSSD_FULL, c > 0);
    if (kUpper) {
      bracket_update(gt, q, lo, hi);
    } else {
      bracket_update(ge, q, lo, hi);
      bracket_update(gt, q, olo, ohi);
    }
  }
  // final round: probe every rank of [lo, hi) (w <= 32); the answer is the
  // first probe satisfying pred, or hi when none does
  const uint64_t w = hi - lo;
  const uint64_t q = lo + lane;
  const int c = (uint64_t)lane < w ? cmp_rank(ds, q, pat, p) : 2;
  const uint32_t ge = __ballot_sync(SSSD_FULL, c >= 0 && c != 2);
  const uint32_t gt = __ballot_sync(SSSD_FULL, c > 0 && c != 2);
  const uint32_t use = kUpper ? gt : ge;
  const uint64_t ans = lo + (use ? (uint64_t)(__ffs(use) - 1) : w);
  if (!kUpper) {
    // these probes cover [lo, hi) completely, so they pin the upper bound when
    // one of them is past the pattern, else only raise its floor
    if (gt) {
      const uint64_t tb = lo + (uint64_t)(__ffs(gt) - 1);
      ohi = min(ohi, tb);
      olo = max(olo, tb);
    } else {
      olo = max(olo, lo + w);
    }
  }
  return ans;
}

__device__ void warp_bounds(const sssd_ds& ds, const uint32_t* pat, int p, uint64_t& out_lo,
                            uint64_t& out_hi) {
  if (ds.kix && p >= 2 && p <= (int)ds.kix_kmax && kix_find(ds, pat, p, out_lo, out_hi) == 1) return;
  uint64_t blo = 0, bhi = ds.n_rows;
  if (ds.bucket) {  // first-token index: rows starting with pat[0] (or >= n_buckets)
    const uint32_t t0 = pat[0];
    if (t0 < ds.n_buckets) {
      blo = ds.bucket[t0];
      bhi = ds.bucket[t0 + 1];
      if (p == 1) {
        out_lo = blo;
        out_hi = bhi;
        return;
      }
    } else {
      blo = ds.bucket[ds.n_buckets];
    }
  }
  uint64_t ulo = blo, uhi = bhi;
  const uint64_t lower = warp_search<false>(ds, pat, p, blo, bhi, ulo, uhi);
  ulo = max(ulo, lower);
  uint64_t d0 = 0, d1 = 0;
  const uint64_t upper = warp_search<true>(ds, pat, p, ulo, uhi, d0, d1);
  out_lo = lower;
  out_hi = upper;
}

// Batched find_range for arbitrary pattern lengths: one warp per pattern.
__global__ void find_ranges_kernel(sssd_ds ds, const uint32_t* pat, const int64_t* pat_off,
                                   const int32_t* pat_len, int32_t B, int64_t* lo_hi) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;
  const int p = pat_len[b];
  uint64_t lo = 0, hi = ds.n_rows;
  if (p > 0) warp_bounds(ds, pat + pat_off[b], p, lo, hi);
  if (lane_id() == 0) {
    lo_hi[2 * b] = (int64_t)(lo + ds.rank_base);
    lo_hi[2 * b + 1] = (int64_t)(hi + ds.rank_base);
  }
}

// --------------------------------------------------------------------------
// block bitonic sort of element indices by (string, orig)
// --------------------------------------------------------------------------

struct ElemLess {
  const sssd_elem* el;
  const uint32_t* tok;
  int n;
  __device__ __forceinline__ bool operator()(uint32_t a, uint32_t b) const {
    if (b >= (uint32_t)n) return a < (uint32_t)n || a < b;  // padding sorts last
    if (a >= (uint32_t)n) return false;
    const sssd_elem ea = el[a], eb = el[b];
    const int r = cmp_str(tok + ea.off, el_len(ea.len_m), tok + eb.off, el_len(eb.len_m));
    if (r != 0) return r < 0;
    return ea.orig < eb.orig;
  }
};

__device__ void block_sort_elems(const sssd_elem* src, sssd_elem* dst, const uint32_t* tok, int n,
                                 uint32_t* idx) {
  int n2 = 1;
  while (n2 < n) n2 <<= 1;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) idx[i] = i;
  __syncthreads();
  const ElemLess less{src, tok, n};
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint32_t a = idx[i], bb = idx[ixj];
          const bool up = (i & k) == 0;
          const bool sw = up ? less(bb, a) : less(a, bb);
          if (sw) {
            idx[i] = bb;
            idx[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[idx[i]];
  __syncthreads();
}

// --------------------------------------------------------------------------
// K2+K3: datastore lookup (ref datastore.py:156-218, A.3 phase-split form)
// --------------------------------------------------------------------------


// Gather the sampled continuations of prefix length p into this request's
// string table (non-empty ones compacted, SA order kept).  Returns the count.
// The warp stages up to `rpl` rows per lane per round in shared memory with
// cp.async (rpl = 4 when it is the batch's only gathering warp and may use the
// whole CTA staging area): 128 samples cost one dependent row round trip.
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}

__device__ int gather_p(const sssd_ds& ds, const KCfg& c, int p, uint64_t lo, uint64_t hi,
                        uint32_t* tab, uint8_t* lens, int64_t* samples, uint32_t* srows, int rpl,
                        const uint32_t* pre_rows) {
  const int lane = lane_id();
  const uint64_t w = hi - lo;
  const int s = (int)min(w, (uint64_t)c.M);
  uint32_t* ptab = tab + (size_t)(p - 1) * c.M * c.TS;
  uint8_t* plen = lens + (size_t)(p - 1) * c.M;
  int cnt = 0;
  for (int k00 = 0; k00 < s; k00 += 32 * rpl) {
    // issue every row fetch of this round first (no register staging)
    for (int u = 0; u < rpl; ++u) {
      const int k = k00 + 32 * u + lane;
      if (k < s) {
        const uint64_t r =
            lo + (w <= (uint64_t)c.M ? (uint64_t)k : ((uint64_t)k * w) / (uint64_t)c.M);
        // sharded mode: the row was fetched by its owning shard into pre_rows[k]
        const uint4* row = pre_rows ? reinterpret_cast<const uint4*>(pre_rows) + (uint64_t)k * 4
                                    : reinterpret_cast<const uint4*>(ds.rows) + (r - ds.rank_base) * 4;
        uint4* sr = reinterpret_cast<uint4*>(srows + (u * 32 + lane) * kRowStride);
#pragma unroll
        for (int h = 0; h < 4; ++h) cp_async16(sr + h, row + h);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    for (int u = 0; u < rpl; ++u) {
      const int k0 = k00 + 32 * u;
      if (k0 >= s) break;
      const int k = k0 + lane;
      const uint32_t* srow = srows + (u * 32 + lane) * kRowStride;
      uint32_t len = 0, pos = 0;
      if (k < s) {
        pos = srow[0];
        if (samples) samples[k] = (int64_t)pos;
        const uint64_t start = (uint64_t)pos + p;
        const uint64_t avail = ds.n_tokens > start ? ds.n_tokens - start : 0;
        const uint32_t lim = (uint32_t)min((uint64_t)c.BL, avail);
        for (uint32_t j = 0; j < lim; ++j) {
          const uint32_t t = (p + j < SSSD_ROW_TOKENS) ? srow[1 + p + j] : __ldg(ds.tokens + start + j);
          if (c.has_sep && t == c.sep) break;
          ++len;
        }
      }
      const bool ne = len > 0;
      const uint32_t bal = __ballot_sync(SSSD_FULL, ne);
      const int idx = cnt + __popc(bal & lanemask_lt());
      if (ne) {
        const uint64_t start = (uint64_t)pos + p;
        uint32_t* dst = ptab + (size_t)idx * c.TS;
        for (uint32_t j = 0; j < len; ++j)
          dst[j] = (p + j < SSSD_ROW_TOKENS) ? srow[1 + p + j] : __ldg(ds.tokens + start + j);
        plen[idx] = (uint8_t)len;
      }
      cnt += __popc(bal);
    }
    __syncwarp();
  }
  return cnt;
}

__device__ __forceinline__ void dedupe_request(const KCfg& c, int b, int n_all, const uint32_t* ds_tab,
                                               const sssd_elem* ds_el, int32_t* ds_n, const Cols& cols, int* gstart);

#ifndef SSSD_LOOKUP_MINB
// 4: up to 128 registers, no spills — this kernel serves small batches (B < 2048: B = 64 lookup
// stage 0.037 -> 0.033 ms against the former 8 / 32-register cap) and the separator / sharded paths
#define SSSD_LOOKUP_MINB 4
#endif
__global__ void __launch_bounds__(32 * SSSD_MAX_P, SSSD_LOOKUP_MINB)
    ds_lookup_kernel(sssd_ds ds, sssd_seqs seqs, KCfg c, uint32_t* ds_tab, uint8_t* ds_len,
                     sssd_elem* ds_el, int32_t* ds_n, sssd_lookup_out lk, sssd_elem* ds_raw,
                     uint32_t* ds_idx, int64_t idx_cap, Cols cols, const int64_t* pre_bounds,
                     const uint32_t* pre_rows) {
  const int b = c.b0 + blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  __shared__ uint32_t s_pat[SSSD_MAX_P];
  __shared__ uint64_t s_lo[SSSD_MAX_P], s_hi[SSSD_MAX_P];
  __shared__ int s_cnt[SSSD_MAX_P];
  extern __shared__ __align__(16) uint32_t s_rows[];  // ds_lookup_smem_words(P, M) words

  const int L = seqs.seq_len[b];
  const uint32_t* seq = seqs.seq + seqs.seq_off[b];
  const int pmax = min(c.P, L);
  if (threadIdx.x < pmax) s_pat[threadIdx.x] = seq[L - pmax + threadIdx.x];
  __syncthreads();

  const int p = warp + 1;
  if (p <= pmax) {
    uint64_t lo, hi;
    if (pre_bounds) {  // sharded mode: global bounds = sum of the shards' local bounds (A.2)
      lo = (uint64_t)pre_bounds[((size_t)b * c.P + warp) * 2] - ds.rank_base;
      hi = (uint64_t)pre_bounds[((size_t)b * c.P + warp) * 2 + 1] - ds.rank_base;
    } else {
      int kf = -1;
      if (ds.kix && !lk.ranges && kix_whole(ds) && p >= 2 && p <= (int)ds.kix_kmax) {
        kf = kix_find(ds, s_pat + (pmax - p), p, lo, hi);
        if (kf == 0) lo = hi = 0;  // absent: empty range (its insertion point is not reported)
      }
      if (kf < 0) warp_bounds(ds, s_pat + (pmax - p), p, lo, hi);
    }
    if (lane == 0) {
      s_lo[warp] = lo + ds.rank_base;
      s_hi[warp] = hi + ds.rank_base;
      s_cnt[warp] = -1;
      if (lk.ranges) {
        lk.ranges[((size_t)b * c.P + warp) * 2] = (int64_t)(lo + ds.rank_base);
        lk.ranges[((size_t)b * c.P + warp) * 2 + 1] = (int64_t)(hi + ds.rank_base);
      }
    }
  } else if (p <= c.P && lane == 0 && lk.ranges) {
    lk.ranges[((size_t)b * c.P + warp) * 2] = -1;
    lk.ranges[((size_t)b * c.P + warp) * 2 + 1] = -1;
  }
  __syncthreads();

  uint32_t* tab = ds_tab + (size_t)b * c.P * c.M * c.TS;
  uint8_t* lens = ds_len + (size_t)b * c.P * c.M;
  int64_t* smp = lk.samples ? lk.samples + (size_t)b * c.P * c.M : nullptr;

  // Gather p = pmax, pmax-1, ... in batches sized by the sample-count upper
  // bound, until the exact non-empty count reaches T (ref datastore.py:216-217).
  int cum = 0, next = pmax, pcut = 1;
  while (next >= 1) {
    int ub = 0, q = next;
    for (; q >= 1; --q) {
      ub += (int)min(s_hi[q - 1] - s_lo[q - 1], (uint64_t)c.M);
      if (cum + ub >= c.T) break;
    }
    const int blo = max(q, 1);
    if (p >= blo && p <= next) {
      // the batch's only gathering warp stages into the whole CTA area
      const bool alone = next == blo;
      const int n = gather_p(ds, c, p, s_lo[warp], s_hi[warp], tab, lens,
                             smp ? smp + (size_t)warp * c.M : nullptr,
                             alone ? s_rows : s_rows + warp * 32 * kRowStride, alone ? c.P : 1,
                             pre_rows ? pre_rows + (((size_t)b * c.P + warp) * c.M) * 16 : nullptr);
      if (lane == 0) s_cnt[warp] = n;
    }
    __syncthreads();
    bool done = false;
    for (int pp = next; pp >= blo; --pp) {
      cum += s_cnt[pp - 1];
      if (cum >= c.T) {
        pcut = pp;
        done = true;
        break;
      }
    }
    if (done) break;
    pcut = blo;
    next = blo - 1;
  }
  if (pmax == 0) pcut = 1;

  // Merge the included per-p runs into one array sorted by (string, list
  // position).  Without a separator every run is already sorted (SA order of
  // the suffixes = order of their cut continuations), so each element's rank
  // is its index plus binary-search counts in the other runs.  A separator
  // breaks that (suffixes [x,0,..] < [x,sep,..] but cut strings [x] < [x,0,..])
  // and the included strings are block-sorted instead.
  int before = 0;  // list position of run p's first element
  for (int q = pmax; q > p; --q)
    if (q >= pcut) before += s_cnt[q - 1];
  int n_all = 0;
  for (int q = pcut; q <= pmax; ++q) n_all += s_cnt[q - 1];
  // the level-synchronous fusion kernel takes the datastore elements with
  // identical continuation strings folded into one weighted element
  // (ds_dedupe_kernel, launched next on the same stream, writes the columns)
  const bool dedupe = cols.meta && ds_dedupe_enabled(c);
  if (c.has_sep) {
    sssd_elem* raw = ds_raw + (size_t)b * c.P * c.M;
    if (p >= pcut && p <= pmax) {
      for (int i = lane; i < s_cnt[warp]; i += 32) {
        sssd_elem e;
        e.off = (uint32_t)(((size_t)(p - 1) * c.M + i) * c.TS);
        e.orig = (uint32_t)(before + i);
        e.len_m = (uint32_t)lens[(size_t)(p - 1) * c.M + i] | (255u << 8);
        e.pad = 0;
        raw[before + i] = e;
      }
    }
    __syncthreads();
    int n = 0;
    for (int q = pcut; q <= pmax; ++q) n += s_cnt[q - 1];
    if (n > 0) {
      int n2 = 1;
      while (n2 < n) n2 <<= 1;
      uint32_t* idx = (n2 <= ds_lookup_smem_words(c.P, c.M)) ? s_rows : ds_idx + (size_t)b * idx_cap;
      sssd_elem* sorted = ds_el + (size_t)b * c.P * c.M;
      block_sort_elems(raw, sorted, tab, n, idx);
      if (cols.meta && !dedupe) {
        const Cols cb{cols.meta + (size_t)b * cols.stride, cols.orig + (size_t)b * cols.stride,
                      cols.tok + (size_t)b * cols.stride * c.BL, cols.stride};
        for (int i = threadIdx.x; i < n; i += blockDim.x) write_cols(cb, i, sorted[i], tab);
      }
    }
  } else if (p >= pcut && p <= pmax) {
    const int cnt = s_cnt[warp];
    for (int i = lane; i < cnt; i += 32) {
      const uint32_t* si = tab + ((size_t)(p - 1) * c.M + i) * c.TS;
      const uint32_t li = lens[(size_t)(p - 1) * c.M + i];
      int rank = i;
      for (int q = pcut; q <= pmax; ++q) {
        if (q == p) continue;
        const int cq = s_cnt[q - 1];
        int a = 0, z = cq;  // first element of run q that comes after string i
        while (a < z) {
          const int mid = (a + z) >> 1;
          const int r = cmp_tab(c, tab + ((size_t)(q - 1) * c.M + mid) * c.TS,
                                lens[(size_t)(q - 1) * c.M + mid], si, li);
          const bool before_i = q > p ? r <= 0 : r < 0;
          if (before_i) a = mid + 1; else z = mid;
        }
        rank += a;
      }
      sssd_elem e;
      e.off = (uint32_t)(((size_t)(p - 1) * c.M + i) * c.TS);
      e.orig = (uint32_t)(before + i);
      e.len_m = li | (255u << 8);
      e.pad = 0;
      ds_el[(size_t)b * c.P * c.M + rank] = e;
      if (cols.meta && !dedupe) {
        const Cols cb{cols.meta + (size_t)b * cols.stride, cols.orig + (size_t)b * cols.stride,
                      cols.tok + (size_t)b * cols.stride * c.BL, cols.stride};
        write_cols(cb, rank, e, tab);
      }
    }
  }
  const int n_out = n_all;  // folded below (or by ds_dedupe_kernel) when dedupe
  if (threadIdx.x == 0) {
    ds_n[b] = n_out;
    if (lk.p_cut) lk.p_cut[b] = pmax > 0 ? pcut : 0;
  }
  if (lk.n_conts && threadIdx.x < c.P) {
    const int q = threadIdx.x + 1;
    lk.n_conts[(size_t)b * c.P + threadIdx.x] = (q <= pmax && s_cnt[threadIdx.x] >= 0) ? s_cnt[threadIdx.x] : -1;
  }
  if (dedupe && ds_dedupe_in_lookup(c.P, c.M)) {
    // fold in place: the sorted elements are in ds_el (visible to the CTA
    // after the barrier); the staged rows are dead, their shared memory holds
    // the group starts (P*M + 1 <= ds_lookup_smem_words)
    __syncthreads();
    dedupe_request(c, b, n_all, ds_tab, ds_el, ds_n, cols, reinterpret_cast<int*>(s_rows));
  }
}

// Fold datastore elements with identical continuation strings (adjacent in
// the sorted array) into one element whose column meta carries the group size
// as its weight (el_wt); the first element of a group has the smallest list
// position, which the fusion kernel's first-appearance order needs.  One CTA
// per request: flags in parallel, compaction by warp 0.  gstart: n_all + 1 ints
// of shared memory.
__device__ __forceinline__ void dedupe_request(const KCfg& c, int b, int n_all, const uint32_t* ds_tab,
                                               const sssd_elem* ds_el, int32_t* ds_n, const Cols& cols, int* gstart) {
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  if (n_all <= 0) return;
  const sssd_elem* sorted = ds_el + (size_t)b * c.P * c.M;
  const uint32_t* tab = ds_tab + (size_t)b * c.P * c.M * c.TS;
  for (int r = threadIdx.x; r < n_all; r += blockDim.x) {
    int st = 1;
    if (r > 0) {
      const sssd_elem x = sorted[r - 1], y = sorted[r];
      st = cmp_tab(c, tab + x.off, el_len(x.len_m), tab + y.off, el_len(y.len_m)) != 0;
    }
    gstart[r] = st;
  }
  __syncthreads();
  if (warp != 0) return;
  int G = 0;
  for (int r0 = 0; r0 < n_all; r0 += 32) {  // compact the flags into group starts (in place: g <= r)
    const int r = r0 + lane;
    const bool st = r < n_all && gstart[r] != 0;
    const uint32_t sm = __ballot_sync(SSSD_FULL, st);
    __syncwarp();
    if (st) gstart[G + __popc(sm & lanemask_lt())] = r;
    G += __popc(sm);
    __syncwarp();
  }
  if (lane == 0) gstart[G] = n_all;
  __syncwarp();
  const Cols cb{cols.meta + (size_t)b * cols.stride, cols.orig + (size_t)b * cols.stride,
                cols.tok + (size_t)b * cols.stride * c.BL, cols.stride};
  for (int g = lane; g < G; g += 32) {
    const sssd_elem e = sorted[gstart[g]];
    write_cols(cb, g, e, tab);
    cb.meta[g] = (e.len_m & 0xffffu) | (uint32_t)(gstart[g + 1] - gstart[g]) << 16;
  }
  if (lane == 0) ds_n[b] = G;
}

__global__ void __launch_bounds__(128)
    ds_dedupe_kernel(KCfg c, const uint32_t* ds_tab, const sssd_elem* ds_el, int32_t* ds_n, Cols cols) {
  extern __shared__ int gstart[];  // [P*M + 1]
  const int b = c.b0 + blockIdx.x;
  dedupe_request(c, b, ds_n[b], ds_tab, ds_el, ds_n, cols, gstart);
}

// --------------------------------------------------------------------------
// K2+K3, one warp per request (the default without a separator): every prefix
// length is searched at the same time by its own group of lanes (a
// (32/groups + 1)-ary search per p), so no warp waits at a CTA barrier for the
// other p's and four times as many requests are in flight per SM as with one
// warp per p.  Same outputs as ds_lookup_kernel (ref datastore.py:156-218).
// --------------------------------------------------------------------------

constexpr int kLkWarps = 4;     // requests per CTA
#ifndef SSSD_LK_STAGE
#define SSSD_LK_STAGE 64
#endif
constexpr int kLkStage = SSSD_LK_STAGE;  // staged suffix rows per warp and round (2 per lane)

#ifndef SSSD_LKW_MINB
#define SSSD_LKW_MINB 8  // <= 64 registers (56, no spills): 64 warps per SM by registers
#endif
#ifdef SSSD_LK_PROBE  // per-phase cycle stamps of the lookup warp (measurement builds only)
__device__ long long* g_lk_cyc;
void lk_probe_set(long long* p) { cudaMemcpyToSymbol(g_lk_cyc, &p, sizeof(p)); }
#define LK_STAMP(i) \
  if (g_lk_cyc && lane == 0) g_lk_cyc[(size_t)b * 8 + (i)] = clock64() - lk_t0;
#else
#define LK_STAMP(i)
#endif
__global__ void __launch_bounds__(32 * kLkWarps, SSSD_LKW_MINB)
    ds_lookup_warp_kernel(sssd_ds ds, sssd_seqs seqs, KCfg c, uint32_t* ds_tab, uint8_t* ds_len,
                          sssd_elem* ds_el, int32_t* ds_n, sssd_lookup_out lk, Cols cols) {
  __shared__ __align__(16) uint32_t s_stage[kLkWarps][kLkStage * kRowStride];
  __shared__ uint32_t s_tail[kLkWarps][SSSD_MAX_P];
  __shared__ uint64_t s_rlo[kLkWarps][SSSD_MAX_P], s_rhi[kLkWarps][SSSD_MAX_P];
  __shared__ int s_cnt[kLkWarps][SSSD_MAX_P];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int b = c.b0 + blockIdx.x * kLkWarps + warp;
  if (b >= c.b1) return;  // (warp-uniform)
#ifdef SSSD_LK_PROBE
  const long long lk_t0 = clock64();
#endif
  const int L = seqs.seq_len[b];
  const uint32_t* seq = seqs.seq + seqs.seq_off[b];
  const int pmax = min(c.P, L);
  uint32_t* tail = s_tail[warp];
  if (lane < pmax) tail[lane] = seq[L - pmax + lane];
  if (lane < SSSD_MAX_P) s_cnt[warp][lane] = -1;
  __syncwarp();

  // first-token bracket of pattern p (its first token is tail[pmax - p])
  auto bracket = [&](int p, uint64_t& blo, uint64_t& bhi) {
    blo = 0;
    bhi = ds.n_rows;
    if (ds.bucket && p >= 1) {
      const uint32_t t0 = tail[pmax - p];
      if (t0 < ds.n_buckets) {
        blo = ds.bucket[t0];
        bhi = ds.bucket[t0 + 1];
      } else {
        blo = ds.bucket[ds.n_buckets];
      }
    }
  };
  // p = 1 needs no probe when its token has a bucket
  const bool p1_free = pmax >= 1 && ds.bucket && tail[pmax - 1] < ds.n_buckets;
  if (lane == 0 && p1_free) {
    uint64_t a, z;
    bracket(1, a, z);
    s_rlo[warp][0] = a;
    s_rhi[warp][0] = z;
  }
  // p = 2 .. kix_kmax: the k-gram index holds the exact range (one slot read
  // + the verification of row lo, which the gather reads next anyway); an
  // absent k-gram is an empty range unless its insertion point is reported
  uint32_t known = p1_free ? 1u : 0u;  // bit p-1: range already known
  if (ds.kix) {
    const int p = lane + 1;
    int kf = -1;
    uint64_t klo = 0, khi = 0;
    if (p >= 2 && p <= pmax && p <= (int)ds.kix_kmax) {
      kf = kix_find(ds, tail + (pmax - p), p, klo, khi);
      if (kf == 0 && (lk.ranges || !kix_whole(ds))) kf = -1;
    }
    if (kf >= 0) {
      s_rlo[warp][p - 1] = kf == 1 ? klo : 0;
      s_rhi[warp][p - 1] = kf == 1 ? khi : 0;
    }
    known |= __ballot_sync(SSSD_FULL, kf >= 0);
  }
  const uint32_t todo = ((pmax >= 32 ? 0u : (1u << pmax)) - 1u) & ~known;  // patterns still searched
  const int ng = __popc(todo);
  if (ng > 0) {
    const int gs = 32 / ng;
    const int gid = lane / gs, gl = lane - gid * gs;
    const bool active = gid < ng;
    int myp = 1;  // group gid searches the gid-th longest pattern still to do
    for (int p = pmax, g = 0; p >= 1; --p)
      if ((todo >> (p - 1)) & 1u) {
        if (g == gid) myp = p;
        ++g;
      }
    if (!active) myp = 1;
    const uint32_t* pat = tail + (pmax - myp);
    const uint32_t gbits = gs >= 32 ? 0xffffffffu : ((1u << gs) - 1u);
    const int gbase = active ? gid * gs : 0;
    uint64_t lo, hi;
    bracket(myp, lo, hi);
    uint64_t ulo = lo, uhi = hi;
    uint64_t q = 0;
    // my group's first satisfying lane j -> bracket update (all lanes execute the shuffles)
    auto upd = [&](uint32_t mask, bool apply, uint64_t& l, uint64_t& h) {
      const uint32_t m = active ? (mask >> gbase) & gbits : 0u;
      const int j = m ? __ffs(m) - 1 : gs;
      const uint64_t qb = __shfl_sync(SSSD_FULL, q, gbase + min(j, gs - 1));
      const uint64_t qa = __shfl_sync(SSSD_FULL, q, gbase + max(j - 1, 0));
      if (apply) {
        if (j == gs) {
          l = max(l, qb + 1);
        } else {
          h = min(h, qb);
          if (j > 0) l = max(l, qa + 1);
        }
      }
    };
    // lower bound (pred c >= 0), tightening the upper bracket (c > 0) from the same probes
    while (true) {
      const bool need = active && hi - lo > (uint64_t)gs;
      if (!__any_sync(SSSD_FULL, need)) break;
      int cv = 2;
      if (need) {
        q = lo + ((hi - lo) * (uint64_t)(gl + 1)) / (uint64_t)(gs + 1);
        cv = cmp_rank(ds, q, pat, myp);
      }
      const uint32_t ge = __ballot_sync(SSSD_FULL, need && cv >= 0);
      const uint32_t gt = __ballot_sync(SSSD_FULL, need && cv > 0);
      upd(ge, need, lo, hi);
      upd(gt, need, ulo, uhi);
    }
    uint64_t lower;
    {
      const uint64_t w = hi - lo;
      const bool v = active && (uint64_t)gl < w;
      q = lo + gl;
      const int cv = v ? cmp_rank(ds, q, pat, myp) : 2;
      const uint32_t ge = (__ballot_sync(SSSD_FULL, v && cv >= 0) >> gbase) & gbits;
      const uint32_t gt = (__ballot_sync(SSSD_FULL, v && cv > 0) >> gbase) & gbits;
      lower = lo + (ge ? (uint64_t)(__ffs(ge) - 1) : w);
      if (gt) {
        const uint64_t tb = lo + (uint64_t)(__ffs(gt) - 1);
        uhi = min(uhi, tb);
        ulo = max(ulo, tb);
      } else {
        ulo = max(ulo, lo + w);
      }
    }
    // upper bound (pred c > 0) from the tightened bracket
    lo = max(ulo, lower);
    hi = uhi;
    while (true) {
      const bool need = active && hi - lo > (uint64_t)gs;
      if (!__any_sync(SSSD_FULL, need)) break;
      int cv = 2;
      if (need) {
        q = lo + ((hi - lo) * (uint64_t)(gl + 1)) / (uint64_t)(gs + 1);
        cv = cmp_rank(ds, q, pat, myp);
      }
      const uint32_t gt = __ballot_sync(SSSD_FULL, need && cv > 0);
      upd(gt, need, lo, hi);
    }
    uint64_t upper;
    {
      const uint64_t w = hi - lo;
      const bool v = active && (uint64_t)gl < w;
      q = lo + gl;
      const int cv = v ? cmp_rank(ds, q, pat, myp) : 2;
      const uint32_t gt = (__ballot_sync(SSSD_FULL, v && cv > 0) >> gbase) & gbits;
      upper = lo + (gt ? (uint64_t)(__ffs(gt) - 1) : w);
    }
    if (active && gl == 0) {
      s_rlo[warp][myp - 1] = lower;
      s_rhi[warp][myp - 1] = upper;
    }
  }
  __syncwarp();
  LK_STAMP(0)
  if (lk.ranges && lane < c.P) {
    const bool ok = lane < pmax;
    lk.ranges[((size_t)b * c.P + lane) * 2] = ok ? (int64_t)(s_rlo[warp][lane] + ds.rank_base) : -1;
    lk.ranges[((size_t)b * c.P + lane) * 2 + 1] = ok ? (int64_t)(s_rhi[warp][lane] + ds.rank_base) : -1;
  }

  uint32_t* tab = ds_tab + (size_t)b * c.P * c.M * c.TS;
  uint8_t* lens = ds_len + (size_t)b * c.P * c.M;
  int64_t* smp = lk.samples ? lk.samples + (size_t)b * c.P * c.M : nullptr;
  uint32_t* stage = s_stage[warp];

  // T cut-off (ref datastore.py:216-217): p = pmax, pmax-1, ... in batches sized
  // by the sample-count upper bound, gathered p by p (rows staged with cp.async,
  // two per lane per round)
  int cum = 0, next = pmax, pcut = 1;
  while (next >= 1) {
    int ub = 0, qq = next;
    for (; qq >= 1; --qq) {
      ub += (int)min(s_rhi[warp][qq - 1] - s_rlo[warp][qq - 1], (uint64_t)c.M);
      if (cum + ub >= c.T) break;
    }
    const int blo = max(qq, 1);
    bool done = false;
    for (int p = next; p >= blo; --p) {
      const uint64_t lo = s_rlo[warp][p - 1], w = s_rhi[warp][p - 1] - lo;
      const int sc = (int)min(w, (uint64_t)c.M);
      uint32_t* ptab = tab + (size_t)(p - 1) * c.M * c.TS;
      uint8_t* plen = lens + (size_t)(p - 1) * c.M;
      int cnt = 0;
      for (int k00 = 0; k00 < sc; k00 += kLkStage) {
        for (int u = 0; u < kLkStage / 32; ++u) {
          const int k = k00 + 32 * u + lane;
          if (k < sc) {
            const uint64_t r = lo + (w <= (uint64_t)c.M ? (uint64_t)k : ((uint64_t)k * w) / (uint64_t)c.M);
            const uint4* row = reinterpret_cast<const uint4*>(ds.rows) + r * 4;
            uint4* sr = reinterpret_cast<uint4*>(stage + (u * 32 + lane) * kRowStride);
#pragma unroll
            for (int h = 0; h < 4; ++h) cp_async16(sr + h, row + h);
          }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        for (int u = 0; u < kLkStage / 32; ++u) {
          const int k0 = k00 + 32 * u;
          if (k0 >= sc) break;
          const int k = k0 + lane;
          const uint32_t* srow = stage + (u * 32 + lane) * kRowStride;
          uint32_t len = 0, pos = 0;
          if (k < sc) {
            pos = srow[0];
            if (smp) smp[(size_t)(p - 1) * c.M + k] = (int64_t)pos;
            const uint64_t start = (uint64_t)pos + p;
            const uint64_t avail = ds.n_tokens > start ? ds.n_tokens - start : 0;
            len = (uint32_t)min((uint64_t)c.BL, avail);  // (no separator on this path)
          }
          const bool ne = len > 0;
          const uint32_t bal = __ballot_sync(SSSD_FULL, ne);
          if (ne) {
            const int idx = cnt + __popc(bal & lanemask_lt());
            const uint64_t start = (uint64_t)pos + p;
            uint32_t* dst = ptab + (size_t)idx * c.TS;
            if (c.tab16) {  // 16-byte stores (the row's tail past len is padding)
              for (uint32_t j = 0; j < len; j += 4) {
                uint32_t v[4];
#pragma unroll
                for (uint32_t k = 0; k < 4; ++k) {
                  const uint32_t jj = j + k;
                  v[k] = jj >= len ? 0u : (p + jj < SSSD_ROW_TOKENS ? srow[1 + p + jj] : __ldg(ds.tokens + start + jj));
                }
                *reinterpret_cast<uint4*>(dst + j) = make_uint4(v[0], v[1], v[2], v[3]);
              }
            } else {
              for (uint32_t j = 0; j < len; ++j)
                dst[j] = (p + j < SSSD_ROW_TOKENS) ? srow[1 + p + j] : __ldg(ds.tokens + start + j);
            }
            plen[idx] = (uint8_t)len;
          }
          cnt += __popc(bal);
        }
        __syncwarp();
      }
      if (lane == 0) s_cnt[warp][p - 1] = cnt;
      cum += cnt;
      if (cum >= c.T) {
        pcut = p;
        done = true;
        break;
      }
    }
    __syncwarp();
    if (done) break;
    pcut = blo;
    next = blo - 1;
  }
  if (pmax == 0) pcut = 1;
  LK_STAMP(1)

  // merge the included runs (each sorted: SA order = order of the cut
  // continuations without a separator): rank = index + binary-searched counts
  // of the other runs (ties: the larger p's run first = list position order)
  int n_all = 0;
  for (int q = pcut; q <= pmax; ++q) n_all += s_cnt[warp][q - 1];
  // folding of identical continuations (see ds_dedupe_kernel) happens below,
  // in this warp, when the group starts fit the staging area
  const bool dedupe = cols.meta && ds_dedupe_enabled(c) && n_all + 1 <= kLkStage * kRowStride;
  const Cols cb{cols.meta ? cols.meta + (size_t)b * cols.stride : nullptr, cols.orig + (size_t)b * cols.stride,
                cols.tok + (size_t)b * cols.stride * c.BL, cols.stride};
  int before = 0;
  for (int p = pmax; p >= pcut; --p) {
    const int cnt = s_cnt[warp][p - 1];
    for (int i = lane; i < cnt; i += 32) {
      const uint32_t* si = tab + ((size_t)(p - 1) * c.M + i) * c.TS;
      const uint32_t li = lens[(size_t)(p - 1) * c.M + i];
      int rank = i;
      for (int q = pcut; q <= pmax; ++q) {
        if (q == p) continue;
        int a = 0, z = s_cnt[warp][q - 1];
        while (a < z) {
          const int mid = (a + z) >> 1;
          const int r = cmp_tab(c, tab + ((size_t)(q - 1) * c.M + mid) * c.TS, lens[(size_t)(q - 1) * c.M + mid], si, li);
          const bool before_i = q > p ? r <= 0 : r < 0;
          if (before_i) a = mid + 1;
          else z = mid;
        }
        rank += a;
      }
      sssd_elem e;
      e.off = (uint32_t)(((size_t)(p - 1) * c.M + i) * c.TS);
      e.orig = (uint32_t)(before + i);
      e.len_m = li | (255u << 8);
      e.pad = 0;
      ds_el[(size_t)b * c.P * c.M + rank] = e;
      if (cb.meta && !dedupe) write_cols(cb, rank, e, tab);
    }
    before += cnt;
  }
  int n_out = n_all;
  LK_STAMP(2)
  if (dedupe) {
    __syncwarp();  // the sorted elements above are this warp's own global writes
    int* gst = reinterpret_cast<int*>(stage);
    const sssd_elem* sorted = ds_el + (size_t)b * c.P * c.M;
    int G = 0;
    for (int r0 = 0; r0 < n_all; r0 += 32) {
      const int r = r0 + lane;
      bool st = false;
      if (r < n_all) {
        if (r == 0) {
          st = true;
        } else {
          const sssd_elem x = sorted[r - 1], y = sorted[r];
          st = cmp_tab(c, tab + x.off, el_len(x.len_m), tab + y.off, el_len(y.len_m)) != 0;
        }
      }
      const uint32_t sm = __ballot_sync(SSSD_FULL, st);
      if (st) gst[G + __popc(sm & lanemask_lt())] = r;
      G += __popc(sm);
    }
    if (lane == 0) gst[G] = n_all;
    __syncwarp();
    for (int g = lane; g < G; g += 32) {
      const sssd_elem e = sorted[gst[g]];
      write_cols(cb, g, e, tab);
      cb.meta[g] = (e.len_m & 0xffffu) | (uint32_t)(gst[g + 1] - gst[g]) << 16;
    }
    n_out = G;
  } else if (cb.meta && ds_dedupe_enabled(c)) {
    __syncwarp();  // (too many continuations to fold here: weight 1 each)
    for (int r = lane; r < n_all; r += 32) write_cols(cb, r, ds_el[(size_t)b * c.P * c.M + r], tab);
  }
  LK_STAMP(3)
#ifdef SSSD_LK_PROBE
  if (g_lk_cyc && lane == 0) {
    g_lk_cyc[(size_t)b * 8 + 4] = n_all;
    g_lk_cyc[(size_t)b * 8 + 5] = pmax - pcut + 1;
    g_lk_cyc[(size_t)b * 8 + 6] = n_out;
  }
#endif
  if (lane == 0) {
    ds_n[b] = n_out;
    if (lk.p_cut) lk.p_cut[b] = pmax > 0 ? pcut : 0;
  }
  if (lk.n_conts && lane < c.P) {
    const int q = lane + 1;
    const int v = (q <= pmax && q >= pcut) ? s_cnt[warp][lane] : -1;
    lk.n_conts[(size_t)b * c.P + lane] = (q <= pmax && s_cnt[warp][lane] >= 0) ? v : -1;
  }
}

// --------------------------------------------------------------------------
// SA-range sharding: local bounds per shard, then the
// owning shard copies each sampled suffix row into an exchange buffer
// --------------------------------------------------------------------------

// bounds[b][p-1] = (#rows < pattern, #rows <= pattern) within this shard;
// patterns are the last p tokens of each (tail) sequence; p > len -> (0, 0)
__global__ void __launch_bounds__(32 * SSSD_MAX_P)
    shard_search_kernel(sssd_ds ds, sssd_seqs seqs, KCfg c, int64_t* bounds) {
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  __shared__ uint32_t s_pat[SSSD_MAX_P];
  const int L = seqs.seq_len[b];
  const uint32_t* seq = seqs.seq + seqs.seq_off[b];
  const int pmax = min(c.P, L);
  if (threadIdx.x < pmax) s_pat[threadIdx.x] = seq[L - pmax + threadIdx.x];
  __syncthreads();
  const int p = warp + 1;
  uint64_t lo = 0, hi = 0;
  if (p <= pmax) warp_bounds(ds, s_pat + (pmax - p), p, lo, hi);
  if (lane == 0) {
    bounds[((size_t)b * c.P + warp) * 2] = (int64_t)lo;
    bounds[((size_t)b * c.P + warp) * 2 + 1] = (int64_t)hi;
  }
}

// xrows[b][p-1][k][16] = suffix row of the k-th sampled global rank when this
// shard owns it, zeros otherwise (so a sum over shards assembles every row)
__global__ void shard_gather_kernel(sssd_ds ds, KCfg c, int B, const int64_t* gbounds, uint32_t* xrows) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one 16B quarter-row per thread
  const int64_t total = (int64_t)B * c.P * c.M * 4;
  if (t >= total) return;
  const int q = (int)(t & 3);
  const int64_t s = t >> 2;
  const int k = (int)(s % c.M);
  const int64_t bp = s / c.M;
  const uint64_t lo = (uint64_t)gbounds[bp * 2], hi = (uint64_t)gbounds[bp * 2 + 1];
  const uint64_t w = hi - lo;
  uint4 v = make_uint4(0, 0, 0, 0);
  if ((uint64_t)k < min(w, (uint64_t)c.M)) {
    const uint64_t r = lo + (w <= (uint64_t)c.M ? (uint64_t)k : ((uint64_t)k * w) / (uint64_t)c.M);
    if (r >= ds.rank_base && r < ds.rank_base + ds.n_rows)
      v = ldg4(reinterpret_cast<const uint4*>(ds.rows) + (r - ds.rank_base) * 4 + q);
  }
  reinterpret_cast<uint4*>(xrows)[t] = v;
}

// Owner-written sample positions (the compact C2 exchange): xpos[b][p-1][k] =
// corpus position + 1 of sampled global rank k of [lo, hi) if this shard owns
// it, else 0, so a sum over shards yields every position exactly once.
__global__ void shard_gather_pos_kernel(sssd_ds ds, KCfg c, int B, const int64_t* gbounds, uint32_t* xpos) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= (int64_t)B * c.P * c.M) return;
  const int k = (int)(s % c.M);
  const int64_t bp = s / c.M;
  const uint64_t lo = (uint64_t)gbounds[bp * 2], hi = (uint64_t)gbounds[bp * 2 + 1];
  const uint64_t w = hi - lo;
  uint32_t v = 0;
  if ((uint64_t)k < min(w, (uint64_t)c.M)) {
    const uint64_t r = lo + (w <= (uint64_t)c.M ? (uint64_t)k : ((uint64_t)k * w) / (uint64_t)c.M);
    if (r >= ds.rank_base && r < ds.rank_base + ds.n_rows) v = __ldg(ds.rows + (r - ds.rank_base) * 16) + 1u;
  }
  xpos[s] = v;
}

// Suffix rows of exchanged positions (pos + 1; 0 = none -> zero row) from the
// replicated token array: the owner rank's requests read their sampled rows
// locally instead of receiving 64 B per sample over NVLink.
__global__ void rows_from_pos_kernel(const uint32_t* tokens, uint64_t n, const uint32_t* xpos, int64_t count,
                                     uint32_t* rows) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one 16 B quarter row per thread
  if (t >= count * 4) return;
  const int q = (int)(t & 3);
  const uint32_t pp = xpos[t >> 2];
  uint32_t v[4] = {0, 0, 0, 0};
  if (pp) {
    const uint64_t pos = pp - 1u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = 4 * q + j;  // column 0 = SA position, 1.. = tokens pos + col - 1
      v[j] = col == 0 ? (uint32_t)pos : (pos + col - 1 < n ? __ldg(tokens + pos + col - 1) : 0u);
    }
  }
  reinterpret_cast<uint4*>(rows)[t] = make_uint4(v[0], v[1], v[2], v[3]);
}

// N2 index build: request b's positions [0, L-1) as keys (token << pb | pos),
// bitonic-sorted in shared memory by one CTA (1024 threads); len[b] = 0 (no
// index: the stateless scan) when L - 1 > SSSD_INDEX_MAX or a token does not
// fit the key.
__global__ void __launch_bounds__(1024) input_index_build_kernel(sssd_seqs seqs, sssd_input_index ix,
                                                                 const int32_t* rows) {
  extern __shared__ __align__(16) uint32_t s_key[];
  __shared__ int s_bad;
  const int b = rows ? rows[blockIdx.x] : (int)blockIdx.x;
  const int n = seqs.seq_len[b] - 1;
  if (n <= 0 || n > SSSD_INDEX_MAX || n > (1 << ix.pos_bits)) {
    if (threadIdx.x == 0) ix.len[b] = 0;
    return;
  }
  const uint32_t* seq = seqs.seq + seqs.seq_off[b];
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  int n2 = 1;
  while (n2 < n) n2 <<= 1;
  const uint32_t tmax = ix.pos_bits >= 32 ? 0u : (1u << (32 - ix.pos_bits));
  for (int j = threadIdx.x; j < n2; j += blockDim.x) {
    if (j < n) {
      const uint32_t t = seq[j];
      if (t >= tmax) s_bad = 1;
      s_key[j] = (t << ix.pos_bits) | (uint32_t)j;
    } else {
      s_key[j] = 0xffffffffu;  // padding sorts last
    }
  }
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) ix.len[b] = 0;
    return;
  }
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const uint32_t a = s_key[i], c2 = s_key[p];
          if ((a > c2) == ((i & k) == 0)) {
            s_key[i] = c2;
            s_key[p] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  uint32_t* out = ix.keys + ix.off[b];
  for (int j = threadIdx.x; j < n; j += blockDim.x) out[j] = s_key[j];
  if (threadIdx.x == 0) ix.len[b] = n;
}

// --------------------------------------------------------------------------
// K4: input scan (ref input_cache.py:88-121, stateless form A.4)
// --------------------------------------------------------------------------

constexpr int kSortSmem = 4096;
#ifndef SSSD_SCAN_MERGE_MIN
#define SSSD_SCAN_MERGE_MIN 32  // occurrence counts above this take the merge sort (when it fits)
#endif
#ifndef SSSD_SCAN_HFIRST
#define SSSD_SCAN_HFIRST 1
#endif

// Launched with 256 threads, or 1024 for long contexts (input_scan_threads);
// dynamic shared memory input_scan_smem_bytes(threads, IBL).
__global__ void __launch_bounds__(1024)
    input_scan_kernel(sssd_seqs seqs, KCfg c, sssd_elem* raw, sssd_elem* sorted, int32_t* in_n,
                      uint32_t* idx_ws, int64_t cap, int64_t cap2, Cols cols) {
  const int b = c.b0 + blockIdx.x;
  const int tid = threadIdx.x, lane = lane_id(), warp = tid >> 5, nw = blockDim.x >> 5;
#ifdef SSSD_LK_PROBE  // measurement builds: scan phases in slots 4-7 of the lookup probe
  const long long sc_t0 = clock64();
#define SC_STAMP(i) \
  if (g_lk_cyc && tid == 0) g_lk_cyc[(size_t)b * 8 + (i)] = clock64() - sc_t0;
#else
#define SC_STAMP(i)
#endif
  __shared__ uint32_t s_tail[SSSD_MAX_P];
  __shared__ int s_wsum[32];
  extern __shared__ __align__(16) uint32_t s_idx[];  // >= kSortSmem words
  const int L = seqs.seq_len[b];
  const uint32_t* seq = seqs.seq + seqs.seq_off[b];
  if (!c.use_in || L < 2) {
    if (tid == 0) in_n[b] = 0;
    return;
  }
  const int jm = min(c.P, L - 1);
  if (tid < jm) s_tail[tid] = seq[L - 1 - tid];
  __syncthreads();
  sssd_elem* r = raw + (size_t)b * cap;
  // Match lengths m[e] (A.4) for end positions e in [1, L): each thread owns
  // kScanV consecutive positions of a 256 * kScanV tile and fetches their
  // first comparison tokens seq[e-1] with independent loads (one memory round
  // trip per tile); only the rare lanes whose first token matches the tail
  // read further back.  A block scan of the per-thread counts places the
  // occurrences in e order.
  constexpr int kScanV = 8;
  const uint32_t t0 = s_tail[0];
  const bool aligned = (reinterpret_cast<uintptr_t>(seq) & 15) == 0;
  static_assert(kScanV == 8, "vector tile loads assume 8 positions per thread");
  int total = 0;
  // N2: with an input index, positions j < L0 come from the sorted keys
  // (binary search for the last token's key range: ascending positions, i.e.
  // e order) and only the tail j >= L0 is scanned below
  int L0 = 0;
  if (c.idx_len) L0 = max(0, min(c.idx_len[b], L - 1));
  if (L0 > 0 && (uint64_t)t0 < (1ull << (32 - c.idx_pb))) {
    const uint32_t* keys = c.idx_keys + c.idx_off[b];
    const uint32_t pmask = (1u << c.idx_pb) - 1u;
    const uint32_t klo = t0 << c.idx_pb, khi = klo | pmask;
    // the key range of the last token by two 17-ary searches in warp 0 (lanes
    // 0-15: first key >= klo, lanes 16-31: first key > khi): ~3 dependent
    // rounds for 2k keys instead of 2 x 11 binary-search steps
    if (warp == 0) {
      const int half = lane >> 4, hl = lane & 15;
      const uint32_t hmask = 0xffffu << (16 * half);
      int lo = 0, hi = L0;
      while (__any_sync(SSSD_FULL, lo < hi)) {
        const int n = hi - lo;
        int p = -1;
        if (n > 0) p = n <= 16 ? (hl < n ? lo + hl : -1) : lo + (int)(((long long)(hl + 1) * n) / 17);
        bool pr = false;
        if (p >= 0) {
          const uint32_t k = keys[p];
          pr = half == 0 ? k < klo : k <= khi;
        }
        const uint32_t bal = (__ballot_sync(SSSD_FULL, pr) & hmask) >> (16 * half);
        const int cnt = __popc(bal);  // predicate is monotone along the probes
        const int plast = __shfl_sync(SSSD_FULL, p, (16 * half) + max(cnt - 1, 0));
        const int pnext = __shfl_sync(SSSD_FULL, p, (16 * half) + min(cnt, 15));
        if (n > 0) {
          if (n <= 16) {
            lo = lo + cnt;
            hi = lo;
          } else {
            if (cnt > 0) lo = plast + 1;
            if (cnt < 16) hi = pnext;
          }
        }
      }
      if (lane == 0) s_wsum[0] = lo;
      if (lane == 16) s_wsum[1] = lo;
    }
    __syncthreads();
    const int a = s_wsum[0];
    const int cnt = s_wsum[1] - a;
    __syncthreads();  // (s_wsum is reused by the tail scan)
    for (int i = tid; i < cnt; i += blockDim.x) {
      const int e = (int)(keys[a + i] & pmask) + 1;  // occurrence of the last token at e - 1
      const int lim = min(jm, e);
      int m = 1;
      while (m < lim && seq[e - 1 - m] == s_tail[m]) ++m;
      sssd_elem el;
      el.off = (uint32_t)e;
      el.orig = (uint32_t)e;
      el.len_m = (uint32_t)min(c.IBL, L - e) | ((uint32_t)m << 8);
      el.pad = 0;
      r[i] = el;
    }
    total = cnt;
  } else {
    L0 = 0;
  }
  for (int tile = (L0 & ~7) + 1; tile < L; tile += (int)blockDim.x * kScanV) {
    const int e0 = tile + tid * kScanV;
    uint32_t v[kScanV];
    if (aligned && e0 + kScanV <= L) {  // two 16-byte loads: seq[e0-1 .. e0+7) (e0-1 is a multiple of 8)
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(seq + e0 - 1));
      const uint4 c2 = __ldg(reinterpret_cast<const uint4*>(seq + e0 + 3));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = c2.x; v[5] = c2.y; v[6] = c2.z; v[7] = c2.w;
    } else {
#pragma unroll
      for (int k = 0; k < kScanV; ++k) v[k] = e0 + k < L ? seq[e0 + k - 1] : ~t0;
    }
    // bit k: position e0 + k matches (m >= 1); positions past the end (e0 + k >= L)
    // and indexed ones (e0 + k <= L0) are masked out
    uint32_t valid = 0xffu;
    if (e0 + kScanV > L) valid = L > e0 ? (1u << (L - e0)) - 1u : 0u;
    if (e0 <= L0) valid &= L0 - e0 + 1 >= kScanV ? 0u : ~((1u << (L0 - e0 + 1)) - 1u);
    uint32_t mk = 0;
#pragma unroll
    for (int k = 0; k < kScanV; ++k) mk |= (v[k] == t0 ? 1u : 0u) << k;
    mk &= valid;
    const int cnt = __popc(mk);
    int inc = cnt;  // block exclusive scan of the counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(SSSD_FULL, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    // warp totals scanned with shuffles (nw <= 32): my warp's base and the tile total
    int wx = lane < nw ? s_wsum[lane] : 0, wi = wx;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(SSSD_FULL, wi, o);
      if (lane >= o) wi += y;
    }
    const int wbase = __shfl_sync(SSSD_FULL, wi - wx, warp);
    const int tsum = __shfl_sync(SSSD_FULL, wi, nw - 1);
    int at = total + wbase + inc - cnt;
    while (mk) {
      const int k = __ffs(mk) - 1;
      mk &= mk - 1;
      const int e = e0 + k;
      const int lim = min(jm, e);
      int m = 1;
      while (m < lim && seq[e - 1 - m] == s_tail[m]) ++m;
      sssd_elem el;
      el.off = (uint32_t)e;
      el.orig = (uint32_t)e;
      el.len_m = (uint32_t)min(c.IBL, L - e) | ((uint32_t)m << 8);
      el.pad = 0;
      r[at++] = el;
    }
    total += tsum;
    __syncthreads();  // s_wsum reuse
  }
  if (tid == 0) in_n[b] = total;
  SC_STAMP(4)
  sssd_elem* out = sorted + (size_t)b * cap;
  if (total == 0) return;
  __syncthreads();
  // Packed path (IBL <= 8, every token < 65535): a continuation string is one
  // 128-bit key (16 bits of token + 1 per depth; an absent token is 0, so a
  // proper prefix sorts first, as cmp_str orders them).  Runs of 32
  // consecutive occurrences are rank-sorted, then each occurrence adds the
  // binary-searched count of smaller keys of every other run (ties: position
  // order = run order).  Any occurrence count that fits shared memory.
  if (c.IBL <= 8 && total * 6 <= input_scan_smem_bytes(blockDim.x, c.IBL) / 4) {
    uint64_t* kh = reinterpret_cast<uint64_t*>(s_idx);
    uint64_t* kl = kh + total;
    uint32_t* srt = reinterpret_cast<uint32_t*>(kl + total);
    uint32_t* lrk = srt + total;
    bool wide = false;
    for (int e = tid; e < total; e += blockDim.x) {
      const sssd_elem el = r[e];
      const uint32_t len = el_len(el.len_m);
      srt[e] = el.off << 4 | el_m(el.len_m);  // (position, m) for the merge path's output (L < 2^28)
      uint64_t h = 0, l = 0;
      for (uint32_t d = 0; d < len; ++d) {
        const uint32_t tk = seq[el.off + d];
        wide |= tk >= 65535u;
        const uint64_t v = (uint64_t)(tk & 0xffffu) + 1;
        if (d < 4) h |= v << (16 * (3 - d));
        else l |= v << (16 * (7 - d));
      }
      kh[e] = h;
      kl[e] = l;
    }
    const bool narrow_keys = !__syncthreads_or(wide);
    SC_STAMP(5)
    const int scan_words = input_scan_smem_bytes(blockDim.x, c.IBL) / 4;
    if (narrow_keys && total > SSSD_SCAN_MERGE_MIN && total * 10 + 2 <= scan_words && L < (1 << 28)) {
      // merge sort (33 to a few thousand occurrences): 32-element runs
      // rank-sorted, then log2(total / 32) merge levels in which every key finds
      // its output slot with one binary search in the partner run (ties: the
      // left run's keys first = position order).  Each thread's chain is
      // ~6 + log2(total) steps per level instead of the run-rank path's
      // (total / 32) binary searches or the bitonic network's shared-memory
      // traffic (cfg4, 32k prompt-heavy contexts: 520 occurrences 17 -> 5 us,
      // 1,047 occurrences 32 -> 6 us).  Keys, then ping-pong (h, l, index)
      // arrays: B aliases kh / kl, A follows (10 words per occurrence).  The
      // payload is (position << 4 | m), so the output needs no global reads:
      // an element's tokens are its key's 16-bit fields.
      uint64_t* Bh = kh;
      uint64_t* Bl = kl;
      uint32_t* Bi = reinterpret_cast<uint32_t*>(kl + total);
      uint64_t* Ah = reinterpret_cast<uint64_t*>(s_idx + ((5 * total + 1) & ~1));
      uint64_t* Al = Ah + total;
      uint32_t* Ai = reinterpret_cast<uint32_t*>(Al + total);
      for (int e = tid; e < total; e += blockDim.x) {
        const int r0 = e & ~31, rn = min(32, total - r0);
        const uint64_t h = kh[e], l = kl[e];
        int lr = 0;
        for (int j = r0; j < r0 + rn; ++j) {
          const uint64_t hj = kh[j], lj = kl[j];
          lr += (hj < h || (hj == h && (lj < l || (lj == l && j < e)))) ? 1 : 0;
        }
        Ah[r0 + lr] = h;
        Al[r0 + lr] = l;
        Ai[r0 + lr] = Bi[e];  // (position, m) stashed by the key build
      }
      __syncthreads();
      uint64_t *sh = Ah, *sl = Al, *dh = Bh, *dl = Bl;
      uint32_t *si = Ai, *di = Bi;
      for (int lw = 5; (1 << lw) < total; ++lw) {
        const int w = 1 << lw;
        for (int i = tid; i < total; i += blockDim.x) {
          const int rid = i >> lw, k = i - (rid << lw), ps = (rid ^ 1) << lw;
          const int pl = max(0, min(w, total - ps));
          const uint64_t h = sh[i], l = sl[i];
          const bool left = (rid & 1) == 0;
          int lo = 0, hi = pl;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
#if SSSD_SCAN_HFIRST  // the low word only on a tie of the high words (half the shared-memory bytes)
            const uint64_t hx = sh[ps + mid];
            bool before = hx < h;
            if (hx == h) {
              const uint64_t lx = sl[ps + mid];
              before = left ? lx < l : lx <= l;
            }
            if (before) lo = mid + 1;
            else hi = mid;
#else
            const uint64_t hx = sh[ps + mid], lx = sl[ps + mid];
            if (hx < h || (hx == h && (left ? lx < l : lx <= l))) lo = mid + 1;
            else hi = mid;
#endif
          }
          const int o = ((rid & ~1) << lw) + k + lo;
          dh[o] = h;
          dl[o] = l;
          di[o] = si[i];
        }
        __syncthreads();
        uint64_t* th = sh;
        sh = dh;
        dh = th;
        uint64_t* tl = sl;
        sl = dl;
        dl = tl;
        uint32_t* ti = si;
        si = di;
        di = ti;
      }
      SC_STAMP(6)
      const Cols cb{cols.meta ? cols.meta + (size_t)b * cols.stride : nullptr,
                    cols.orig + (size_t)b * cols.stride, cols.tok + (size_t)b * cols.stride * c.IBL, cols.stride};
      for (int i = tid; i < total; i += blockDim.x) {
        const uint32_t pm = si[i], pos = pm >> 4;
        sssd_elem el;
        el.off = pos;
        el.orig = pos;
        el.len_m = (uint32_t)min(c.IBL, L - (int)pos) | (pm & 15u) << 8;
        el.pad = 0;
        out[i] = el;
        if (cb.meta) {
          cb.meta[i] = el.len_m & 0xffffu;
          cb.orig[i] = pos;
          const uint64_t h = sh[i], l = sl[i];
          const uint32_t len = el_len(el.len_m);
          for (uint32_t d = 0; d < len; ++d)
            cb.tok[d * cb.stride + i] = (uint32_t)(((d < 4 ? h >> (16 * (3 - d)) : l >> (16 * (7 - d))) & 0xffffu) - 1);
        }
      }
      SC_STAMP(7)
      return;
    }
    if (narrow_keys && total > 1024) {
      // many occurrences (prompt-heavy long contexts): a bitonic sort of the
      // (key, position) triples in shared memory, O(n log^2 n) instead of
      // the runs' O(n^2 / 32) binary searches; all-ascending form, so
      // positions >= total act as +infinity without being stored
      uint32_t* ix = srt;
      for (int e = tid; e < total; e += blockDim.x) ix[e] = (uint32_t)e;
      __syncthreads();
      int n2 = 1;
      while (n2 < total) n2 <<= 1;
      for (int lk = 1; (1 << lk) <= n2; ++lk) {
        for (int lj = lk - 1; lj >= 0; --lj) {
          for (int q = tid; q < n2 / 2; q += blockDim.x) {
            const int pb = q >> lj, pr = q & ((1 << lj) - 1);
            int lo, hi;
            if (lj == lk - 1) {
              lo = (pb << lk) + pr;
              hi = (pb << lk) + (1 << lk) - 1 - pr;
            } else {
              lo = (pb << (lj + 1)) + pr;
              hi = lo + (1 << lj);
            }
            if (hi >= total) continue;
            const uint64_t ha = kh[lo], la = kl[lo], hb = kh[hi], lb = kl[hi];
            const uint32_t ia = ix[lo], ib = ix[hi];
            if (hb < ha || (hb == ha && (lb < la || (lb == la && ib < ia)))) {
              kh[lo] = hb, kl[lo] = lb, ix[lo] = ib;
              kh[hi] = ha, kl[hi] = la, ix[hi] = ia;
            }
          }
          __syncthreads();
        }
      }
      SC_STAMP(6)
      const Cols cb{cols.meta ? cols.meta + (size_t)b * cols.stride : nullptr,
                    cols.orig + (size_t)b * cols.stride, cols.tok + (size_t)b * cols.stride * c.IBL, cols.stride};
      for (int i = tid; i < total; i += blockDim.x) {
        const sssd_elem el = r[ix[i]];
        out[i] = el;
        if (cb.meta) write_cols(cb, i, el, seq);
      }
      SC_STAMP(7)
      return;
    }
    if (narrow_keys) {
      for (int e = tid; e < total; e += blockDim.x) {
        const int r0 = e & ~31, rn = min(32, total - r0);
        const uint64_t h = kh[e], l = kl[e];
        int lr = 0;
        for (int j = r0; j < r0 + rn; ++j) {
          const uint64_t hj = kh[j], lj = kl[j];
          lr += (hj < h || (hj == h && (lj < l || (lj == l && j < e)))) ? 1 : 0;
        }
        srt[r0 + lr] = (uint32_t)e;
        lrk[e] = (uint32_t)lr;
      }
      __syncthreads();
      SC_STAMP(6)
      const Cols cb{cols.meta ? cols.meta + (size_t)b * cols.stride : nullptr,
                    cols.orig + (size_t)b * cols.stride, cols.tok + (size_t)b * cols.stride * c.IBL, cols.stride};
      for (int e = tid; e < total; e += blockDim.x) {
        const int r0 = e & ~31;
        const uint64_t h = kh[e], l = kl[e];
        int rank = (int)lrk[e];
        for (int q0 = 0; q0 < total; q0 += 32) {
          if (q0 == r0) continue;
          int lo = 0, hi = min(32, total - q0);  // elements of run q0 that sort before mine
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const uint32_t x = srt[q0 + mid];
            const uint64_t hx = kh[x], lx = kl[x];
            if (hx < h || (hx == h && (lx < l || (lx == l && q0 < r0)))) lo = mid + 1;
            else hi = mid;
          }
          rank += lo;
        }
        const sssd_elem el = r[e];
        out[rank] = el;
        if (cb.meta) write_cols(cb, rank, el, seq);
      }
      SC_STAMP(7)
      return;
    }
    __syncthreads();  // the key area is reused below
  }
  if (total <= (int)blockDim.x && total * (c.IBL + 6) <= input_scan_smem_bytes(blockDim.x, c.IBL) / 4) {
    // the common case (<= blockDim occurrences): continuation strings staged in
    // shared memory; warp w rank-sorts occurrences [32w, 32w + 32), then each
    // occurrence adds, per other run, a binary-searched count of the run's
    // smaller strings (ties: position order, i.e. run order).  When every
    // token is < 65535 and IBL <= 8, a string is compared as one 128-bit key
    // (16 bits of token + 1 per depth; an absent token is 0, so a proper
    // prefix sorts first, as cmp_str orders them).
    uint32_t* str = s_idx;  // [total][IBL] strings, [total] lengths, [total] run-sorted indices, keys
    uint32_t* slen = s_idx + total * c.IBL;
    uint32_t* srt = slen + total;
    uint64_t* kh = reinterpret_cast<uint64_t*>(s_idx + ((total * (c.IBL + 2) + 1) & ~1));
    uint64_t* kl = kh + total;
    sssd_elem me{};
    uint32_t ml = 0;
    const uint32_t* mine = str + tid * c.IBL;
    bool wide = false;
    if (tid < total) {
      me = r[tid];
      ml = el_len(me.len_m);
      slen[tid] = ml;
      for (uint32_t d = 0; d < ml; ++d) {
        const uint32_t tk = seq[me.off + d];
        str[tid * c.IBL + d] = tk;
        wide |= tk >= 65535u;
      }
    }
    const bool packed = !__syncthreads_or(wide || c.IBL > 8);
    uint64_t mh = 0, mlo = 0;
    if (packed && tid < total) {
      for (uint32_t d = 0; d < ml; ++d) {
        const uint64_t v = (uint64_t)(mine[d] + 1);
        if (d < 4) mh |= v << (16 * (3 - d));
        else mlo |= v << (16 * (7 - d));
      }
      kh[tid] = mh;
      kl[tid] = mlo;
    }
    if (packed) __syncthreads();
    // does occurrence j sort before mine?  (q_before: j's run precedes mine on ties)
    auto before = [&](uint32_t j, bool q_before) {
      if (packed) {
        const uint64_t h = kh[j], l = kl[j];
        return h < mh || (h == mh && (l < mlo || (l == mlo && q_before)));
      }
      const int cr = cmp_str(str + j * c.IBL, slen[j], mine, ml);
      return cr < 0 || (cr == 0 && q_before);
    };
    const int r0 = warp * 32, rn = min(32, total - r0);
    int lr = 0;
    if (tid < total) {
      for (int jj = r0; jj < r0 + rn; ++jj) lr += before((uint32_t)jj, jj < tid) ? 1 : 0;
      srt[r0 + lr] = (uint32_t)tid;
    }
    __syncthreads();
    if (tid < total) {
      int rank = lr;
      for (int q0 = 0; q0 < total; q0 += 32) {
        if (q0 == r0) continue;
        const int qn = min(32, total - q0);
        int lo = 0, hi = qn;  // elements of run q that sort before mine
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (before(srt[q0 + mid], q0 < r0)) lo = mid + 1;
          else hi = mid;
        }
        rank += lo;
      }
      out[rank] = me;
      if (cols.meta) {
        const Cols cb{cols.meta + (size_t)b * cols.stride, cols.orig + (size_t)b * cols.stride,
                      cols.tok + (size_t)b * cols.stride * c.IBL, cols.stride};
        cb.meta[rank] = me.len_m & 0xffffu;
        cb.orig[rank] = me.orig;
        for (uint32_t d = 0; d < ml; ++d) cb.tok[d * cb.stride + rank] = mine[d];
      }
    }
    return;
  }
  int n2 = 1;
  while (n2 < total) n2 <<= 1;
  uint32_t* idx = (n2 <= kSortSmem) ? s_idx : idx_ws + (size_t)b * cap2;
  block_sort_elems(r, out, seq, total, idx);
  if (cols.meta) {
    const Cols cb{cols.meta + (size_t)b * cols.stride, cols.orig + (size_t)b * cols.stride,
                  cols.tok + (size_t)b * cols.stride * c.IBL, cols.stride};
    for (int i = tid; i < total; i += blockDim.x) write_cols(cb, i, out[i], seq);
  }
}

// Sort caller-provided source paths (sssd_merge): one CTA per (request, source).
__global__ void __launch_bounds__(256)
    sort_sources_kernel(const uint32_t* tok, const sssd_elem* el, const int64_t* el_off,
                        const int32_t* el_n, sssd_elem* sorted, uint32_t* idx_ws, int64_t idx_cap,
                        Cols cols) {
  __shared__ uint32_t s_idx[kSortSmem];
  const int bs = blockIdx.x;
  const int n = el_n[bs];
  if (n <= 0) return;
  const int64_t o = el_off[bs];
  uint32_t* idx = (n <= kSortSmem) ? s_idx : idx_ws + o * 2;  // idx_ws holds 2*total entries
  (void)idx_cap;
  block_sort_elems(el + o, sorted + o, tok, n, idx);
  for (int i = threadIdx.x; i < n; i += blockDim.x) write_cols(cols, o + i, sorted[o + i], tok);
}

}  // namespace sssd
