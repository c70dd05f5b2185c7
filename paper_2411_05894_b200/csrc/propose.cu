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
//   draft_kernel       one warp per request: best-first fusion over tries that
//                      are never materialised — a trie node is a range of its
//                      source's sorted element array and is expanded lazily into
//                      a sibling group when popped — followed by DFS
//                      flattening and u64 ancestor masks.  Replaces merge /
//                      flatten (ref fusion.py:209-261, draft.py:67-86).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "propose.cuh"

namespace sssd {

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
  uint64_t ulo = 0, uhi = ds.n_rows;
  const uint64_t lower = warp_search<false>(ds, pat, p, 0, ds.n_rows, ulo, uhi);
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

constexpr int kRowStride = 16;  // u32 per staged row in smem

// Gather the sampled continuations of prefix length p into this request's
// string table (non-empty ones compacted, SA order kept).  Returns the count.
__device__ int gather_p(const sssd_ds& ds, const KCfg& c, int p, uint64_t lo, uint64_t hi,
                        uint32_t* tab, uint8_t* lens, int64_t* samples, uint32_t* srows) {
  const int lane = lane_id();
  const uint64_t w = hi - lo;
  const int s = (int)min(w, (uint64_t)c.M);
  uint32_t* ptab = tab + (size_t)(p - 1) * c.M * c.BL;
  uint8_t* plen = lens + (size_t)(p - 1) * c.M;
  uint32_t* srow = srows + lane * kRowStride;
  int cnt = 0;
  for (int k0 = 0; k0 < s; k0 += 32) {
    const int k = k0 + lane;
    const bool valid = k < s;
    uint32_t len = 0, pos = 0;
    if (valid) {
      const uint64_t r =
          lo + (w <= (uint64_t)c.M ? (uint64_t)k : ((uint64_t)k * w) / (uint64_t)c.M);
      const uint4* row = reinterpret_cast<const uint4*>(ds.rows) + (r - ds.rank_base) * 4;
      uint4* sr = reinterpret_cast<uint4*>(srow);
      sr[0] = ldg4(row);
      sr[1] = ldg4(row + 1);
      sr[2] = ldg4(row + 2);
      sr[3] = ldg4(row + 3);
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
      uint32_t* dst = ptab + (size_t)idx * c.BL;
      for (uint32_t j = 0; j < len; ++j)
        dst[j] = (p + j < SSSD_ROW_TOKENS) ? srow[1 + p + j] : __ldg(ds.tokens + start + j);
      plen[idx] = (uint8_t)len;
    }
    cnt += __popc(bal);
    __syncwarp();
  }
  return cnt;
}

__global__ void __launch_bounds__(32 * SSSD_MAX_P)
    ds_lookup_kernel(sssd_ds ds, sssd_seqs seqs, KCfg c, uint32_t* ds_tab, uint8_t* ds_len,
                     sssd_elem* ds_el, int32_t* ds_n, sssd_lookup_out lk, sssd_elem* ds_raw,
                     uint32_t* ds_idx, int64_t idx_cap) {
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  __shared__ uint32_t s_pat[SSSD_MAX_P];
  __shared__ uint64_t s_lo[SSSD_MAX_P], s_hi[SSSD_MAX_P];
  __shared__ int s_cnt[SSSD_MAX_P];
  __shared__ __align__(16) uint32_t s_rows[SSSD_MAX_P * 32 * kRowStride];

  const int L = seqs.seq_len[b];
  const uint32_t* seq = seqs.seq + seqs.seq_off[b];
  const int pmax = min(c.P, L);
  if (threadIdx.x < pmax) s_pat[threadIdx.x] = seq[L - pmax + threadIdx.x];
  __syncthreads();

  const int p = warp + 1;
  if (p <= pmax) {
    uint64_t lo, hi;
    warp_bounds(ds, s_pat + (pmax - p), p, lo, hi);
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

  uint32_t* tab = ds_tab + (size_t)b * c.P * c.M * c.BL;
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
      const int n = gather_p(ds, c, p, s_lo[warp], s_hi[warp], tab, lens,
                             smp ? smp + (size_t)warp * c.M : nullptr, s_rows + warp * 32 * kRowStride);
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
  if (c.has_sep) {
    sssd_elem* raw = ds_raw + (size_t)b * c.P * c.M;
    if (p >= pcut && p <= pmax) {
      for (int i = lane; i < s_cnt[warp]; i += 32) {
        sssd_elem e;
        e.off = (uint32_t)(((size_t)(p - 1) * c.M + i) * c.BL);
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
      uint32_t* idx = (n <= SSSD_MAX_P * 32 * kRowStride) ? s_rows : ds_idx + (size_t)b * idx_cap;
      block_sort_elems(raw, ds_el + (size_t)b * c.P * c.M, tab, n, idx);
    }
  } else if (p >= pcut && p <= pmax) {
    const int cnt = s_cnt[warp];
    for (int i = lane; i < cnt; i += 32) {
      const uint32_t* si = tab + ((size_t)(p - 1) * c.M + i) * c.BL;
      const uint32_t li = lens[(size_t)(p - 1) * c.M + i];
      int rank = i;
      for (int q = pcut; q <= pmax; ++q) {
        if (q == p) continue;
        const int cq = s_cnt[q - 1];
        int a = 0, z = cq;  // first element of run q that comes after string i
        while (a < z) {
          const int mid = (a + z) >> 1;
          const int r = cmp_str(tab + ((size_t)(q - 1) * c.M + mid) * c.BL,
                                lens[(size_t)(q - 1) * c.M + mid], si, li);
          const bool before_i = q > p ? r <= 0 : r < 0;
          if (before_i) a = mid + 1; else z = mid;
        }
        rank += a;
      }
      sssd_elem e;
      e.off = (uint32_t)(((size_t)(p - 1) * c.M + i) * c.BL);
      e.orig = (uint32_t)(before + i);
      e.len_m = li | (255u << 8);
      e.pad = 0;
      ds_el[(size_t)b * c.P * c.M + rank] = e;
    }
  }
  if (threadIdx.x == 0) {
    int n = 0;
    for (int q = pcut; q <= pmax; ++q) n += s_cnt[q - 1];
    ds_n[b] = n;
    if (lk.p_cut) lk.p_cut[b] = pmax > 0 ? pcut : 0;
  }
  if (lk.n_conts && threadIdx.x < c.P) {
    const int q = threadIdx.x + 1;
    lk.n_conts[(size_t)b * c.P + threadIdx.x] = (q <= pmax && s_cnt[threadIdx.x] >= 0) ? s_cnt[threadIdx.x] : -1;
  }
}

// --------------------------------------------------------------------------
// K4: input scan (ref input_cache.py:88-121, stateless form A.4)
// --------------------------------------------------------------------------

constexpr int kSortSmem = 4096;

__global__ void __launch_bounds__(256)
    input_scan_kernel(sssd_seqs seqs, KCfg c, sssd_elem* raw, sssd_elem* sorted, int32_t* in_n,
                      uint32_t* idx_ws, int64_t cap, int64_t cap2) {
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  __shared__ uint32_t s_tail[SSSD_MAX_P];
  __shared__ int s_wsum[8];
  __shared__ uint32_t s_idx[kSortSmem];
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
  int base = 0;
  for (int e0 = 1; e0 < L; e0 += blockDim.x) {
    const int e = e0 + tid;
    int m = 0;
    if (e < L) {
      const int lim = min(jm, e);
      while (m < lim && seq[e - 1 - m] == s_tail[m]) ++m;
    }
    const bool f = m > 0;
    const uint32_t bal = __ballot_sync(SSSD_FULL, f);
    if (lane == 0) s_wsum[warp] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (w < warp) off += s_wsum[w];
      tot += s_wsum[w];
    }
    if (f) {
      sssd_elem el;
      el.off = (uint32_t)e;
      el.orig = (uint32_t)e;
      el.len_m = (uint32_t)min(c.IBL, L - e) | ((uint32_t)m << 8);
      el.pad = 0;
      r[base + off + __popc(bal & lanemask_lt())] = el;
    }
    base += tot;
    __syncthreads();
  }
  if (tid == 0) in_n[b] = base;
  sssd_elem* out = sorted + (size_t)b * cap;
  if (base == 0) return;
  uint32_t* idx = (base <= kSortSmem) ? s_idx : idx_ws + (size_t)b * cap2;
  block_sort_elems(r, out, seq, base, idx);
}

// Sort caller-provided source paths (sssd_merge): one CTA per (request, source).
__global__ void __launch_bounds__(256)
    sort_sources_kernel(const uint32_t* tok, const sssd_elem* el, const int64_t* el_off,
                        const int32_t* el_n, sssd_elem* sorted, uint32_t* idx_ws, int64_t idx_cap) {
  __shared__ uint32_t s_idx[kSortSmem];
  const int bs = blockIdx.x;
  const int n = el_n[bs];
  if (n <= 0) return;
  const int64_t o = el_off[bs];
  uint32_t* idx = (n <= kSortSmem) ? s_idx : idx_ws + o * 2;  // idx_ws holds 2*total entries
  (void)idx_cap;
  block_sort_elems(el + o, sorted + o, tok, n, idx);
}

// --------------------------------------------------------------------------
// K5: fusion + flatten (ref fusion.py:209-261, draft.py:67-86; A.5, A.6)
// --------------------------------------------------------------------------

struct Child {  // one candidate of a sibling group (32 B, global arena)
  double pp;       // path probability (ref fusion.py:244,259)
  uint32_t first;  // first-appearance position = reference child order
  uint32_t count;  // node count in its source trie
  uint32_t token;
  uint32_t a, b;   // element range [a, b) of the node in the source array
  uint32_t pad;
};

struct Group {  // sibling group header (40 B, shared memory)
  double prio;    // head priority
  Child* ch;
  uint32_t first;  // head first-appearance
  int32_t head;    // head child index, -1 when exhausted
  uint32_t nch;
  uint32_t meta;     // depth << 26 | rank << 22 | sequence
  uint32_t dparent;  // draft node the children hang under
  uint32_t pad;
};

__device__ __forceinline__ uint32_t g_depth(uint32_t meta) { return meta >> 26; }
__device__ __forceinline__ uint32_t g_rank(uint32_t meta) { return (meta >> 22) & 0xf; }

struct Arena {
  Child* slab;
  uint32_t used, cap;
  Child* pool;
  unsigned long long* cursor;
  uint64_t pool_cap;
  int32_t* err;
  __device__ Child* alloc(uint32_t n) {  // warp-uniform
    if (used + n <= cap) {
      Child* p = slab + used;
      used += n;
      return p;
    }
    unsigned long long at = 0;
    if (lane_id() == 0) at = atomicAdd(cursor, (unsigned long long)n);
    at = __shfl_sync(SSSD_FULL, at, 0);
    if (at + n > pool_cap) {
      if (lane_id() == 0) atomicExch(err, SSSD_E_WORKSPACE);
      return nullptr;
    }
    return pool + at;
  }
  // return the unused tail [p + keep, p + n) of the latest slab allocation
  __device__ void shrink(Child* p, uint32_t n, uint32_t keep) {
    if (p + n == slab + used) used -= n - keep;
  }
};

// better(a, b): higher priority first, then smaller first-appearance (ticket)
__device__ __forceinline__ bool child_better(double pa, uint32_t fa, double pb, uint32_t fb) {
  return pa > pb || (pa == pb && fa < fb);
}

__device__ __forceinline__ void warp_best(double& p, uint32_t& f, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double op = __shfl_xor_sync(SSSD_FULL, p, o);
    const uint32_t of = __shfl_xor_sync(SSSD_FULL, f, o);
    const int oi = __shfl_xor_sync(SSSD_FULL, i, o);
    if (oi >= 0 && (i < 0 || child_better(op, of, p, f))) {
      p = op;
      f = of;
      i = oi;
    }
  }
}

// Expand the node covering [a, z) of source sd at depth D-1 into the sibling
// group of its depth-D children (sub-runs by token index D-1).  Creates a
// group (appended at *G) when the node has at least one child.
__device__ void expand(const SrcDesc& sd, uint32_t rank, uint32_t D, uint32_t a, uint32_t z,
                       bool seed, double ppar, uint32_t pcount, uint32_t dparent, double disc,
                       Group* groups, int& G, Arena& ar) {
  const int lane = lane_id();
  Child* ch = ar.alloc(z - a);
  if (!ch) return;
  uint32_t nch = 0;
  double bp = -1.0;
  uint32_t bf = 0xffffffffu;
  int bi = -1;
  bool c_open = false;
  uint32_t c_tok = 0, c_cnt = 0, c_first = 0xffffffffu, c_start = 0;
  const double dpc = (double)pcount;

  auto emit = [&](bool pred, uint32_t tok, uint32_t cnt, uint32_t first, uint32_t s, uint32_t e) {
    const bool live = pred && cnt > 0;
    const uint32_t bal = __ballot_sync(SSSD_FULL, live);
    if (live) {
      const uint32_t k = nch + __popc(bal & lanemask_lt());
      const double ratio = __ddiv_rn((double)cnt, dpc);
      const double pp = seed ? ratio : __dmul_rn(ppar, ratio);
      const double pr = __dmul_rn(pp, disc);
      Child cc;
      cc.pp = pp;
      cc.first = first;
      cc.count = cnt;
      cc.token = tok;
      cc.a = s;
      cc.b = e;
      cc.pad = 0;
      ch[k] = cc;
      if (bi < 0 || child_better(pr, first, bp, bf)) {
        bp = pr;
        bf = first;
        bi = (int)k;
      }
    }
    nch += __popc(bal);
  };

  for (uint32_t base = a; base < z; base += 32) {
    const uint32_t i = base + lane;
    bool has = false;
    uint32_t t = 0, wgt = 0, orig = 0xffffffffu;
    if (i < z) {
      const sssd_elem e = sd.el[i];
      if (el_len(e.len_m) >= D) {
        has = true;
        t = sd.tok[e.off + D - 1];
        if ((int)el_m(e.len_m) >= sd.thr) {
          wgt = 1;
          orig = e.orig;
        }
      }
    }
    const uint32_t hasm = __ballot_sync(SSSD_FULL, has);
    if (!hasm) continue;
    const uint32_t tprev = __shfl_up_sync(SSSD_FULL, t, 1);
    bool head;
    if (lane == 0) head = has && !(c_open && c_tok == t);
    else head = has && (!((hasm >> (lane - 1)) & 1u) || tprev != t);
    const uint32_t headm = __ballot_sync(SSSD_FULL, head);
    // a pending carry run ends where this chunk starts a new run
    if (c_open && (headm & 1u)) {
      emit(lane == 0, c_tok, c_cnt, c_first, c_start, base);
      c_open = false;
    }
    const uint32_t le = headm & (lanemask_lt() | (1u << lane));
    const int seg = le ? 31 - __clz(le) : -1;
    uint32_t cnt = wgt, fm = orig;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t oc = __shfl_up_sync(SSSD_FULL, cnt, o);
      const uint32_t of = __shfl_up_sync(SSSD_FULL, fm, o);
      if (lane >= o && lane - o >= seg) {
        cnt += oc;
        fm = min(fm, of);
      }
    }
    uint32_t start = base + (seg < 0 ? 0 : seg);
    if (seg < 0) {  // continuation of the carried run
      cnt += c_cnt;
      fm = min(fm, c_first);
      start = c_start;
    }
    const bool nxt_has = lane < 31 ? ((hasm >> (lane + 1)) & 1u) : false;
    const bool nxt_head = lane < 31 ? ((headm >> (lane + 1)) & 1u) : false;
    const bool tail = has && (lane == 31 || !nxt_has || nxt_head);
    const bool open = tail && lane == 31 && i + 1 < z;
    emit(tail && !open, t, cnt, fm, start, i + 1);
    const uint32_t ob = __ballot_sync(SSSD_FULL, open);
    if (ob) {
      c_tok = __shfl_sync(SSSD_FULL, t, 31);
      c_cnt = __shfl_sync(SSSD_FULL, cnt, 31);
      c_first = __shfl_sync(SSSD_FULL, fm, 31);
      c_start = __shfl_sync(SSSD_FULL, start, 31);
      c_open = true;
    } else {
      c_open = false;
    }
  }
  if (c_open) emit(lane == 0, c_tok, c_cnt, c_first, c_start, z);
  ar.shrink(ch, z - a, nch);
  if (nch == 0) return;
  warp_best(bp, bf, bi);
  if (lane == 0) {
    Group g;
    g.prio = bp;
    g.ch = ch;
    g.first = bf;
    g.head = bi;
    g.nch = nch;
    g.meta = (D << 26) | (rank << 22) | (uint32_t)G;
    g.dparent = dparent;
    g.pad = 0;
    groups[G] = g;
  }
  ++G;
  __syncwarp();
}

__global__ void __launch_bounds__(32)
    draft_kernel(const SrcDesc* desc, const uint32_t* root_tok, KCfg c, Child* slabs,
                 uint32_t slab_cap, Child* pool, unsigned long long* cursor, uint64_t pool_cap,
                 int32_t* err, sssd_draft_out out) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int b = blockIdx.x;
  const int lane = lane_id();
  const int S = c.S;
  const int W = (S + 63) >> 6;
  const int Gmax = (c.P + 1) * S + c.P + 1;
  Group* groups = reinterpret_cast<Group*>(smem);
  uint32_t* d_tok = reinterpret_cast<uint32_t*>(groups + Gmax);
  int16_t* d_par = reinterpret_cast<int16_t*>(d_tok + S);
  int16_t* d_fc = d_par + S;
  int16_t* d_ns = d_fc + S;
  int16_t* d_lc = d_ns + S;
  int16_t* d_dep = d_lc + S;
  int16_t* pre = d_dep + S;
  int16_t* n2p = pre + S;
  int16_t* stk = n2p + S;

  Arena ar{slabs + (size_t)b * slab_cap, 0, slab_cap, pool, cursor, pool_cap, err};
  if (lane == 0) {
    d_tok[0] = root_tok[b];
    d_par[0] = -1;
    d_fc[0] = d_ns[0] = d_lc[0] = -1;
    d_dep[0] = 0;
  }
  __syncwarp();
  int G = 0;
  int size = 1;
  const SrcDesc* sds = desc + (size_t)b * (c.P + 1);

  // Seeds: datastore (rank 0), then input trees p = n_trees..1 (rank P-p+1).
  if (S > 1) {
    for (int rk = 0; rk <= c.P; ++rk) {
      const SrcDesc sd = sds[rk];
      if (sd.n <= 0) continue;
      uint32_t rc = 0;
      for (int i = lane; i < sd.n; i += 32) rc += (int)el_m(sd.el[i].len_m) >= sd.thr ? 1u : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rc += __shfl_xor_sync(SSSD_FULL, rc, o);
      if (rc == 0) continue;
      expand(sd, rk, 1, 0, sd.n, true, 0.0, rc, 0, c.disc[rk * c.disc_stride + 1], groups, G, ar);
    }
  }

  while (size < S) {
    // pop: min over group heads of (-prio, depth, rank, sequence)
    double bp = -1.0;
    uint32_t bm = 0xffffffffu;
    int bg = -1;
    for (int gi = lane; gi < G; gi += 32) {
      const Group& g = groups[gi];
      if (g.head < 0) continue;
      if (bg < 0 || g.prio > bp || (g.prio == bp && g.meta < bm)) {
        bp = g.prio;
        bm = g.meta;
        bg = gi;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double op = __shfl_xor_sync(SSSD_FULL, bp, o);
      const uint32_t om = __shfl_xor_sync(SSSD_FULL, bm, o);
      const int og = __shfl_xor_sync(SSSD_FULL, bg, o);
      if (og >= 0 && (bg < 0 || op > bp || (op == bp && om < bm))) {
        bp = op;
        bm = om;
        bg = og;
      }
    }
    if (bg < 0) break;
    const Group g = groups[bg];
    const Child h = g.ch[g.head];
    const uint32_t D = g_depth(g.meta), rk = g_rank(g.meta);
    const double dsc = c.disc[rk * c.disc_stride + D];
    // draft insert: an existing (parent, token) keeps the first node (ref fusion.py:185-198)
    const int par = (int)g.dparent;
    int found = -1;
    for (int i0 = 1; i0 < size; i0 += 32) {
      const int i = i0 + lane;
      const bool hit = i < size && d_par[i] == par && d_tok[i] == h.token;
      const uint32_t hb = __ballot_sync(SSSD_FULL, hit);
      if (hb) {
        found = i0 + __ffs(hb) - 1;
        break;
      }
    }
    int nid = found;
    if (found < 0) {
      nid = size++;
      if (lane == 0) {
        d_tok[nid] = h.token;
        d_par[nid] = (int16_t)par;
        d_fc[nid] = d_ns[nid] = d_lc[nid] = -1;
        d_dep[nid] = (int16_t)(d_dep[par] + 1);
        if (d_lc[par] < 0) d_fc[par] = (int16_t)nid;
        else d_ns[d_lc[par]] = (int16_t)nid;
        d_lc[par] = (int16_t)nid;
      }
    }
    // advance the popped group's head: best child strictly after (h.prio, h.first)
    {
      const double hp = __dmul_rn(h.pp, dsc);
      double np = -1.0;
      uint32_t nf = 0xffffffffu;
      int ni = -1;
      for (uint32_t k = lane; k < g.nch; k += 32) {
        const Child ck = g.ch[k];
        const double pk = __dmul_rn(ck.pp, dsc);
        if (child_better(hp, h.first, pk, ck.first) && (ni < 0 || child_better(pk, ck.first, np, nf))) {
          np = pk;
          nf = ck.first;
          ni = (int)k;
        }
      }
      warp_best(np, nf, ni);
      if (lane == 0) {
        groups[bg].head = ni;
        groups[bg].prio = np;
        groups[bg].first = nf;
      }
    }
    __syncwarp();
    // push the popped source node's children (ref fusion.py:258-259)
    if (h.b - h.a > 0) {
      const SrcDesc sd = sds[rk];
      if (D + 1 < (uint32_t)c.disc_stride)
        expand(sd, rk, D + 1, h.a, h.b, false, h.pp, h.count, (uint32_t)nid,
               c.disc[rk * c.disc_stride + D + 1], groups, G, ar);
    }
    __syncwarp();
  }

  // DFS pre-order flatten, children in insertion order (ref draft.py:67-86)
  if (lane == 0) {
    int sp = 0, k = 0;
    stk[sp++] = 0;
    while (sp > 0) {
      const int nid = stk[--sp];
      pre[k] = (int16_t)nid;
      n2p[nid] = (int16_t)k;
      ++k;
      int cnt = 0;
      for (int ch = d_fc[nid]; ch >= 0; ch = d_ns[ch]) ++cnt;
      int j = 0;
      for (int ch = d_fc[nid]; ch >= 0; ch = d_ns[ch], ++j) stk[sp + cnt - 1 - j] = (int16_t)ch;
      sp += cnt;
    }
  }
  __syncwarp();
  uint32_t* o_tok = out.tokens + (size_t)b * S;
  int32_t* o_par = out.parents + (size_t)b * S;
  int32_t* o_dep = out.depths + (size_t)b * S;
  uint64_t* o_mask = out.mask + (size_t)b * S * W;
  for (int k = lane; k < S; k += 32) {
    if (k < size) {
      const int nid = pre[k];
      o_tok[k] = d_tok[nid];
      o_par[k] = nid == 0 ? -1 : (int32_t)n2p[d_par[nid]];
      o_dep[k] = d_dep[nid];
      uint64_t mw[SSSD_MAX_DRAFT / 64] = {0, 0, 0, 0};
      for (int x = nid; x >= 0; x = d_par[x]) {
        const int pk = n2p[x];
        mw[pk >> 6] |= 1ull << (pk & 63);
      }
      for (int w = 0; w < W; ++w) o_mask[(size_t)k * W + w] = mw[w];
    } else {
      o_tok[k] = 0;
      o_par[k] = -1;
      o_dep[k] = -1;
      for (int w = 0; w < W; ++w) o_mask[(size_t)k * W + w] = 0;
    }
  }
  if (lane == 0) out.size[b] = size;
}

}  // namespace sssd
