// Shared device helpers for libsssd (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "sssd.h"

#define SSSD_FULL 0xffffffffu

namespace sssd {

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint4 ldg4(const uint4* p) { return __ldg(p); }

__device__ __forceinline__ uint32_t el_len(uint32_t len_m) { return len_m & 0xffu; }
__device__ __forceinline__ uint32_t el_m(uint32_t len_m) { return (len_m >> 8) & 0xffu; }
// column meta words carry a multiplicity in bits 16..31 (0 = 1): identical
// datastore continuations folded into one element (level-synchronous fusion)
__device__ __forceinline__ uint32_t el_wt(uint32_t meta) { return max(meta >> 16, 1u); }

// Lexicographic compare of two token strings with "shorter sorts first"
// (a proper prefix precedes its extensions; ref datastore.py:129-141 and the
// continuation-list order of A.3/A.4).  Returns -1/0/+1.
__device__ __forceinline__ int cmp_str(const uint32_t* a, uint32_t la, const uint32_t* b,
                                       uint32_t lb) {
  const uint32_t l = la < lb ? la : lb;
  for (uint32_t j = 0; j < l; ++j) {
    const uint32_t x = a[j], y = b[j];
    if (x != y) return x < y ? -1 : 1;
  }
  return la < lb ? -1 : (la > lb ? 1 : 0);
}

// cmp_str for 16-byte aligned rows whose allocation extends to a multiple of 4
// tokens (the gathered continuation table, KCfg::TS): 4 tokens per load, so a
// long common prefix costs ceil(l / 4) dependent loads instead of l.
__device__ __forceinline__ int cmp_row16(const uint32_t* a, uint32_t la, const uint32_t* b, uint32_t lb) {
  const uint32_t l = la < lb ? la : lb;
  for (uint32_t j = 0; j < l; j += 4) {
    const uint4 x = *reinterpret_cast<const uint4*>(a + j), y = *reinterpret_cast<const uint4*>(b + j);
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (uint32_t k = 0; k < 4; ++k)
      if (j + k < l && xs[k] != ys[k]) return xs[k] < ys[k] ? -1 : 1;
  }
  return la < lb ? -1 : (la > lb ? 1 : 0);
}

// Depth-major columns of one sorted source array (the fusion kernel's input):
// element i's metadata, insertion position and token at depth d live at
// meta[i], orig[i], tok[d * stride + i], so the lanes of a warp expanding a
// trie node read 3 coalesced, mutually independent words per element.
struct Cols {
  uint32_t* meta;  // len | m << 8
  uint32_t* orig;
  uint32_t* tok;
  int64_t stride;
};

__device__ __forceinline__ void write_cols(const Cols& c, int64_t i, const sssd_elem& e,
                                           const uint32_t* tokbuf) {
  const uint32_t len = el_len(e.len_m);
  c.meta[i] = e.len_m & 0xffffu;
  c.orig[i] = e.orig;
  for (uint32_t d = 0; d < len; ++d) c.tok[d * c.stride + i] = tokbuf[e.off + d];
}

// Per-(request, source) view used by the fusion kernel: n sorted elements in
// columns; an element counts toward this source's tree when its backward-match
// length m >= thr (input tree p: thr = p; datastore and caller trees: thr = 0).
struct SrcDesc {
  const uint32_t* meta;
  const uint32_t* orig;
  const uint32_t* tok;
  int64_t stride;
  int32_t n;
  int32_t thr;
  int32_t depth;  // token columns (no element is longer): nodes at this depth have no children
  int32_t pad;
};

// cnt / pc as the correctly rounded double (bit-identical to __ddiv_rn) for
// integers below 2^24, in 8 instructions instead of __ddiv_rn's 14 with a
// range check: a float reciprocal refined once in double (relative error
// < 2^-44), q0 = RN(cnt * r), the exact fma residual cnt - q0 * pc and one
// correction fma.  The quotient of two integers below 2^24 is never a rounding
// midpoint and lies at least ulp / 2^25 from one, far beyond the corrected
// value's error (< 2^-40 ulp), so the final rounding is RN(cnt / pc).
// Larger operands take __ddiv_rn.  (Checked against exact rational fma
// arithmetic on 120k operand pairs with the float reciprocal perturbed by
// +-1 ulp; the fusion's priorities are pinned to the oracle by the GPU tests.)
__device__ __forceinline__ double ratio_rn(uint32_t cnt, uint32_t pc) {
  if ((cnt | pc) >= (1u << 24)) return __ddiv_rn((double)cnt, (double)pc);
  const double x = (double)cnt, y = (double)pc;
  float rf;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rf) : "f"((float)pc));
  const double r0 = (double)rf;
  const double r = __fma_rn(r0, __fma_rn(-y, r0, 1.0), r0);
  const double q0 = __dmul_rn(x, r);
  return __fma_rn(__fma_rn(-q0, y, x), r, q0);
}

// k-gram range index (sssd_kix_build): 64-bit hash of (k, t[0..k)), never 0
// (0 marks an empty slot).
__host__ __device__ __forceinline__ uint64_t kix_hash(const uint32_t* t, int k) {
  uint64_t h = 0x9E3779B97F4A7C15ull * (uint64_t)(k + 1);
  for (int j = 0; j < k; ++j) {
    h ^= t[j];
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 32;
  }
  h ^= h >> 29;
  h *= 0xc4ceb9fe1a85ec53ull;
  h ^= h >> 32;
  return h | 1ull;
}

// The table covers the whole corpus (not an SA-range shard, whose absent
// patterns still need their local insertion points for the summed bounds).
__device__ __forceinline__ bool kix_whole(const sssd_ds& ds) { return ds.rank_base == 0 && ds.n_rows == ds.n_tokens; }

// Rows [lo, hi) whose suffix starts with pat[0..k) (2 <= k <= ds.kix_kmax):
// returns 1 (found, lo / hi set), 0 (no suffix starts with the k-gram: the
// range is empty, its insertion point unknown) or -1 (the slot of this hash
// belongs to another k-gram -- a 64-bit collision: search instead).
__device__ __forceinline__ int kix_find(const sssd_ds& ds, const uint32_t* pat, int k, uint64_t& lo, uint64_t& hi) {
  const uint64_t h = kix_hash(pat, k);
  const uint4* tab = reinterpret_cast<const uint4*>(ds.kix);
  for (uint64_t s = h & ds.kix_mask;; s = (s + 1) & ds.kix_mask) {
    const uint4 e = __ldg(tab + s);
    const uint64_t key = (uint64_t)e.y << 32 | e.x;
    if (key == 0) return 0;
    if (key == h) {
      const uint32_t* row = ds.rows + (uint64_t)e.z * 16;  // verify: row lo starts with the k-gram
      if (ds.n_tokens - row[0] < (uint64_t)k) return -1;
      for (int j = 0; j < k; ++j)
        if (row[1 + j] != pat[j]) return -1;
      lo = e.z;
      hi = e.w;
      return 1;
    }
  }
}

}  // namespace sssd
