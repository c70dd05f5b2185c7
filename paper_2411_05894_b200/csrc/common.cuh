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

}  // namespace sssd
