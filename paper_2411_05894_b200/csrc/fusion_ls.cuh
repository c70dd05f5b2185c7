// Level-synchronous fusion: shared level / parent / top-list records and the
// warp sort, used by the one-warp kernels (fusion_ls.cu) and the CTA-per-request
// kernel (fusion_cta.cu).  Algorithm: fusion_ls.cu header, DESIGN.md 3.1.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "propose.cuh"

namespace sssd {

// the level phases are inlined: as separate calls (__noinline__) the kernel
// spilled across them and took 0.515 instead of 0.485 ms per cfg2 step
#ifndef SSSD_LS_CALL
#define SSSD_LS_CALL __forceinline__
#endif

// One level's nodes, structure of arrays over one base pointer (fields are
// recomputed from (base, cap), which keeps them out of registers).
// k0/k1/ord/tbr/pid are indexed by sorted position, pp/a/z/cnt/tok/ppid by
// generation index (ord maps).
//   k0  ~bits(priority)
//   k1  rank<<56 | parent tb<<32 | first; path key ppid<<32 | tok after the class pass
//   pp  path probability (ref fusion.py:244,259)
//   tbr rank << 22 | class position tb;  pid: path id (0 = the root path)
struct LsLevel {
  uint8_t* p;
  uint32_t cap;
  __device__ __forceinline__ uint64_t* k0() const { return reinterpret_cast<uint64_t*>(p); }
  __device__ __forceinline__ uint64_t* k1() const { return reinterpret_cast<uint64_t*>(p) + cap; }
  __device__ __forceinline__ double* pp() const { return reinterpret_cast<double*>(p) + 2 * cap; }
  __device__ __forceinline__ uint32_t* f(int i) const {
    return reinterpret_cast<uint32_t*>(reinterpret_cast<double*>(p) + 3 * cap) + i * cap;
  }
  __device__ __forceinline__ uint32_t* a() const { return f(0); }
  __device__ __forceinline__ uint32_t* z() const { return f(1); }
  __device__ __forceinline__ uint32_t* cnt() const { return f(2); }
  __device__ __forceinline__ uint32_t* tok() const { return f(3); }
  __device__ __forceinline__ uint32_t* ppid() const { return f(4); }
  __device__ __forceinline__ uint32_t* ord() const { return f(5); }
  __device__ __forceinline__ uint32_t* tbr() const { return f(6); }
  __device__ __forceinline__ uint32_t* pid() const { return f(7); }
};
static_assert(kLsLevelBytes == 3 * 8 + 8 * 4, "level record");

__device__ __forceinline__ LsLevel level_carve(uint8_t* p, uint32_t cap) { return LsLevel{p, cap}; }

// The expanded prefix of the previous level (the parents of this level);
// off = exclusive scan of the element-range sizes.
struct LsPar {
  uint8_t* p;
  uint32_t cap;
  __device__ __forceinline__ double* pp() const { return reinterpret_cast<double*>(p); }
  __device__ __forceinline__ uint32_t* f(int i) const {
    return reinterpret_cast<uint32_t*>(reinterpret_cast<double*>(p) + cap) + i * cap;
  }
  __device__ __forceinline__ uint32_t* a() const { return f(0); }
  __device__ __forceinline__ uint32_t* z() const { return f(1); }
  __device__ __forceinline__ uint32_t* cnt() const { return f(2); }
  __device__ __forceinline__ uint32_t* tbr() const { return f(3); }
  __device__ __forceinline__ uint32_t* pid() const { return f(4); }
  __device__ __forceinline__ uint32_t* off() const { return f(5); }
};
static_assert(kLsParBytes == 8 + 6 * 4, "parent record");

__device__ __forceinline__ LsPar par_carve(uint8_t* p, uint32_t cap) { return LsPar{p, cap}; }

// Running top list: the best (dec_len-1) distinct paths in G order;
// g1 = depth << 26 | rank << 22 | tb.
struct LsTop {
  uint8_t* p;
  int S;
  __device__ __forceinline__ uint64_t* g0() const { return reinterpret_cast<uint64_t*>(p); }
  __device__ __forceinline__ uint32_t* f(int i) const {
    return reinterpret_cast<uint32_t*>(reinterpret_cast<uint64_t*>(p) + S) + i * S;
  }
  __device__ __forceinline__ uint32_t* g1() const { return f(0); }
  __device__ __forceinline__ uint32_t* pid() const { return f(1); }
  __device__ __forceinline__ uint32_t* tok() const { return f(2); }
  __device__ __forceinline__ uint32_t* ppid() const { return f(3); }
};

__device__ __forceinline__ LsTop top_carve(uint8_t* p, int S) { return LsTop{p, S}; }

__device__ __forceinline__ bool g_less(uint64_t a0, uint32_t a1, uint64_t b0, uint32_t b1) {
  return a0 < b0 || (a0 == b0 && a1 < b1);
}
__device__ __forceinline__ bool k_less(uint64_t a0, uint64_t a1, uint64_t b0, uint64_t b1) {
  return a0 < b0 || (a0 == b0 && a1 < b1);
}

constexpr uint32_t kTbBits = 22;
constexpr uint32_t kTbMask = (1u << kTbBits) - 1;

// Lane bounds [lo, hi] of this lane's run of equal (parent j, token) keys in a
// generation chunk.  Runs are lane intervals (a parent's elements are sorted
// by their depth-d token; lanes without an element are runs of one), so a run
// starts where the key differs from the previous lane's: one ballot of the run
// heads (measured 2 % faster at cfg2 than __match_any_sync on the 64-bit key).
__device__ __forceinline__ void run_bounds(bool has, uint32_t j, uint32_t tk, int& lo_l, int& hi_l) {
  const int lane = lane_id();
  const uint32_t kj = has ? j : 0xffffffffu, kt = has ? tk : (uint32_t)lane;
  const uint32_t pj = __shfl_up_sync(SSSD_FULL, kj, 1), pt = __shfl_up_sync(SSSD_FULL, kt, 1);
  const uint32_t heads = __ballot_sync(SSSD_FULL, lane == 0 || !has || pj != kj || pt != kt);
  const uint32_t le = lanemask_lt() | (1u << lane), above = heads & ~le;
  lo_l = 31 - __clz(heads & le);
  hi_l = above ? __ffs(above) - 2 : 31;
}

__host__ __device__ inline int top_bytes(int S) { return (S * 24 + 15) / 16 * 16; }


// Bump-allocate `bytes` from the fusion pool (warp-uniform); nullptr + status
// word on exhaustion.
__device__ __forceinline__ uint8_t* pool_take(uint8_t* pool, unsigned long long* cursor, uint64_t pool_bytes,
                                              int32_t* err, unsigned long long bytes) {
  unsigned long long at = 0;
  if (lane_id() == 0) at = atomicAdd(cursor, bytes);
  at = __shfl_sync(SSSD_FULL, at, 0);
  if (at + bytes > pool_bytes) {
    if (lane_id() == 0) atomicExch(err, SSSD_E_WORKSPACE);
    return nullptr;
  }
  return pool + at;
}

// Sort positions [0, n) by (k0, k1), carrying ord (n <= 32: ranks in
// registers; otherwise a bitonic network).
__device__ SSSD_LS_CALL void ls_sort(LsLevel L, uint32_t n) {
  const int lane = lane_id();
  if (n <= 32) {
    uint64_t m0 = ~0ull, m1 = ~0ull;
    if (lane < (int)n) {
      m0 = L.k0()[lane];
      m1 = L.k1()[lane];
    }
    uint32_t r = 0;
    for (uint32_t q = 0; q < n; ++q) {
      const uint64_t q0 = __shfl_sync(SSSD_FULL, m0, q), q1 = __shfl_sync(SSSD_FULL, m1, q);
      r += k_less(q0, q1, m0, m1) ? 1u : 0u;
    }
    __syncwarp();
    if (lane < (int)n) {
      L.k0()[r] = m0;
      L.k1()[r] = m1;
      L.ord()[r] = (uint32_t)lane;
    }
    __syncwarp();
    return;
  }
  // bitonic network in its all-ascending form (each merge starts by
  // comparing i with the mirror position of its block), so positions >= n act
  // as +infinity without being stored: a comparator reaching past n is a no-op
  uint32_t N2 = 64;
  while (N2 < n) N2 <<= 1;
  for (uint32_t lk = 1; (1u << lk) <= N2; ++lk) {
    const uint32_t kk = 1u << lk;
    for (int lj = (int)lk - 1; lj >= 0; --lj) {
      const uint32_t jj = 1u << lj;
      for (uint32_t p = lane; p < N2 / 2; p += 32) {
        const uint32_t pb = p >> lj, pr = p & (jj - 1);
        uint32_t lo, hi;
        if (lj == (int)lk - 1) {
          lo = (pb << lk) + pr;
          hi = (pb << lk) + kk - 1 - pr;
        } else {
          lo = (pb << (lj + 1)) + pr;
          hi = lo + jj;
        }
        if (hi >= n) continue;
        const uint64_t a0 = L.k0()[lo], a1 = L.k1()[lo], b0 = L.k0()[hi], b1 = L.k1()[hi];
        if (k_less(b0, b1, a0, a1)) {
          const uint32_t oa = L.ord()[lo], ob = L.ord()[hi];
          L.k0()[lo] = b0;
          L.k1()[lo] = b1;
          L.ord()[lo] = ob;
          L.k0()[hi] = a0;
          L.k1()[hi] = a1;
          L.ord()[hi] = oa;
        }
      }
      __syncwarp();
    }
  }
}

}  // namespace sssd
