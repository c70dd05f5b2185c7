// Tree-attention verification on B200: tcgen05.mma (kind::f16, bf16 inputs,
// fp32 accumulators in TMEM) fed by TMA.  Semantics of ref draft.py:205-210 —
// every draft node i attends to the committed prefix [0, ctx) and to its
// ancestors-or-self among the S tree keys [ctx, ctx + S) (u64 ancestor rows
// from the fusion kernel), so one forward gives all s_q greedy predictions.
//
// One CTA = (row tile of 128 query rows, batch * kv-head, KV split).  The
// G = Hq/Hkv query heads sharing a kv head are packed with the S tree queries
// into the MMA M dimension (row r = head_in_group * S + i): K/V are read once
// per kv head (GQA).  Warp roles (10 warps):
//   warps 0-7  softmax, two warpgroups: warpgroup g takes key blocks j = g,
//              g+2, ... with its own online-softmax state (m, l) and its own O
//              accumulator O[g] in TMEM — an intra-CTA split of the keys that
//              doubles softmax issue width without a per-block cross-warpgroup
//              sync; one thread per query row reads S with tcgen05.ld and
//              writes P (bf16 pairs) back over the S columns it has read with
//              tcgen05.st, rescales O[g] lazily (only when the running max
//              grows by > 2^8); the epilogue merges (m0, l0, O[0]) and
//              (m1, l1, O[1])
//   warp 8     TMA producer: K and V blocks of 128 keys into separate rings
//              (2 K slots, 4 V slots of 32 KB, 128B swizzle), mbarrier
//              complete_tx; a K slot is released when Q K^T completed, a V
//              slot when P V completed
//   warp 9     MMA issuer: S[j%2] = Q K_j^T (M128 N128 K16 x 8) as soon as the
//              K slot lands, so Q K^T of block j+1 overlaps the softmax of j;
//              O[j%2] += P_j V_j with P read from TMEM (the A-from-TMEM form)
//              and V as an MN-major shared-memory operand once P_j is ready
// TMEM: S0 | S1 | O0 | O1 (4 x 128 fp32 columns; P_j aliases the first 64
// columns of its S).  Split-KV partials (unnormalised O, row max, row sum)
// are merged by the log-sum-exp combine kernel.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>

#include "common.cuh"

namespace sssd {
int fail(int code, const char* fmt, ...);
int cuda_check(cudaError_t e, const char* what);

namespace attn {

constexpr int kD = 128;             // head dim
constexpr int kM = 128;             // rows per tile (UMMA M)
constexpr int kN = 128;             // keys per block (UMMA N of QK^T, K of PV)
constexpr int kTile = kM * kD * 2;  // 32 KB per bf16 128x128 tile
constexpr int kHalf = kTile / 2;    // 16 KB: 128 rows x 64 columns (one 128B-swizzled TMA box)
// K and V rings (separate barriers): a K slot is free once Q K_j^T has
// completed, a V slot once P_j V_j has; 6 x 32 KB slots + the Q tile = 224 KB
#ifndef SSSD_ATTN_KSTAGES
#define SSSD_ATTN_KSTAGES 2
#endif
constexpr int kKStages = SSSD_ATTN_KSTAGES;
constexpr int kVStages = 6 - kKStages;
static_assert(kKStages >= 1 && kVStages >= 2, "ring split");
constexpr int kWgWarps = 4;                  // one softmax warpgroup = 128 rows
constexpr int kWgThreads = 32 * kWgWarps;
constexpr int kTmaWarp = 2 * kWgWarps;       // warp 8
constexpr int kMmaWarp = 2 * kWgWarps + 1;   // warp 9
constexpr int kThreads = 32 * (kMmaWarp + 1);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 128B-swizzled K-major tile of 128 rows x 128 bf16 columns, stored as two
// [128 x 64] halves (16 KB each, = the TMA SWIZZLE_128B box layout): element
// (r, c) at half(c/64) + r*128 + (((c%64)/8) ^ (r%8))*16 + (c%8)*2.
__device__ __forceinline__ uint32_t sw_off(int r, int c8) {
  return (uint32_t)((c8 >> 3) * kHalf + r * 128 + (((c8 & 7) ^ (r & 7)) << 4));
}

// UMMA shared-memory descriptor, SWIZZLE_128B (layout type 2), version 1
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46) | (2ull << 61);
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, M = 128, N = 128
__device__ __forceinline__ uint32_t idesc_bf16(bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) | ((128u >> 3) << 17) |
         ((128u >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// A operand from TMEM (K-major: lane = row, one 32-bit column = 2 bf16 along K)
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

// bounded wait: a pipeline stage that never completes traps instead of hanging
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  for (uint32_t it = 0; !mbar_try(bar, phase); ++it) {
    if (it > (1u << 26)) {
      printf("sssd tree_attn: mbarrier timeout block (%d,%d,%d) thread %d phase %u\n", blockIdx.x, blockIdx.y,
             blockIdx.z, threadIdx.x, phase);
      __trap();
    }
  }
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float fast_exp2(float x) {
#ifdef SSSD_ATTN_FAKE_EXP  // timing experiment only: softmax without the MUFU (wrong results)
  return fmaf(x, 1e-3f, 1.0f);
#else
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#endif
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])),
      "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
      "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])),
      "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}

// 16 consecutive 32-bit columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

struct Params {
  const uint16_t* q;     // [B][S][Hq][D]
  const uint64_t* mask;  // [B][S][W]
  const int32_t* ctx;    // [B]
  uint16_t* o;           // [B][S][Hq][D]
  float* part_o;         // [splits][B][Hq][S][D]   (splits > 1)
  float* part_ml;        // [splits][B][Hq][S][2]
  int B, S, Hq, Hkv, G, max_pos, W, splits, split_len;
  float scale_log2;
};

struct Smem {  // 1024-aligned dynamic shared memory layout (224 KB)
  uint8_t q[kTile];           // Q tile; reused for the warpgroup merge once all MMAs completed
  uint8_t k[kKStages][kTile];
  uint8_t v[kVStages][kTile];
  uint64_t kfull[kKStages], kempty[kKStages], vfull[kVStages], vempty[kVStages];
  uint64_t s_full[2], s_free[2], p_ready[2], pv_done[2];
  uint32_t tmem;
};

__device__ __forceinline__ void wg_bar() {  // both softmax warpgroups (256 threads)
  asm volatile("bar.sync 1, %0;" ::"n"(2 * kWgThreads) : "memory");
}

// One key block of one softmax warpgroup (one thread per query row): the
// visibility words of the block's 4 x 32 keys (prefix keys visible, tree key t
// iff ancestor bit t), then P = 2^(S*scale - m) in bf16, written back into
// TMEM over the S columns already read (P V then takes A from TMEM, so no
// shared-memory P and the K slot is free as soon as Q K^T completed), and the
// running (m, l) with a lazy rescale of O.
//   * one pass over S (TMEM's read port is the scarce resource): P relative
//     to the running max, kept in registers until the block max is known to
//     stay within 2^8 of it — the lazy-rescale rule then keeps m and P
//     unchanged; the first block of a row and the rare block that raises the
//     max further take the two-pass form (warp-uniform: tcgen05.ld/st are
//     warp-collective) over the still intact S;
//   * a warp whose rows are all padding (G*S < 128) skips the block (its P
//     rows keep stale S bits; P V rows are independent);
//   * fully visible 32-key chunks (every prefix chunk) skip the per-key masks;
//   * max / sum use 4 independent chains.
__device__ __forceinline__ void softmax_block(uint64_t* s_full, uint64_t* s_free, uint64_t* pv_done,
                                              uint64_t* p_ready, bool row_ok, const uint64_t* mrow, int S,
                                              int ctx, int k0, int kv1, uint32_t tS, uint32_t tO, int it,
                                              bool has_prev, float sl2, float& m_run, float& l_run) {
  uint32_t visw[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int key0 = k0 + c * 32;
    // padding rows (row_ok false) see every key: their lanes then take the
    // same mask-free branch as the live rows of a prefix chunk (no divergence
    // in a partly filled warp); their P rows only feed padding rows of O
    uint32_t w = 0xffffffffu;
    if (row_ok) {
      const int lim = min(32, kv1 - key0);
      w = lim >= 32 ? 0xffffffffu : (lim > 0 ? (1u << lim) - 1u : 0u);
      if (key0 + 32 > ctx) {
        uint32_t tree = 0;
#pragma unroll 1
        for (int jj = max(0, ctx - key0); jj < 32; ++jj) {
          const int t = key0 + jj - ctx;
          if (t < S && ((mrow[t >> 6] >> (t & 63)) & 1ull)) tree |= 1u << jj;
        }
        const uint32_t pref = ctx - key0 >= 32 ? 0xffffffffu : (ctx > key0 ? (1u << (ctx - key0)) - 1u : 0u);
        w &= pref | tree;
      }
    }
    visw[c] = w;
  }
  mbar_wait(s_full, it & 1);
  fence_after();
#ifdef SSSD_ATTN_NO_SOFTMAX  // timing experiment only: the pipeline without softmax work (wrong results)
  const bool live = false;
#else
  const bool live = __any_sync(SSSD_FULL, row_ok);
#endif
  float m_use = m_run, corr = 1.f, psum = 0.f;
  if (live) {
    bool two_pass = __any_sync(SSSD_FULL, row_ok && m_run == -INFINITY);
    if (!two_pass) {
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY}, ps[4] = {0.f, 0.f, 0.f, 0.f};
      uint32_t pk[64];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float sv[32];
        tmem_ld32(tS + c * 32, sv);
        const uint32_t w = visw[c];
        if (w == 0xffffffffu) {
#pragma unroll
          for (int jj = 0; jj < 32; jj += 2) {
            const int a = (jj >> 1) & 3;
            mx[a] = fmaxf(mx[a], fmaxf(sv[jj], sv[jj + 1]));
            const float e0 = fast_exp2(fmaf(sv[jj], sl2, -m_run));
            const float e1 = fast_exp2(fmaf(sv[jj + 1], sl2, -m_run));
            ps[a] += e0 + e1;
            const __nv_bfloat162 h2 = __floats2bfloat162_rn(e0, e1);
            pk[c * 16 + (jj >> 1)] = *reinterpret_cast<const uint32_t*>(&h2);
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < 32; jj += 2) {
            const int a = (jj >> 1) & 3;
            const bool v0 = (w >> jj) & 1u, v1 = (w >> (jj + 1)) & 1u;
            mx[a] = fmaxf(mx[a], fmaxf(v0 ? sv[jj] : -INFINITY, v1 ? sv[jj + 1] : -INFINITY));
            const float e0 = v0 ? fast_exp2(fmaf(sv[jj], sl2, -m_run)) : 0.f;
            const float e1 = v1 ? fast_exp2(fmaf(sv[jj + 1], sl2, -m_run)) : 0.f;
            ps[a] += e0 + e1;
            const __nv_bfloat162 h2 = __floats2bfloat162_rn(e0, e1);
            pk[c * 16 + (jj >> 1)] = *reinterpret_cast<const uint32_t*>(&h2);
          }
        }
      }
      psum = (ps[0] + ps[1]) + (ps[2] + ps[3]);
      const float m4 = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      const float bmax = (m4 == -INFINITY) ? m4 : m4 * sl2;
      two_pass = __any_sync(SSSD_FULL, bmax > m_run + 8.f);
      if (!two_pass) {
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_st16(tS + c * 16, pk + c * 16);
      }
    }
    if (two_pass) {
      float sv[32];
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        tmem_ld32(tS + c * 32, sv);
        const uint32_t w = visw[c];
        if (w == 0xffffffffu) {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) mx[jj & 3] = fmaxf(mx[jj & 3], sv[jj]);
        } else {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) mx[jj & 3] = fmaxf(mx[jj & 3], ((w >> jj) & 1u) ? sv[jj] : -INFINITY);
        }
      }
      float bmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      bmax = (bmax == -INFINITY) ? bmax : bmax * sl2;
      // lazy rescale: keep the running max unless the block max exceeds it by
      // more than 2^8 (P <= 256 stays exact in bf16 range; O / l is unchanged)
      if (bmax > m_run + 8.f) {
        corr = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - bmax);
        m_use = bmax;
      }
      float ps[4] = {0.f, 0.f, 0.f, 0.f};
      // chunk c's P goes to columns [16c, 16c + 16): S columns this pass has read
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        tmem_ld32(tS + c * 32, sv);
        const uint32_t w = (m_use == -INFINITY) ? 0u : visw[c];
        uint32_t pk[16];
#pragma unroll
        for (int jj = 0; jj < 32; jj += 2) {
          float e0 = fast_exp2(fmaf(sv[jj], sl2, -m_use));
          float e1 = fast_exp2(fmaf(sv[jj + 1], sl2, -m_use));
          e0 = ((w >> jj) & 1u) ? e0 : 0.f;
          e1 = ((w >> (jj + 1)) & 1u) ? e1 : 0.f;
          ps[(jj >> 1) & 3] += e0 + e1;
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(e0, e1);
          pk[jj >> 1] = *reinterpret_cast<const uint32_t*>(&h2);
        }
        tmem_st16(tS + c * 16, pk);
      }
      psum = (ps[0] + ps[1]) + (ps[2] + ps[3]);
    }
  }
  l_run = l_run * corr + psum;
  // O[g] is stable once this warpgroup's previous P V completed
  if (has_prev && live) {
    mbar_wait(pv_done, (it - 1) & 1);
    fence_after();
    if (__any_sync(SSSD_FULL, corr != 1.f)) {  // warp-collective TMEM ld/st
      float ov[32];
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        tmem_ld32(tO + c * 32, ov);
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) ov[jj] *= corr;
        tmem_st32(tO + c * 32, ov);
      }
    }
  }
  m_run = m_use;
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  fence_before();
  mbar_arrive(s_free);
  mbar_arrive(p_ready);
}

__global__ void __launch_bounds__(kThreads, 1)
    tree_attn_kernel(Params p, const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tile = blockIdx.x, bh = blockIdx.y, split = blockIdx.z;
  const int b = bh / p.Hkv, kvh = bh % p.Hkv;
  const int rows = p.G * p.S;
  const int ctx = p.ctx[b];
  const int total = ctx + p.S;
  const int kv0 = split * p.split_len;
  const int kv1 = min(total, kv0 + p.split_len);
  const int nblk = kv1 > kv0 ? (kv1 - kv0 + kN - 1) / kN : 0;

  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(&sm.kfull[s], 1);
      mbar_init(&sm.kempty[s], 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(&sm.vfull[s], 1);
      mbar_init(&sm.vempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.s_full[s], 1);
      mbar_init(&sm.s_free[s], kWgThreads);
      mbar_init(&sm.p_ready[s], kWgThreads);
      mbar_init(&sm.pv_done[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Q tile (swizzled K-major): row r = (head_in_group, query i) -> q[b][i][kvh*G + hl][:]
  if (warp < 2 * kWgWarps) {
    for (int idx = tid; idx < kM * 16; idx += 2 * kWgThreads) {
      const int rr = idx >> 4, c8 = idx & 15;
      const int gr = tile * kM + rr;
      uint4 val = make_uint4(0, 0, 0, 0);
      if (gr < rows) {
        const int h2 = kvh * p.G + gr / p.S, i2 = gr % p.S;
        val = __ldg(reinterpret_cast<const uint4*>(p.q + (((int64_t)b * p.S + i2) * p.Hq + h2) * kD) + c8);
      }
      *reinterpret_cast<uint4*>(sm.q + sw_off(rr, c8)) = val;
    }
    fence_async_smem();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = sm.tmem;
  const int64_t row0 = (int64_t)(b * p.Hkv + kvh) * p.max_pos;  // first K/V row of this (b, kv head)

  if (warp == kTmaWarp) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      for (int j = 0; j < nblk; ++j) {
        const int y = (int)(row0 + kv0 + j * kN);
        const int sk = j % kKStages, sv = j % kVStages;
        if (j >= kKStages) mbar_wait(&sm.kempty[sk], ((j / kKStages) - 1) & 1);
        mbar_expect_tx(&sm.kfull[sk], kTile);
        tma_load_2d(sm.k[sk], &kmap, 0, y, &sm.kfull[sk]);
        tma_load_2d(sm.k[sk] + kHalf, &kmap, 64, y, &sm.kfull[sk]);
        if (j >= kVStages) mbar_wait(&sm.vempty[sv], ((j / kVStages) - 1) & 1);
        mbar_expect_tx(&sm.vfull[sv], kTile);
        tma_load_2d(sm.v[sv], &vmap, 0, y, &sm.vfull[sv]);
        tma_load_2d(sm.v[sv] + kHalf, &vmap, 64, y, &sm.vfull[sv]);
      }
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer ----------------
    // block j: S[j&1] = Q K_j^T, O[j&1] += P_j V_j (warpgroup j&1 owns S/O[j&1])
    if (lane == 0) {
      const uint32_t id_qk = idesc_bf16(false), id_pv = idesc_bf16(true);
      const uint32_t aQ = smem_u32(sm.q);
      for (int j = -1; j < nblk; ++j) {
        const int jn = j + 1;  // Q K^T of the next block goes first so it overlaps softmax(j)
        if (jn < nblk) {
          const int st = jn % kKStages, g = jn & 1;
          mbar_wait(&sm.kfull[st], (jn / kKStages) & 1);
          if (jn >= 2) mbar_wait(&sm.s_free[g], ((jn >> 1) - 1) & 1);
          fence_after();
          const uint32_t aK = smem_u32(sm.k[st]);
          const uint32_t tS = tbase + g * kN;
#pragma unroll
          for (int ks = 0; ks < kD / 16; ++ks) {
            const uint32_t off = (ks >> 2) * kHalf + (ks & 3) * 32;  // K step of 16 columns
            mma_bf16(tS, sw128_desc(aQ + off, 16, 1024), sw128_desc(aK + off, 16, 1024), id_qk, ks > 0);
          }
          mma_commit(&sm.s_full[g]);
          mma_commit(&sm.kempty[st]);
        }
        if (j < 0) continue;
        const int g = j & 1;
        const int sv = j % kVStages;
        mbar_wait(&sm.vfull[sv], (j / kVStages) & 1);
        mbar_wait(&sm.p_ready[g], (j >> 1) & 1);
        fence_after();
        const uint32_t aV = smem_u32(sm.v[sv]);
        const uint32_t tO = tbase + 2 * kN + g * kD, tP = tbase + g * kN;
#pragma unroll
        for (int ks = 0; ks < kN / 16; ++ks) {
          // P from TMEM (16 keys = 8 packed columns per step); V: MN-major, 8-key groups of 1024 B.
          // Q K^T of block j+2 (into the same S/P columns) is issued after this
          // in program order; tcgen05.mma from one thread executes in order
          mma_bf16_ts(tO, tP + ks * 8, sw128_desc(aV + ks * 2048, kHalf, 1024), id_pv, (j >= 2 || ks > 0) ? 1u : 0u);
        }
        mma_commit(&sm.pv_done[g]);
        mma_commit(&sm.vempty[sv]);
      }
    }
  } else {
    // ---------------- softmax: warpgroup g takes blocks j = g, g+2, ... ----------------
    // one thread per query row; each warpgroup keeps its own (m, l, O[g]) — an
    // intra-CTA split of the keys merged in the epilogue
    const int g = warp / kWgWarps, rt = tid - g * kWgThreads;
    const int r = tile * kM + rt;
    const bool row_ok = r < rows;
    const int hl = row_ok ? r / p.S : 0, qi = row_ok ? r % p.S : 0;
    const int head = kvh * p.G + hl;
    const uint64_t* mrow = p.mask + ((int64_t)b * p.S + qi) * p.W;
    const uint32_t lane_off = (uint32_t)((warp % kWgWarps) * 32) << 16;
    const uint32_t tS = tbase + g * kN + lane_off, tO = tbase + 2 * kN + g * kD + lane_off;
    const float sl2 = p.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;
    int it = 0;
    for (int j = g; j < nblk; j += 2, ++it) {
      softmax_block(&sm.s_full[g], &sm.s_free[g], &sm.pv_done[g], &sm.p_ready[g], row_ok, mrow, p.S, ctx,
                    kv0 + j * kN, kv1, tS, tO, it, it > 0, sl2, m_run, l_run);
    }
    if (it > 0) mbar_wait(&sm.pv_done[g], (it - 1) & 1);
    // ---------------- epilogue: merge the two warpgroups ----------------
    // every MMA has completed once both warpgroups passed their last pv_done
    // (commit tracks all earlier tcgen05 ops), so the Q tile is free for (m, l)
    float* xm = reinterpret_cast<float*>(sm.q);  // [2][kM] m, then [2][kM] l
    wg_bar();
    xm[g * kM + rt] = m_run;
    xm[2 * kM + g * kM + rt] = l_run;
    wg_bar();
    fence_after();
    const float m0 = xm[rt], m1 = xm[kM + rt];
    const float mm = fmaxf(m0, m1);
    const float w0 = (m0 == -INFINITY) ? 0.f : fast_exp2(m0 - mm);
    const float w1 = (m1 == -INFINITY) ? 0.f : fast_exp2(m1 - mm);
    const float l = w0 * xm[2 * kM + rt] + w1 * xm[3 * kM + rt];
    const bool has0 = nblk > 0, has1 = nblk > 1;  // warpgroup 1 owns no block when nblk == 1
    const uint32_t tO0 = tbase + 2 * kN + lane_off, tO1 = tO0 + kD;
    // warpgroup g writes output columns [64 g, 64 g + 64)
    const int64_t prow = (((int64_t)split * p.B + b) * p.Hq + head) * p.S + qi;
    const float inv = (l > 0.f) ? 1.f / l : 0.f;
    for (int c = 2 * g; c < 2 * g + 2; ++c) {
      float o0[32], o1[32];
      if (has0) tmem_ld32(tO0 + c * 32, o0);
      if (has1) tmem_ld32(tO1 + c * 32, o1);
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) o0[jj] = (has0 ? w0 * o0[jj] : 0.f) + (has1 ? w1 * o1[jj] : 0.f);
      if (!row_ok) continue;
      if (p.splits == 1) {
        uint32_t pk[16];
#pragma unroll
        for (int jj = 0; jj < 32; jj += 2) {
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(o0[jj] * inv, o0[jj + 1] * inv);
          pk[jj >> 1] = *reinterpret_cast<const uint32_t*>(&h2);
        }
        uint4* dst = reinterpret_cast<uint4*>(p.o + (((int64_t)b * p.S + qi) * p.Hq + head) * kD + c * 32);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) dst[q4] = make_uint4(pk[q4 * 4], pk[q4 * 4 + 1], pk[q4 * 4 + 2], pk[q4 * 4 + 3]);
      } else {
        float4* dst = reinterpret_cast<float4*>(p.part_o + prow * kD + c * 32);
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) dst[q4] = make_float4(o0[q4 * 4], o0[q4 * 4 + 1], o0[q4 * 4 + 2], o0[q4 * 4 + 3]);
      }
    }
    if (p.splits > 1 && row_ok && g == 0) {
      p.part_ml[prow * 2] = mm;
      p.part_ml[prow * 2 + 1] = l;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == kMmaWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
}

// merge split-KV partials: O = sum_s 2^(m_s - M) O_s / sum_s 2^(m_s - M) l_s
__global__ void tree_attn_combine_kernel(Params p) {
  const int64_t row = (int64_t)blockIdx.x;  // (b, head, i)
  const int d = threadIdx.x;                // 0..127
  const int total_rows = p.B * p.Hq * p.S;
  if (row >= total_rows) return;
  const int i = (int)(row % p.S);
  const int head = (int)((row / p.S) % p.Hq);
  const int b = (int)(row / ((int64_t)p.S * p.Hq));
  float M = -INFINITY;
  for (int s = 0; s < p.splits; ++s) M = fmaxf(M, p.part_ml[((int64_t)s * total_rows + row) * 2]);
  float num = 0.f, den = 0.f;
  for (int s = 0; s < p.splits; ++s) {
    const int64_t pr = (int64_t)s * total_rows + row;
    const float ms = p.part_ml[pr * 2], ls = p.part_ml[pr * 2 + 1];
    const float w = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
    num += w * p.part_o[pr * kD + d];
    den += w * ls;
  }
  const float out = den > 0.f ? num / den : 0.f;
  p.o[(((int64_t)b * p.S + i) * p.Hq + head) * kD + d] = __bfloat16_as_ushort(__float2bfloat16_rn(out));
}

constexpr int kSmem = (int)sizeof(Smem) + 1024;

// TMA descriptor over a [rows][128] bf16 cache viewed as 2D, box 64 x 128, 128B swizzle
static int make_kv_map(CUtensorMap* map, const void* base, uint64_t rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(SSSD_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)kD, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)kD * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)kN};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SSSD_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SSSD_OK;
}

}  // namespace attn
}  // namespace sssd

using namespace sssd;

extern "C" {

static int attn_max_splits(int32_t max_pos) {  // every split keeps >= 1024 keys (bounds the workspace)
  int cap = 1;
  while (cap < 64 && (max_pos / (cap * 2)) >= 1024) cap *= 2;
  return cap;
}

// Split count minimising waves x (key blocks per CTA + fixed per-CTA cost).
// The fixed cost (TMEM alloc, Q tile, pipeline fill, epilogue, partial
// write-back) was measured at ~4.5 key blocks on B200 (cfg3: 1 split beats 2;
// cfg4: 2 beat 4 and 8).
static int attn_splits(int32_t B, int32_t Hq, int32_t Hkv, int32_t S, int32_t max_pos) {
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n_sm <= 0) n_sm = 148;
  }
  const int G = Hq / Hkv;
  const int tiles = (G * S + attn::kM - 1) / attn::kM;
  const int64_t ctas = (int64_t)tiles * B * Hkv;
  const int nb = (max_pos + attn::kN - 1) / attn::kN;
  const int cap = attn_max_splits(max_pos);
  int best = 1;
  double best_cost = 1e300;
  for (int s = 1; s <= cap; ++s) {
    const double waves = (double)((ctas * s + n_sm - 1) / n_sm);
    const double cost = waves * ((nb + s - 1) / s + 4.5);
    if (cost < best_cost * 0.999) best_cost = cost, best = s;
  }
  return best;
}

size_t sssd_tree_attention_workspace(int32_t B, int32_t S, int32_t Hq, int32_t max_pos) {
  const int splits = attn_max_splits(max_pos);  // upper bound of attn_splits
  return (size_t)splits * B * Hq * S * (attn::kD + 2) * sizeof(float) + 256;
}

int sssd_tree_attention(const uint16_t* q, const uint16_t* k, const uint16_t* v, const uint64_t* mask,
                        const int32_t* ctx_len, int32_t B, int32_t S, int32_t Hq, int32_t Hkv,
                        int32_t max_pos, int32_t head_dim, float scale, uint16_t* o, void* workspace,
                        size_t workspace_bytes, void* stream) {
  if (head_dim != attn::kD) return fail(SSSD_E_LIMIT, "tree attention supports head_dim 128, got %d", head_dim);
  if (B <= 0 || S <= 0 || Hq <= 0 || Hkv <= 0 || Hq % Hkv) return fail(SSSD_E_ARG, "bad attention shape");
  if (S > SSSD_MAX_DRAFT) return fail(SSSD_E_LIMIT, "S=%d exceeds %d", S, SSSD_MAX_DRAFT);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  attn::Params p;
  p.q = q;
  p.mask = mask;
  p.ctx = ctx_len;
  p.o = o;
  p.B = B;
  p.S = S;
  p.Hq = Hq;
  p.Hkv = Hkv;
  p.G = Hq / Hkv;
  p.max_pos = max_pos;
  p.W = (S + 63) / 64;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.splits = attn_splits(B, Hq, Hkv, S, max_pos);
  p.split_len = ((max_pos + p.splits - 1) / p.splits + attn::kN - 1) / attn::kN * attn::kN;
  const size_t need = (size_t)p.splits * B * Hq * S * (attn::kD + 2) * sizeof(float) + 256;
  if (p.splits > 1) {
    if (!workspace || workspace_bytes < need)
      return fail(SSSD_E_WORKSPACE, "tree attention needs %zu workspace bytes, got %zu", need, workspace_bytes);
    p.part_o = static_cast<float*>(workspace);
    p.part_ml = p.part_o + (size_t)p.splits * B * Hq * S * attn::kD;
  } else {
    p.part_o = nullptr;
    p.part_ml = nullptr;
  }
  CUtensorMap kmap, vmap;
  const uint64_t rows = (uint64_t)B * Hkv * max_pos;
  int rc = attn::make_kv_map(&kmap, k, rows);
  if (!rc) rc = attn::make_kv_map(&vmap, v, rows);
  if (rc) return rc;
  const int tiles = (p.G * S + attn::kM - 1) / attn::kM;
  rc = cuda_check(cudaFuncSetAttribute(attn::tree_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       attn::kSmem),
                  "tree_attn smem attribute");
  if (rc) return rc;
  attn::tree_attn_kernel<<<dim3(tiles, B * Hkv, p.splits), attn::kThreads, attn::kSmem, st>>>(p, kmap, vmap);
  if ((rc = cuda_check(cudaGetLastError(), "tree_attn_kernel launch"))) return rc;
  if (p.splits > 1) {
    attn::tree_attn_combine_kernel<<<B * Hq * S, attn::kD, 0, st>>>(p);
    if ((rc = cuda_check(cudaGetLastError(), "tree_attn_combine launch"))) return rc;
  }
  return SSSD_OK;
}

}  // extern "C"
