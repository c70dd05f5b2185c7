// Tree-attention verification on B200: tcgen05.mma (kind::f16, bf16 inputs,
// fp32 accumulators in TMEM), semantics of ref draft.py:205-210 — every draft
// node i attends to the committed prefix [0, ctx) and to its ancestors-or-self
// among the S tree keys [ctx, ctx + S) (u64 ancestor rows from the fusion
// kernel), so one forward gives all s_q greedy predictions.
//
// One CTA = (row tile of 128 query rows, batch * kv-head, KV split).  The
// G = Hq/Hkv query heads sharing a kv head are packed with the S tree queries
// into the MMA M dimension (row r = head_in_group * S + i), so K/V are read
// once per kv head (GQA).  Per 128-key block:
//   stage K, V (global -> smem, core-matrix layout)          all threads
//   S = Q K^T        8 x tcgen05.mma M128 N128 K16 -> TMEM    thread 0
//   online softmax   tcgen05.ld S rows, mask, exp2, P -> smem  1 thread / row
//   O *= corr        tcgen05.ld/st of the O accumulator rows
//   O += P V         8 x tcgen05.mma (V as an MN-major operand)
// Splits write unnormalised partial O + (max, sum); a combine kernel merges
// them with the log-sum-exp rule.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"

namespace sssd {
int fail(int code, const char* fmt, ...);
int cuda_check(cudaError_t e, const char* what);

namespace attn {

constexpr int kD = 128;       // head dim
constexpr int kM = 128;       // rows per tile (UMMA M)
constexpr int kN = 128;       // keys per block (UMMA N of QK^T, K of PV)
constexpr int kTile = kM * kD * 2;  // 32 KB per bf16 128x128 tile
constexpr int kThreads = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Core-matrix ("interleave", no swizzle) layout of a 128 x 128 bf16 tile:
// element (r, c) lives at (r/8)*2048 + (c/8)*128 + (r%8)*16 + (c%8)*2.
// As a K-major operand (rows = M or N, c = K): LBO = 128 B, SBO = 2048 B.
// As an MN-major operand (rows = K, c = N):    LBO = 2048 B, SBO = 128 B.
__device__ __forceinline__ uint32_t tile_off(int r, int c8) { return (r >> 3) * 2048 + c8 * 128 + (r & 7) * 16; }

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);  // version 1, no swizzle
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

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
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

// bounded wait: a tensor-core op that never completes traps instead of hanging
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  for (uint32_t it = 0; !mbar_try(bar, phase); ++it) {
    if (it > (1u << 24)) {
      printf("sssd tree_attn: mbarrier timeout block (%d,%d,%d) phase %u\n", blockIdx.x, blockIdx.y, blockIdx.z, phase);
      __trap();
    }
  }
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
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

struct Params {
  const uint16_t* q;   // [B][S][Hq][D]
  const uint16_t* k;   // [B][Hkv][max_pos][D]
  const uint16_t* v;
  const uint64_t* mask;  // [B][S][W]
  const int32_t* ctx;    // [B]
  uint16_t* o;           // [B][S][Hq][D]
  float* part_o;         // [splits][B][Hq][S][D]   (splits > 1)
  float* part_ml;        // [splits][B][Hq][S][2]
  int B, S, Hq, Hkv, G, max_pos, W, splits, split_len;
  float scale_log2;
};

// asynchronous staging of rows [0, nrows) of a 128 x 128 bf16 tile into the
// core-matrix layout (cp.async, 16 B per op, all in flight); rows >= nrows are
// zero-filled (src-size 0) so masked keys contribute 0 * 0 to P V
__device__ __forceinline__ void stage_tile_async(uint8_t* tile, const uint16_t* src, int64_t row_stride,
                                                 int nrows) {
#pragma unroll 4
  for (int idx = threadIdx.x; idx < kM * 16; idx += kThreads) {
    const int r = idx >> 4, c8 = idx & 15;
    const uint16_t* g = src + (int64_t)(r < nrows ? r : 0) * row_stride + c8 * 8;
    const uint32_t bytes = r < nrows ? 16u : 0u;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(tile + tile_off(r, c8))), "l"(g),
                 "r"(bytes)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(kThreads, 1) tree_attn_kernel(Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sKb[2] = {smem + kTile, smem + 2 * kTile};
  uint8_t* sVb[2] = {smem + 3 * kTile, smem + 4 * kTile};
  uint8_t* sP = smem + 5 * kTile;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 6 * kTile);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int tile = blockIdx.x;               // row tile
  const int bh = blockIdx.y;                 // b * Hkv + kvh
  const int split = blockIdx.z;
  const int b = bh / p.Hkv, kvh = bh % p.Hkv;
  const int rows = p.G * p.S;
  const int r = tile * kM + tid;             // this thread's query row
  const bool row_ok = r < rows;
  const int hl = row_ok ? r / p.S : 0, qi = row_ok ? r % p.S : 0;
  const int head = kvh * p.G + hl;
  const int ctx = p.ctx[b];
  const int total = ctx + p.S;
  const int kv0 = split * p.split_len;
  const int kv1 = min(total, kv0 + p.split_len);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Q tile: row r = (head_in_group, query i) -> q[b][i][kvh*G + hl][:]
  for (int idx = tid; idx < kM * 16; idx += kThreads) {
    const int rr = idx >> 4, c8 = idx & 15;
    const int gr = tile * kM + rr;
    uint4 val = make_uint4(0, 0, 0, 0);
    if (gr < rows) {
      const int h2 = kvh * p.G + gr / p.S, i2 = gr % p.S;
      val = __ldg(reinterpret_cast<const uint4*>(p.q + (((int64_t)b * p.S + i2) * p.Hq + h2) * kD) + c8);
    }
    *reinterpret_cast<uint4*>(sQ + tile_off(rr, c8)) = val;
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t tS = tbase, tO = tbase + 128;

  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  const uint64_t* mrow_all = p.mask + ((int64_t)b * p.S + qi) * p.W;

  const uint32_t id_qk = idesc_bf16(false), id_pv = idesc_bf16(true);
  const uint32_t aQ = smem_u32(sQ), aP = smem_u32(sP);
  const int64_t kv_stride = (int64_t)p.max_pos * kD;
  const uint16_t* kbase = p.k + ((int64_t)b * p.Hkv + kvh) * kv_stride;
  const uint16_t* vbase = p.v + ((int64_t)b * p.Hkv + kvh) * kv_stride;

  float m_run = -INFINITY, l_run = 0.f;
  uint32_t phase = 0;
  bool first = true;
  if (kv0 < kv1) {  // prefetch block 0
    const int nk = min(kN, kv1 - kv0);
    stage_tile_async(sKb[0], kbase + (int64_t)kv0 * kD, kD, nk);
    stage_tile_async(sVb[0], vbase + (int64_t)kv0 * kD, kD, nk);
  }
  int buf = 0;
  for (int k0 = kv0; k0 < kv1; k0 += kN, buf ^= 1) {
    // prefetch the next block into the other buffer (its last readers, the
    // MMAs of the previous block, completed before this iteration)
    if (k0 + kN < kv1) {
      const int nk2 = min(kN, kv1 - (k0 + kN));
      stage_tile_async(sKb[buf ^ 1], kbase + (int64_t)(k0 + kN) * kD, kD, nk2);
      stage_tile_async(sVb[buf ^ 1], vbase + (int64_t)(k0 + kN) * kD, kD, nk2);
      asm volatile("cp.async.wait_group 2;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    const uint32_t aK = smem_u32(sKb[buf]), aV = smem_u32(sVb[buf]);
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      fence_after();
#pragma unroll
      for (int ks = 0; ks < kD / 16; ++ks)
        mma_bf16(tS, smem_desc(aQ + ks * 256, 128, 2048), smem_desc(aK + ks * 256, 128, 2048), id_qk, ks > 0);
      mma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    fence_after();

    // online softmax over this block (one thread per query row).  Visibility of
    // the 32 keys of chunk c is one word: prefix keys are all visible, tree key
    // t is visible iff bit t of this row's ancestor mask is set.
    uint32_t visw[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int key0 = k0 + c * 32;
      uint32_t w = 0;
      if (row_ok) {
        const int lim = min(32, kv1 - key0);  // keys past the range are invisible
        w = lim >= 32 ? 0xffffffffu : (lim > 0 ? (1u << lim) - 1u : 0u);
        if (key0 + 32 > ctx) {  // chunk overlaps the tree region
          uint32_t tree = 0;
#pragma unroll 1
          for (int jj = max(0, ctx - key0); jj < 32; ++jj) {
            const int t = key0 + jj - ctx;
            if (t < p.S && ((mrow_all[t >> 6] >> (t & 63)) & 1ull)) tree |= 1u << jj;
          }
          const uint32_t pref = ctx - key0 >= 32 ? 0xffffffffu : (ctx > key0 ? (1u << (ctx - key0)) - 1u : 0u);
          w &= pref | tree;
        }
      }
      visw[c] = w;
    }
    float sv[32];
    float bmax = -INFINITY;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      tmem_ld32(tS + lane_off + c * 32, sv);
      const uint32_t w = visw[c];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if ((w >> j) & 1u) bmax = fmaxf(bmax, sv[j]);
    }
    bmax = (bmax == -INFINITY) ? bmax : bmax * p.scale_log2;
    const float m_new = fmaxf(m_run, bmax);
    const float corr = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - m_new);
    float psum = 0.f;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      tmem_ld32(tS + lane_off + c * 32, sv);
      const uint32_t w = (m_new == -INFINITY) ? 0u : visw[c];
      uint32_t pk[16];
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float e0 = ((w >> j) & 1u) ? fast_exp2(fmaf(sv[j], p.scale_log2, -m_new)) : 0.f;
        const float e1 = ((w >> (j + 1)) & 1u) ? fast_exp2(fmaf(sv[j + 1], p.scale_log2, -m_new)) : 0.f;
        psum += e0 + e1;
        const __nv_bfloat162 h2 = __floats2bfloat162_rn(e0, e1);
        pk[j >> 1] = *reinterpret_cast<const uint32_t*>(&h2);
      }
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4)
        *reinterpret_cast<uint4*>(sP + tile_off(tid, c * 4 + q4)) =
            make_uint4(pk[q4 * 4], pk[q4 * 4 + 1], pk[q4 * 4 + 2], pk[q4 * 4 + 3]);
    }
    l_run = l_run * corr + psum;
    // rescale the running O rows; tcgen05.ld/st are warp-collective, so the
    // whole warp takes the branch when any of its rows needs it
    if (!first && __any_sync(SSSD_FULL, corr != 1.f)) {
      float ov[32];
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        tmem_ld32(tO + lane_off + c * 32, ov);
#pragma unroll
        for (int j = 0; j < 32; ++j) ov[j] *= corr;
        tmem_st32(tO + lane_off + c * 32, ov);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    m_run = m_new;
    fence_async_smem();
    fence_before();
    __syncthreads();
    if (tid == 0) {
      fence_after();
#pragma unroll
      for (int ks = 0; ks < kN / 16; ++ks)
        mma_bf16(tO, smem_desc(aP + ks * 256, 128, 2048), smem_desc(aV + ks * 4096, 2048, 128), id_pv,
                 (!first || ks > 0) ? 1u : 0u);
      mma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    fence_after();
    first = false;
  }

  // epilogue: O row from TMEM
  float ov[32];
  if (p.splits == 1) {
    const float inv = (l_run > 0.f) ? 1.f / l_run : 0.f;
    for (int c = 0; c < 4; ++c) {
      if (first) {
#pragma unroll
        for (int j = 0; j < 32; ++j) ov[j] = 0.f;
      } else {
        tmem_ld32(tO + lane_off + c * 32, ov);
      }
      if (row_ok) {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(ov[j] * inv, ov[j + 1] * inv);
          pk[j >> 1] = *reinterpret_cast<const uint32_t*>(&h2);
        }
        uint4* dst = reinterpret_cast<uint4*>(p.o + (((int64_t)b * p.S + qi) * p.Hq + head) * kD + c * 32);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) dst[q4] = make_uint4(pk[q4 * 4], pk[q4 * 4 + 1], pk[q4 * 4 + 2], pk[q4 * 4 + 3]);
      }
    }
  } else {
    const int64_t prow = (((int64_t)split * p.B + b) * p.Hq + head) * p.S + qi;
    for (int c = 0; c < 4; ++c) {
      if (first) {
#pragma unroll
        for (int j = 0; j < 32; ++j) ov[j] = 0.f;
      } else {
        tmem_ld32(tO + lane_off + c * 32, ov);
      }
      if (row_ok) {
        float4* dst = reinterpret_cast<float4*>(p.part_o + prow * kD + c * 32);
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) dst[q4] = make_float4(ov[q4 * 4], ov[q4 * 4 + 1], ov[q4 * 4 + 2], ov[q4 * 4 + 3]);
      }
    }
    if (row_ok) {
      p.part_ml[prow * 2] = m_run;
      p.part_ml[prow * 2 + 1] = l_run;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(256));
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

constexpr int kSmem = 6 * kTile + 64;

}  // namespace attn
}  // namespace sssd

using namespace sssd;

extern "C" {

static int attn_splits(int32_t B, int32_t Hq, int32_t Hkv, int32_t S, int32_t max_pos) {
  const int G = Hq / Hkv;
  const int tiles = (G * S + attn::kM - 1) / attn::kM;
  const int ctas = tiles * B * Hkv;
  int splits = 1;
  while (ctas * splits < 2 * 148 && (max_pos / (splits * 2)) >= 1024) splits *= 2;
  return splits;
}

size_t sssd_tree_attention_workspace(int32_t B, int32_t S, int32_t Hq, int32_t max_pos) {
  // worst case over Hkv: splits chosen for Hkv = 1
  int splits = 1;
  while (splits < 64 && (max_pos / (splits * 2)) >= 1024) splits *= 2;
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
  p.k = k;
  p.v = v;
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
  const int tiles = (p.G * S + attn::kM - 1) / attn::kM;
  int rc = cuda_check(cudaFuncSetAttribute(attn::tree_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           attn::kSmem),
                      "tree_attn smem attribute");
  if (rc) return rc;
  attn::tree_attn_kernel<<<dim3(tiles, B * Hkv, p.splits), attn::kThreads, attn::kSmem, st>>>(p);
  if ((rc = cuda_check(cudaGetLastError(), "tree_attn_kernel launch"))) return rc;
  if (p.splits > 1) {
    attn::tree_attn_combine_kernel<<<B * Hq * S, attn::kD, 0, st>>>(p);
    if ((rc = cuda_check(cudaGetLastError(), "tree_attn_combine launch"))) return rc;
  }
  return SSSD_OK;
}

}  // extern "C"
