// Fused elementwise stages of the verification forward (model.py): one
// HBM pass each instead of the 5-15 PyTorch ops they replace (the glue
// between the cuBLAS projections and the tcgen05 tree attention).
//   sssd_rmsnorm_bf16   y = x * rsqrt(mean(x^2) + eps) * w           (fp32 math)
//   sssd_rope_kv_bf16   rotary embedding of q and k from the fused qkv
//                       projection; q to [b][S][Hq][d], k and v straight
//                       into the KV cache at slots ctx + s (the tree slots)
//   sssd_swiglu_bf16    a = silu(g) * u from the fused gate|up projection
// Rounding follows the PyTorch ops they replace (fp32 math, one bf16 rounding
// per PyTorch op boundary where that op materialised bf16).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"

namespace sssd {
int fail(int code, const char* fmt, ...);
int cuda_check(cudaError_t e, const char* what);

// one CTA per row; blockDim = 256, h a multiple of 8
__global__ void __launch_bounds__(256) rmsnorm_kernel(const __nv_bfloat16* x, const __nv_bfloat16* w,
                                                      __nv_bfloat16* y, int h, float eps) {
  __shared__ float s_part[8];
  const int64_t row = blockIdx.x;
  const __nv_bfloat16* xr = x + row * h;
  float ss = 0.f;
  for (int i = threadIdx.x * 8; i < h; i += blockDim.x * 8) {
    const uint4 v = *reinterpret_cast<const uint4*>(xr + i);
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(p[k]);
      ss += f.x * f.x + f.y * f.y;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(SSSD_FULL, ss, o);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) tot += s_part[i];
  const float r = rsqrtf(tot / (float)h + eps);
  for (int i = threadIdx.x * 8; i < h; i += blockDim.x * 8) {
    const uint4 v = *reinterpret_cast<const uint4*>(xr + i);
    const uint4 wv = *reinterpret_cast<const uint4*>(w + i);
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
    const __nv_bfloat162* q = reinterpret_cast<const __nv_bfloat162*>(&wv);
    uint4 o;
    __nv_bfloat162* po = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(p[k]), g = __bfloat1622float2(q[k]);
      po[k] = __floats2bfloat162_rn(f.x * r * g.x, f.y * r * g.y);
    }
    *reinterpret_cast<uint4*>(y + row * h + i) = o;
  }
}

// grid = b * S, block = 128.  The d/2 rotation angles of the token are
// computed once into shared memory; each thread then rotates bf16 pairs
// (i, i+1) against (i+half, i+half+1) of the Hq + Hkv rotated heads, and the
// Hkv value heads are copied 16 bytes at a time (d % 8 == 0, d <= 256).
__global__ void __launch_bounds__(128) rope_kv_kernel(const __nv_bfloat16* qkv, const int64_t* pos,
                                                      const int32_t* ctx_len, const int64_t* rows,
                                                      __nv_bfloat16* q_out, __nv_bfloat16* k_cache,
                                                      __nv_bfloat16* v_cache, int S, int hq, int hkv, int d,
                                                      int max_pos, float theta) {
  __shared__ float s_cos[128], s_sin[128];
  const int bs = blockIdx.x, bi = bs / S, s = bs - bi * S;
  const int half = d >> 1, hp = half >> 1;
  const int width = (hq + 2 * hkv) * d;
  const __nv_bfloat16* src = qkv + (int64_t)bs * width;
  const int64_t row = rows ? rows[bi] : bi;  // row < 0: rotate q only, write no K/V (a padding request)
  const int64_t slot = (int64_t)ctx_len[bi] + s;
  if (threadIdx.x < half) {
    // torch: inv = 1 / theta ** (arange(0, d, 2) / d); ang = pos * inv  (float32)
    const int i = threadIdx.x;
    const float ang = (float)pos[bs] * (1.0f / powf(theta, (float)(2 * i) / (float)d));
    s_cos[i] = cosf(ang);
    s_sin[i] = sinf(ang);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < (hq + hkv) * hp; t += blockDim.x) {
    const int hh = t / hp, i = 2 * (t - hh * hp);
    const float2 x1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(src + hh * d + i));
    const float2 x2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(src + hh * d + i + half));
    const float c0 = s_cos[i], c1 = s_cos[i + 1], n0 = s_sin[i], n1 = s_sin[i + 1];
    const __nv_bfloat162 y1 = __floats2bfloat162_rn(x1.x * c0 - x2.x * n0, x1.y * c1 - x2.y * n1);
    const __nv_bfloat162 y2 = __floats2bfloat162_rn(x1.x * n0 + x2.x * c0, x1.y * n1 + x2.y * c1);
    if (hh >= hq && row < 0) continue;
    __nv_bfloat16* dst = hh < hq ? q_out + ((int64_t)bs * hq + hh) * d
                                 : k_cache + ((row * hkv + (hh - hq)) * max_pos + slot) * d;
    *reinterpret_cast<__nv_bfloat162*>(dst + i) = y1;
    *reinterpret_cast<__nv_bfloat162*>(dst + i + half) = y2;
  }
  if (row < 0) return;
  const int d8 = d >> 3;
  for (int t = threadIdx.x; t < hkv * d8; t += blockDim.x) {
    const int hh = t / d8, i = (t - hh * d8) * 8;
    *reinterpret_cast<uint4*>(v_cache + ((row * hkv + hh) * max_pos + slot) * d + i) =
        *reinterpret_cast<const uint4*>(src + (hq + hkv + hh) * d + i);
  }
}

// Row argmax of fp32 logits (the greedy prediction of every draft node), same
// result as torch.argmax: the first index of the maximum, a NaN counting as
// the maximum (its first index).  One CTA per row, 16-byte loads.
__device__ __forceinline__ bool am_better(float v, int i, float bv, int bi) {
  const bool vn = v != v, bn = bv != bv;
  if (vn || bn) return vn && (!bn || i < bi);
  return v > bv || (v == bv && i < bi);
}

__global__ void __launch_bounds__(256) argmax_kernel(const float* x, int cols, int32_t* out, bool vec) {
  const float* row = x + (int64_t)blockIdx.x * cols;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  if (vec) {  // 4 independent 16-byte loads in flight per thread per round
    const float4* r4 = reinterpret_cast<const float4*>(row);
    const int n4 = cols / 4;
    for (int j0 = threadIdx.x; j0 < n4; j0 += 4 * blockDim.x) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u * blockDim.x;
        v[u] = j < n4 ? __ldg(r4 + j) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = 4 * (j0 + u * blockDim.x);
        if (am_better(v[u].x, i, bv, bi)) bv = v[u].x, bi = i;
        if (am_better(v[u].y, i + 1, bv, bi)) bv = v[u].y, bi = i + 1;
        if (am_better(v[u].z, i + 2, bv, bi)) bv = v[u].z, bi = i + 2;
        if (am_better(v[u].w, i + 3, bv, bi)) bv = v[u].w, bi = i + 3;
      }
    }
  } else {
    for (int i = threadIdx.x; i < cols; i += blockDim.x) {
      const float v = row[i];
      if (am_better(v, i, bv, bi)) bv = v, bi = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v = __shfl_down_sync(0xffffffffu, bv, o);
    const int i = __shfl_down_sync(0xffffffffu, bi, o);
    if (am_better(v, i, bv, bi)) bv = v, bi = i;
  }
  __shared__ float s_v[8];
  __shared__ int s_i[8];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) s_v[w] = bv, s_i[w] = bi;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (am_better(s_v[k], s_i[k], bv, bi)) bv = s_v[k], bi = s_i[k];
    out[blockIdx.x] = bi == 0x7fffffff ? 0 : bi;
  }
}

__device__ __forceinline__ float silu_bf16(float g) {
  // torch: silu in fp32 on the bf16 gate, rounded to bf16 (F.silu output dtype)
  return __bfloat162float(__float2bfloat16_rn(g / (1.0f + expf(-g))));
}

// a[r][j] = bf16(bf16(silu(g)) * u) with g = gu[r][j], u = gu[r][m + j];
// 8 outputs per thread (m % 8 == 0), 16-byte loads and stores
__global__ void __launch_bounds__(256) swiglu_kernel(const __nv_bfloat16* gu, __nv_bfloat16* a, int64_t rows,
                                                     int m) {
  const int m8 = m >> 3;
  const int64_t n = rows * (int64_t)m8;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / m8;
    const int j = (int)(t - r * m8) * 8;
    const __nv_bfloat16* gr = gu + r * 2 * m;
    const uint4 gv = *reinterpret_cast<const uint4*>(gr + j);
    const uint4 uv = *reinterpret_cast<const uint4*>(gr + m + j);
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
    const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uv);
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 g = __bfloat1622float2(g2[k]), u = __bfloat1622float2(u2[k]);
      o2[k] = __floats2bfloat162_rn(silu_bf16(g.x) * u.x, silu_bf16(g.y) * u.y);
    }
    *reinterpret_cast<uint4*>(a + r * m + j) = o;
  }
}

}  // namespace sssd

using namespace sssd;

extern "C" {

int sssd_rmsnorm_bf16(const void* x, const void* w, void* y, int64_t rows, int32_t h, float eps, void* stream) {
  if (!x || !w || !y || rows < 0 || h <= 0 || h % 8) return fail(SSSD_E_ARG, "rmsnorm: bad arguments");
  if (rows == 0) return SSSD_OK;
  rmsnorm_kernel<<<(unsigned)rows, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w), static_cast<__nv_bfloat16*>(y),
      h, eps);
  return cuda_check(cudaGetLastError(), "rmsnorm launch");
}

int sssd_rope_kv_bf16(const void* qkv, const int64_t* pos, const int32_t* ctx_len, const int64_t* rows,
                      void* q_out, void* k_cache, void* v_cache, int32_t b, int32_t S, int32_t hq, int32_t hkv,
                      int32_t d, int32_t max_pos, float theta, void* stream) {
  if (!qkv || !pos || !ctx_len || !q_out || !k_cache || !v_cache || b < 0 || S <= 0 || d % 8 || d > 256)
    return fail(SSSD_E_ARG, "rope_kv: bad arguments");
  if (b == 0) return SSSD_OK;
  rope_kv_kernel<<<(unsigned)(b * S), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(qkv), pos, ctx_len, rows, static_cast<__nv_bfloat16*>(q_out),
      static_cast<__nv_bfloat16*>(k_cache), static_cast<__nv_bfloat16*>(v_cache), S, hq, hkv, d, max_pos, theta);
  return cuda_check(cudaGetLastError(), "rope_kv launch");
}

int sssd_argmax_f32(const float* x, int64_t rows, int32_t cols, int32_t* out, void* stream) {
  if (!x || !out || rows < 0 || cols <= 0) return fail(SSSD_E_ARG, "argmax: bad arguments");
  if (rows == 0) return SSSD_OK;
  const bool vec = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && cols % 4 == 0;
  argmax_kernel<<<(unsigned)rows, 256, 0, static_cast<cudaStream_t>(stream)>>>(x, cols, out, vec);
  return cuda_check(cudaGetLastError(), "argmax launch");
}

int sssd_swiglu_bf16(const void* gu, void* a, int64_t rows, int32_t m, void* stream) {
  if (!gu || !a || rows < 0 || m <= 0 || m % 8) return fail(SSSD_E_ARG, "swiglu: bad arguments");
  if (rows == 0) return SSSD_OK;
  const int64_t n = rows * (int64_t)(m / 8);
  const unsigned blocks = (unsigned)min((n + 255) / 256, (int64_t)148 * 32);
  swiglu_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const __nv_bfloat16*>(gu),
                                                                       static_cast<__nv_bfloat16*>(a), rows, m);
  return cuda_check(cudaGetLastError(), "swiglu launch");
}

}  // extern "C"
