// Datastore index construction on the GPU (replaces ref datastore.py:81-109
// build_suffix_array and the in-memory layout of datastore.py:144-154).
//
// Suffix array: prefix doubling with group refinement on our own radix sort
// (csrc/sa_build.cu); the SA of a sequence is unique, so the result is
// bit-identical to the reference.
//
// Suffix rows: the lookup layout.  Row r (64 B, one aligned 2-sector line) =
// {pos = SA[r], tokens[pos .. pos+15)} so a search probe or a sampled
// continuation is ONE independent 64 B access instead of an SA load followed
// by a dependent token load.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace sssd {
int fail(int code, const char* fmt, ...);
int cuda_check(cudaError_t e, const char* what);

__global__ void rows_build_kernel(const uint32_t* tokens, uint64_t n, const uint32_t* sa,
                                  uint32_t* rows) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint32_t pos = sa[r];
  uint32_t t[16];
  t[0] = pos;
#pragma unroll
  for (int j = 0; j < SSSD_ROW_TOKENS; ++j) t[j + 1] = (uint64_t)pos + j < n ? __ldg(tokens + pos + j) : 0u;
  uint4* dst = reinterpret_cast<uint4*>(rows) + r * 4;
  dst[0] = make_uint4(t[0], t[1], t[2], t[3]);
  dst[1] = make_uint4(t[4], t[5], t[6], t[7]);
  dst[2] = make_uint4(t[8], t[9], t[10], t[11]);
  dst[3] = make_uint4(t[12], t[13], t[14], t[15]);
}

__global__ void rows_sa64_kernel(const uint32_t* rows, uint64_t n, uint64_t* out) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) out[r] = rows[r * 16];
}

// Full-size suffix-array verification (a size-independent parity property:
// an array that is a permutation of [0, n) with every adjacent pair of
// suffixes strictly increasing IS the unique suffix array, ref
// datastore.py:81-109 / SURVEY A.1).  Adjacent rows compare on their inline
// tokens, then on the corpus tokens past them; a proper prefix sorts first.
__global__ void sa_check_order_kernel(const uint32_t* tokens, uint64_t n, const uint32_t* rows, uint64_t n_rows,
                                      unsigned long long* bad) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r + 1 >= n_rows) return;
  const uint32_t* a = rows + r * 16;
  const uint32_t* b = a + 16;
  const uint64_t pa = a[0], pb = b[0];
  const uint64_t la = n - pa, lb = n - pb;  // suffix lengths
  int c = 0;
  const uint64_t inl = min((uint64_t)SSSD_ROW_TOKENS, min(la, lb));
  for (uint64_t j = 0; j < inl && c == 0; ++j)
    if (a[1 + j] != b[1 + j]) c = a[1 + j] < b[1 + j] ? -1 : 1;
  for (uint64_t j = inl; c == 0 && j < min(la, lb); ++j) {  // rare: longer common prefixes
    const uint32_t x = __ldg(tokens + pa + j), y = __ldg(tokens + pb + j);
    if (x != y) c = x < y ? -1 : 1;
  }
  if (c == 0) c = la < lb ? -1 : 1;  // equal prefix: the shorter suffix first (la != lb for pa != pb)
  if (c >= 0 || pa == pb) atomicAdd(bad, 1ull);
}

__global__ void sa_check_mark_kernel(const uint32_t* rows, uint64_t n_rows, uint64_t n, uint32_t* bits,
                                     unsigned long long* bad) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const uint64_t p = rows[r * 16];
  if (p >= n) {
    atomicAdd(bad, 1ull);
    return;
  }
  atomicOr(bits + (p >> 5), 1u << (p & 31));
}

__global__ void sa_check_count_kernel(const uint32_t* bits, uint64_t n, unsigned long long* missing) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t words = (n + 31) / 32;
  if (w >= words) return;
  uint32_t want = 0xffffffffu;
  if (w == words - 1 && (n & 31)) want = (1u << (n & 31)) - 1u;
  const uint32_t miss = want & ~bits[w];
  if (miss) atomicAdd(missing, (unsigned long long)__popc(miss));
}

size_t sa_build_workspace2(uint64_t n);
int sa_build2(const uint32_t* tokens, uint64_t n, uint32_t* sa_out, void* workspace, size_t workspace_bytes,
              cudaStream_t st, int* rounds_out);

}  // namespace sssd

using namespace sssd;

// bucket[t] = first row whose first token is >= t: row r writes the entries
// (tok0(r-1), tok0(r)] (clamped to n_buckets); the last row also closes the
// table with n_rows.  Rows are sorted, so the writes cover [0, n_buckets].
__global__ void bucket_build_kernel(const uint32_t* rows, uint64_t n, uint32_t nb, uint32_t* bucket) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t t = rows[r * 16 + 1];
  const int64_t prev = r > 0 ? (int64_t)rows[(r - 1) * 16 + 1] : -1;
  for (int64_t u = prev + 1; u <= t && u <= (int64_t)nb; ++u) bucket[u] = (uint32_t)r;
  if (r == n - 1)
    for (int64_t u = t + 1; u <= (int64_t)nb; ++u) bucket[u] = (uint32_t)n;
}

// ---- k-gram range index (sssd_kix_*) -------------------------------------------
// Row r starts a k-group when its suffix has >= k tokens and row r-1's first k
// tokens differ (or row r-1's suffix is shorter than k); the group runs to the
// next row that is not in it.  Rows hold their first 15 tokens inline, so every
// test reads the first 32 B sector of two adjacent rows (coalesced).
__device__ __forceinline__ bool kix_starts(const uint32_t* rows, uint64_t r, uint64_t n_tokens, int k) {
  const uint32_t* a = rows + r * 16;
  if (n_tokens - a[0] < (uint64_t)k) return false;
  if (r == 0) return true;
  const uint32_t* b = a - 16;
  if (n_tokens - b[0] < (uint64_t)k) return true;
  for (int j = 1; j <= k; ++j)
    if (a[j] != b[j]) return true;
  return false;
}

__global__ void kix_count_kernel(const uint32_t* rows, uint64_t n, uint64_t n_tokens, int kmax,
                                 unsigned long long* count) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t c = 0;
  if (r < n)
    for (int k = 2; k <= kmax; ++k) c += kix_starts(rows, r, n_tokens, k) ? 1u : 0u;
  c = __reduce_add_sync(SSSD_FULL, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}

__global__ void kix_insert_kernel(const uint32_t* rows, uint64_t n, uint64_t n_tokens, int kmax, uint4* tab,
                                  uint64_t mask) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int k = 2; k <= kmax; ++k) {
    if (!kix_starts(rows, r, n_tokens, k)) continue;
    const uint64_t h = kix_hash(rows + r * 16 + 1, k);
    for (uint64_t s = h & mask;; s = (s + 1) & mask) {
      unsigned long long* key = reinterpret_cast<unsigned long long*>(tab + s);
      const unsigned long long old = atomicCAS(key, 0ull, (unsigned long long)h);
      if (old == 0ull) {
        tab[s].z = (uint32_t)r;
        break;
      }
      if (old == h) break;  // a colliding k-gram holds the slot: its lookups verify and search
    }
  }
}

// hi of the group that row r-1 belongs to, written by the first row after it
// (or by the last row): the slot is found by the hash and checked to be that
// group's (its lo row has the same k tokens) before hi is written.
__global__ void kix_ends_kernel(const uint32_t* rows, uint64_t n, uint64_t n_tokens, int kmax, uint4* tab,
                                uint64_t mask) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r > n || r == 0) return;
  const uint32_t* p = rows + (r - 1) * 16;
  for (int k = 2; k <= kmax; ++k) {
    if (n_tokens - p[0] < (uint64_t)k) continue;               // row r-1 is in no k-group
    if (r < n && !kix_starts(rows, r, n_tokens, k)) {          // row r continues the group...
      if (n_tokens - rows[r * 16] >= (uint64_t)k) continue;   // ...unless it is shorter than k
    }
    const uint64_t h = kix_hash(p + 1, k);
    for (uint64_t s = h & mask;; s = (s + 1) & mask) {
      const uint4 e = tab[s];
      const uint64_t key = (uint64_t)e.y << 32 | e.x;
      if (key == 0) break;
      if (key == h) {
        const uint32_t* lr = rows + (uint64_t)e.z * 16;
        bool same = n_tokens - lr[0] >= (uint64_t)k;
        for (int j = 1; j <= k && same; ++j) same = lr[j] == p[j];
        if (same) tab[s].w = (uint32_t)r;
        break;
      }
    }
  }
}

// u16 -> u32 token widening: 4 tokens per thread per step (8 B in, 16 B out)
// when both pointers are suitably aligned, grid-stride, scalar tail.
__global__ void widen_u16_kernel(const uint16_t* src, uint32_t* dst, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool vec = (reinterpret_cast<uintptr_t>(src) % 8 == 0) && (reinterpret_cast<uintptr_t>(dst) % 16 == 0);
  int64_t done = 0;
  if (vec) {
    const int64_t n4 = n / 4;
    const uint2* s4 = reinterpret_cast<const uint2*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int64_t i = t0; i < n4; i += stride) {
      const uint2 v = s4[i];
      d4[i] = make_uint4(v.x & 0xffffu, v.x >> 16, v.y & 0xffffu, v.y >> 16);
    }
    done = n4 * 4;
  }
  for (int64_t i = done + t0; i < n; i += stride) dst[i] = src[i];
}

// Last min(P, len) tokens of every request, right-aligned in a [B][P] u32
// array, plus the (offset, length) view the datastore lookup reads them
// through.  `seq` may be pinned host memory (read over PCIe, zero-copy): the
// lookup needs only these tokens, so it can start before the contexts are
// uploaded.
__global__ void gather_tails_kernel(const void* seq, int elem_bytes, const int64_t* off, const int32_t* len, int B,
                                    int P, uint32_t* tails, int64_t* toff, int32_t* tlen) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int L = len[b];
  const int pm = L < P ? (L > 0 ? L : 0) : P;
  const int64_t end = off[b] + L;
  for (int j = 0; j < pm; ++j) {
    const int64_t i = end - pm + j;
    tails[(int64_t)b * P + (P - pm) + j] = elem_bytes == 2 ? (uint32_t)static_cast<const uint16_t*>(seq)[i]
                                                            : static_cast<const uint32_t*>(seq)[i];
  }
  toff[b] = (int64_t)b * P + (P - pm);
  tlen[b] = pm;
}

extern "C" {

size_t sssd_sa_build_workspace(uint64_t n) { return sa_build_workspace2(n ? n : 1); }

int sssd_sa_build(const uint32_t* tokens, uint64_t n, uint32_t* sa_out, void* workspace,
                  size_t workspace_bytes, void* stream) {
  if (n == 0) return fail(SSSD_E_ARG, "empty corpus");
  if (n >= 0xffffffffull) return fail(SSSD_E_LIMIT, "corpus longer than 2^32-1 tokens");
  if (!tokens || !sa_out) return fail(SSSD_E_ARG, "NULL buffer");
  return sa_build2(tokens, n, sa_out, workspace, workspace_bytes, static_cast<cudaStream_t>(stream), nullptr);
}

int sssd_sa_build_ex(const uint32_t* tokens, uint64_t n, uint32_t* sa_out, void* workspace, size_t workspace_bytes,
                     void* stream, int32_t* rounds) {
  if (n == 0) return fail(SSSD_E_ARG, "empty corpus");
  if (n >= 0xffffffffull) return fail(SSSD_E_LIMIT, "corpus longer than 2^32-1 tokens");
  if (!tokens || !sa_out) return fail(SSSD_E_ARG, "NULL buffer");
  int r = 1;
  const int rc = sa_build2(tokens, n, sa_out, workspace, workspace_bytes, static_cast<cudaStream_t>(stream), &r);
  if (rounds) *rounds = r;
  return rc;
}

int sssd_rows_build(const uint32_t* tokens, uint64_t n, const uint32_t* sa, uint32_t* rows,
                    void* stream) {
  if (n == 0) return fail(SSSD_E_ARG, "empty corpus");
  if (reinterpret_cast<uintptr_t>(rows) % 64) return fail(SSSD_E_ARG, "rows must be 64-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rows_build_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(tokens, n, sa, rows);
  return cuda_check(cudaGetLastError(), "rows_build launch");
}

int sssd_bucket_build(const uint32_t* rows, uint64_t n_rows, uint32_t n_buckets, uint32_t* bucket,
                      void* stream) {
  if (!rows || !bucket) return fail(SSSD_E_ARG, "bucket_build needs rows and an output table");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n_rows == 0)
    return cuda_check(cudaMemsetAsync(bucket, 0, ((size_t)n_buckets + 1) * 4, st), "bucket memset");
  if (n_rows >= 0xffffffffull) return fail(SSSD_E_LIMIT, "bucket index needs < 2^32 rows");
  bucket_build_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, st>>>(rows, n_rows, n_buckets, bucket);
  return cuda_check(cudaGetLastError(), "bucket_build launch");
}

int sssd_kix_count(const uint32_t* rows, uint64_t n_rows, uint64_t n_tokens, uint32_t kmax, uint64_t* count,
                   void* stream) {
  if (!rows || !count) return fail(SSSD_E_ARG, "kix_count needs rows and a count word");
  if (kmax < 2 || kmax > 7) return fail(SSSD_E_ARG, "kix kmax must be in 2..7");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = cuda_check(cudaMemsetAsync(count, 0, 8, st), "kix count memset");
  if (rc || n_rows == 0) return rc;
  kix_count_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, st>>>(
      rows, n_rows, n_tokens, (int)kmax, reinterpret_cast<unsigned long long*>(count));
  return cuda_check(cudaGetLastError(), "kix_count launch");
}

int sssd_kix_build(const uint32_t* rows, uint64_t n_rows, uint64_t n_tokens, uint32_t kmax, uint32_t* table,
                   uint64_t cap, void* stream) {
  if (!rows || !table) return fail(SSSD_E_ARG, "kix_build needs rows and a table");
  if (kmax < 2 || kmax > 7) return fail(SSSD_E_ARG, "kix kmax must be in 2..7");
  if (cap == 0 || (cap & (cap - 1))) return fail(SSSD_E_ARG, "kix capacity must be a power of two");
  if (n_rows >= 0xffffffffull) return fail(SSSD_E_LIMIT, "kix needs < 2^32 rows");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = cuda_check(cudaMemsetAsync(table, 0, cap * 16, st), "kix memset");
  if (rc || n_rows == 0) return rc;
  uint4* tab = reinterpret_cast<uint4*>(table);
  kix_insert_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, st>>>(rows, n_rows, n_tokens, (int)kmax, tab, cap - 1);
  kix_ends_kernel<<<(unsigned)((n_rows + 256) / 256), 256, 0, st>>>(rows, n_rows, n_tokens, (int)kmax, tab, cap - 1);
  return cuda_check(cudaGetLastError(), "kix_build launch");
}

int sssd_widen_u16(const uint16_t* src, uint32_t* dst, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!src || !dst))) return fail(SSSD_E_ARG, "widen_u16: bad buffers");
  if (n == 0) return SSSD_OK;
  const int64_t n4 = n / 4;
  const unsigned blocks = (unsigned)min((n4 + 255) / 256 + 1, (int64_t)148 * 16);
  widen_u16_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, n);
  return cuda_check(cudaGetLastError(), "widen_u16 launch");
}

int sssd_gather_tails(const void* seq, int32_t elem_bytes, const int64_t* off, const int32_t* len, int32_t B,
                      int32_t P, uint32_t* tails, int64_t* tails_off, int32_t* tails_len, void* stream) {
  if (B < 0 || P < 1 || P > SSSD_MAX_P || (elem_bytes != 2 && elem_bytes != 4))
    return fail(SSSD_E_ARG, "gather_tails: bad arguments");
  if (B == 0) return SSSD_OK;
  if (!seq || !off || !len || !tails || !tails_off || !tails_len) return fail(SSSD_E_ARG, "gather_tails: null buffer");
  gather_tails_kernel<<<(B + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(seq, elem_bytes, off, len, B, P,
                                                                                        tails, tails_off, tails_len);
  return cuda_check(cudaGetLastError(), "gather_tails launch");
}

size_t sssd_sa_check_workspace(uint64_t n) { return ((n + 31) / 32) * 4 + 64; }

int sssd_sa_check(const uint32_t* tokens, uint64_t n, const uint32_t* rows, uint64_t n_rows, void* workspace,
                  size_t workspace_bytes, unsigned long long* counts, void* stream) {
  if (!tokens || !rows || !counts) return fail(SSSD_E_ARG, "sa_check needs tokens, rows and counts");
  if (!workspace || workspace_bytes < sssd_sa_check_workspace(n))
    return fail(SSSD_E_WORKSPACE, "sa_check needs %zu workspace bytes", sssd_sa_check_workspace(n));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint32_t* bits = static_cast<uint32_t*>(workspace);
  const uint64_t words = (n + 31) / 32;
  int rc = cuda_check(cudaMemsetAsync(bits, 0, words * 4, st), "sa_check memset");
  if (!rc) rc = cuda_check(cudaMemsetAsync(counts, 0, 3 * sizeof(unsigned long long), st), "sa_check memset");
  if (rc) return rc;
  if (n_rows > 1)
    sa_check_order_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, st>>>(tokens, n, rows, n_rows, counts);
  if (n_rows)
    sa_check_mark_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, st>>>(rows, n_rows, n, bits, counts + 2);
  if (words) sa_check_count_kernel<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(bits, n, counts + 1);
  return cuda_check(cudaGetLastError(), "sa_check launch");
}

int sssd_rows_sa64(const uint32_t* rows, uint64_t n, uint64_t* sa64_out, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n == 0) return SSSD_OK;
  rows_sa64_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rows, n, sa64_out);
  return cuda_check(cudaGetLastError(), "rows_sa64 launch");
}

}  // extern "C"
