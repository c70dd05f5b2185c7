// Verification side of the decode step (ref draft.py:114-138 verify_greedy,
// draft.py:202-216 GenerationSession.step, harness.py:49-67 TeacherForcedOracle).
//
//   teacher_predict_kernel  node predictions of a teacher-forced greedy model
//   accept_kernel           one warp per request: greedy walk, bonus token and
//                           in-place append of the emitted tokens
//   kv_compact_kernel       move the accepted tree rows of the KV cache to the
//                           contiguous positions after the committed prefix
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace sssd {
int fail(int code, const char* fmt, ...);
int cuda_check(cudaError_t e, const char* what);

constexpr uint32_t kExhausted = 0xffffffffu;  // ref harness.py:29-32

__global__ void teacher_predict_kernel(const int32_t* depths, const int32_t* size, int32_t S,
                                       const uint32_t* ref, const int64_t* ref_off,
                                       const int32_t* ref_len, const int32_t* seq_len,
                                       const int32_t* prompt_len, int32_t B, uint32_t* pred) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * S) return;
  const int b = (int)(t / S), i = (int)(t % S);
  uint32_t v = kExhausted;
  if (i < size[b]) {
    const int64_t idx = (int64_t)seq_len[b] - prompt_len[b] + depths[t];
    if (idx >= 0 && idx < ref_len[b]) v = ref[ref_off[b] + idx];
  }
  pred[t] = v;
}

__global__ void accept_kernel(const uint32_t* tokens, const int32_t* parents, const int32_t* size,
                              int32_t S, const uint32_t* pred, int32_t B, uint32_t* seq,
                              const int64_t* seq_off, int32_t* seq_len, const int32_t* seq_cap,
                              int32_t* path, int32_t* n_acc, uint32_t* bonus, int32_t* emitted) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = lane_id();
  if (b >= B) return;
  const uint32_t* tk = tokens + (size_t)b * S;
  const int32_t* pa = parents + (size_t)b * S;
  const uint32_t* pr = pred + (size_t)b * S;
  int32_t* pth = path + (size_t)b * S;
  const int n = size[b];
  int cur = 0, k = 0;
  while (true) {
    const uint32_t want = pr[cur];
    int nxt = -1;
    for (int j0 = cur + 1; j0 < n; j0 += 32) {  // children follow their parent in DFS order
      const int j = j0 + lane;
      const bool hit = j < n && pa[j] == cur && tk[j] == want;
      const uint32_t hb = __ballot_sync(SSSD_FULL, hit);
      if (hb) {
        nxt = j0 + __ffs(hb) - 1;
        break;
      }
    }
    if (nxt < 0) break;
    if (lane == 0) pth[k] = nxt;
    ++k;
    cur = nxt;
  }
  if (lane == 0) {
    const uint32_t bon = pr[cur];
    n_acc[b] = k;
    bonus[b] = bon;
    emitted[b] = k + 1;
    int L = seq_len[b];
    uint32_t* s = seq + seq_off[b];
    const int cap = seq_cap[b];
    for (int j = 0; j < k && L < cap; ++j) s[L++] = tk[pth[j]];
    if (L < cap) s[L++] = bon;
    seq_len[b] = L;
  }
}

// kv: [layer][b][head][max_pos][d] bf16 (as u16).  For each request, rows
// base + path[k] (k < n_acc) move to base + 1 + k; path is increasing so the
// copy is done in order by one warp per (layer, b, head).
__global__ void kv_compact_kernel(uint16_t* kv, int32_t n_layers, int32_t B, int32_t n_heads,
                                  int32_t max_pos, int32_t head_dim, const int32_t* base,
                                  const int32_t* path, const int32_t* n_acc, int32_t S) {
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = lane_id();
  if (w >= (int64_t)n_layers * B * n_heads) return;
  const int h = (int)(w % n_heads);
  const int b = (int)((w / n_heads) % B);
  const int layer = (int)(w / ((int64_t)n_heads * B));
  uint16_t* rows = kv + (((int64_t)layer * B + b) * n_heads + h) * (int64_t)max_pos * head_dim;
  const int na = n_acc[b];
  for (int k = 0; k < na; ++k) {
    const int src = base[b] + path[(size_t)b * S + k];
    const int dst = base[b] + 1 + k;
    if (src == dst) continue;
    for (int d = lane; d < head_dim; d += 32) rows[(int64_t)dst * head_dim + d] = rows[(int64_t)src * head_dim + d];
    __syncwarp();
  }
}

}  // namespace sssd

using namespace sssd;

extern "C" {

int sssd_teacher_predict(const int32_t* depths, const int32_t* size, int32_t S,
                         const uint32_t* ref, const int64_t* ref_off, const int32_t* ref_len,
                         const int32_t* seq_len, const int32_t* prompt_len, int32_t B,
                         uint32_t* pred, void* stream) {
  if (B <= 0 || S <= 0) return B == 0 ? SSSD_OK : fail(SSSD_E_ARG, "bad batch");
  const int64_t n = (int64_t)B * S;
  teacher_predict_kernel<<<(unsigned)((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      depths, size, S, ref, ref_off, ref_len, seq_len, prompt_len, B, pred);
  return cuda_check(cudaGetLastError(), "teacher_predict launch");
}

int sssd_accept(const uint32_t* tokens, const int32_t* parents, const int32_t* size, int32_t S,
                const uint32_t* pred, int32_t B, uint32_t* seq, const int64_t* seq_off,
                int32_t* seq_len, const int32_t* seq_cap, int32_t* path, int32_t* n_acc,
                uint32_t* bonus, int32_t* emitted, void* stream) {
  if (B <= 0) return B == 0 ? SSSD_OK : fail(SSSD_E_ARG, "bad batch");
  accept_kernel<<<(B + 3) / 4, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      tokens, parents, size, S, pred, B, seq, seq_off, seq_len, seq_cap, path, n_acc, bonus, emitted);
  return cuda_check(cudaGetLastError(), "accept launch");
}

int sssd_kv_compact(uint16_t* kv, int32_t n_layers, int32_t B, int32_t n_heads, int32_t max_pos,
                    int32_t head_dim, const int32_t* base, const int32_t* path,
                    const int32_t* n_acc, int32_t S, void* stream) {
  const int64_t warps = (int64_t)n_layers * B * n_heads;
  if (warps <= 0) return SSSD_OK;
  kv_compact_kernel<<<(unsigned)((warps + 3) / 4), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      kv, n_layers, B, n_heads, max_pos, head_dim, base, path, n_acc, S);
  return cuda_check(cudaGetLastError(), "kv_compact launch");
}

}  // extern "C"
