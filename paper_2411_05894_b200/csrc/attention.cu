// Tree-attention verification (placeholder until the tcgen05 kernel lands).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace sssd {
int fail(int code, const char* fmt, ...);
}

extern "C" {

size_t sssd_tree_attention_workspace(int32_t B, int32_t S, int32_t Hq, int32_t max_pos) {
  (void)B; (void)S; (void)Hq; (void)max_pos;
  return 0;
}

int sssd_tree_attention(const uint16_t* q, const uint16_t* k, const uint16_t* v,
                        const uint64_t* mask, const int32_t* ctx_len, int32_t B, int32_t S,
                        int32_t Hq, int32_t Hkv, int32_t max_pos, int32_t head_dim, float scale,
                        uint16_t* o, void* workspace, size_t workspace_bytes, void* stream) {
  return sssd::fail(SSSD_E_ARG, "tree attention not built yet");
}

}
