// Kernel-side configuration and launch declarations of the propose path.
#pragma once
#include <stdint.h>

#include "common.cuh"

namespace sssd {

struct KCfg {
  int b0, b1;  // request range [b0, b1) handled by this launch (blockIdx.x is relative to b0)
  int P, S, BL, IBL, M, T, use_ds, use_in, n_trees, has_sep;
  int TS;     // row stride of the gathered continuation table (propose: BL rounded up to 4)
  int tab16;  // table rows 16-byte aligned with TS % 4 == 0 (vector compares)
  uint32_t sep;
  int disc_stride;
  const double* disc;
  int fusion;  // 0 = level-synchronous (fusion_ls.cu), 1 = heap order (fusion.cu)
  const int32_t* seq_len;  // [B] live lengths for position ids (nullptr: pos = depth)
  // optional input index (N2, sssd_input_index); idx_len == nullptr: stateless scan
  const uint32_t* idx_keys;
  const int64_t* idx_off;
  const int32_t* idx_len;
  int idx_pb;
};

// Optional per-node outputs of a flattened draft (priority / source rank /
// position id, see sssd_draft_out); shared by both fusion kernels.
__device__ __forceinline__ void write_node_extra(const sssd_draft_out& out, const KCfg& c, int b, int k,
                                                 double prio, int32_t src, int32_t depth) {
  const size_t o = (size_t)b * c.S + k;
  if (out.priority) out.priority[o] = prio;
  if (out.source) out.source[o] = src;
  if (out.pos) out.pos[o] = depth < 0 ? -1 : (c.seq_len ? c.seq_len[b] - 1 : 0) + depth;
}

// Source descriptors of request b (rank 0 = datastore, rank r >= 1 = input
// tree p = P - r + 1), written by propose_setup_kernel -- or built in place by
// the CTA fusion kernel for small launches (one launch fewer on the latency
// path).
struct SetupSrc {
  sssd_seqs seqs;
  Cols dsc, inc;
  const int32_t* ds_n;
  const int32_t* in_n;
};
__device__ __forceinline__ SrcDesc make_src_desc(const SetupSrc& u, const KCfg& c, int b, int rk) {
  SrcDesc d;
  if (rk == 0) {
    d.meta = u.dsc.meta + (size_t)b * u.dsc.stride;
    d.orig = u.dsc.orig + (size_t)b * u.dsc.stride;
    d.tok = u.dsc.tok + (size_t)b * u.dsc.stride * c.BL;
    d.stride = u.dsc.stride;
    d.n = c.use_ds ? u.ds_n[b] : 0;
    d.thr = 0;
    d.depth = c.BL;
  } else {
    const int p = c.P - rk + 1;
    d.meta = u.inc.meta + (size_t)b * u.inc.stride;
    d.orig = u.inc.orig + (size_t)b * u.inc.stride;
    d.tok = u.inc.tok + (size_t)b * u.inc.stride * c.IBL;
    d.stride = u.inc.stride;
    d.n = (c.use_in && p <= c.n_trees) ? u.in_n[b] : 0;
    d.thr = p;
    d.depth = c.IBL;
  }
  d.pad = 0;
  return d;
}

struct Child;
#ifdef SSSD_LK_PROBE
void lk_probe_set(long long* p);  // measurement builds: per-phase cycles of ds_lookup_warp_kernel
#endif

__global__ void find_ranges_kernel(sssd_ds ds, const uint32_t* pat, const int64_t* pat_off,
                                   const int32_t* pat_len, int32_t B, int64_t* lo_hi);

__global__ void ds_lookup_kernel(sssd_ds ds, sssd_seqs seqs, KCfg c, uint32_t* ds_tab,
                                 uint8_t* ds_len, sssd_elem* ds_el, int32_t* ds_n,
                                 sssd_lookup_out lk, sssd_elem* ds_raw, uint32_t* ds_idx,
                                 int64_t idx_cap, Cols cols, const int64_t* pre_bounds,
                                 const uint32_t* pre_rows);
// datastore element folding for the level-synchronous fusion (weights <= 65535)
__host__ __device__ inline bool ds_dedupe_enabled(const KCfg& c) { return c.fusion == 0 && c.P * c.M <= 12000; }

__global__ void ds_dedupe_kernel(KCfg c, const uint32_t* ds_tab, const sssd_elem* ds_el, int32_t* ds_n, Cols cols);
__global__ void ds_lookup_warp_kernel(sssd_ds ds, sssd_seqs seqs, KCfg c, uint32_t* ds_tab, uint8_t* ds_len,
                                      sssd_elem* ds_el, int32_t* ds_n, sssd_lookup_out lk, Cols cols);
__global__ void shard_search_kernel(sssd_ds ds, sssd_seqs seqs, KCfg c, int64_t* bounds);
__global__ void shard_gather_kernel(sssd_ds ds, KCfg c, int B, const int64_t* gbounds, uint32_t* xrows);
__global__ void shard_gather_pos_kernel(sssd_ds ds, KCfg c, int B, const int64_t* gbounds, uint32_t* xpos);
__global__ void rows_from_pos_kernel(const uint32_t* tokens, uint64_t n, const uint32_t* xpos, int64_t count,
                                     uint32_t* rows);

// scratch of the datastore lookup when a separator forces a block sort
__host__ __device__ inline int64_t ds_idx_cap(int P, int M) {
  int64_t n = (int64_t)P * M, p2 = 1;
  while (p2 < n) p2 <<= 1;
  return p2;
}
constexpr int kRowStride = 16;  // u32 per staged suffix row in shared memory
// dynamic shared memory of ds_lookup_kernel (u32 words): one staged row per
// thread, and room for the separator sort's index array up to 4096 entries
__host__ __device__ inline int ds_lookup_smem_words(int P, int M) {
  const int64_t cap = ds_idx_cap(P, M);
  const int rows = P * 32 * kRowStride;
  return rows > (cap < 4096 ? (int)cap : 4096) ? rows : (cap < 4096 ? (int)cap : 4096);
}
// ds_lookup_kernel folds in place (its dynamic shared memory holds the group
// starts) instead of leaving it to a separate ds_dedupe_kernel launch
__host__ __device__ inline bool ds_dedupe_in_lookup(int P, int M) { return P * M + 1 <= ds_lookup_smem_words(P, M); }
// input scan launch shape: 1024 threads once a context spans several
// 2048-position tiles (fewer sequential tiles, wider occurrence sort)
inline int input_scan_threads(int max_len) { return max_len > 4096 ? 1024 : 256; }
__host__ __device__ inline int input_scan_smem_bytes(int threads, int ibl) {
  int need = threads * (ibl + 6);
  // long contexts (1024 threads, 2 CTAs per SM): room for the packed keys of
  // up to 4096 occurrences (6 words each), sorted in shared memory
  if (threads >= 1024 && need < 4096 * 6) need = 4096 * 6;
  return 4 * (need > 4096 ? need : 4096);
}
__global__ void input_scan_kernel(sssd_seqs seqs, KCfg c, sssd_elem* raw, sssd_elem* sorted,
                                  int32_t* in_n, uint32_t* idx_ws, int64_t cap, int64_t cap2,
                                  Cols cols);
__global__ void input_index_build_kernel(sssd_seqs seqs, sssd_input_index ix, const int32_t* rows);
__global__ void sort_sources_kernel(const uint32_t* tok, const sssd_elem* el,
                                    const int64_t* el_off, const int32_t* el_n, sssd_elem* sorted,
                                    uint32_t* idx_ws, int64_t idx_cap, Cols cols);
struct Group;
__global__ void draft_kernel(const SrcDesc* desc, const uint32_t* root_tok, KCfg c, Child* slabs,
                             uint32_t slab_cap, Child* pool, unsigned long long* cursor,
                             uint64_t pool_cap, int32_t* err, uint8_t* gover, int64_t gover_bytes,
                             sssd_draft_out out, long long* cycles, const int32_t* order);
__device__ __forceinline__ int lpt_bucket(const SrcDesc* d, int P) {
  long long cost = d[0].n;
  for (int r = 1; r <= P; ++r) cost += d[r].n;
  return 63 - min(63, 2 * (63 - __clzll(cost + 1)));  // 2 buckets per octave, largest first
}
__global__ void lpt_scatter_kernel(const uint8_t* bucket, const int32_t* hist, int32_t* fill, int b0, int b1,
                                   int32_t* order);

// level-synchronous fusion: level-node and parent record bytes, and how many
// of each a warp keeps in shared memory (larger levels use the fusion pool)
constexpr int kLsLevelBytes = 56;
constexpr int kLsParBytes = 32;
#ifndef SSSD_LS_CAP
// 96 nodes (9.8 KB per warp with the parent / top buffers): 24 warps per SM
// at 80 registers; 128 nodes (20 warps) drafts cfg2 4.7 % slower, B = 64
// batches ~6 % faster (fewer regenerations of cut levels)
#define SSSD_LS_CAP 96
#endif
constexpr int kLsCap = SSSD_LS_CAP;
#ifndef SSSD_LS_PARCAP
#define SSSD_LS_PARCAP 32  // 8.7 KB per warp: 24 warps per SM (64 parents: 21; cfg2 fusion 0.479 -> 0.469 ms)
#endif
constexpr int kLsParCap = SSSD_LS_PARCAP;
constexpr int kLsRankWords = SSSD_MAX_P + 1;  // per-rank class counters (ranks 0..P)
int ls_smem_bytes(int P, int S);
__global__ void draft_ls_kernel(const SrcDesc* desc, const uint32_t* root_tok, KCfg c, uint8_t* pool,
                                unsigned long long* cursor, uint64_t pool_bytes, int32_t* err,
                                sssd_draft_out out, long long* cycles, const int32_t* order,
                                const int32_t* order_count = nullptr);
// the same kernel for small launches: element loads issued one chunk ahead
__global__ void draft_ls_small_kernel(const SrcDesc* desc, const uint32_t* root_tok, KCfg c, uint8_t* pool,
                                      unsigned long long* cursor, uint64_t pool_bytes, int32_t* err,
                                      sssd_draft_out out, long long* cycles, const int32_t* order,
                                      const int32_t* order_count = nullptr);

// CTA-per-request form (fusion_cta.cu): the same level-synchronous fusion with
// a level's generation and sort spread over the warps of one CTA (small launches)
int cta_smem_bytes(int P, int S);
int cta_threads();
// use_su: build the source descriptors and root tokens from su in the kernel
// (desc / root_tok unused)
__global__ void draft_cta_kernel(const SrcDesc* desc, const uint32_t* root_tok, KCfg c, uint8_t* pool,
                                 unsigned long long* cursor, uint64_t pool_bytes, int32_t* err, sssd_draft_out out,
                                 long long* cycles, const int32_t* order, SetupSrc su, int use_su);

// all-nodes fusion (fusion_ane.cu): every live source node of a request in
// shared memory, threshold + sort instead of level-by-level expansion; the
// requests that outgrow these tables go to draft_ls_kernel through fb
// (fb[0] = count, fb[1..] = requests)
constexpr int kAneNodes = 2048;
constexpr int kAneElems = 1024;
constexpr int kAneCands = 256;
int ane_smem_bytes();
__global__ void draft_ane_kernel(const SrcDesc* desc, const uint32_t* root_tok, KCfg c, sssd_draft_out out,
                                 int32_t* fb);

constexpr int kChildBytes = 32;
constexpr int kGroupBytes = 16;  // cold group record
constexpr int kGroupSmem = 128;  // groups kept in shared memory; later ones spill to global
constexpr int kChildSmem = 48;   // child records in the shared-memory slab

// Upper bound on sibling groups: one per source seed plus one per pop, and a
// draft node can be popped at most once per source.
__host__ __device__ inline int draft_max_groups(int P, int S) { return (P + 1) * S + P + 1; }

inline int draft_smem_bytes(int P, int S) {
  const int G = draft_max_groups(P, S);
  const int Gs = G < kGroupSmem ? G : kGroupSmem;
  return kChildSmem * kChildBytes + Gs * (kGroupBytes + 12) + S * 4 + S * 2 * 8 + 16;
}

// global overflow bytes per request: cold records + live-list slots beyond kGroupSmem
inline int64_t draft_group_overflow_bytes(int P, int S) {
  const int G = draft_max_groups(P, S);
  const int Go = G > kGroupSmem ? G - kGroupSmem : 0;
  return ((int64_t)Go * (kGroupBytes + 12) + 127) / 128 * 128;
}

}  // namespace sssd
