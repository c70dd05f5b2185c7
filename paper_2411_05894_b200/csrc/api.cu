// C-ABI entry points of libsssd.so (see include/sssd.h): argument validation,
// workspace carving and kernel launches.  No allocation, no synchronisation
// (except the explicit sssd_workspace_status).
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

#include <string>

#include "common.cuh"
#include "propose.cuh"

namespace sssd {

static thread_local std::string g_err;
static long long* g_cycles = nullptr;  // optional per-request fusion-kernel cycle counts

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SSSD_OK;
  return fail(SSSD_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bump-carve a workspace; with base == nullptr it only measures.
struct Carver {
  uint8_t* base;
  size_t off;
  template <class T>
  T* take(size_t n) {
    off = align_up(off, 128);
    // with base == nullptr the returned "pointer" is the byte offset
    T* p = reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(base) + off);
    off += n * sizeof(T);
    return p;
  }
};

static int validate_cfg(const sssd_cfg* c) {
  if (!c) return fail(SSSD_E_ARG, "cfg is NULL");
  if (c->P < 1) return fail(SSSD_E_ARG, "P must be >= 1, got %d", c->P);
  if (c->P > SSSD_MAX_P) return fail(SSSD_E_LIMIT, "P=%d exceeds the compiled limit %d", c->P, SSSD_MAX_P);
  if (c->dec_len < 1) return fail(SSSD_E_ARG, "dec_len must be >= 1, got %d", c->dec_len);
  if (c->dec_len > SSSD_MAX_DRAFT)
    return fail(SSSD_E_LIMIT, "dec_len=%d exceeds the compiled limit %d", c->dec_len, SSSD_MAX_DRAFT);
  if (c->branch_len < 1) return fail(SSSD_E_ARG, "branch_len must be >= 1, got %d", c->branch_len);
  if (c->input_branch_len < 1)
    return fail(SSSD_E_ARG, "input_branch_len must be >= 1, got %d", c->input_branch_len);
  if (c->branch_len > SSSD_MAX_DEPTH || c->input_branch_len > SSSD_MAX_DEPTH)
    return fail(SSSD_E_LIMIT, "branch lengths exceed the compiled limit %d", SSSD_MAX_DEPTH);
  if (c->M < 1) return fail(SSSD_E_ARG, "M must be >= 1, got %d", c->M);
  if (c->T < 1) return fail(SSSD_E_ARG, "T must be >= 1, got %d", c->T);
  if (c->n_input_trees < 0 || c->n_input_trees > c->P)
    return fail(SSSD_E_ARG, "got %d input trees for P=%d", c->n_input_trees, c->P);
  const int md = c->branch_len > c->input_branch_len ? c->branch_len : c->input_branch_len;
  if (c->disc_stride < md + 1) return fail(SSSD_E_ARG, "disc_stride %d < max depth + 1", c->disc_stride);
  if (!c->disc) return fail(SSSD_E_ARG, "discount table is NULL");
  if (c->fusion != 0 && c->fusion != 1) return fail(SSSD_E_ARG, "fusion must be 0 or 1, got %d", c->fusion);
  return SSSD_OK;
}

static int merge_depth(const sssd_cfg* cfg) { return cfg->disc_stride - 1; }

static KCfg kcfg(const sssd_cfg* c) {
  KCfg k;
  k.b0 = 0;
  k.b1 = 0;
  k.P = c->P;
  k.S = c->dec_len;
  k.BL = c->branch_len;
  k.TS = (c->branch_len + 3) & ~3;
  k.tab16 = 1;
  k.IBL = c->input_branch_len;
  k.M = c->M;
  k.T = c->T;
  k.use_ds = c->use_datastore;
  k.use_in = c->use_input;
  k.n_trees = c->n_input_trees;
  k.has_sep = c->has_separator;
  k.sep = c->separator;
  k.disc_stride = c->disc_stride;
  k.disc = c->disc;
  k.fusion = c->fusion;
  k.seq_len = nullptr;
  k.idx_keys = nullptr;
  k.idx_off = nullptr;
  k.idx_len = nullptr;
  k.idx_pb = 0;
  return k;
}

constexpr uint32_t kSlabChildren = 2048;

struct DraftWs {
  int32_t* order;
  int32_t* fb;  // all-nodes fusion fallback list: [0] = count, [1..] = requests
  uint8_t* bucket;
  int32_t* hist;  // [64] histogram + [64] fill cursors (zeroed with the status words)
  uint8_t* gover;
  int64_t gover_bytes;
  SrcDesc* desc;
  uint32_t* root;
  Child* slabs;
  Child* pool;
  unsigned long long* cursor;
  int32_t* err;
  uint64_t pool_cap;
};

// Fusion arena: a per-request slab (stack of sibling-group child lists) plus a
// shared overflow pool.  An expansion reserves its element-range size and
// returns the unused tail, so the slab holds the typical request; long
// contexts (huge input-tree roots) spill into the pool, sized by max_len.
// Status block (cursor, err, LPT histogram): always the first 528 bytes of a
// propose or merge workspace, so the status word sits at a fixed offset
// (kStatusErrOffset) whatever B / max_len the workspace was carved for.
constexpr size_t kStatusWords = 2 + 64;
constexpr size_t kStatusErrOffset = 8;
static unsigned long long* carve_status(Carver& cv) { return cv.take<unsigned long long>(kStatusWords); }

static DraftWs carve_draft(Carver& cv, unsigned long long* status, int P, int S, int B, int64_t max_len = 0) {
  DraftWs d;
  d.order = cv.take<int32_t>((size_t)B);
  d.fb = cv.take<int32_t>((size_t)B + 1);
  d.bucket = cv.take<uint8_t>((size_t)B);
  d.gover_bytes = draft_group_overflow_bytes(P, S);
  d.gover = cv.take<uint8_t>((size_t)B * (d.gover_bytes ? d.gover_bytes : 1));
  d.desc = cv.take<SrcDesc>((size_t)B * (P + 1));
  d.root = cv.take<uint32_t>((size_t)B);
  d.slabs = reinterpret_cast<Child*>(cv.take<uint8_t>((size_t)B * kSlabChildren * kChildBytes));
  d.pool_cap = (1u << 16) + (uint64_t)B * 1024 +
               (max_len > (int64_t)kSlabChildren ? (uint64_t)B * (P + 1) * (uint64_t)max_len : 0);
  d.pool = reinterpret_cast<Child*>(cv.take<uint8_t>((size_t)d.pool_cap * kChildBytes));
  d.cursor = status;  // cursor + err (status words) + LPT histogram
  d.err = reinterpret_cast<int32_t*>(d.cursor + 1);
  d.hist = reinterpret_cast<int32_t*>(d.cursor + 2);
  return d;
}

struct PropWs {
  uint32_t* ds_tab;
  uint8_t* ds_len;
  sssd_elem* ds_el;
  int32_t* ds_n;
  sssd_elem* ds_raw;
  uint32_t* ds_idx;
  int64_t ds_idx_cap;
  sssd_elem* in_raw;
  sssd_elem* in_el;
  int32_t* in_n;
  uint32_t* idx;
  Cols ds_cols, in_cols;
  int64_t cap, cap2;
  DraftWs d;
  size_t bytes;
};

static PropWs carve_propose(uint8_t* base, const sssd_cfg* c, int B, int max_len) {
  Carver cv{base, 0};
  unsigned long long* status = carve_status(cv);
  PropWs w;
  const size_t PM = (size_t)c->P * c->M;
  w.ds_tab = cv.take<uint32_t>((size_t)B * PM * ((c->branch_len + 3) & ~3));  // 16-byte rows (KCfg::TS)
  w.ds_len = cv.take<uint8_t>((size_t)B * PM);
  w.ds_el = cv.take<sssd_elem>((size_t)B * PM);
  w.ds_n = cv.take<int32_t>((size_t)B);
  const bool sep = c->has_separator != 0;
  w.ds_idx_cap = ds_idx_cap(c->P, c->M);
  w.ds_raw = cv.take<sssd_elem>(sep ? (size_t)B * PM : 1);
  w.ds_idx = cv.take<uint32_t>(sep && w.ds_idx_cap > ds_lookup_smem_words(c->P, c->M) ? (size_t)B * w.ds_idx_cap : 1);
  w.cap = max_len > 1 ? max_len : 1;
  int64_t p2 = 1;
  while (p2 < w.cap) p2 <<= 1;
  w.cap2 = w.cap > 4096 ? p2 : 0;
  w.in_raw = cv.take<sssd_elem>((size_t)B * w.cap);
  w.in_el = cv.take<sssd_elem>((size_t)B * w.cap);
  w.in_n = cv.take<int32_t>((size_t)B);
  w.idx = cv.take<uint32_t>((size_t)B * (w.cap2 ? w.cap2 : 1));
  w.ds_cols.stride = (int64_t)PM;
  w.ds_cols.meta = cv.take<uint32_t>((size_t)B * PM);
  w.ds_cols.orig = cv.take<uint32_t>((size_t)B * PM);
  w.ds_cols.tok = cv.take<uint32_t>((size_t)B * PM * c->branch_len);
  w.in_cols.stride = w.cap;
  w.in_cols.meta = cv.take<uint32_t>((size_t)B * w.cap);
  w.in_cols.orig = cv.take<uint32_t>((size_t)B * w.cap);
  w.in_cols.tok = cv.take<uint32_t>((size_t)B * w.cap * c->input_branch_len);
  w.d = carve_draft(cv, status, c->P, c->dec_len, B, w.cap);
  w.bytes = align_up(cv.off, 256);
  return w;
}

__global__ void propose_setup_kernel(sssd_seqs seqs, KCfg c, Cols dsc, const int32_t* ds_n,
                                     Cols inc, const int32_t* in_n, SrcDesc* desc, uint32_t* root,
                                     uint8_t* bucket, int32_t* hist) {
  __shared__ int sh[64];  // block histogram of LPT buckets (one global atomic per bucket and block)
  if (bucket && threadIdx.x < 64) sh[threadIdx.x] = 0;
  if (bucket) __syncthreads();
  const int b = c.b0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (b < c.b1) {
    const int L = seqs.seq_len[b];
    root[b] = seqs.seq[seqs.seq_off[b] + L - 1];
    SrcDesc* d = desc + (size_t)b * (c.P + 1);
    const SetupSrc u{seqs, dsc, inc, ds_n, in_n};
    for (int rk = 0; rk <= c.P; ++rk) d[rk] = make_src_desc(u, c, b, rk);
    if (bucket) {
      const int k = lpt_bucket(d, c.P);
      bucket[b] = (uint8_t)k;
      atomicAdd(&sh[k], 1);
    }
  }
  if (bucket) {
    __syncthreads();
    if (threadIdx.x < 64 && sh[threadIdx.x]) atomicAdd(&hist[threadIdx.x], sh[threadIdx.x]);
  }
}

__global__ void merge_setup_kernel(Cols cols, const int64_t* el_off, const int32_t* el_n,
                                   const uint32_t* roots, int B, KCfg c, SrcDesc* desc,
                                   uint32_t* root) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  root[b] = roots[b];
  SrcDesc* d = desc + (size_t)b * (c.P + 1);
  for (int rk = 0; rk <= c.P; ++rk) {
    const int s = rk == 0 ? 0 : c.P - rk + 1;  // source slot: 0 = datastore, p = input tree p
    const bool live = rk == 0 || s <= c.n_trees;
    const size_t bs = (size_t)b * (c.P + 1) + s;
    const int64_t o = live ? el_off[bs] : 0;
    d[rk].meta = cols.meta + o;
    d[rk].orig = cols.orig + o;
    d[rk].tok = cols.tok + o;
    d[rk].stride = cols.stride;
    d[rk].n = live ? el_n[bs] : 0;
    d[rk].thr = 0;
    d[rk].depth = (int32_t)(c.disc_stride - 1);
    d[rk].pad = 0;
  }
}

static int input_scan_attr(int ibl) {
  return cuda_check(cudaFuncSetAttribute(input_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         input_scan_smem_bytes(1024, ibl)), "input_scan_kernel smem attribute");
}

static int fusion_smem_attr(const KCfg& k) {
  if (k.fusion == 1)
    return cuda_check(cudaFuncSetAttribute(draft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           draft_smem_bytes(k.P, k.S)), "draft_kernel smem attribute");
  if (int rc = cuda_check(cudaFuncSetAttribute(draft_ane_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               ane_smem_bytes()), "draft_ane_kernel smem attribute"))
    return rc;
  if (int rc = cuda_check(cudaFuncSetAttribute(draft_ls_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               ls_smem_bytes(k.P, k.S)), "draft_ls_small_kernel smem attribute"))
    return rc;
  if (int rc = cuda_check(cudaFuncSetAttribute(draft_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               cta_smem_bytes(k.P, k.S)), "draft_cta_kernel smem attribute"))
    return rc;
  return cuda_check(cudaFuncSetAttribute(draft_ls_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         ls_smem_bytes(k.P, k.S)), "draft_ls_kernel smem attribute");
}

// Fusion form switch (A/B and cross-checks; identical drafts in every form):
// -1 = automatic (CTA-per-request form for launches of <= cta_max() requests,
// one warp per request above), 0 = one warp per request only, 1 = all-nodes
// kernel first (fusion_ane.cu), 2 = CTA-per-request form for every launch.
// SSSD_FUSION_FORM (or the older SSSD_FUSION_ANE=0/1) sets the start value.
static int g_fusion_form = [] {
  const char* e = getenv("SSSD_FUSION_FORM");
  if (!e) e = getenv("SSSD_FUSION_ANE");
  return e && e[0] >= '0' && e[0] <= '2' ? e[0] - '0' : -1;
}();
static bool ane_enabled(int) { return g_fusion_form == 1; }

// Launches of at most this many requests use draft_ls_small_kernel (few warps
// per SM: load latency, not issue slots, bounds them); SSSD_LS_SMALL overrides.
static int ls_small_max() {
  static const int v = getenv("SSSD_LS_SMALL") ? atoi(getenv("SSSD_LS_SMALL")) : 1024;
  return v;
}

// Launches of at most this many requests use draft_cta_kernel (one CTA of
// cta_threads() per request: the latency of a small batch is its slowest
// request's dependency chain, which the CTA form shortens).
static int cta_max() {
  static const int v = getenv("SSSD_CTA_MAX") ? atoi(getenv("SSSD_CTA_MAX")) : 512;
  return v;
}
static bool getenv_cached_no_inline_setup() {  // A/B switch: SSSD_NO_INLINE_SETUP keeps the setup kernel
  static const bool v = getenv("SSSD_NO_INLINE_SETUP") != nullptr;
  return v;
}
static bool cta_enabled(int nb) { return g_fusion_form == 2 || (g_fusion_form < 0 && nb <= cta_max()); }

// One fusion + flatten launch over requests [k.b0, k.b0 + nb) (or order[] of them).
static void launch_fusion(const DraftWs& d, const KCfg& k, int nb, const sssd_draft_out* out,
                          cudaStream_t st, long long* cyc, const int32_t* order, const SetupSrc* su = nullptr) {
  if (k.fusion == 1)
    draft_kernel<<<nb, 32, draft_smem_bytes(k.P, k.S), st>>>(d.desc, d.root, k, d.slabs, kSlabChildren, d.pool,
                                                             d.cursor, d.pool_cap, d.err, d.gover, d.gover_bytes,
                                                             *out, cyc, order);
  else
  {
    // the level-synchronous kernel uses the heap form's slabs + pool as one pool
    uint8_t* lo = reinterpret_cast<uint8_t*>(d.slabs);
    uint8_t* hi = reinterpret_cast<uint8_t*>(d.pool) + d.pool_cap * kChildBytes;
    if (ane_enabled(nb)) {
      // all-nodes fusion; the requests it lists in d.fb go to the level-synchronous kernel
      cudaMemsetAsync(d.fb, 0, sizeof(int32_t), st);
      draft_ane_kernel<<<nb, 32, ane_smem_bytes(), st>>>(d.desc, d.root, k, *out, d.fb);
      draft_ls_kernel<<<nb, 32, ls_smem_bytes(k.P, k.S), st>>>(d.desc, d.root, k, lo, d.cursor,
                                                               (uint64_t)(hi - lo), d.err, *out, cyc,
                                                               d.fb + 1 - k.b0, d.fb);
      return;
    }
    if (cta_enabled(nb))
      draft_cta_kernel<<<nb, cta_threads(), cta_smem_bytes(k.P, k.S), st>>>(d.desc, d.root, k, lo, d.cursor,
                                                                           (uint64_t)(hi - lo), d.err, *out, cyc,
                                                                           order, su ? *su : SetupSrc{},
                                                                           su != nullptr);
    else if (nb <= ls_small_max())
      draft_ls_small_kernel<<<nb, 32, ls_smem_bytes(k.P, k.S), st>>>(d.desc, d.root, k, lo, d.cursor,
                                                                     (uint64_t)(hi - lo), d.err, *out, cyc, order);
    else
      draft_ls_kernel<<<nb, 32, ls_smem_bytes(k.P, k.S), st>>>(d.desc, d.root, k, lo, d.cursor,
                                                               (uint64_t)(hi - lo), d.err, *out, cyc, order);
  }
}

static int launch_draft(const DraftWs& d, const KCfg& k, int B, const sssd_draft_out* out,
                        cudaStream_t st) {
  int rc = fusion_smem_attr(k);
  if (rc) return rc;
  launch_fusion(d, k, B, out, st, nullptr, nullptr);
  return cuda_check(cudaGetLastError(), "fusion kernel launch");
}

static int validate_out(const sssd_draft_out* out) {
  if (!out || !out->size || !out->tokens || !out->parents || !out->depths || !out->mask)
    return fail(SSSD_E_ARG, "draft output buffers must all be non-NULL");
  return SSSD_OK;
}

}  // namespace sssd

using namespace sssd;

extern "C" {

const char* sssd_error_string(int code) {
  switch (code) {
    case SSSD_OK: return "ok";
    case SSSD_E_ARG: return "invalid argument";
    case SSSD_E_LIMIT: return "compiled limit exceeded";
    case SSSD_E_CUDA: return "CUDA error";
    case SSSD_E_WORKSPACE: return "workspace too small";
    default: return "unknown error";
  }
}

const char* sssd_last_error(void) { return g_err.c_str(); }

int sssd_version(void) { return 1; }

size_t sssd_propose_workspace(const sssd_cfg* cfg, int32_t B, int32_t max_len) {
  if (!cfg || B < 0) return 0;
  return carve_propose(nullptr, cfg, B, max_len).bytes;
}

// Library-internal streams used to fork the independent propose stages off the
// caller's stream (joined back with events, so the caller sees stream order).
// One set per (host thread, device): concurrent proposes from several host
// threads never share fork streams or events (unbounded
// concurrent readers), and lazy creation needs no lock.  (The set lives as
// long as its thread; a thread keeps at most one per device.)
struct Aux {
  cudaStream_t s[2];
  cudaEvent_t fork;
  cudaEvent_t done[2][8];
};

static Aux* aux_streams() {
  thread_local Aux aux[16];
  thread_local bool ready[16] = {false};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
  if (!ready[dev]) {
    Aux& x = aux[dev];
    for (auto& s : x.s)
      if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    if (cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    for (auto& row : x.done)
      for (auto& e : row)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    ready[dev] = true;
  }
  return &aux[dev];
}

static int propose_impl(const sssd_ds* ds, const sssd_seqs* seqs, const sssd_cfg* cfg,
                        const sssd_draft_out* out, const sssd_lookup_out* lookup, void* workspace,
                        size_t workspace_bytes, void* stream, cudaEvent_t* ev,
                        const int64_t* pre_bounds = nullptr, const uint32_t* pre_rows = nullptr,
                        const sssd_input_index* index = nullptr);

int sssd_propose(const sssd_ds* ds, const sssd_seqs* seqs, const sssd_cfg* cfg,
                 const sssd_draft_out* out, const sssd_lookup_out* lookup, void* workspace,
                 size_t workspace_bytes, void* stream) {
  return propose_impl(ds, seqs, cfg, out, lookup, workspace, workspace_bytes, stream, nullptr);
}

int sssd_propose_ex(const sssd_ds* ds, const sssd_seqs* seqs, const sssd_input_index* index, const sssd_cfg* cfg,
                    const sssd_draft_out* out, const sssd_lookup_out* lookup, void* workspace,
                    size_t workspace_bytes, void* stream, float* stage_ms) {
  if (!stage_ms)
    return propose_impl(ds, seqs, cfg, out, lookup, workspace, workspace_bytes, stream, nullptr, nullptr, nullptr,
                        index);
  cudaEvent_t ev[5];
  for (auto& e : ev) cudaEventCreate(&e);
  int rc = propose_impl(ds, seqs, cfg, out, lookup, workspace, workspace_bytes, stream, ev, nullptr, nullptr, index);
  if (!rc) rc = cuda_check(cudaEventSynchronize(ev[4]), "profile sync");
  if (!rc)
    for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&stage_ms[i], ev[i], ev[i + 1]);
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

int sssd_input_index_build(const sssd_seqs* seqs, const sssd_input_index* index, const int32_t* rows,
                           int32_t n_rows, void* stream) {
  if (!seqs || !index || !index->keys || !index->off || !index->len)
    return fail(SSSD_E_ARG, "input index build needs sequences and index buffers");
  if (index->pos_bits < 1 || index->pos_bits > 24) return fail(SSSD_E_ARG, "pos_bits must be in 1..24");
  if (n_rows <= 0) return n_rows == 0 ? SSSD_OK : fail(SSSD_E_ARG, "bad row count");
  const int attr = cuda_check(cudaFuncSetAttribute(input_index_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   4 * SSSD_INDEX_MAX), "index build smem attribute");
  if (attr) return attr;
  input_index_build_kernel<<<n_rows, 1024, 4 * SSSD_INDEX_MAX, static_cast<cudaStream_t>(stream)>>>(*seqs, *index,
                                                                                                    rows);
  return cuda_check(cudaGetLastError(), "input index build launch");
}

int sssd_propose_profile(const sssd_ds* ds, const sssd_seqs* seqs, const sssd_cfg* cfg,
                         const sssd_draft_out* out, void* workspace, size_t workspace_bytes,
                         void* stream, float* stage_ms) {
  cudaEvent_t ev[5];
  for (auto& e : ev) cudaEventCreate(&e);
  int rc = propose_impl(ds, seqs, cfg, out, nullptr, workspace, workspace_bytes, stream, ev);
  if (!rc) rc = cuda_check(cudaEventSynchronize(ev[4]), "profile sync");
  if (!rc)
    for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&stage_ms[i], ev[i], ev[i + 1]);
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

// Per-range fusion state: arena cursor and LPT histogram + fill cursors (one
// launch instead of two memsets; the status word between them is kept).
__global__ void fuse_reset_kernel(unsigned long long* cursor, int32_t* hist) {
  if (threadIdx.x == 0) *cursor = 0;
  hist[threadIdx.x] = 0;  // blockDim = 128: [64] histogram + [64] fill cursors
}

// The three stages over a request range [b0, b1) of a batch whose workspace
// was carved for all of it (outputs and stage buffers are indexed by request).
static void lookup_range(const PropWs& w, const KCfg& k, const sssd_cfg* cfg, const sssd_ds* ds,
                         const sssd_seqs* seqs, const sssd_lookup_out& lk, const int64_t* pre_bounds,
                         const uint32_t* pre_rows, cudaStream_t s, int b0, int b1) {
  KCfg kk = k;
  kk.b0 = b0;
  kk.b1 = b1;
  // one warp per request (lane groups per p) for throughput; small batches
  // keep one warp per p (lower latency per request when SMs are idle)
  if (!cfg->has_separator && !pre_bounds && b1 - b0 >= 2048)
    ds_lookup_warp_kernel<<<(b1 - b0 + 3) / 4, 128, 0, s>>>(*ds, *seqs, kk, w.ds_tab, w.ds_len, w.ds_el, w.ds_n,
                                                              lk, w.ds_cols);
  else
    ds_lookup_kernel<<<b1 - b0, 32 * cfg->P, 4 * ds_lookup_smem_words(cfg->P, cfg->M), s>>>(
        *ds, *seqs, kk, w.ds_tab, w.ds_len, w.ds_el, w.ds_n, lk, w.ds_raw, w.ds_idx, w.ds_idx_cap, w.ds_cols,
        pre_bounds, pre_rows);
  if (ds_dedupe_enabled(kk) && (cfg->has_separator || pre_bounds || b1 - b0 < 2048) &&
      !ds_dedupe_in_lookup(cfg->P, cfg->M))  // (the warp kernel and, below 4096 samples, ds_lookup_kernel fold themselves)
    ds_dedupe_kernel<<<b1 - b0, 128, 4 * (cfg->P * cfg->M + 1), s>>>(kk, w.ds_tab, w.ds_el, w.ds_n, w.ds_cols);
}

static void scan_range(const PropWs& w, const KCfg& k, const sssd_cfg* cfg, const sssd_seqs* seqs, cudaStream_t s,
                       int b0, int b1) {
  KCfg kk = k;
  kk.b0 = b0;
  kk.b1 = b1;
  const int th = input_scan_threads(seqs->max_len);
  input_scan_kernel<<<b1 - b0, th, input_scan_smem_bytes(th, cfg->input_branch_len), s>>>(
      *seqs, kk, w.in_raw, w.in_el, w.in_n, w.idx, w.cap, w.cap2, w.in_cols);
}

// Setup (sources, roots), longest-first order over the range when it spans
// several waves, fusion.  The LPT histogram is per launch: ranges of one
// workspace run in stream order (sssd_propose_phase zeroes it per range).
static void fuse_range(const PropWs& w, const KCfg& k, const sssd_seqs* seqs, const sssd_draft_out* out,
                       cudaStream_t s, int b0, int b1) {
  KCfg kk = k;
  kk.b0 = b0;
  kk.b1 = b1;
  kk.seq_len = seqs->seq_len;
  static const bool no_lpt = getenv("SSSD_NO_LPT") != nullptr;  // A/B switch
  const bool lpt = !no_lpt && b1 - b0 >= 2048;                   // order only pays with several waves
  if (!lpt && kk.fusion == 0 && cta_enabled(b1 - b0) && !getenv_cached_no_inline_setup()) {
    // the CTA fusion kernel builds its source descriptors itself: one launch
    // fewer between the lookup / scan join and the fusion (latency path)
    const SetupSrc su{*seqs, w.ds_cols, w.in_cols, w.ds_n, w.in_n};
    launch_fusion(w.d, kk, b1 - b0, out, s, g_cycles, nullptr, &su);
    return;
  }
  propose_setup_kernel<<<(b1 - b0 + 127) / 128, 128, 0, s>>>(*seqs, kk, w.ds_cols, w.ds_n, w.in_cols, w.in_n,
                                                               w.d.desc, w.d.root, lpt ? w.d.bucket : nullptr,
                                                               w.d.hist);
  if (lpt)
    lpt_scatter_kernel<<<(b1 - b0 + 255) / 256, 256, 0, s>>>(w.d.bucket, w.d.hist, w.d.hist + 64, b0, b1,
                                                               w.d.order);
  launch_fusion(w.d, kk, b1 - b0, out, s, g_cycles, lpt ? w.d.order : nullptr);
}

static int propose_impl(const sssd_ds* ds, const sssd_seqs* seqs, const sssd_cfg* cfg,
                        const sssd_draft_out* out, const sssd_lookup_out* lookup, void* workspace,
                        size_t workspace_bytes, void* stream, cudaEvent_t* ev, const int64_t* pre_bounds,
                        const uint32_t* pre_rows, const sssd_input_index* index) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  if ((rc = validate_out(out))) return rc;
  if (!seqs || seqs->B < 0) return fail(SSSD_E_ARG, "bad sequence batch");
  if (cfg->use_datastore) {
    if (!ds || !ds->rows) return fail(SSSD_E_ARG, "use_datastore requires a datastore");
    if (ds->n_rows == 0 || ds->n_tokens == 0) return fail(SSSD_E_ARG, "empty corpus");
    if (ds->n_tokens >= 0xffffffffull) return fail(SSSD_E_LIMIT, "corpus longer than 2^32-1 tokens");
    if (cfg->P + cfg->branch_len > SSSD_ROW_TOKENS && !ds->tokens)
      return fail(SSSD_E_ARG, "P + branch_len > %d needs the token array", SSSD_ROW_TOKENS);
  }
  const int B = seqs->B;
  if (B == 0) return SSSD_OK;
  const PropWs w = carve_propose(static_cast<uint8_t*>(workspace), cfg, B, seqs->max_len);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(SSSD_E_WORKSPACE, "propose needs %zu workspace bytes, got %zu", w.bytes, workspace_bytes);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  KCfg k = kcfg(cfg);
  if (index) {
    if (!index->keys || !index->off || !index->len || index->pos_bits < 1 || index->pos_bits > 24)
      return fail(SSSD_E_ARG, "bad input index (keys / off / len, pos_bits in 1..24)");
    k.idx_keys = index->keys;
    k.idx_off = index->off;
    k.idx_len = index->len;
    k.idx_pb = index->pos_bits;
  }
  sssd_lookup_out lk{};
  if (lookup) lk = *lookup;
  if ((rc = cuda_check(cudaMemsetAsync(w.d.cursor, 0, 16 + 512, st), "memset status"))) return rc;
  if ((rc = fusion_smem_attr(k))) return rc;
  if ((rc = input_scan_attr(cfg->input_branch_len))) return rc;

  auto launch_lookup = [&](cudaStream_t s, int b0, int b1) {
    lookup_range(w, k, cfg, ds, seqs, lk, pre_bounds, pre_rows, s, b0, b1);
  };
  auto launch_scan = [&](cudaStream_t s, int b0, int b1) { scan_range(w, k, cfg, seqs, s, b0, b1); };
  auto launch_fuse = [&](cudaStream_t s, int b0, int b1) { fuse_range(w, k, seqs, out, s, b0, b1); };

  if (ev) {  // profiling: stages back to back on the caller's stream
    cudaEventRecord(ev[0], st);
    if (cfg->use_datastore) launch_lookup(st, 0, B);
    cudaEventRecord(ev[1], st);
    if (cfg->use_input) launch_scan(st, 0, B);
    cudaEventRecord(ev[2], st);
    KCfg kk = k;
    kk.b0 = 0;
    kk.b1 = B;
    kk.seq_len = seqs->seq_len;
    const bool lpt = getenv("SSSD_NO_LPT") == nullptr && B >= 2048;
    propose_setup_kernel<<<(B + 127) / 128, 128, 0, st>>>(*seqs, kk, w.ds_cols, w.ds_n, w.in_cols, w.in_n,
                                                            w.d.desc, w.d.root, lpt ? w.d.bucket : nullptr,
                                                            w.d.hist);
    if (lpt) lpt_scatter_kernel<<<(B + 255) / 256, 256, 0, st>>>(w.d.bucket, w.d.hist, w.d.hist + 64, 0, B, w.d.order);
    cudaEventRecord(ev[3], st);
    launch_fusion(w.d, kk, B, out, st, g_cycles, lpt ? w.d.order : nullptr);
    cudaEventRecord(ev[4], st);
    return cuda_check(cudaGetLastError(), "propose launch");
  }

  // The lookup and the input scan are independent and both latency-bound: run
  // them on two forked streams, chunk the batch, and let the fusion kernel of
  // chunk i (caller's stream) overlap the lookup / scan of chunk i+1.
  Aux* ax = aux_streams();
  if (!ax) return fail(SSSD_E_CUDA, "could not create auxiliary streams");
  // chunked pipelining measured slower (each chunk pays a fusion-kernel tail);
  // SSSD_PROPOSE_CHUNKS (A/B switch, <= 8) re-measures it
  static const int env_chunks = getenv("SSSD_PROPOSE_CHUNKS") ? atoi(getenv("SSSD_PROPOSE_CHUNKS")) : 1;
  const int chunks = B >= 4096 ? max(1, min(8, env_chunks)) : 1;
  const int per = (B + chunks - 1) / chunks;
  cudaEventRecord(ax->fork, st);
  cudaStreamWaitEvent(ax->s[0], ax->fork, 0);
  cudaStreamWaitEvent(ax->s[1], ax->fork, 0);
  for (int ci = 0; ci < chunks; ++ci) {
    const int b0 = ci * per, b1 = min(B, b0 + per);
    if (b0 >= b1) break;
    if (cfg->use_datastore) launch_lookup(ax->s[0], b0, b1);
    if (cfg->use_input) launch_scan(ax->s[1], b0, b1);
    cudaEventRecord(ax->done[0][ci], ax->s[0]);
    cudaEventRecord(ax->done[1][ci], ax->s[1]);
    cudaStreamWaitEvent(st, ax->done[0][ci], 0);
    cudaStreamWaitEvent(st, ax->done[1][ci], 0);
    if (ci > 0) fuse_reset_kernel<<<1, 128, 0, st>>>(w.d.cursor, w.d.hist);  // per-range arena + LPT histogram
    launch_fuse(st, b0, b1);
  }
  return cuda_check(cudaGetLastError(), "propose launch");
}

// Returns the device status word of the last propose / merge that used this
// workspace (synchronising on `stream`): 0 or SSSD_E_WORKSPACE.  The word sits
// at a fixed offset (status block first), so cfg / B / max_len / is_merge /
// total_elems are accepted for ABI stability but no longer needed.
int sssd_workspace_status(const sssd_cfg* cfg, int32_t B, int32_t max_len, const void* workspace,
                          int32_t is_merge, int64_t total_elems, void* stream) {
  (void)cfg, (void)B, (void)max_len, (void)is_merge, (void)total_elems;
  if (!workspace) return fail(SSSD_E_ARG, "null workspace");
  int32_t v = 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = cuda_check(cudaMemcpyAsync(&v, static_cast<const uint8_t*>(workspace) + kStatusErrOffset, 4,
                                      cudaMemcpyDeviceToHost, st), "status copy");
  if (rc) return rc;
  if ((rc = cuda_check(cudaStreamSynchronize(st), "status sync"))) return rc;
  if (v) return fail(v, "device workspace overflow (fusion arena)");
  return SSSD_OK;
}

size_t sssd_merge_workspace(const sssd_cfg* cfg, int32_t B, int64_t total_elems) {
  if (!cfg || B < 0) return 0;
  Carver cv{nullptr, 0};
  unsigned long long* status = carve_status(cv);
  const size_t te = (size_t)(total_elems > 0 ? total_elems : 1);
  cv.take<sssd_elem>(te);
  cv.take<uint32_t>(2 * te);
  cv.take<uint32_t>(te * (2 + merge_depth(cfg)));
  carve_draft(cv, status, cfg->P, cfg->dec_len, B);
  return align_up(cv.off, 256);
}

int sssd_merge(const uint32_t* tok, const sssd_elem* el, const int64_t* el_off,
                const int32_t* el_n, int64_t total_elems, const uint32_t* root_tokens, int32_t B,
                const sssd_cfg* cfg, const sssd_draft_out* out, void* workspace,
                size_t workspace_bytes, void* stream) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  if ((rc = validate_out(out))) return rc;
  if (B < 0) return fail(SSSD_E_ARG, "bad batch size %d", B);
  if (B == 0) return SSSD_OK;
  Carver cv{static_cast<uint8_t*>(workspace), 0};
  unsigned long long* status = carve_status(cv);
  const size_t te = (size_t)(total_elems > 0 ? total_elems : 1);
  sssd_elem* sorted = cv.take<sssd_elem>(te);
  uint32_t* idx = cv.take<uint32_t>(2 * te);
  uint32_t* colbuf = cv.take<uint32_t>(te * (2 + merge_depth(cfg)));
  Cols cols{colbuf, colbuf + te, colbuf + 2 * te, (int64_t)te};
  DraftWs d = carve_draft(cv, status, cfg->P, cfg->dec_len, B);
  const size_t need = align_up(cv.off, 256);
  if (!workspace || workspace_bytes < need)
    return fail(SSSD_E_WORKSPACE, "merge needs %zu workspace bytes, got %zu", need, workspace_bytes);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const KCfg k = kcfg(cfg);
  if ((rc = cuda_check(cudaMemsetAsync(d.cursor, 0, 16, st), "memset status"))) return rc;
  sort_sources_kernel<<<B * (cfg->P + 1), 256, 0, st>>>(tok, el, el_off, el_n, sorted, idx, 2 * te, cols);
  if ((rc = cuda_check(cudaGetLastError(), "sort_sources_kernel launch"))) return rc;
  merge_setup_kernel<<<(B + 127) / 128, 128, 0, st>>>(cols, el_off, el_n, root_tokens, B, k, d.desc, d.root);
  if ((rc = cuda_check(cudaGetLastError(), "merge_setup_kernel launch"))) return rc;
  return launch_draft(d, k, B, out, st);
}


size_t sssd_ds_lookup_workspace(const sssd_cfg* cfg, int32_t B) {
  if (!cfg || B < 0) return 0;
  const int64_t cap = ds_idx_cap(cfg->P, cfg->M);
  return (size_t)B * cfg->P * cfg->M * sizeof(sssd_elem) + 256 + (size_t)B * cap * 4;
}

int sssd_ds_lookup(const sssd_ds* ds, const sssd_seqs* seqs, const sssd_cfg* cfg, uint32_t* tab,
                   uint8_t* lens, sssd_elem* el, int32_t* n_el, const sssd_lookup_out* lookup,
                   void* workspace, size_t workspace_bytes, void* stream) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  if (!ds || !ds->rows || ds->n_rows == 0) return fail(SSSD_E_ARG, "empty corpus");
  if (cfg->P + cfg->branch_len > SSSD_ROW_TOKENS && !ds->tokens)
    return fail(SSSD_E_ARG, "P + branch_len > %d needs the token array", SSSD_ROW_TOKENS);
  if (!seqs || seqs->B < 0) return fail(SSSD_E_ARG, "bad sequence batch");
  if (seqs->B == 0) return SSSD_OK;
  const size_t need = sssd_ds_lookup_workspace(cfg, seqs->B);
  if (!workspace || workspace_bytes < need)
    return fail(SSSD_E_WORKSPACE, "ds_lookup needs %zu workspace bytes, got %zu", need, workspace_bytes);
  sssd_lookup_out lk{};
  if (lookup) lk = *lookup;
  sssd_elem* raw = static_cast<sssd_elem*>(workspace);
  uint32_t* idx = reinterpret_cast<uint32_t*>(
      align_up(reinterpret_cast<uintptr_t>(raw + (size_t)seqs->B * cfg->P * cfg->M), 256));
  KCfg kk = kcfg(cfg);
  kk.b0 = 0;
  kk.b1 = seqs->B;
  kk.TS = cfg->branch_len;  // the caller's table layout: [B][P][M][branch_len]
  kk.tab16 = (cfg->branch_len % 4 == 0 && (reinterpret_cast<uintptr_t>(tab) & 15) == 0) ? 1 : 0;
  if (!cfg->has_separator)
    ds_lookup_warp_kernel<<<(seqs->B + 3) / 4, 128, 0, static_cast<cudaStream_t>(stream)>>>(
        *ds, *seqs, kk, tab, lens, el, n_el, lk, Cols{});
  else
    ds_lookup_kernel<<<seqs->B, 32 * cfg->P, 4 * ds_lookup_smem_words(cfg->P, cfg->M),
                       static_cast<cudaStream_t>(stream)>>>(*ds, *seqs, kk, tab, lens, el, n_el, lk, raw, idx,
                                                            ds_idx_cap(cfg->P, cfg->M), Cols{}, nullptr, nullptr);
  return cuda_check(cudaGetLastError(), "ds_lookup_kernel launch");
}

size_t sssd_input_scan_workspace(int32_t B, int32_t max_len) {
  const int64_t cap = max_len > 1 ? max_len : 1;
  int64_t p2 = 1;
  while (p2 < cap) p2 <<= 1;
  return (size_t)B * cap * sizeof(sssd_elem) + (size_t)B * (cap > 4096 ? p2 : 1) * 4 + 256;
}

int sssd_input_scan(const sssd_seqs* seqs, const sssd_cfg* cfg, sssd_elem* el, int32_t* n_el,
                    void* workspace, size_t workspace_bytes, void* stream) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  if (!seqs || seqs->B < 0) return fail(SSSD_E_ARG, "bad sequence batch");
  if (seqs->B == 0) return SSSD_OK;
  const size_t need = sssd_input_scan_workspace(seqs->B, seqs->max_len);
  if (!workspace || workspace_bytes < need)
    return fail(SSSD_E_WORKSPACE, "input_scan needs %zu workspace bytes, got %zu", need, workspace_bytes);
  const int64_t cap = seqs->max_len > 1 ? seqs->max_len : 1;
  int64_t p2 = 1;
  while (p2 < cap) p2 <<= 1;
  sssd_elem* raw = static_cast<sssd_elem*>(workspace);
  uint32_t* idx = reinterpret_cast<uint32_t*>(raw + (size_t)seqs->B * cap);
  KCfg k = kcfg(cfg);
  k.use_in = 1;
  const int th = input_scan_threads(seqs->max_len);
  if ((rc = input_scan_attr(cfg->input_branch_len))) return rc;
  input_scan_kernel<<<seqs->B, th, input_scan_smem_bytes(th, cfg->input_branch_len),
                      static_cast<cudaStream_t>(stream)>>>(
      *seqs, k, raw, el, n_el, idx, cap, cap > 4096 ? p2 : 0, Cols{});
  return cuda_check(cudaGetLastError(), "input_scan_kernel launch");
}

int sssd_find_ranges(const sssd_ds* ds, const uint32_t* pat, const int64_t* pat_off,
                     const int32_t* pat_len, int32_t B, int64_t* lo_hi, void* stream) {
  if (!ds || !ds->rows || ds->n_rows == 0) return fail(SSSD_E_ARG, "empty corpus");
  if (B <= 0) return B == 0 ? SSSD_OK : fail(SSSD_E_ARG, "bad batch");
  find_ranges_kernel<<<(B + 3) / 4, 128, 0, static_cast<cudaStream_t>(stream)>>>(*ds, pat, pat_off,
                                                                                 pat_len, B, lo_hi);
  return cuda_check(cudaGetLastError(), "find_ranges_kernel launch");
}


int sssd_shard_search(const sssd_ds* ds, const sssd_seqs* tails, const sssd_cfg* cfg, int64_t* bounds,
                      void* stream) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  if (!ds || !ds->rows) return fail(SSSD_E_ARG, "shard has no rows");
  if (!tails || tails->B < 0) return fail(SSSD_E_ARG, "bad sequence batch");
  if (tails->B == 0) return SSSD_OK;
  if (ds->n_rows == 0)
    return cuda_check(cudaMemsetAsync(bounds, 0, sizeof(int64_t) * 2 * tails->B * cfg->P,
                                      static_cast<cudaStream_t>(stream)), "bounds memset");
  shard_search_kernel<<<tails->B, 32 * cfg->P, 0, static_cast<cudaStream_t>(stream)>>>(*ds, *tails, kcfg(cfg),
                                                                                       bounds);
  return cuda_check(cudaGetLastError(), "shard_search_kernel launch");
}

int sssd_shard_gather(const sssd_ds* ds, const sssd_cfg* cfg, int32_t B, const int64_t* gbounds, uint32_t* xrows,
                      void* stream) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  if (B <= 0) return B == 0 ? SSSD_OK : fail(SSSD_E_ARG, "bad batch");
  const int64_t total = (int64_t)B * cfg->P * cfg->M * 4;
  shard_gather_kernel<<<(unsigned)((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      *ds, kcfg(cfg), B, gbounds, xrows);
  return cuda_check(cudaGetLastError(), "shard_gather_kernel launch");
}

int sssd_shard_gather_pos(const sssd_ds* ds, const sssd_cfg* cfg, int32_t B, const int64_t* gbounds, uint32_t* xpos,
                          void* stream) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  if (!ds || (!ds->rows && ds->n_rows)) return fail(SSSD_E_ARG, "shard has no rows");
  if (B <= 0) return B == 0 ? SSSD_OK : fail(SSSD_E_ARG, "bad batch");
  const int64_t total = (int64_t)B * cfg->P * cfg->M;
  shard_gather_pos_kernel<<<(unsigned)((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      *ds, kcfg(cfg), B, gbounds, xpos);
  return cuda_check(cudaGetLastError(), "shard_gather_pos_kernel launch");
}

int sssd_rows_from_pos(const uint32_t* tokens, uint64_t n_tokens, const uint32_t* xpos, int64_t count, uint32_t* rows,
                       void* stream) {
  if (!tokens || !xpos || !rows) return fail(SSSD_E_ARG, "rows_from_pos needs tokens, positions and rows");
  if (count <= 0) return count == 0 ? SSSD_OK : fail(SSSD_E_ARG, "bad count");
  rows_from_pos_kernel<<<(unsigned)((count * 4 + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      tokens, n_tokens, xpos, count, rows);
  return cuda_check(cudaGetLastError(), "rows_from_pos_kernel launch");
}

int sssd_propose_pre(const sssd_ds* ds, const sssd_seqs* seqs, const sssd_cfg* cfg, const int64_t* gbounds,
                     const uint32_t* rows, const sssd_draft_out* out, const sssd_lookup_out* lookup,
                     void* workspace, size_t workspace_bytes, void* stream) {
  if (!gbounds || !rows) return fail(SSSD_E_ARG, "sharded propose needs global bounds and assembled rows");
  if (cfg && cfg->P + cfg->branch_len > SSSD_ROW_TOKENS)
    return fail(SSSD_E_LIMIT, "sharded lookup needs P + branch_len <= %d", SSSD_ROW_TOKENS);
  return propose_impl(ds, seqs, cfg, out, lookup, workspace, workspace_bytes, stream, nullptr, gbounds, rows);
}

// Stage-by-stage propose over request ranges of one batch (host-buffer
// pipelines: the datastore lookup of every request can run from its context
// tail before the contexts themselves are uploaded; the input scan and the
// fusion then follow the uploads range by range).  The workspace is carved
// for (B, max_len) = the whole batch; `seqs` holds B requests (for LOOKUP it
// may be a tail view, sssd_gather_tails).  FUSE ranges of one workspace must
// be stream-ordered.
int sssd_propose_phase(const sssd_ds* ds, const sssd_seqs* seqs, const sssd_cfg* cfg, const sssd_draft_out* out,
                       const sssd_lookup_out* lookup, void* workspace, size_t workspace_bytes, int32_t phases,
                       int32_t B, int32_t max_len, int32_t b0, int32_t b1, void* stream) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  if ((rc = validate_out(out))) return rc;
  if (!seqs || seqs->B != B || B < 0 || max_len < 0) return fail(SSSD_E_ARG, "bad sequence batch");
  if (b0 < 0 || b1 < b0 || b1 > B) return fail(SSSD_E_ARG, "bad request range [%d, %d) of %d", b0, b1, B);
  if (phases & ~(SSSD_PHASE_LOOKUP | SSSD_PHASE_SCAN | SSSD_PHASE_FUSE | SSSD_PHASE_BEGIN))
    return fail(SSSD_E_ARG, "unknown phase bits 0x%x", phases);
  if ((phases & SSSD_PHASE_LOOKUP) && cfg->use_datastore) {
    if (!ds || !ds->rows) return fail(SSSD_E_ARG, "use_datastore requires a datastore");
    if (ds->n_rows == 0 || ds->n_tokens == 0) return fail(SSSD_E_ARG, "empty corpus");
    if (ds->n_tokens >= 0xffffffffull) return fail(SSSD_E_LIMIT, "corpus longer than 2^32-1 tokens");
    if (cfg->P + cfg->branch_len > SSSD_ROW_TOKENS && !ds->tokens)
      return fail(SSSD_E_ARG, "P + branch_len > %d needs the token array", SSSD_ROW_TOKENS);
  }
  if (B == 0) return SSSD_OK;
  const PropWs w = carve_propose(static_cast<uint8_t*>(workspace), cfg, B, max_len);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(SSSD_E_WORKSPACE, "propose needs %zu workspace bytes, got %zu", w.bytes, workspace_bytes);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const KCfg k = kcfg(cfg);
  sssd_lookup_out lk{};
  if (lookup) lk = *lookup;
  if (phases & SSSD_PHASE_BEGIN)  // cursor, status word, LPT histogram
    if ((rc = cuda_check(cudaMemsetAsync(w.d.cursor, 0, 16 + 512, st), "memset status"))) return rc;
  if (b1 == b0) return cuda_check(cudaGetLastError(), "propose phase");
  if ((phases & SSSD_PHASE_LOOKUP) && cfg->use_datastore)
    lookup_range(w, k, cfg, ds, seqs, lk, nullptr, nullptr, st, b0, b1);
  if ((phases & SSSD_PHASE_SCAN) && cfg->use_input) {
    if ((rc = input_scan_attr(cfg->input_branch_len))) return rc;
    scan_range(w, k, cfg, seqs, st, b0, b1);
  }
  if (phases & SSSD_PHASE_FUSE) {
    if ((rc = fusion_smem_attr(k))) return rc;
    // a fusion launch's arena slices die with it: the cursor restarts per
    // range; the status word (offset 8) accumulates
    fuse_reset_kernel<<<1, 128, 0, st>>>(w.d.cursor, w.d.hist);
    fuse_range(w, k, seqs, out, st, b0, b1);
  }
  return cuda_check(cudaGetLastError(), "propose phase");
}

// Measurement aid: when set (device pointer, [B] int64), the fusion kernel
// records clock64 cycles per request; NULL disables.
#ifdef SSSD_LK_PROBE
void sssd_set_lookup_probe(long long* cycles) { sssd::lk_probe_set(cycles); }
#endif
void sssd_set_cycle_probe(long long* cycles) { g_cycles = cycles; }
void sssd_set_fusion_form(int form) { g_fusion_form = form < 0 ? -1 : (form > 2 ? 2 : form); }

}  // extern "C"
