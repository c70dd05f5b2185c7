/*
 * sssd.h — C ABI of libsssd.so, the B200 (sm_100a) implementation of the SSSD
 * speculation-and-verification hot path.
 *
 * The reference (`specdraft`, /root/reference/pkg/src/specdraft) is a pure
 * Python package: its "plugin boundary" is its public Python API
 * (`__init__.py:10-111`).  Each entry point below is the batched device
 * equivalent of one reference function; the comment names the reference
 * interface it replaces.  The Python package `paper_2411_05894_b200` binds this
 * header with ctypes and mirrors the reference API on top.
 *
 * Conventions
 *   - Every pointer argument is a DEVICE pointer owned by the caller (the
 *     library never allocates persistent memory); `stream` is a cudaStream_t.
 *   - All launches are asynchronous on `stream`; return value is 0 or a
 *     negative SSSD_E_* code (argument validation happens before any launch).
 *     `sssd_error_string(code)` gives the message.
 *   - Token ids are uint32 (the reference's on-disk `<u4`, datastore.py:17).
 *   - No torch types cross this boundary.
 */
#ifndef SSSD_H
#define SSSD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSSD_OK 0
#define SSSD_E_ARG (-1)        /* invalid argument (message has details)          */
#define SSSD_E_LIMIT (-2)      /* a configured size exceeds a compiled limit      */
#define SSSD_E_CUDA (-3)       /* a CUDA runtime call failed                      */
#define SSSD_E_WORKSPACE (-4)  /* workspace too small; sssd_*_workspace() sizes it */

/* Compiled limits (checked on every call). */
#define SSSD_MAX_P 8           /* max prefix length P (FusionConfig.P)           */
#define SSSD_MAX_DEPTH 32      /* max branch_len / input_branch_len              */
#define SSSD_MAX_DRAFT 256     /* max dec_len (draft nodes incl. root)           */
#define SSSD_ROW_TOKENS 15     /* tokens inlined per suffix row                  */

const char* sssd_error_string(int code);
/* Last detailed message of a failed call on this thread. */
const char* sssd_last_error(void);
int sssd_version(void);

/* ------------------------------------------------------------------------ */
/* Datastore index (replaces datastore.py:81-109 build_suffix_array,       */
/* datastore.py:229-242 build)                                              */
/* ------------------------------------------------------------------------ */

/* Bytes of scratch for sssd_sa_build on n tokens. */
size_t sssd_sa_build_workspace(uint64_t n);

/* Suffix array of tokens[0..n) by radix-sort prefix doubling (own LSD radix
 * sort; each round re-sorts only the positions of not-yet-singleton groups).
 * sa_out: uint32[n] (n < 2^32).  Bit-identical to the reference SA (unique). */
int sssd_sa_build(const uint32_t* tokens, uint64_t n, uint32_t* sa_out, void* workspace,
                  size_t workspace_bytes, void* stream);

/* sssd_sa_build reporting the number of prefix-doubling rounds (host int,
 * the reference loop's iteration count for this corpus). */
int sssd_sa_build_ex(const uint32_t* tokens, uint64_t n, uint32_t* sa_out, void* workspace, size_t workspace_bytes,
                     void* stream, int32_t* rounds);

/* Suffix rows: row r = {sa[r], tokens[sa[r] .. sa[r]+15)} as 16 x uint32 (64 B,
 * tokens past the corpus end are 0; validity is n - pos).  `rows` must be
 * 64-byte aligned, n*64 bytes.  The lookup kernels read only rows (and
 * `tokens` when P + branch_len > 15). */
int sssd_rows_build(const uint32_t* tokens, uint64_t n, const uint32_t* sa, uint32_t* rows,
                    void* stream);

/* First-token index of the suffix rows: bucket[t] (t = 0 .. n_buckets) = the
 * first local row whose first token is >= t, so rows starting with token t < n_buckets
 * are exactly [bucket[t], bucket[t+1]).  A search accelerator for find_range
 * (ref datastore.py:156-183): the same bounds with fewer probes. */
int sssd_bucket_build(const uint32_t* rows, uint64_t n_rows, uint32_t n_buckets, uint32_t* bucket,
                      void* stream);

/* k-gram range index over sorted suffix rows (a find_range accelerator,
 * ref datastore.py:156-183): every k-gram g (2 <= k <= kmax <= 7) that starts
 * a suffix gets one open-addressing slot {64-bit hash of (k, g), lo, hi} with
 * [lo, hi) = the local rows whose suffix starts with g.  sssd_kix_count
 * writes the number of such k-grams to *count (device u64, synchronise
 * before reading); sssd_kix_build fills a zeroed table of cap = 2^j >=
 * 2 * count slots (16 B each).  Lookups verify the tokens of row lo, so a
 * hash collision costs a search, never a wrong range. */
int sssd_kix_count(const uint32_t* rows, uint64_t n_rows, uint64_t n_tokens, uint32_t kmax, uint64_t* count,
                   void* stream);
int sssd_kix_build(const uint32_t* rows, uint64_t n_rows, uint64_t n_tokens, uint32_t kmax, uint32_t* table,
                   uint64_t cap, void* stream);

/* Widen n uint16 token ids to uint32 (device to device): the compact host
 * format of a propose_pinned batch whose vocabulary fits 16 bits, uploaded at
 * half the PCIe bytes and widened next to the kernels that read it. */
int sssd_widen_u16(const uint16_t* src, uint32_t* dst, int64_t n, void* stream);

/* Full-size verification of a built index (a size-independent parity
 * property: a permutation of [0, n) whose adjacent suffixes strictly increase
 * is the unique suffix array of ref datastore.py:81-109).  counts (device,
 * 3 x u64): [0] adjacent rows not strictly increasing, [1] corpus positions
 * missing from the SA column, [2] SA entries >= n.  All zero <=> correct. */
size_t sssd_sa_check_workspace(uint64_t n);
int sssd_sa_check(const uint32_t* tokens, uint64_t n, const uint32_t* rows, uint64_t n_rows, void* workspace,
                  size_t workspace_bytes, unsigned long long* counts, void* stream);

/* Copy the SA column of rows out as uint64 (the SSSD v1 file's `<u8` array). */
int sssd_rows_sa64(const uint32_t* rows, uint64_t n, uint64_t* sa64_out, void* stream);

/* ------------------------------------------------------------------------ */
/* Draft configuration (FusionConfig fusion.py:29-88 + query cfg             */
/* datastore.py:46-78)                                                       */
/* ------------------------------------------------------------------------ */
typedef struct sssd_cfg {
  int32_t P;                /* max prefix length                                 */
  int32_t dec_len;          /* draft node budget incl. root                      */
  int32_t branch_len;       /* datastore continuation length                     */
  int32_t input_branch_len; /* input-cache continuation length                   */
  int32_t M;                /* sample cap per prefix length                      */
  int32_t T;                /* min continuations before shortening stops         */
  int32_t use_datastore;    /* GenerationSession flags (draft.py:150-151)        */
  int32_t use_input;
  int32_t n_input_trees;    /* input trees passed to merge (<= P); P in propose  */
  int32_t has_separator;
  uint32_t separator;
  int32_t disc_stride;      /* = max depth + 1                                   */
  const double* disc;       /* device [(P+1)][disc_stride]: rank 0 = datastore,
                               rank r = input p=P-r+1 (fusion.py:141-155)        */
  int32_t fusion;           /* 0 = level-synchronous fusion (needs every disc row
                               non-increasing in depth, which FusionConfig's
                               ranges guarantee); 1 = heap-order fusion         */
} sssd_cfg;

/* Per-element record of a source's sorted element array:
 * a continuation path = tok[off .. off+len) of the source's token buffer,
 * `orig` = position in the reference's insertion order, `m` = backward match
 * length (input source; 255 for datastore / user paths). */
typedef struct sssd_elem {
  uint32_t off;
  uint32_t orig;
  uint32_t len_m; /* len | (m << 8) */
  uint32_t pad;
} sssd_elem;

/* Datastore view: rows over global SA ranks [rank_base, rank_base + n_rows),
 * n_tokens = corpus length.  A single GPU holds all ranks (rank_base = 0). */
typedef struct sssd_ds {
  const uint32_t* rows;
  const uint32_t* tokens; /* needed only when P + branch_len > 15 */
  uint64_t n_tokens;
  uint64_t rank_base;
  uint64_t n_rows;
  const uint32_t* bucket; /* optional (NULL = none): [n_buckets + 1] first-token index,
                             bucket[t] = first local row whose first token >= t
                             (sssd_bucket_build); narrows every range search */
  uint32_t n_buckets;
  const uint32_t* kix;    /* optional (NULL = none): k-gram range table (sssd_kix_build),
                             [kix_mask + 1] slots of 4 u32 {hash lo, hash hi, lo, hi}:
                             the local row range of every k-gram (2 <= k <= kix_kmax)
                             that starts a suffix; a pattern of <= kix_kmax tokens
                             found there needs no search */
  uint64_t kix_mask;
  uint32_t kix_kmax;
} sssd_ds;

/* Sequences: request b's live sequence is seq[seq_off[b] .. seq_off[b]+seq_len[b]). */
typedef struct sssd_seqs {
  const uint32_t* seq;
  const int64_t* seq_off;
  const int32_t* seq_len;
  int32_t B;
  int32_t max_len; /* upper bound of seq_len[] (workspace sizing) */
} sssd_seqs;

/* Outputs of one propose batch (FlattenedDraft draft.py:48-64, one per request). */
typedef struct sssd_draft_out {
  int32_t* size;     /* [B]                                     */
  uint32_t* tokens;  /* [B][S]   S = dec_len                    */
  int32_t* parents;  /* [B][S]   -1 for the root                */
  int32_t* depths;   /* [B][S]                                  */
  uint64_t* mask;    /* [B][S][W] W = ceil(S/64); bit j of row i = j is i or an ancestor */
  /* Optional per-node outputs (NULL = not written):                        */
  double* priority;  /* [B][S] DraftNode.priority (fusion.py:158-198): the path
                        probability x discount of the node's first insertion;
                        +inf for the root, 0 for padding                     */
  int32_t* source;   /* [B][S] DraftNode.source as its merge rank (fusion.py:
                        245-249): 0 = datastore, r >= 1 = input tree p = P-r+1;
                        -1 for the root and padding                          */
  int32_t* pos;      /* [B][S] position id L-1+depth (L = seq_len[b]; depth
                        alone for sssd_merge); -1 for padding                */
} sssd_draft_out;

/* Optional lookup diagnostics for parity (any pointer may be NULL). */
typedef struct sssd_lookup_out {
  int64_t* ranges;   /* [B][P][2] (lo, hi) for every p <= min(P, L) (find_range)  */
  int64_t* samples;  /* [B][P][M] corpus positions of the sampled ranks, -1 pad   */
  int32_t* n_conts;  /* [B][P] non-empty continuations per p                      */
  int32_t* p_cut;    /* [B] smallest evaluated p (get_conts shortening stop)      */
} sssd_lookup_out;

/* Incremental per-request input index (the stateful
 * analogue of InputCache._push, ref input_cache.py:46-63).  Request b's
 * positions [0, len[b]) are kept sorted as u32 keys (token << pos_bits | pos)
 * in keys[off[b] .. off[b] + len[b]); a propose then finds the occurrences of
 * the last token by binary search instead of scanning the context, and scans
 * only the tail [len[b], L-1) appended since the index was built (the decode
 * loop's accepted tokens).  Results are identical to the stateless scan.
 * len[b] = 0 means "no index" (full scan): the build leaves it 0 when the
 * prefix exceeds SSSD_INDEX_MAX positions or a token does not fit the key. */
#define SSSD_INDEX_MAX 32768
typedef struct sssd_input_index {
  uint32_t* keys;
  const int64_t* off;
  int32_t* len;
  int32_t pos_bits; /* 1..24: positions < 2^pos_bits, tokens < 2^(32 - pos_bits) */
} sssd_input_index;

/* Build the index of positions [0, seq_len[b] - 1) for requests rows[i]
 * (i < n_rows; rows NULL = requests 0 .. n_rows-1): one CTA per request,
 * a shared-memory bitonic sort. */
int sssd_input_index_build(const sssd_seqs* seqs, const sssd_input_index* index, const int32_t* rows,
                           int32_t n_rows, void* stream);

/* sssd_propose with an input index (NULL = the stateless scan) and, when
 * stage_ms is non-NULL, the per-stage device times of sssd_propose_profile
 * (synchronises). */
int sssd_propose_ex(const sssd_ds* ds, const sssd_seqs* seqs, const sssd_input_index* index, const sssd_cfg* cfg,
                    const sssd_draft_out* out, const sssd_lookup_out* lookup, void* workspace,
                    size_t workspace_bytes, void* stream, float* stage_ms);

/* Workspace bytes for sssd_propose on this batch shape. */
size_t sssd_propose_workspace(const sssd_cfg* cfg, int32_t B, int32_t max_len);

/* One batched propose (GenerationSession.propose, draft.py:183-200, over B
 * sessions): datastore range search + sampling + continuation lists
 * (Datastore.get_conts datastore.py:156-218), input-cache trees
 * (InputCache.get_conts input_cache.py:88-113), best-first fusion
 * (merge fusion.py:209-261) and flatten + ancestor masks (draft.py:67-86). */
int sssd_propose(const sssd_ds* ds, const sssd_seqs* seqs, const sssd_cfg* cfg,
                 const sssd_draft_out* out, const sssd_lookup_out* lookup, void* workspace,
                 size_t workspace_bytes, void* stream);

/* The same propose, stage by stage over request ranges [b0, b1) of one batch
 * of B requests whose workspace is sssd_propose_workspace(cfg, B, max_len):
 * SSSD_PHASE_BEGIN once per batch (status reset), then LOOKUP / SCAN / FUSE
 * for any ranges in dependency order (FUSE of a range after its LOOKUP and
 * SCAN; FUSE ranges stream-ordered).  LOOKUP reads only the last P tokens of
 * each request, so `seqs` may then be the tail view of sssd_gather_tails.
 * Replaces the reference's per-request GenerationSession.propose
 * (draft.py:183-200) for host-buffer pipelines (DraftEngine.propose_pinned). */
#define SSSD_PHASE_LOOKUP 1
#define SSSD_PHASE_SCAN 2
#define SSSD_PHASE_FUSE 4
#define SSSD_PHASE_BEGIN 8
int sssd_propose_phase(const sssd_ds* ds, const sssd_seqs* seqs, const sssd_cfg* cfg,
                       const sssd_draft_out* out, const sssd_lookup_out* lookup, void* workspace,
                       size_t workspace_bytes, int32_t phases, int32_t B, int32_t max_len, int32_t b0,
                       int32_t b1, void* stream);

/* Tail view for the lookup: the last min(P, len[b]) tokens of request b
 * (seq: u16 if elem_bytes == 2 else u32; device memory or pinned host
 * memory, read zero-copy) right-aligned in tails[B][P], with
 * tails_off[b] / tails_len[b] describing them as a sequence batch. */
int sssd_gather_tails(const void* seq, int32_t elem_bytes, const int64_t* off, const int32_t* len,
                      int32_t B, int32_t P, uint32_t* tails, int64_t* tails_off, int32_t* tails_len,
                      void* stream);

/* Stage entry points (the single-request reference API is built on these). */

/* Batched Datastore.find_range (datastore.py:156-183): pattern b =
 * pat[pat_off[b] .. + pat_len[b]); lo_hi[b] = (lo, hi) global SA ranks. */
int sssd_find_ranges(const sssd_ds* ds, const uint32_t* pat, const int64_t* pat_off,
                     const int32_t* pat_len, int32_t B, int64_t* lo_hi, void* stream);

/* Datastore.get_conts (datastore.py:185-218) for B prefixes (the last
 * min(P, len) tokens of each sequence): continuation strings tab[B][P][M][BL],
 * lengths lens[B][P][M], and the evaluated ones as elements el[B][P*M] sorted
 * by (string, insertion order), n_el[B] of them (el.orig = insertion order). */
size_t sssd_ds_lookup_workspace(const sssd_cfg* cfg, int32_t B);
int sssd_ds_lookup(const sssd_ds* ds, const sssd_seqs* seqs, const sssd_cfg* cfg, uint32_t* tab,
                   uint8_t* lens, sssd_elem* el, int32_t* n_el, const sssd_lookup_out* lookup,
                   void* workspace, size_t workspace_bytes, void* stream);

/* InputCache.get_conts (input_cache.py:88-113) for B sequences: every earlier
 * occurrence e of the last token (m = backward match length >= 1), as elements
 * el[B][max_len] sorted by (seq[e:e+len], e); n_el[B] of them.  Tree p holds
 * the elements with m >= p (el.orig = e = insertion order). */
size_t sssd_input_scan_workspace(int32_t B, int32_t max_len);
int sssd_input_scan(const sssd_seqs* seqs, const sssd_cfg* cfg, sssd_elem* el, int32_t* n_el,
                    void* workspace, size_t workspace_bytes, void* stream);

/* sssd_propose with CUDA events between its launches; synchronises and writes
 * the device time of each stage: [0] ds_lookup_kernel, [1] input_scan_kernel,
 * [2] propose_setup_kernel, [3] draft_kernel (ms).  Measurement aid only. */
int sssd_propose_profile(const sssd_ds* ds, const sssd_seqs* seqs, const sssd_cfg* cfg,
                         const sssd_draft_out* out, void* workspace, size_t workspace_bytes,
                         void* stream, float* stage_ms);

/* SA-range sharding.  A shard is an sssd_ds over global
 * ranks [rank_base, rank_base + n_rows) with n_tokens = the global corpus
 * length.  Per step:
 *   sssd_shard_search   local bounds[b][p-1] = (#shard rows < pattern, <=) of the
 *                       last p tokens of each tail sequence;  SUM over shards =
 *                       global [lo, hi) exactly (A.2)          -> NCCL all-reduce
 *   sssd_shard_gather   xrows[b][p-1][k][16] = suffix row of sampled global rank
 *                       k of [lo, hi) if this shard owns it, else 0
 *                                                   -> NCCL reduce-scatter (sum)
 *   sssd_propose_pre    sssd_propose for this rank's requests with the global
 *                       bounds and assembled rows instead of a local search. */
int sssd_shard_search(const sssd_ds* ds, const sssd_seqs* tails, const sssd_cfg* cfg, int64_t* bounds,
                      void* stream);
int sssd_shard_gather(const sssd_ds* ds, const sssd_cfg* cfg, int32_t B, const int64_t* gbounds, uint32_t* xrows,
                      void* stream);
/* The compact C2 exchange (what sharded.py uses): 4 B per sample instead of
 * a 64 B row.  sssd_shard_gather_pos writes xpos[b][p-1][k] = corpus position
 * + 1 of sampled global rank k if this shard owns it, else 0 -> NCCL
 * reduce-scatter (sum); sssd_rows_from_pos then rebuilds the `count` suffix
 * rows (64 B each, zero for 0) from the replicated token array for
 * sssd_propose_pre. */
int sssd_shard_gather_pos(const sssd_ds* ds, const sssd_cfg* cfg, int32_t B, const int64_t* gbounds, uint32_t* xpos,
                          void* stream);
int sssd_rows_from_pos(const uint32_t* tokens, uint64_t n_tokens, const uint32_t* xpos, int64_t count, uint32_t* rows,
                       void* stream);
int sssd_propose_pre(const sssd_ds* ds, const sssd_seqs* seqs, const sssd_cfg* cfg, const int64_t* gbounds,
                     const uint32_t* rows, const sssd_draft_out* out, const sssd_lookup_out* lookup,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Measurement aid: device int64[B][8] receiving, per request of subsequent
 * sssd_propose calls, the fusion kernel's {total cycles, seeding cycles,
 * best-first loop cycles, flatten cycles, pops, elements scanned by
 * expansions, peak live sibling groups, allocations spilled out of shared
 * memory}; NULL disables. */
void sssd_set_cycle_probe(long long* cycles);

/* Fusion form of the level-synchronous path (cfg fusion = 0): -1 = automatic
 * (one CTA per request for launches of <= SSSD_CTA_MAX requests, default 512;
 * one warp per request above), 0 = one warp per request only, 1 = all-nodes
 * kernel first (requests outgrowing its shared-memory tables fall back to the
 * level-synchronous kernel), 2 = one CTA per request for every launch.
 * Identical drafts in every form; a process-wide tuning switch, initialised
 * from SSSD_FUSION_FORM. */
void sssd_set_fusion_form(int form);

/* Fusion of caller-provided source trees (merge fusion.py:209-261 + flatten).
 * Each tree is given as its multiset of root-to-end paths in DFS order (first
 * appearance order = the tree's child order): paths of request b / source s
 * are elements el[el_off[b*(P+1)+s] .. + el_n[...]) over token buffer `tok`;
 * source 0 = datastore tree, source s>=1 = input tree p=s.  The library sorts
 * them on the device and runs the same fusion kernel as sssd_propose. */
size_t sssd_merge_workspace(const sssd_cfg* cfg, int32_t B, int64_t total_elems);
int sssd_merge(const uint32_t* tok, const sssd_elem* el, const int64_t* el_off,
               const int32_t* el_n, int64_t total_elems, const uint32_t* root_tokens, int32_t B,
               const sssd_cfg* cfg, const sssd_draft_out* out, void* workspace,
               size_t workspace_bytes, void* stream);

/* Synchronises `stream` and returns the device status word left in a propose
 * or merge workspace by the last call that used it: 0, or SSSD_E_WORKSPACE
 * when the fusion arena overflowed (outputs are then invalid).  The word is an
 * int32 at byte offset SSSD_STATUS_OFFSET of every workspace (callers that
 * pipeline several proposes through one workspace copy it after each call);
 * the size arguments are ignored. */
#define SSSD_STATUS_OFFSET 8
int sssd_workspace_status(const sssd_cfg* cfg, int32_t B, int32_t max_len, const void* workspace,
                          int32_t is_merge, int64_t total_elems, void* stream);

/* ------------------------------------------------------------------------ */
/* Verification (verify_greedy draft.py:114-138, step draft.py:202-216)      */
/* ------------------------------------------------------------------------ */

/* Teacher-forced node predictions (TeacherForcedOracle harness.py:49-67):
 * pred[b][i] = ref[b][L_b - plen_b + depth[b][i]] or 0xFFFFFFFF. */
int sssd_teacher_predict(const int32_t* depths, const int32_t* size, int32_t S,
                         const uint32_t* ref, const int64_t* ref_off, const int32_t* ref_len,
                         const int32_t* seq_len, const int32_t* prompt_len, int32_t B,
                         uint32_t* pred, void* stream);

/* Greedy accept + append: walks the draft with pred[b][*], writes the accepted
 * node indices (path[b][0..n_acc)), the bonus token, and appends
 * accepted tokens + bonus to the sequence buffer in place (seq_len updated,
 * clipped to seq_cap[b]).  emitted[b] = n_acc + 1 before clipping. */
int sssd_accept(const uint32_t* tokens, const int32_t* parents, const int32_t* size, int32_t S,
                const uint32_t* pred, int32_t B, uint32_t* seq, const int64_t* seq_off,
                int32_t* seq_len, const int32_t* seq_cap, int32_t* path, int32_t* n_acc,
                uint32_t* bonus, int32_t* emitted, void* stream);

/* KV compaction after acceptance: for each request, copy cache rows of the
 * accepted draft nodes (positions base_b + path[b][k]) to base_b + 1 + k, for
 * every layer / kv head: kv[layer][b][head][pos][d] layout (bf16). */
int sssd_kv_compact(uint16_t* kv, int32_t n_layers, int32_t B, int32_t n_heads, int32_t max_pos,
                    int32_t head_dim, const int32_t* base, const int32_t* path,
                    const int32_t* n_acc, int32_t S, void* stream);

/* ------------------------------------------------------------------------ */
/* Tree attention (verification forward; semantics draft.py:205-210)         */
/* ------------------------------------------------------------------------ */
/* q:  [B][S][Hq][D] bf16, k/v cache: [B][Hkv][max_pos][D] bf16 holding the
 * prefix rows [0, ctx_len[b]) and the S tree rows at [ctx_len[b], +S);
 * mask [B][S][W] u64 ancestor bitmask; o: [B][S][Hq][D] bf16.  D = 128. */
int sssd_tree_attention(const uint16_t* q, const uint16_t* k, const uint16_t* v,
                        const uint64_t* mask, const int32_t* ctx_len, int32_t B, int32_t S,
                        int32_t Hq, int32_t Hkv, int32_t max_pos, int32_t head_dim, float scale,
                        uint16_t* o, void* workspace, size_t workspace_bytes, void* stream);
size_t sssd_tree_attention_workspace(int32_t B, int32_t S, int32_t Hq, int32_t max_pos);

/* ------------------------------------------------------------------------ */
/* Fused elementwise stages of the verification forward (bf16 tensors;      */
/* the projections around them are cuBLAS GEMMs)                            */
/* ------------------------------------------------------------------------ */
/* y[r] = x[r] * rsqrt(mean(x[r]^2) + eps) * w, h % 8 == 0 */
int sssd_rmsnorm_bf16(const void* x, const void* w, void* y, int64_t rows, int32_t h, float eps, void* stream);
/* qkv [b*S][(hq + 2 hkv) d] (fused projection) -> rotary q into q_out [b][S][hq][d]; rotary k and v
 * into the caches [B][hkv][max_pos][d] at row rows[i] (NULL = i), slot ctx_len[i] + s;
 * pos [b][S] int64 positions, theta = rope base. */
int sssd_rope_kv_bf16(const void* qkv, const int64_t* pos, const int32_t* ctx_len, const int64_t* rows,
                      void* q_out, void* k_cache, void* v_cache, int32_t b, int32_t S, int32_t hq, int32_t hkv,
                      int32_t d, int32_t max_pos, float theta, void* stream);
/* a[r][j] = silu(gu[r][j]) * gu[r][m + j] (fused gate|up projection) */
int sssd_swiglu_bf16(const void* gu, void* a, int64_t rows, int32_t m, void* stream);
/* Row argmax of fp32 logits [rows][cols] -> int32 [rows]: torch.argmax semantics
 * (first index of the maximum; a NaN is the maximum).  The greedy predictions
 * of a verify step (the oracle of draft.py:205-210). */
int sssd_argmax_f32(const float* x, int64_t rows, int32_t cols, int32_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SSSD_H */
