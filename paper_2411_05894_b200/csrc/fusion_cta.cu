// K5, CTA-per-request form of the level-synchronous fusion (sm_100a), for
// small launches (a B = 64 or B = 8 batch: one warp per request leaves most of
// the GPU idle, and the slowest request's single-warp chain is the batch's
// latency).  Same algorithm and bit-identical output as draft_ls_kernel
// (fusion_ls.cu header; ref fusion.py:209-261, draft.py:67-86);
// what changes is who does the work of a level:
//
//   * generation: the expanded parents are split into kCtaWarps contiguous
//     slices of about equal element count (runs never cross a parent, so the
//     slices are independent); every warp scans its slice with the one-warp
//     chunk loop and appends its children to the shared level buffer through
//     a shared counter -- the order of the appended records is irrelevant,
//     the sort that follows is a total order on (k0, k1);
//   * the level buffer is large (kCtaLevCap nodes), so a level is never cut
//     and re-sorted while it is generated (the one-warp kernel's 96-node
//     buffer sorts + cuts repeatedly on big prompt-heavy levels); a level
//     beyond it is generated again into a pool buffer;
//   * levels of more than 64 nodes are sorted by a CTA-wide bitonic network;
//   * class positions, the top-list merge and tau stay on warp 0 (they are
//     short), the parent copy and the flatten rank / mask passes use every
//     thread.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "fusion_ls.cuh"
#include "propose.cuh"

#ifndef SSSD_CTA_RANK_MAX  // levels of (kCtaSortWarp, this] nodes: rank sort (<= 2 * kCtaThreads)
#define SSSD_CTA_RANK_MAX (2 * kCtaThreads)
#endif

namespace sssd {

#ifndef SSSD_CTA_WARPS
#define SSSD_CTA_WARPS 8
#endif
constexpr int kCtaWarps = SSSD_CTA_WARPS;
constexpr int kCtaThreads = 32 * kCtaWarps;
constexpr int kCtaLevCap = 1024;  // level nodes in shared memory
constexpr int kCtaParCap = 256;  // parents in shared memory
constexpr int kCtaSortWarp = 64; // levels up to this size are sorted by warp 0

// CTA scratch words: counters and broadcasts between the phases
struct CtaShared {
  uint32_t nb, n;           // level records written / children generated
  uint32_t E, has_empty;    // element count of the level, a parent without elements
  uint32_t nexp, stop;      // next level's parents, early exit
  uint32_t next_pid, t;     // class pass / merge results (warp 0)
  uint8_t* glev;            // pool buffers (level / parents), grown on demand
  uint8_t* gpar;
  uint32_t glev_cap, gpar_cap;
  uint32_t jb[kCtaWarps + 1];  // generation slices (parent index bounds)
};

int cta_threads() { return kCtaThreads; }

// (staging the source element columns in shared memory first was measured:
// no gain at B = 64 -- the level chains are bound by their own dependent
// steps, not by the L2 loads -- and one CTA per SM fewer at B >= 256)
int cta_smem_bytes(int P, int S) {
  return kLsLevelBytes * kCtaLevCap + kLsParBytes * kCtaParCap + (P + 1) * (int)sizeof(SrcDesc) + top_bytes(S) +
         S * 8 + 16 * 4 + (int)((sizeof(CtaShared) + 15) / 16 * 16);
}

// Sort positions [0, n) by (k0, k1), carrying ord: the all-ascending bitonic
// network of ls_sort over every thread of the CTA.
__device__ __forceinline__ void cta_sort(LsLevel L, uint32_t n) {
  uint32_t N2 = 64;
  while (N2 < n) N2 <<= 1;
  for (uint32_t lk = 1; (1u << lk) <= N2; ++lk) {
    const uint32_t kk = 1u << lk;
    for (int lj = (int)lk - 1; lj >= 0; --lj) {
      const uint32_t jj = 1u << lj;
      for (uint32_t p = threadIdx.x; p < N2 / 2; p += kCtaThreads) {
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
      __syncthreads();
    }
  }
}

// Levels of up to 2 * kCtaThreads nodes: every thread ranks (up to) two nodes
// against all n keys (broadcast shared-memory reads; (k0, k1) keys are unique),
// then writes them to their ranks -- two barriers instead of the bitonic
// network's one per stage.
static_assert(SSSD_CTA_RANK_MAX <= 2 * kCtaThreads, "two nodes per thread");
__device__ __forceinline__ void cta_rank_sort(LsLevel L, uint32_t n) {
  uint64_t m0[2] = {~0ull, ~0ull}, m1[2] = {~0ull, ~0ull};
  uint32_t r[2] = {0, 0}, o[2] = {0, 0};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t i = threadIdx.x + h * kCtaThreads;
    if (i < n) {
      m0[h] = L.k0()[i];
      m1[h] = L.k1()[i];
      o[h] = L.ord()[i];
    }
  }
  for (uint32_t q = 0; q < n; ++q) {
    const uint64_t q0 = L.k0()[q], q1 = L.k1()[q];
#pragma unroll
    for (int h = 0; h < 2; ++h) r[h] += k_less(q0, q1, m0[h], m1[h]) ? 1u : 0u;
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t i = threadIdx.x + h * kCtaThreads;
    if (i < n) {
      L.k0()[r[h]] = m0[h];
      L.k1()[r[h]] = m1[h];
      L.ord()[r[h]] = o[h];
    }
  }
  __syncthreads();
}

// One warp's share of a level's generation: parents [jb, je), whose elements
// are the flat positions [xb, xe) (ls_generate's chunk loop over a slice).
// Children go to L at positions reserved from sh->nb (records past cap are
// counted, not written); every generated child is counted in sh->n.
__device__ __forceinline__ void cta_generate(const LsPar par, int jb, int je, uint32_t xb, uint32_t xe, LsLevel L,
                                             uint32_t cap, const SrcDesc* sd, const double* disc, int disc_stride,
                                             int d, bool has_empty, bool has_tau, uint64_t tau0, uint32_t tau_dr,
                                             CtaShared* sh) {
  const int lane = lane_id();
  const uint32_t lt = lanemask_lt();
  uint32_t n = 0;
  const double* drow = disc + d;
  auto emit = [&](bool pred, int j, uint32_t tk, uint32_t cnt, uint32_t first, uint32_t s, uint32_t e) {
    bool live = pred && cnt > 0;
    if (!__ballot_sync(SSSD_FULL, live)) return;
    uint64_t k0 = ~0ull, k1 = ~0ull;
    double pp = 0.0;
    uint32_t pid = 0;
    if (live) {
      const uint32_t tr = par.tbr()[j], rk = tr >> kTbBits, pc = par.cnt()[j];
      const double ratio = ratio_rn(cnt, pc);  // ref fusion.py:259
      pp = __dmul_rn(par.pp()[j], ratio);
      const double pr = __dmul_rn(pp, drow[rk * disc_stride]);  // ref fusion.py:246
      k0 = ~(uint64_t)__double_as_longlong(pr);
      k1 = (uint64_t)rk << 56 | (uint64_t)(tr & kTbMask) << 32 | first;
      pid = par.pid()[j];
      const uint32_t dr = (uint32_t)d << 26 | rk << kTbBits;
      if (has_tau && (k0 > tau0 || (k0 == tau0 && dr > tau_dr))) live = false;
    }
    const uint32_t km = __ballot_sync(SSSD_FULL, live);
    if (!km) return;
    n += __popc(km);
    uint32_t at = 0;
    if (lane == 0) at = atomicAdd(&sh->nb, (uint32_t)__popc(km));
    at = __shfl_sync(SSSD_FULL, at, 0);
    if (live) {
      const uint32_t pos = at + __popc(km & lt);
      if (pos < cap) {
        L.k0()[pos] = k0;
        L.k1()[pos] = k1;
        L.pp()[pos] = pp;
        L.a()[pos] = s;
        L.z()[pos] = e;
        L.cnt()[pos] = cnt;
        L.tok()[pos] = tk;
        L.ppid()[pos] = pid;
        L.ord()[pos] = pos;
      }
    }
  };
  bool c_open = false;
  uint32_t c_cnt = 0, c_first = 0, c_start = 0;
  auto parent_of = [&](uint32_t x) {  // last parent in [jb, je) whose offset is <= x
    int lo = jb, hi = je;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (par.off()[mid] <= x) lo = mid;
      else hi = mid;
    }
    return lo;
  };
  struct Ld {
    int j;
    uint32_t i, lm, tk, og, th;
  };
  auto load_chunk = [&](uint32_t base, int jprev) {
    Ld r{0, 0, 0, 0, 0xffffffffu, 0};
    const uint32_t x = base + lane;
    if (!has_empty) {
      const int q = jprev + 1 + lane;
      uint32_t bit = 0;
      if (q < je) {
        const uint32_t st = par.off()[q] - base;
        if (st < 32) bit = 1u << st;
      }
      const uint32_t heads = __reduce_or_sync(SSSD_FULL, bit);
      r.j = jprev + __popc(heads & (0xffffffffu >> (31 - lane)));
    }
    if (x < xe) {
      if (has_empty) r.j = parent_of(x);
      const SrcDesc& sc = sd[par.tbr()[r.j] >> kTbBits];
      r.i = par.a()[r.j] + (x - par.off()[r.j]);
      r.th = (uint32_t)sc.thr;
      r.lm = sc.meta[r.i];
      r.tk = sc.tok[(int64_t)(d - 1) * sc.stride + r.i];
      r.og = sc.orig[r.i];
    }
    return r;
  };
  if (xb < xe) {
    Ld cur = load_chunk(xb, jb - 1);
    for (uint32_t base = xb; base < xe; base += 31) {
      const uint32_t x = base + lane;
      const bool last = base + 32 >= xe;
      const bool owned = x < xe && (lane < 31 || last);
      const int jprev = __shfl_sync(SSSD_FULL, cur.j, 30);
      Ld nxt{};
      if (!last) nxt = load_chunk(base + 31, jprev);  // one chunk ahead: a lone warp hides the load latency
      const int j = cur.j;
      const uint32_t i = cur.i, lm = cur.lm, tk = cur.tk, og = cur.og, th = cur.th;
      const bool has = x < xe && el_len(lm) >= (uint32_t)d;
      const bool w = owned && has && el_m(lm) >= th;
      const uint32_t orig = w ? og : 0xffffffffu;
      const uint32_t wt = w ? el_wt(lm) : 0u;
      const uint32_t hasm = __ballot_sync(SSSD_FULL, has);
      if (hasm) {
        int lo_l, hi_l;
        run_bounds(has, (uint32_t)j, tk, lo_l, hi_l);
        uint32_t fm = orig, cnt = wt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_down_sync(SSSD_FULL, fm, o);
          const uint32_t z = __shfl_down_sync(SSSD_FULL, cnt, o);
          if (lane + o <= hi_l) {
            fm = min(fm, y);
            cnt += z;
          }
        }
        fm = __shfl_sync(SSSD_FULL, fm, lo_l);
        cnt = __shfl_sync(SSSD_FULL, cnt, lo_l);
        uint32_t start = i - (uint32_t)(lane - lo_l);
        if (c_open && lo_l == 0) {
          cnt += c_cnt;
          fm = min(fm, c_first);
          start = c_start;
        }
        const bool to_next = !last && has && hi_l == 31;
        emit(owned && has && lane == hi_l && !to_next, j, tk, cnt, fm, start, i + 1);
        c_open = __ballot_sync(SSSD_FULL, lane == 30 && to_next) != 0;
        if (c_open) {
          c_cnt = __shfl_sync(SSSD_FULL, cnt, 30);
          c_first = __shfl_sync(SSSD_FULL, fm, 30);
          c_start = __shfl_sync(SSSD_FULL, start, 30);
        }
      }
      if (last) break;
      cur = nxt;
    }
  }
  if (lane == 0 && n) atomicAdd(&sh->n, n);
}

// All warps: generate level d from the parents in par (slices in sh->jb).
__device__ __forceinline__ void cta_generate_all(const LsPar par, int np, LsLevel L, uint32_t cap, const SrcDesc* sd,
                                                 const KCfg& c, int d, bool has_tau, uint64_t tau0, uint32_t tau_dr,
                                                 CtaShared* sh) {
  const int warp = threadIdx.x >> 5;
  const int jb = (int)sh->jb[warp], je = (int)sh->jb[warp + 1];
  const uint32_t xb = jb < np ? par.off()[jb] : sh->E;
  const uint32_t xe = je < np ? par.off()[je] : sh->E;
  cta_generate(par, jb, je, xb, xe, L, cap, sd, c.disc, c.disc_stride, d, sh->has_empty != 0, has_tau, tau0, tau_dr,
               sh);
}

__global__ void __launch_bounds__(kCtaThreads, 1)
    draft_cta_kernel(const SrcDesc* desc, const uint32_t* root_tok, KCfg c, uint8_t* pool,
                     unsigned long long* cursor, uint64_t pool_bytes, int32_t* err, sssd_draft_out out,
                     long long* cycles, const int32_t* order, SetupSrc su, int use_su) {
  extern __shared__ __align__(16) uint8_t smem[];
  const long long t_start = clock64();
  const int b = order ? order[c.b0 + blockIdx.x] : c.b0 + blockIdx.x;
  const int tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const uint32_t lt = lanemask_lt();
  const int S = c.S, K = S - 1;
  const int NR = c.P + 1;

  uint8_t* sp = smem;
  const LsLevel Ls = level_carve(sp, kCtaLevCap);
  sp += kLsLevelBytes * kCtaLevCap;
  uint8_t* par_smem = sp;
  LsPar par = par_carve(sp, kCtaParCap);
  sp += kLsParBytes * kCtaParCap;
  SrcDesc* sd = reinterpret_cast<SrcDesc*>(sp);
  sp += NR * sizeof(SrcDesc);
  const LsTop T = top_carve(sp, S);
  sp += top_bytes(S);
  uint32_t* nl = reinterpret_cast<uint32_t*>(sp);  // sorted positions of the level's new paths
  sp += S * 4;
  uint32_t* npos = reinterpret_cast<uint32_t*>(sp);  // their slots in the merged top list
  sp += S * 4;
  uint32_t* rcnt = reinterpret_cast<uint32_t*>(sp);  // per-rank class counters
  sp += 16 * 4;
  CtaShared* sh = reinterpret_cast<CtaShared*>(sp);

  __shared__ uint32_t s_root;
  if (use_su) {
    for (int r = tid; r < NR; r += kCtaThreads) sd[r] = make_src_desc(su, c, b, r);
    if (tid == 0) s_root = su.seqs.seq[su.seqs.seq_off[b] + su.seqs.seq_len[b] - 1];
  } else {
    for (int r = tid; r < NR; r += kCtaThreads) sd[r] = desc[(size_t)b * NR + r];
    if (tid == 0) s_root = root_tok[b];
  }
  if (tid == 0) {
    sh->glev = nullptr;
    sh->gpar = nullptr;
    sh->glev_cap = sh->gpar_cap = 0;
    sh->stop = 0;
  }
  __syncthreads();
  // level 0: warp r sums source r's root count (ref fusion.py:244: seeds are
  // count / root_count); parents are appended in rank order by warp 0
  uint32_t* rc_s = rcnt;  // scratch before the first class pass (NR <= 9 words)
  for (int rk = warp; rk < NR; rk += kCtaWarps) {
    uint32_t rc = 0;
    if (K > 0)
      for (int i = lane; i < sd[rk].n; i += 32) {
        const uint32_t mt = sd[rk].meta[i];
        rc += (int)el_m(mt) >= sd[rk].thr ? el_wt(mt) : 0u;
      }
    rc = __reduce_add_sync(SSSD_FULL, rc);
    if (lane == 0) rc_s[rk] = sd[rk].n > 0 ? rc : 0u;
  }
  __syncthreads();
  int np = 0;
  for (int rk = 0; rk < NR; ++rk) {
    const uint32_t rc = rc_s[rk];
    if (rc == 0) continue;
    if (tid == 0) {
      par.a()[np] = 0;
      par.z()[np] = (uint32_t)sd[rk].n;
      par.cnt()[np] = rc;
      par.pp()[np] = 1.0;
      par.tbr()[np] = (uint32_t)rk << kTbBits;
      par.pid()[np] = 0;
    }
    ++np;
  }
  __syncthreads();

  int t = 0;
  uint32_t next_pid = 1;
  uint32_t gen_total = 0, max_level = 0, levels = 0;
  uint32_t ph_gen = 0, ph_sort = 0, ph_cls = 0, ph_merge = 0;  // thread 0's phase cycles (cycle probe)
  uint32_t tp = (uint32_t)clock();

  for (int d = 1; np > 0 && d < c.disc_stride; ++d) {
    // 1. exclusive scan of the parents' element-range sizes (warp 0), and the
    //    generation slices: warp w starts at the first parent whose offset is
    //    >= w * E / kCtaWarps
    if (warp == 0) {
      uint32_t E = 0;
      bool has_empty = false;
      for (int j0 = 0; j0 < np; j0 += 32) {
        const int j = j0 + lane;
        uint32_t e = 0;
        if (j < np && d <= sd[par.tbr()[j] >> kTbBits].depth) e = par.z()[j] - par.a()[j];
        has_empty |= __ballot_sync(SSSD_FULL, j < np && e == 0) != 0;
        uint32_t inc = e;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(SSSD_FULL, inc, o);
          if (lane >= o) inc += y;
        }
        if (j < np) par.off()[j] = E + inc - e;
        E += __shfl_sync(SSSD_FULL, inc, 31);
      }
      __syncwarp();
      if (lane <= kCtaWarps) {
        uint32_t jw = (uint32_t)np;
        if (lane < kCtaWarps) {
          const uint32_t tw = (uint32_t)(((uint64_t)E * lane) / kCtaWarps);
          int lo = 0, hi = np;  // first parent with off >= tw
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (par.off()[mid] < tw) lo = mid + 1;
            else hi = mid;
          }
          jw = lane == 0 ? 0u : (uint32_t)lo;
        }
        sh->jb[lane] = jw;
      }
      if (lane == 0) {
        sh->E = E;
        sh->has_empty = has_empty;
        sh->nb = 0;
        sh->n = 0;
      }
    }
    __syncthreads();
    const uint32_t E = sh->E;
    if (E == 0) break;
    ++levels;

    tp = (uint32_t)clock();
    // 2. generate into shared memory; a level beyond kCtaLevCap is generated
    //    again into a pool buffer
    const bool has_tau = t == K;
    const uint64_t tau0 = has_tau ? T.g0()[K - 1] : 0ull;
    const uint32_t tau_dr = has_tau ? T.g1()[K - 1] & ~kTbMask : 0u;
    cta_generate_all(par, np, Ls, kCtaLevCap, sd, c, d, has_tau, tau0, tau_dr, sh);
    __syncthreads();
    const uint32_t n_all = sh->n;
    if (n_all == 0) break;
    LsLevel L = Ls;
    if (n_all > (uint32_t)kCtaLevCap) {
      __syncthreads();  // every thread has read sh->n
      if (tid == 0) {
        uint32_t need = 64;
        while (need < n_all) need <<= 1;
        if (sh->glev_cap < need) {
          unsigned long long at = atomicAdd(cursor, (unsigned long long)need * kLsLevelBytes);
          if (at + (unsigned long long)need * kLsLevelBytes > pool_bytes) {
            atomicExch(err, SSSD_E_WORKSPACE);
            sh->stop = 1;
          } else {
            sh->glev = pool + at;
            sh->glev_cap = need;
          }
        }
        sh->nb = 0;
        sh->n = 0;
      }
      __syncthreads();
      if (sh->stop) break;
      L = level_carve(sh->glev, sh->glev_cap);
      cta_generate_all(par, np, L, sh->glev_cap, sd, c, d, has_tau, tau0, tau_dr, sh);
      __syncthreads();
    }
    const uint32_t n = n_all;
    if (n > kTbMask) {
      if (tid == 0) atomicExch(err, SSSD_E_LIMIT);
      break;
    }

    ph_gen += (uint32_t)clock() - tp;
    tp = (uint32_t)clock();
    // 3. sort the level by (k0, k1) = (~priority, rank, parent tb, first)
    if (n > (uint32_t)SSSD_CTA_RANK_MAX) {
      cta_sort(L, n);
    } else if (n > (uint32_t)kCtaSortWarp) {
      cta_rank_sort(L, n);
    } else {
      if (warp == 0) ls_sort(L, n);
      __syncthreads();
    }

    ph_sort += (uint32_t)clock() - tp;
    tp = (uint32_t)clock();
    // 4-6 on warp 0: class positions and path ids, top-list merge, next parents
    if (warp == 0) {
      uint32_t nnew = 0;
      // nodes past the chunk holding the level's K-th new path can be neither
      // listed nor expanded (their G exceeds that path's, which bounds tau):
      // the class pass stops there (ne), so its cost follows the draft budget,
      // not the level size
      uint32_t ne = n;
      if (lane < 16) rcnt[lane] = 0;
      __syncwarp();
      for (uint32_t s0 = 0; s0 < n; s0 += 32) {
        const uint32_t s = s0 + lane;
        const bool v = s < n;
        uint32_t rk = 0, tb = 0;
        unsigned long long pk = 1ull << 63 | (unsigned)lane;
        if (v) {
          rk = (uint32_t)(L.k1()[s] >> 56);
          const uint32_t g = L.ord()[s];
          pk = (unsigned long long)L.ppid()[g] << 32 | L.tok()[g];
        }
        const uint32_t rm = __match_any_sync(SSSD_FULL, v ? rk : 64u + lane);
        if (v) tb = rcnt[rk] + __popc(rm & lt);
        const uint32_t pm = __match_any_sync(SSSD_FULL, pk);
        const int rep = __ffs(pm) - 1;
        int found = -1;
        if (v && lane == rep && s0 > 0) {  // an earlier chunk holds the path?
          for (uint32_t q = 0; q < s0; ++q)
            if (L.k1()[q] == pk) {
              found = (int)q;
              break;
            }
        }
        const uint32_t newm = __ballot_sync(SSSD_FULL, v && lane == rep && found < 0);
        uint32_t id = 0;
        if (v && lane == rep) id = found >= 0 ? L.pid()[found] : next_pid + __popc(newm & lt);
        id = __shfl_sync(SSSD_FULL, id, rep);
        if ((newm >> lane) & 1u) {
          const uint32_t at = nnew + __popc(newm & lt);
          if (at < (uint32_t)K) nl[at] = s;
        }
        next_pid += __popc(newm);
        nnew += __popc(newm);
        __syncwarp();
        if (v) {
          if (lane == 31 - __clz(rm)) rcnt[rk] += __popc(rm);
          L.tbr()[s] = rk << kTbBits | tb;
          L.pid()[s] = id;
          L.k1()[s] = pk;
        }
        __syncwarp();
        if (nnew >= (uint32_t)K) {
          ne = min(n, s0 + 32);
          break;
        }
      }

      ph_cls += (uint32_t)clock() - tp;
      // merge the level's new paths (already in G order) into the top list
      const uint32_t dd = (uint32_t)d << 26;
      uint32_t u = min(nnew, (uint32_t)K);
      uint32_t lb = (uint32_t)t;
      if (u > 0 && t > 0) {
        const uint64_t f0 = L.k0()[nl[0]];
        const uint32_t f1 = dd | L.tbr()[nl[0]];
        uint32_t cntl = 0;
        for (int i0 = 0; i0 < t; i0 += 32) {
          const int i = i0 + lane;
          cntl += __popc(__ballot_sync(SSSD_FULL, i < t && g_less(T.g0()[i], T.g1()[i], f0, f1)));
        }
        lb = cntl;
        if (lb >= (uint32_t)K) u = 0;
      }
      uint32_t ue = 0;
      for (uint32_t m0 = 0; m0 < u; m0 += 32) {
        const uint32_t m = m0 + lane;
        uint32_t slot = 0xffffffffu;
        if (m < u) {
          const uint32_t sm = nl[m];
          const uint64_t x0 = L.k0()[sm];
          const uint32_t x1 = dd | L.tbr()[sm];
          uint32_t lo = lb, hi = (uint32_t)t;
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (g_less(T.g0()[mid], T.g1()[mid], x0, x1)) lo = mid + 1;
            else hi = mid;
          }
          slot = m + lo;
          npos[m] = slot;
        }
        const uint32_t okm = __ballot_sync(SSSD_FULL, slot < (uint32_t)K);
        ue += __popc(okm);
        if (okm != SSSD_FULL) break;
      }
      __syncwarp();
      for (int c0 = ((t - 1) >> 5) << 5; c0 >= (int)(lb & ~31u) && t > 0 && ue > 0; c0 -= 32) {
        const int i = c0 + lane;
        uint64_t x0 = 0;
        uint32_t x1 = 0, xp = 0, xt = 0, xq = 0, pos = 0xffffffffu;
        if (i < t && i >= (int)lb) {
          x0 = T.g0()[i];
          x1 = T.g1()[i];
          xp = T.pid()[i];
          xt = T.tok()[i];
          xq = T.ppid()[i];
          uint32_t lo = 0, hi = ue;
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (npos[mid] - mid <= (uint32_t)i) lo = mid + 1;
            else hi = mid;
          }
          pos = (uint32_t)i + lo;
        }
        __syncwarp();
        if (pos < (uint32_t)K) {
          T.g0()[pos] = x0;
          T.g1()[pos] = x1;
          T.pid()[pos] = xp;
          T.tok()[pos] = xt;
          T.ppid()[pos] = xq;
        }
        __syncwarp();
      }
      for (uint32_t m = lane; m < ue; m += 32) {
        const uint32_t pos = npos[m], sm = nl[m], g = L.ord()[sm];
        T.g0()[pos] = L.k0()[sm];
        T.g1()[pos] = dd | L.tbr()[sm];
        T.pid()[pos] = L.pid()[sm];
        T.tok()[pos] = L.tok()[g];
        T.ppid()[pos] = L.ppid()[g];
      }
      t = min(K, t + (int)u);
      __syncwarp();

      // the parents of the next level: the prefix at or below the threshold
      uint32_t nexp = ne;
      if (t == K) {
        const uint64_t tau0n = T.g0()[K - 1];
        const uint32_t tau1n = T.g1()[K - 1];
        nexp = 0;
        for (uint32_t s0 = 0; s0 < ne; s0 += 32) {
          const uint32_t s = s0 + lane;
          const bool ok = s < ne && !g_less(tau0n, tau1n, L.k0()[s], dd | L.tbr()[s]);
          const uint32_t okm = __ballot_sync(SSSD_FULL, ok);
          nexp += __popc(okm);
          if (okm != SSSD_FULL) break;
        }
      }
      if (lane == 0) {
        sh->nexp = nexp;
        sh->next_pid = next_pid;
        sh->t = (uint32_t)t;
        if (nexp > (uint32_t)kCtaParCap && sh->gpar_cap < nexp) {
          uint32_t need = 2 * kCtaParCap;
          while (need < nexp) need <<= 1;
          unsigned long long at = atomicAdd(cursor, (unsigned long long)need * kLsParBytes);
          if (at + (unsigned long long)need * kLsParBytes > pool_bytes) {
            atomicExch(err, SSSD_E_WORKSPACE);
            sh->stop = 1;
          } else {
            sh->gpar = pool + at;
            sh->gpar_cap = need;
          }
        }
      }
    }
    __syncthreads();
    // t and next_pid were computed by warp 0: every thread reads them back
    t = (int)sh->t;
    next_pid = sh->next_pid;
    if (sh->stop) break;
    const uint32_t nexp = sh->nexp;
    par = nexp > (uint32_t)kCtaParCap ? par_carve(sh->gpar, sh->gpar_cap) : par_carve(par_smem, kCtaParCap);
    for (uint32_t j = tid; j < nexp; j += kCtaThreads) {
      const uint32_t g = L.ord()[j];
      par.pp()[j] = L.pp()[g];
      par.a()[j] = L.a()[g];
      par.z()[j] = L.z()[g];
      par.cnt()[j] = L.cnt()[g];
      par.tbr()[j] = L.tbr()[j];
      par.pid()[j] = L.pid()[j];
    }
    gen_total += n_all;
    max_level = max(max_level, n_all);
    np = (int)nexp;
    __syncthreads();
    ph_merge += (uint32_t)clock() - tp;
  }
  __syncthreads();
  const long long t_levels = clock64();

  // 7. flatten: node v = 1..t is top entry v-1 (insertion order = G order)
  int* f_par = reinterpret_cast<int*>(smem);  // the level buffer is free now
  int* f_fc = f_par + S;
  int* f_ns = f_fc + S;
  int* f_pos = f_ns + S;
  int* f_dep = f_pos + S;
  int* pmap = f_dep + S;  // path id -> node (path ids < next_pid)
  const int size = t + 1;
  const bool use_map = (int)next_pid <= (kLsLevelBytes * kCtaLevCap) / 4 - 5 * S;
  if (use_map)
    for (int v = 1 + tid; v < size; v += kCtaThreads) pmap[T.pid()[v - 1]] = v;
  __syncthreads();
  for (int v = tid; v < size; v += kCtaThreads) {
    int pr = -1, dv = 0;
    if (v > 0) {
      const uint32_t pp = T.ppid()[v - 1];
      pr = 0;
      if (pp != 0) {
        if (use_map) {
          pr = pmap[pp];
        } else {
          for (int u = 0; u < v - 1; ++u)
            if (T.pid()[u] == pp) {
              pr = u + 1;
              break;
            }
        }
      }
      dv = (int)(T.g1()[v - 1] >> 26);
    }
    f_par[v] = pr;
    f_dep[v] = dv;
    f_fc[v] = -1;
  }
  __syncthreads();
  uint32_t* o_tok = out.tokens + (size_t)b * S;
  int32_t* o_par = out.parents + (size_t)b * S;
  int32_t* o_dep = out.depths + (size_t)b * S;
  int maxd = 0;
  for (int v = tid; v < size; v += kCtaThreads) maxd = max(maxd, f_dep[v]);
  maxd = __syncthreads_or(maxd > 8) ? 9 : 0;
  const bool extra = out.priority || out.source || out.pos;
  auto node_extra = [&](int v, int k) {
    if (v == 0) {
      write_node_extra(out, c, b, k, __longlong_as_double(0x7ff0000000000000ll), -1, 0);
    } else {
      write_node_extra(out, c, b, k, __longlong_as_double((long long)~T.g0()[v - 1]),
                       (int32_t)((T.g1()[v - 1] >> kTbBits) & 15u), f_dep[v]);
    }
  };
  if (maxd <= 8 && size <= 127) {
    // pre-order position = rank of the node's ancestor-index path (7 bits per depth)
    uint64_t* kk = reinterpret_cast<uint64_t*>(smem + ((20 * S + 7) & ~7));
    for (int v = tid; v < size; v += kCtaThreads) {
      uint64_t key = 0;
      for (int u = v; u > 0; u = f_par[u]) key |= (uint64_t)u << (7 * (8 - f_dep[u]));
      kk[v] = key;
    }
    __syncthreads();
    for (int v = tid; v < size; v += kCtaThreads) {
      const uint64_t kv = kk[v];
      int r = 0;
      for (int q = 0; q < size; ++q) r += kk[q] < kv ? 1 : 0;
      f_pos[v] = r;
    }
    __syncthreads();
    for (int v = tid; v < size; v += kCtaThreads) {
      const int k = f_pos[v];
      o_tok[k] = v == 0 ? s_root : T.tok()[v - 1];
      o_par[k] = v == 0 ? -1 : f_pos[f_par[v]];
      o_dep[k] = f_dep[v];
      if (extra) node_extra(v, k);
    }
  } else if (warp == 0) {
    for (int v = lane; v < size; v += 32) f_pos[v] = -1;
    __syncwarp();
    for (int c0 = ((size - 1) >> 5) << 5; c0 >= 0; c0 -= 32) {
      const int v = c0 + lane;
      const bool ok = v >= 1 && v < size;
      const int p = ok ? f_par[v] : -2 - lane;
      const uint32_t mm = __match_any_sync(SSSD_FULL, p);
      const uint32_t above = mm & ~((2u << lane) - 1u);
      int ns = -1;
      if (ok) ns = above ? c0 + __ffs(above) - 1 : f_pos[p];
      __syncwarp();
      if (ok) {
        f_ns[v] = ns;
        if (lane == __ffs(mm) - 1) f_pos[p] = v;
      }
      __syncwarp();
    }
    for (int v = lane; v < size; v += 32) f_fc[v] = f_pos[v];
    __syncwarp();
    if (lane == 0) {  // DFS walk: first child, else next sibling of the nearest ancestor that has one
      int v = 0, k = 0;
      while (true) {
        f_pos[v] = k;
        o_tok[k] = v == 0 ? s_root : T.tok()[v - 1];
        o_par[k] = v == 0 ? -1 : f_pos[f_par[v]];
        o_dep[k] = f_dep[v];
        if (extra) node_extra(v, k);
        ++k;
        int nx = f_fc[v];
        if (nx < 0) {
          int u = v;
          while (u > 0 && f_ns[u] < 0) u = f_par[u];
          if (u <= 0) break;
          nx = f_ns[u];
        }
        v = nx;
      }
    }
  }
  __syncthreads();
  const int W = (S + 63) >> 6;
  uint64_t* o_mask = out.mask + (size_t)b * S * W;
  for (int v = tid; v < size; v += kCtaThreads) {  // mask row = ancestors-or-self (ref draft.py:80-84)
    const int k = f_pos[v];
    for (int w = 0; w < W; ++w) {
      uint64_t m = 0;
      for (int x = v; x >= 0; x = f_par[x]) {
        const int pk = f_pos[x];
        if ((pk >> 6) == w) m |= 1ull << (pk & 63);
      }
      o_mask[(size_t)k * W + w] = m;
    }
  }
  for (int k = size + tid; k < S; k += kCtaThreads) {
    o_tok[k] = 0;
    o_par[k] = -1;
    o_dep[k] = -1;
    for (int w = 0; w < W; ++w) o_mask[(size_t)k * W + w] = 0;
    if (extra) write_node_extra(out, c, b, k, 0.0, -1, -1);
  }
  if (tid == 0) {
    out.size[b] = size;
    if (cycles) {
      long long* st = cycles + (size_t)b * 8;
      const long long t_end = clock64();
      st[0] = t_end - t_start;
      st[1] = ph_gen;
      st[2] = ph_sort + ph_cls;
      st[3] = t_end - t_levels;
      st[4] = ph_merge - ph_cls;  // merge + parents (ph_merge spans the class pass too)
      st[5] = levels | (long long)max_level << 16;
      st[6] = gen_total;
      st[7] = ph_cls;
    }
  }
}

}  // namespace sssd
