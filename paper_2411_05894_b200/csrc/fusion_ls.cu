// K5, level-synchronous form: fusion + DFS flatten for SSSD drafts (sm_100a).
// Replaces ref fusion.py:209-261 (merge) and draft.py:67-86 (flatten) with the
// same output bit for bit; tests/ls_model.py states the algorithm over the
// oracle's tries and DESIGN.md 3.1 the equivalence argument:
//
//  * a source node's key (-priority, depth, rank, ticket) exceeds its parent's
//    (count ratios <= 1, discount rows non-increasing in depth), so the
//    reference heap pops all source-trie nodes in global key order;
//  * tickets of equal (priority, depth, rank) order by the parent's pop order,
//    then child order, so inside one (depth, rank) class the order is
//    (-priority, parent's class position, child first-appearance) -- one sort
//    per level gives each node its class position tb and its global key
//    G = (~bits(priority), depth, rank, tb);
//  * the draft is the first dec_len-1 distinct token paths in G order and a
//    path's parent path precedes it, so only nodes with G <= the current
//    (dec_len-1)-th best distinct-path key are ever expanded.
//
// One warp per request, one trie level per iteration: the children of every
// expanded node of the level are generated together (element ranges of the
// sorted source arrays, flattened over the lanes), sorted, given class
// positions and path ids, and merged into the running top list.  The heap
// form (fusion.cu) needs ~78 dependent pops per cfg2 request; this form needs
// <= branch_len levels of lane-parallel work, all in shared memory unless a
// level outgrows kLsCap nodes (then the request's global pool slice).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "propose.cuh"
#include "fusion_ls.cuh"

namespace sssd {

int ls_smem_bytes(int P, int S) {
  return kLsLevelBytes * kLsCap + kLsParBytes * kLsParCap + (P + 1) * (int)sizeof(SrcDesc) +
         top_bytes(S) + S * 8 + kLsRankWords * 4;
}


// Cut a full level buffer to its smallest `keepn` (<= kLsCap - 32) nodes, moved to
// slots [0, keepn) in order; returns keepn and the first cut key.
__device__ SSSD_LS_CALL uint32_t ls_cut(LsLevel L, uint32_t nb, uint32_t keepn, uint64_t* th0, uint64_t* th1) {
  const uint32_t lane = (uint32_t)lane_id();
  __syncwarp();  // order the level records this warp emitted before the sort reads them (racecheck)
  ls_sort(L, nb);
  *th0 = L.k0()[keepn];
  *th1 = L.k1()[keepn];
  // read the whole kept prefix (registers of every round) before any write:
  // a record may move into a slot another lane still has to read
  constexpr int R = (kLsCap - 32 + 31) / 32;
  uint32_t a[R], z[R], c[R], t[R], p[R];
  double q[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t s = lane + 32 * r;
    if (s < keepn) {
      const uint32_t g = L.ord()[s];
      q[r] = L.pp()[g];
      a[r] = L.a()[g];
      z[r] = L.z()[g];
      c[r] = L.cnt()[g];
      t[r] = L.tok()[g];
      p[r] = L.ppid()[g];
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t s = lane + 32 * r;
    if (s < keepn) {
      L.pp()[s] = q[r];
      L.a()[s] = a[r];
      L.z()[s] = z[r];
      L.cnt()[s] = c[r];
      L.tok()[s] = t[r];
      L.ppid()[s] = p[r];
    }
  }
  for (uint32_t s = lane; s < keepn; s += 32) L.ord()[s] = s;
  __syncwarp();
  return keepn;
}

// Generate the depth-d children of parents [0, np) (element ranges scanned
// flat over the lanes; runs of equal token inside one parent's range are
// one child) into L.  Returns (nodes kept in L, all children).
// With keepn == 0, nodes past `cap` are counted but not written.  With keepn
// (the shared-memory buffer, dec_len - 1 <= keepn <= cap - 32), a full buffer
// is sorted and cut to its smallest keepn nodes, and later children at or
// above the cut key are discarded: L always holds a prefix of the level's
// (k0, k1) order, which is all the level needs whenever that prefix holds
// dec_len - 1 distinct paths (the caller checks and otherwise regenerates).
template <bool kPF>
__device__ SSSD_LS_CALL uint2 ls_generate(const LsPar par, int np, uint32_t E, LsLevel L, uint32_t cap,
                                          uint32_t keepn, const SrcDesc* sd, const double* disc,
                                          int disc_stride, int d, bool has_empty, bool has_tau, uint64_t tau0,
                                          uint32_t tau_dr) {
  const int lane = lane_id();
  const uint32_t lt = lanemask_lt();
  uint32_t n = 0, nb = 0;
  uint64_t th0 = ~0ull, th1 = ~0ull;  // cut key: children >= it are discarded
  const double* drow = disc + d;
  // A child whose (~priority, depth, rank) already exceeds the top list's
  // (dec_len-1)-th key tau (from earlier levels; tau only decreases) can be
  // neither expanded nor listed, and it sorts after every node that can:
  // it is not generated at all (a tie on all three keeps the node, tb decides).
  auto emit = [&](bool pred, int j, uint32_t tk, uint32_t cnt, uint32_t first, uint32_t s, uint32_t e) {
    bool live = pred && cnt > 0;
    if (!__ballot_sync(SSSD_FULL, live)) return;
    uint64_t k0 = ~0ull, k1 = ~0ull;
    double pp = 0.0;
    uint32_t pid = 0;
    if (live) {
      const uint32_t tr = par.tbr()[j], rk = tr >> kTbBits, pc = par.cnt()[j];
      const double ratio = ratio_rn(cnt, pc);  // == __ddiv_rn (common.cuh)
      pp = __dmul_rn(par.pp()[j], ratio);                                           // ref fusion.py:259
      const double pr = __dmul_rn(pp, drow[rk * disc_stride]);                    // ref fusion.py:246
      k0 = ~(uint64_t)__double_as_longlong(pr);
      k1 = (uint64_t)rk << 56 | (uint64_t)(tr & kTbMask) << 32 | first;
      pid = par.pid()[j];
      const uint32_t dr = (uint32_t)d << 26 | rk << kTbBits;
      if (has_tau && (k0 > tau0 || (k0 == tau0 && dr > tau_dr))) live = false;
    }
    const uint32_t bal = __ballot_sync(SSSD_FULL, live);
    if (!bal) return;
    n += __popc(bal);
    bool keep = live && k_less(k0, k1, th0, th1);
    uint32_t km = __ballot_sync(SSSD_FULL, keep);
    if (keepn && nb + __popc(km) > cap) {  // cut the full buffer to its smallest keepn
      nb = ls_cut(L, nb, keepn, &th0, &th1);
      keep = live && k_less(k0, k1, th0, th1);
      km = __ballot_sync(SSSD_FULL, keep);
    }
    if (keep) {
      const uint32_t pos = nb + __popc(km & lt);
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
    nb += __popc(km);
  };
  // Chunks of 32 lanes advance by 31 elements: lane 31 holds the next chunk's
  // first element as a look-ahead, so a run reaching lane 30 knows whether it
  // continues; every run is emitted once, by its last owned lane, with the
  // count / first / start carried in from earlier chunks.
  bool c_open = false;
  uint32_t c_cnt = 0, c_first = 0, c_start = 0;
  auto parent_of = [&](uint32_t x) {  // last parent whose offset is <= x
    int lo = 0, hi = np;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (par.off()[mid] <= x) lo = mid;
      else hi = mid;
    }
    return lo;
  };
  // Without empty parents every parent starting inside a chunk owns a distinct
  // element, so the chunk's parent starts form a 32-bit head mask (one OR
  // reduction) and an element's parent is the carried parent plus the heads
  // at or before it; a level with empty (depth-capped) parents binary-searches.
  // one chunk's parents and element loads (kPF: issued one chunk ahead, so a
  // lone warp overlaps the global-load latency with the previous chunk's work)
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
      if (q < np) {
        const uint32_t st = par.off()[q] - base;
        if (st < 32) bit = 1u << st;
      }
      const uint32_t heads = __reduce_or_sync(SSSD_FULL, bit);
      r.j = jprev + __popc(heads & (0xffffffffu >> (31 - lane)));
    }
    if (x < E) {
      if (has_empty) r.j = parent_of(x);
      const SrcDesc& sc = sd[par.tbr()[r.j] >> kTbBits];
      r.i = par.a()[r.j] + (x - par.off()[r.j]);
      r.th = (uint32_t)sc.thr;
      r.lm = sc.meta[r.i];  // independent loads; column d-1 exists (d <= source depth)
      r.tk = sc.tok[(int64_t)(d - 1) * sc.stride + r.i];
      r.og = sc.orig[r.i];
    }
    return r;
  };
  Ld cur = load_chunk(0, -1);
  for (uint32_t base = 0; base < E; base += 31) {
    const uint32_t x = base + lane;
    const bool last = base + 32 >= E;  // no look-ahead: lane 31 (if any) is the final element
    const bool owned = x < E && (lane < 31 || last);
    const int jprev = __shfl_sync(SSSD_FULL, cur.j, 30);  // parent of the next chunk's element base + 30
    Ld nxt{};
    if (kPF && !last) nxt = load_chunk(base + 31, jprev);
    const int j = cur.j;
    const uint32_t i = cur.i, lm = cur.lm, tk = cur.tk, og = cur.og, th = cur.th;
    const bool has = x < E && el_len(lm) >= (uint32_t)d;
    const bool w = owned && has && el_m(lm) >= th;
    const uint32_t orig = w ? og : 0xffffffffu;
    const uint32_t wt = w ? el_wt(lm) : 0u;
    const uint32_t hasm = __ballot_sync(SSSD_FULL, has);
    if (hasm) {  // (a carried run always continues at lane 0, so none is open otherwise)
      int lo_l, hi_l;
      run_bounds(has, (uint32_t)j, tk, lo_l, hi_l);
      // run minimum of orig and run sum of weights (segmented down-scans;
      // runs are lane intervals)
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
      if (c_open && lo_l == 0) {  // the run carried in from the previous chunk
        cnt += c_cnt;
        fm = min(fm, c_first);
        start = c_start;
      }
      const bool to_next = !last && has && hi_l == 31;  // my run reaches the look-ahead
      emit(owned && has && lane == hi_l && !to_next, j, tk, cnt, fm, start, i + 1);
      c_open = __ballot_sync(SSSD_FULL, lane == 30 && to_next) != 0;
      if (c_open) {
        c_cnt = __shfl_sync(SSSD_FULL, cnt, 30);
        c_first = __shfl_sync(SSSD_FULL, fm, 30);
        c_start = __shfl_sync(SSSD_FULL, start, 30);
      }
    }
    if (last) break;
    cur = kPF ? nxt : load_chunk(base + 31, jprev);
  }
  __syncwarp();
  return make_uint2(nb, n);
}

#ifndef SSSD_LS_MINB
#define SSSD_LS_MINB 24  // 80 registers, no spills (the level phases are inlined)
#endif
#ifdef SSSD_LS_PROBE  // per-phase cycle counts in the cycle probe (costs registers)
#define LS_PROBE(...) __VA_ARGS__
#else
#define LS_PROBE(...)
#endif

template <bool kPF>
__device__ __forceinline__ void draft_ls_body(const SrcDesc* desc, const uint32_t* root_tok, const KCfg& c,
                                              uint8_t* pool, unsigned long long* cursor, uint64_t pool_bytes,
                                              int32_t* err, const sssd_draft_out& out, long long* cycles,
                                              const int32_t* order, const int32_t* order_count) {
  extern __shared__ __align__(16) uint8_t smem[];
  const long long t_start = clock64();
#ifdef SSSD_LS_TIMELINE  // measurement builds: global start / end stamps per request (cycle probe slots 6, 7)
  unsigned long long g_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
#endif
  if (order_count && (int)blockIdx.x >= *order_count) return;  // a list filled on the device
  const int b = order ? order[c.b0 + blockIdx.x] : c.b0 + blockIdx.x;
  const int lane = lane_id();
  const uint32_t lt = lanemask_lt();
  const int S = c.S, K = S - 1;
  const int NR = c.P + 1;

  uint8_t* sp = smem;
  const LsLevel Ls = level_carve(sp, kLsCap);
  sp += kLsLevelBytes * kLsCap;
  LsPar par = par_carve(sp, kLsParCap);
  sp += kLsParBytes * kLsParCap;
  SrcDesc* sd = reinterpret_cast<SrcDesc*>(sp);
  sp += NR * sizeof(SrcDesc);
  const LsTop T = top_carve(sp, S);
  sp += top_bytes(S);
  uint32_t* nl = reinterpret_cast<uint32_t*>(sp);  // sorted positions of the level's new paths
  sp += S * 4;
  uint32_t* npos = reinterpret_cast<uint32_t*>(sp);  // their slots in the merged top list
  sp += S * 4;
  uint32_t* rcnt = reinterpret_cast<uint32_t*>(sp);  // per-rank class counters

  for (int r = lane; r < NR; r += 32) sd[r] = desc[(size_t)b * NR + r];
  __syncwarp();

  // level 0: the source roots are the parents of the seeds (path prob 1.0, so
  // pp * (count / root_count) is the seed's count / root_count exactly)
  int np = 0;
  if (K > 0) {
    for (int rk = 0; rk < NR; ++rk) {
      if (sd[rk].n <= 0) continue;
      uint32_t rc = 0;
      for (int i = lane; i < sd[rk].n; i += 32) {
        const uint32_t mt = sd[rk].meta[i];
        rc += (int)el_m(mt) >= sd[rk].thr ? el_wt(mt) : 0u;
      }
      rc = __reduce_add_sync(SSSD_FULL, rc);
      if (rc == 0) continue;
      if (lane == 0) {
        par.a()[np] = 0;
        par.z()[np] = (uint32_t)sd[rk].n;
        par.cnt()[np] = rc;
        par.pp()[np] = 1.0;
        par.tbr()[np] = (uint32_t)rk << kTbBits;
        par.pid()[np] = 0;
      }
      ++np;
    }
  }
  __syncwarp();

  uint8_t* glev = nullptr;  // global level / parent buffers (pool), grown on demand
  uint32_t glev_cap = 0;
  uint8_t* gpar = nullptr;
  uint32_t gpar_cap = 0;
  int t = 0;
  uint32_t next_pid = 1;
  uint32_t gen_total = 0, max_level = 0, gallocs = 0, levels = 0;
  uint32_t ph_gen = 0, ph_sort = 0, ph_merge = 0;  // probe: generation, sort + classes, merge + parents

  for (int d = 1; np > 0 && d < c.disc_stride; ++d) {
    // 1. exclusive scan of the parents' element-range sizes
    uint32_t E = 0;
    bool has_empty = false;  // a parent with no element at this depth (shares its offset)
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
    if (E == 0) break;
    ++levels;

    // 2. generate into shared memory (keeping the smallest nodes when the level
    //    outgrows it); a level whose kept prefix is too short, or that cannot
    //    drop (dec_len - 1 > kLsCap - 32), is generated again in full into a
    //    global buffer
    LsLevel L = Ls;
    // a cut keeps cap - 32 nodes: smaller prefixes (fewer cuts for small
    // drafts) measured worse on prompt-heavy levels, whose duplicate paths
    // across the P+1 sources then force the full regeneration
    const uint32_t keepn = K <= kLsCap - 32 ? (uint32_t)(kLsCap - 32) : 0u;
    const bool drop = keepn != 0;
    LS_PROBE(uint32_t tp = (uint32_t)clock());
    const bool has_tau = t == K;
    const uint64_t tau0 = has_tau ? T.g0()[K - 1] : 0ull;
    const uint32_t tau_dr = has_tau ? T.g1()[K - 1] & ~kTbMask : 0u;
    const uint2 gr = ls_generate<kPF>(par, np, E, Ls, kLsCap, keepn, sd, c.disc, c.disc_stride, d, has_empty, has_tau, tau0,
                                 tau_dr);
    LS_PROBE(ph_gen += (uint32_t)clock() - tp; tp = (uint32_t)clock());
    uint32_t n = gr.x, n_all = gr.y;
    if (n_all == 0) break;
    bool global = !drop && n_all > (uint32_t)kLsCap;
    const uint32_t pid0 = next_pid;
    uint32_t nnew = 0;
    bool fail = false;
    for (int attempt = 0; attempt < 2; ++attempt) {
      if (global) {
        uint32_t need = 64;
        while (need < n_all) need <<= 1;
        if (glev_cap < need) {
          glev = pool_take(pool, cursor, pool_bytes, err, (unsigned long long)need * kLsLevelBytes);
          if (!glev) {
            fail = true;
            break;
          }
          glev_cap = need;
          ++gallocs;
        }
        L = level_carve(glev, glev_cap);
        n = ls_generate<kPF>(par, np, E, L, glev_cap, 0u, sd, c.disc, c.disc_stride, d, has_empty, has_tau, tau0,
                        tau_dr).x;
      }
      if (n > kTbMask) {  // class positions must fit their field
        if (lane == 0) atomicExch(err, SSSD_E_LIMIT);
        fail = true;
        break;
      }

      LS_PROBE(ph_gen += (uint32_t)clock() - tp; tp = (uint32_t)clock());
      // 3. sort the level by (k0, k1) = (~priority, rank, parent tb, first)
      ls_sort(L, n);

      // 4. class positions, path ids (first occurrence in G order wins), new paths
      next_pid = pid0;
      nnew = 0;
      if (lane < kLsRankWords) rcnt[lane] = 0;
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
      }
      if (n < n_all && nnew < (uint32_t)K) {  // the kept prefix lacks dec_len - 1 paths
        global = true;
        continue;
      }
      break;
    }
    if (fail) break;
    LS_PROBE(ph_sort += (uint32_t)clock() - tp; tp = (uint32_t)clock());
    gen_total += n_all;
    max_level = max(max_level, n_all);

    // 5. merge the level's new paths (already in G order) into the top list,
    //    in place: new paths find their slots against the old list, old
    //    entries move up chunk by chunk from the end (pos >= i), then the new
    //    paths land in the gaps
    const uint32_t dd = (uint32_t)d << 26;
    {
      uint32_t u = min(nnew, (uint32_t)K);
      // top entries below the level's best new path keep their slots: lb of them
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
        if (lb >= (uint32_t)K) u = 0;  // the top list is full of better paths: nothing enters
      }
      // slots of the new paths against the old list; they increase with m, so
      // the paths that land inside the list (slot < K) are a prefix of ue
      uint32_t ue = 0;
      for (uint32_t m0 = 0; m0 < u; m0 += 32) {
        const uint32_t m = m0 + lane;
        uint32_t slot = 0xffffffffu;
        if (m < u) {
          const uint32_t sm = nl[m];
          const uint64_t x0 = L.k0()[sm];
          const uint32_t x1 = dd | L.tbr()[sm];
          uint32_t lo = lb, hi = (uint32_t)t;  // top entries with G < x
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
      // an old entry i moves up by the landing new paths that precede it:
      // #{m < ue : npos[m] - m <= i} (non-decreasing in m); entries pushed past
      // K drop out.  Chunks go from the end so no unread entry is overwritten.
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
    }

    // 6. the parents of the next level: the prefix at or below the threshold
    uint32_t nexp = n;
    if (t == K) {
      const uint64_t tau0 = T.g0()[K - 1];
      const uint32_t tau1 = T.g1()[K - 1];
      nexp = 0;
      for (uint32_t s0 = 0; s0 < n; s0 += 32) {
        const uint32_t s = s0 + lane;
        const bool ok = s < n && !g_less(tau0, tau1, L.k0()[s], dd | L.tbr()[s]);
        const uint32_t okm = __ballot_sync(SSSD_FULL, ok);
        nexp += __popc(okm);
        if (okm != SSSD_FULL) break;
      }
    }
    if (nexp > (uint32_t)kLsParCap) {
      if (gpar_cap < nexp) {
        uint32_t need = 2 * kLsParCap;
        while (need < nexp) need <<= 1;
        gpar = pool_take(pool, cursor, pool_bytes, err, (unsigned long long)need * kLsParBytes);
        if (!gpar) break;
        gpar_cap = need;
        ++gallocs;
      }
      par = par_carve(gpar, gpar_cap);
    } else {
      par = par_carve(smem + kLsLevelBytes * kLsCap, kLsParCap);
    }
    for (uint32_t j = lane; j < nexp; j += 32) {
      const uint32_t g = L.ord()[j];
      par.pp()[j] = L.pp()[g];
      par.a()[j] = L.a()[g];
      par.z()[j] = L.z()[g];
      par.cnt()[j] = L.cnt()[g];
      par.tbr()[j] = L.tbr()[j];
      par.pid()[j] = L.pid()[j];
    }
    __syncwarp();
    np = (int)nexp;
    LS_PROBE(ph_merge += (uint32_t)clock() - tp);
  }
  __syncwarp();
  const long long t_levels = clock64();

  // 7. flatten: node v = 1..t is top entry v-1 (insertion order = G order;
  //    a parent path precedes its children, siblings insert in index order)
  int* f_par = reinterpret_cast<int*>(smem);  // the level buffer is free now
  int* f_fc = f_par + S;                      // first child
  int* f_ns = f_fc + S;                       // next sibling
  int* f_pos = f_ns + S;                      // pre-order position
  int* f_dep = f_pos + S;
  int* pmap = f_dep + S;  // path id -> node (path ids < next_pid)
  const int size = t + 1;
  const bool use_map = (int)next_pid <= (kLsLevelBytes * kLsCap) / 4 - 5 * S;
  if (use_map)
    for (int v = 1 + lane; v < size; v += 32) pmap[T.pid()[v - 1]] = v;
  __syncwarp();
  int maxd = 0;
  for (int v = lane; v < size; v += 32) {
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
    maxd = max(maxd, dv);
  }
  __syncwarp();
  uint32_t* o_tok = out.tokens + (size_t)b * S;
  int32_t* o_par = out.parents + (size_t)b * S;
  int32_t* o_dep = out.depths + (size_t)b * S;
  maxd = __reduce_max_sync(SSSD_FULL, maxd);
  // per-node priority (the top entry's key holds ~bits(priority)) and merge
  // rank of the node's first insertion (ref fusion.py:185-198), position id
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
    // pre-order position = rank of the node's ancestor-index path (7 bits per
    // depth, index order = sibling insertion order, a prefix sorts first)
    uint64_t* kk = reinterpret_cast<uint64_t*>(smem + ((20 * S + 7) & ~7));
    for (int v = lane; v < size; v += 32) {
      uint64_t key = 0;
      for (int u = v; u > 0; u = f_par[u]) key |= (uint64_t)u << (7 * (8 - f_dep[u]));
      kk[v] = key;
    }
    __syncwarp();
    for (int v = lane; v < size; v += 32) {
      const uint64_t kv = kk[v];
      int r = 0;
      for (int q = 0; q < size; ++q) r += kk[q] < kv ? 1 : 0;
      f_pos[v] = r;
    }
    __syncwarp();
    for (int v = lane; v < size; v += 32) {
      const int k = f_pos[v];
      o_tok[k] = v == 0 ? root_tok[b] : T.tok()[v - 1];
      o_par[k] = v == 0 ? -1 : f_pos[f_par[v]];
      o_dep[k] = f_dep[v];
      if (extra) node_extra(v, k);
    }
  } else {
    // next sibling = the next index with the same parent: inside a chunk by
    // match_any, across chunks through a first-index-per-parent table built
    // from the last chunk backwards (f_pos doubles as that table)
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
        if (lane == __ffs(mm) - 1) f_pos[p] = v;  // first index with parent p so far
      }
      __syncwarp();
    }
    for (int v = lane; v < size; v += 32) f_fc[v] = f_pos[v];
    __syncwarp();
    if (lane == 0) {  // DFS walk: first child, else next sibling of the nearest ancestor that has one
      int v = 0, k = 0;
      while (true) {
        f_pos[v] = k;
        o_tok[k] = v == 0 ? root_tok[b] : T.tok()[v - 1];
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
  __syncwarp();
  const int W = (S + 63) >> 6;
  uint64_t* o_mask = out.mask + (size_t)b * S * W;
  for (int v = lane; v < size; v += 32) {  // mask row = ancestors-or-self (ref draft.py:80-84)
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
  for (int k = size + lane; k < S; k += 32) {
    o_tok[k] = 0;
    o_par[k] = -1;
    o_dep[k] = -1;
    for (int w = 0; w < W; ++w) o_mask[(size_t)k * W + w] = 0;
    if (extra) write_node_extra(out, c, b, k, 0.0, -1, -1);
  }
  if (lane == 0) {
    out.size[b] = size;
    if (cycles) {  // per-request profile (optional): see sssd_set_cycle_probe
      long long* st = cycles + (size_t)b * 8;
      const long long t_end = clock64();
      st[0] = t_end - t_start;
      st[1] = ph_gen;
      st[2] = ph_sort;
      st[3] = t_end - t_levels;  // flatten
      st[4] = ph_merge;
      st[5] = levels | (long long)max_level << 16;
#ifdef SSSD_LS_TIMELINE
      unsigned long long g_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
      st[6] = (long long)g_start;
      st[7] = (long long)g_end;
#else
      st[6] = gen_total;
      st[7] = gallocs;
#endif
    }
  }
}

__global__ void __launch_bounds__(32, SSSD_LS_MINB)
    draft_ls_kernel(const SrcDesc* desc, const uint32_t* root_tok, KCfg c, uint8_t* pool,
                    unsigned long long* cursor, uint64_t pool_bytes, int32_t* err, sssd_draft_out out,
                    long long* cycles, const int32_t* order, const int32_t* order_count) {
  draft_ls_body<false>(desc, root_tok, c, pool, cursor, pool_bytes, err, out, cycles, order, order_count);
}

// Small launches (a warp alone on its SM sub-partition: latency, not issue
// slots, bounds it): element loads one chunk ahead, no register cap.
__global__ void __launch_bounds__(32, 1)
    draft_ls_small_kernel(const SrcDesc* desc, const uint32_t* root_tok, KCfg c, uint8_t* pool,
                          unsigned long long* cursor, uint64_t pool_bytes, int32_t* err, sssd_draft_out out,
                          long long* cycles, const int32_t* order, const int32_t* order_count) {
  draft_ls_body<true>(desc, root_tok, c, pool, cursor, pool_bytes, err, out, cycles, order, order_count);
}

}  // namespace sssd
