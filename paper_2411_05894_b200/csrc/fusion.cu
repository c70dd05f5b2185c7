// K5: best-first fusion + DFS flatten for SSSD drafts (sm_100a).
// Replaces ref fusion.py:209-261 (merge) and draft.py:67-86 (flatten); the
// tie-break and float semantics follow SURVEY.md A.5 / A.6 exactly.
//
// One warp per request.  Source tries are never materialised: a trie node is
// a range [a, z) of its source's element array sorted by (string, insertion
// order), so a node's children are the runs of equal token at its depth.
//
// Frontier.  The reference heap orders candidates by (-priority, depth, rank,
// ticket).  Children pushed by one pop share depth, rank and parent and hold
// consecutive tickets, so the frontier is kept as *sibling groups*: the heap
// minimum is the minimum over group heads of (-priority, depth, rank, group
// creation order), and inside a group candidates pop in (priority desc,
// first-appearance asc) order.  Keys are compared as 96-bit integers
// (~bits(priority) is monotone for priorities >= 0) with three REDUX
// (__reduce_min_sync) steps instead of shuffle trees; groups of <= 32
// children are stored in pop order at creation so advancing a head is O(1).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "propose.cuh"

namespace sssd {

struct Child {  // one candidate (32 B, global arena)
  double pp;       // path probability (ref fusion.py:244,259)
  uint32_t first;  // first-appearance position = reference child order
  uint32_t count;  // node count in its source trie
  uint32_t token;
  uint32_t a, b;   // element range of the candidate node in the source array
  uint32_t pad;
};

// A sibling group is split into a hot key (always in shared memory, scanned
// every pop) and a cold record (children pointer and cursor; shared memory for
// the first kGroupSmem groups, global overflow after).
struct Group {  // cold record (16 B)
  Child* ch;
  uint32_t head;  // head child index (low 24 bits) | draft parent << 24
  uint32_t nch;   // children (low 31 bits) | stored-in-pop-order flag << 31
};
static_assert(sizeof(Child) == kChildBytes, "Child layout");
static_assert(sizeof(Group) == kGroupBytes, "Group layout");
constexpr uint32_t kExhausted = 0xffffffffu;  // meta of a group with no candidates left

__device__ __forceinline__ uint32_t g_depth(uint32_t meta) { return meta >> 26; }
__device__ __forceinline__ uint32_t g_rank(uint32_t meta) { return (meta >> 22) & 0xf; }

__device__ __forceinline__ void prio_key(double pr, uint32_t& hi, uint32_t& lo) {
  const uint64_t k = ~(uint64_t)__double_as_longlong(pr);
  hi = (uint32_t)(k >> 32);
  lo = (uint32_t)k;
}

__device__ __forceinline__ bool key_less(uint32_t ah, uint32_t al, uint32_t at, uint32_t bh,
                                         uint32_t bl, uint32_t bt) {
  return ah < bh || (ah == bh && (al < bl || (al == bl && at < bt)));
}

// Lane holding the minimum (hi, lo, tie) among valid lanes (ties are unique),
// or -1 when no lane is valid.
__device__ __forceinline__ int warp_argmin3(bool valid, uint32_t hi, uint32_t lo, uint32_t tie) {
  if (!__ballot_sync(SSSD_FULL, valid)) return -1;
  if (!valid) hi = lo = tie = 0xffffffffu;
  const uint32_t mh = __reduce_min_sync(SSSD_FULL, hi);
  bool c = valid && hi == mh;
  const uint32_t ml = __reduce_min_sync(SSSD_FULL, c ? lo : 0xffffffffu);
  c = c && lo == ml;
  const uint32_t mt = __reduce_min_sync(SSSD_FULL, c ? tie : 0xffffffffu);
  c = c && tie == mt;
  return __ffs(__ballot_sync(SSSD_FULL, c)) - 1;
}

struct Arena {
  // child lists: a shared-memory slab first, then the request's global slab,
  // then the shared overflow pool
  Child* sslab;
  uint32_t sused, scap;
  Child* slab;
  uint32_t used, cap;
  Child* pool;
  unsigned long long* cursor;
  uint64_t pool_cap;
  int32_t* err;
  uint32_t spill = 0;    // probe: allocations served outside shared memory
  uint32_t scanned = 0;  // probe: elements scanned by expansions
  __device__ Child* alloc(uint32_t n) {  // warp-uniform
    scanned += n;
    if (sused + n <= scap) {
      Child* p = sslab + sused;
      sused += n;
      return p;
    }
    ++spill;
    if (used + n <= cap) {
      Child* p = slab + used;
      used += n;
      return p;
    }
    unsigned long long at = 0;
    if (lane_id() == 0) at = atomicAdd(cursor, (unsigned long long)n);
    at = __shfl_sync(SSSD_FULL, at, 0);
    if (at + n > pool_cap) {
      if (lane_id() == 0) atomicExch(err, SSSD_E_WORKSPACE);
      return nullptr;
    }
    return pool + at;
  }
  // give back the unused tail [p + keep, p + n) of the latest allocation
  __device__ void shrink(Child* p, uint32_t n, uint32_t keep) {
    if (p + n == sslab + sused) sused -= n - keep;
    else if (p + n == slab + used) used -= n - keep;
  }
};

// Frontier: hot keys of the *live* groups form a compact list in shared memory
// (an exhausted group is swapped out), so a pop scans only groups that still
// hold candidates.  Cold records are indexed by group id: ids < kGroupSmem in
// shared memory, later ids in the request's global overflow area.
struct Frontier {
  uint32_t *kh, *kl, *km;     // live list slots [0, kGroupSmem): ~bits(prio) hi / lo, meta
  uint32_t *gkh, *gkl, *gkm;  // live list slots >= kGroupSmem (global, rare)
  Group* sc;
  Group* gc;
  int G;  // groups created
  int A;  // live groups
  __device__ __forceinline__ Group* cold(int i) const { return i < kGroupSmem ? sc + i : gc + (i - kGroupSmem); }
  __device__ __forceinline__ void put(int q, uint32_t h, uint32_t l, uint32_t m) {
    if (q < kGroupSmem) { kh[q] = h; kl[q] = l; km[q] = m; }
    else { gkh[q - kGroupSmem] = h; gkl[q - kGroupSmem] = l; gkm[q - kGroupSmem] = m; }
  }
  __device__ __forceinline__ void get(int q, uint32_t& h, uint32_t& l, uint32_t& m) const {
    if (q < kGroupSmem) { h = kh[q]; l = kl[q]; m = km[q]; }
    else { h = gkh[q - kGroupSmem]; l = gkl[q - kGroupSmem]; m = gkm[q - kGroupSmem]; }
  }
};

// Expand the node covering [a, z) of source sd at depth D-1 into the group of
// its depth-D children (runs of equal token index D-1).  seed: the node is the
// source root (path prob = count / root_count, ref fusion.py:244); otherwise
// path prob = ppar * (count / pcount) (ref fusion.py:259).
__device__ void expand(const SrcDesc& sd, uint32_t rank, uint32_t D, uint32_t a, uint32_t z,
                       bool seed, double ppar, uint32_t pcount, uint32_t dparent, double disc,
                       Frontier& fr, Arena& ar) {
  const int lane = lane_id();
  const double dpc = (double)pcount;
  const uint32_t n = z - a;
  const uint32_t* tokD = sd.tok + (int64_t)(D - 1) * sd.stride;
  Child* ch = nullptr;
  uint32_t nch = 0;

  if (n == 1) {  // single element: at most one child, count 1
    const uint32_t lm = sd.meta[a], t = tokD[a], o = sd.orig[a];
    if (el_len(lm) < D || (int)el_m(lm) < sd.thr) return;
    ch = ar.alloc(1);
    if (!ch) return;
    if (lane == 0) {
      const double ratio = pcount == 1 ? 1.0 : __ddiv_rn(1.0, dpc);  // c/c == 1.0 exactly
      Child c;
      c.pp = seed ? ratio : __dmul_rn(ppar, ratio);
      c.first = o;
      c.count = 1;
      c.token = t;
      c.a = a;
      c.b = z;
      c.pad = 0;
      ch[0] = c;
    }
    nch = 1;
  } else {
    ch = ar.alloc(n);
    if (!ch) return;
    auto emit = [&](bool pred, uint32_t tok, uint32_t cnt, uint32_t first, uint32_t s, uint32_t e) {
      const bool live = pred && cnt > 0;
      const uint32_t bal = __ballot_sync(SSSD_FULL, live);
      if (live) {
        const double ratio = cnt == pcount ? 1.0 : __ddiv_rn((double)cnt, dpc);  // exact shortcut
        Child c;
        c.pp = seed ? ratio : __dmul_rn(ppar, ratio);
        c.first = first;
        c.count = cnt;
        c.token = tok;
        c.a = s;
        c.b = e;
        c.pad = 0;
        ch[nch + __popc(bal & lanemask_lt())] = c;
      }
      nch += __popc(bal);
    };
    bool c_open = false;
    uint32_t c_tok = 0, c_cnt = 0, c_first = 0xffffffffu, c_start = 0;
    for (uint32_t base = a; base < z; base += 32) {
      const uint32_t i = base + lane;
      bool has = false, w = false;
      uint32_t t = 0, orig = 0xffffffffu;
      if (i < z) {
        const uint32_t lm = sd.meta[i], tv = tokD[i], ov = sd.orig[i];
        if (el_len(lm) >= D) {
          has = true;
          t = tv;
          if ((int)el_m(lm) >= sd.thr) {
            w = true;
            orig = ov;
          }
        }
      }
      const uint32_t hasm = __ballot_sync(SSSD_FULL, has);
      if (!hasm) continue;
      // runs of equal token are contiguous (the range is sorted); lanes without
      // a token at this depth get a private key
      const unsigned long long key = has ? (0x100000000ull | t) : (0x200000000ull + (unsigned)lane);
      const uint32_t gm = __match_any_sync(SSSD_FULL, key);
      const uint32_t wm = __ballot_sync(SSSD_FULL, w);
      const int lo_l = __ffs(gm) - 1, hi_l = 31 - __clz(gm);
      // run minimum of orig: segmented down-scan (lane lo_l ends with the
      // minimum over [lo_l, hi_l]); runs are contiguous lane intervals
      uint32_t fm = orig;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_down_sync(SSSD_FULL, fm, o);
        if (lane + o <= hi_l) fm = min(fm, x);
      }
      fm = __shfl_sync(SSSD_FULL, fm, lo_l);
      uint32_t cnt = __popc(gm & wm);
      const uint32_t t0 = __shfl_sync(SSSD_FULL, t, 0);
      if (c_open && !((hasm & 1u) && t0 == c_tok)) {  // the carried run ended at the chunk edge
        emit(lane == 0, c_tok, c_cnt, c_first, c_start, base);
        c_open = false;
      }
      uint32_t start = base + lo_l;
      if (c_open && has && lo_l == 0) {  // continuation of the carried run
        cnt += c_cnt;
        fm = min(fm, c_first);
        start = c_start;
      }
      const bool to_next = has && hi_l == 31 && base + 32 < z;
      emit(has && lane == hi_l && !to_next, t, cnt, fm, start, base + hi_l + 1);
      if (__ballot_sync(SSSD_FULL, lane == 31 && to_next)) {
        c_tok = __shfl_sync(SSSD_FULL, t, 31);
        c_cnt = __shfl_sync(SSSD_FULL, cnt, 31);
        c_first = __shfl_sync(SSSD_FULL, fm, 31);
        c_start = __shfl_sync(SSSD_FULL, start, 31);
        c_open = true;
      } else {
        c_open = false;
      }
    }
    if (c_open) emit(lane == 0, c_tok, c_cnt, c_first, c_start, z);
    ar.shrink(ch, n, nch);
    if (nch == 0) return;
  }
  __syncwarp();

  uint32_t head = 0, kh = 0xffffffffu, kl = 0xffffffffu;
  uint32_t sorted = 1;
  if (nch == 1) {
    prio_key(__dmul_rn(ch[0].pp, disc), kh, kl);
  } else if (nch <= 32) {
    // store the group in pop order: rank of each child by (priority desc, first asc)
    const bool v = (uint32_t)lane < nch;
    Child cc;
    uint32_t h = 0xffffffffu, l = 0xffffffffu, f = 0xffffffffu;
    if (v) {
      cc = ch[lane];
      prio_key(__dmul_rn(cc.pp, disc), h, l);
      f = cc.first;
    }
    uint32_t r = 0;
    for (uint32_t j = 0; j < nch; ++j) {
      const uint32_t jh = __shfl_sync(SSSD_FULL, h, j), jl = __shfl_sync(SSSD_FULL, l, j),
                     jf = __shfl_sync(SSSD_FULL, f, j);
      r += key_less(jh, jl, jf, h, l, f) ? 1u : 0u;
    }
    __syncwarp();
    if (v) ch[r] = cc;
    const int src = __ffs(__ballot_sync(SSSD_FULL, v && r == 0)) - 1;
    kh = __shfl_sync(SSSD_FULL, h, src);
    kl = __shfl_sync(SSSD_FULL, l, src);
    __syncwarp();
  } else {
    // large group: keep emission order, find heads by scanning
    sorted = 0;
    uint32_t bh = 0xffffffffu, bl = 0xffffffffu, bf = 0xffffffffu, bi = 0;
    bool bv = false;
    for (uint32_t k = lane; k < nch; k += 32) {
      const Child c = ch[k];
      uint32_t h, l;
      prio_key(__dmul_rn(c.pp, disc), h, l);
      if (!bv || key_less(h, l, c.first, bh, bl, bf)) {
        bh = h;
        bl = l;
        bf = c.first;
        bi = k;
        bv = true;
      }
    }
    const int win = warp_argmin3(bv, bh, bl, bf);
    head = __shfl_sync(SSSD_FULL, bi, win);
    kh = __shfl_sync(SSSD_FULL, bh, win);
    kl = __shfl_sync(SSSD_FULL, bl, win);
  }
  if (lane == 0) {
    Group g;
    g.ch = ch;
    g.head = head | (dparent << 24);
    g.nch = nch | (sorted << 31);
    *fr.cold(fr.G) = g;
    fr.put(fr.A, kh, kl, (D << 26) | (rank << 22) | (uint32_t)fr.G);
  }
  ++fr.G;
  ++fr.A;
  __syncwarp();
}

#ifndef SSSD_DRAFT_MINB
#define SSSD_DRAFT_MINB 24  // resident requests per SM the register budget is sized for (24: best measured)
#endif

__global__ void __launch_bounds__(32, SSSD_DRAFT_MINB)
    draft_kernel(const SrcDesc* desc, const uint32_t* root_tok, KCfg c, Child* slabs,
                 uint32_t slab_cap, Child* pool, unsigned long long* cursor, uint64_t pool_cap,
                 int32_t* err, uint8_t* gover, int64_t gover_bytes, sssd_draft_out out,
                 long long* cycles, const int32_t* order) {
  extern __shared__ __align__(16) uint8_t smem[];
  const long long t_start = clock64();
  const int b = order ? order[c.b0 + blockIdx.x] : c.b0 + blockIdx.x;  // longest-first launch order
  const int lane = lane_id();
  const int S = c.S;
  const int W = (S + 63) >> 6;
  const int Gmax = draft_max_groups(c.P, S);
  const int Gs = min(Gmax, kGroupSmem);
  Child* sslab = reinterpret_cast<Child*>(smem);
  Group* sc = reinterpret_cast<Group*>(sslab + kChildSmem);
  uint32_t* skh = reinterpret_cast<uint32_t*>(sc + Gs);
  uint32_t* skl = skh + Gs;
  uint32_t* skm = skl + Gs;
  uint32_t* d_tok = skm + Gs;
  int16_t* d_par = reinterpret_cast<int16_t*>(d_tok + S);
  int16_t* d_fc = d_par + S;  // first child
  int16_t* d_lc = d_fc + S;   // last child
  int16_t* d_ps = d_lc + S;   // previous sibling
  int16_t* d_dep = d_ps + S;
  int16_t* pre = d_dep + S;   // pre-order position -> node
  int16_t* n2p = pre + S;     // node -> pre-order position
  int16_t* stk = n2p + S;

  const int Go = Gmax - Gs;
  Group* gc = reinterpret_cast<Group*>(gover + (size_t)b * gover_bytes);  // cold overflow
  uint32_t* gkh = reinterpret_cast<uint32_t*>(gc + (Go > 0 ? Go : 0));     // live-list overflow
  uint32_t* gkl = gkh + (Go > 0 ? Go : 0);
  uint32_t* gkm = gkl + (Go > 0 ? Go : 0);

  Arena ar{sslab, 0, kChildSmem, slabs + (size_t)b * slab_cap, 0, slab_cap, pool, cursor, pool_cap, err};
  Frontier fr{skh, skl, skm, gkh, gkl, gkm, sc, gc, 0, 0};
  if (lane == 0) {
    d_tok[0] = root_tok[b];
    d_par[0] = -1;
    d_fc[0] = d_lc[0] = d_ps[0] = -1;
    d_dep[0] = 0;
  }
  __syncwarp();
  int size = 1;
  const SrcDesc* sds = desc + (size_t)b * (c.P + 1);

  // seeds: datastore (rank 0), then input trees p = n_trees..1 (rank P-p+1)
  if (S > 1) {
    for (int rk = 0; rk <= c.P; ++rk) {
      const SrcDesc sd = sds[rk];
      if (sd.n <= 0) continue;
      uint32_t rc = 0;
      for (int i = lane; i < sd.n; i += 32) rc += (int)el_m(sd.meta[i]) >= sd.thr ? 1u : 0u;
      rc = __reduce_add_sync(SSSD_FULL, rc);
      if (rc == 0) continue;
      expand(sd, rk, 1, 0, sd.n, true, 0.0, rc, 0, c.disc[rk * c.disc_stride + 1], fr, ar);
    }
  }

  const long long t_seeded = clock64();
  uint32_t pops = 0, max_live = fr.A;
  while (size < S) {
    ++pops;
    max_live = max(max_live, (uint32_t)fr.A);
    // pop: minimum over group heads of (~prio, depth|rank|sequence); exhausted
    // groups carry meta = kExhausted and lose every comparison
    uint32_t bh = 0xffffffffu, bl = 0xffffffffu, bm = kExhausted;
    int bp = 0;
    const int A1 = min(fr.A, kGroupSmem);
    for (int q = lane; q < A1; q += 32) {
      const uint32_t h = skh[q], l = skl[q], m = skm[q];
      if (key_less(h, l, m, bh, bl, bm)) {
        bh = h;
        bl = l;
        bm = m;
        bp = q;
      }
    }
    for (int q = kGroupSmem + lane; q < fr.A; q += 32) {
      const int o = q - kGroupSmem;
      const uint32_t h = gkh[o], l = gkl[o], m = gkm[o];
      if (key_less(h, l, m, bh, bl, bm)) {
        bh = h;
        bl = l;
        bm = m;
        bp = q;
      }
    }
    const int win = warp_argmin3(bm != kExhausted, bh, bl, bm);
    if (win < 0) break;
    const uint32_t meta = __shfl_sync(SSSD_FULL, bm, win);
    const uint32_t pkh = __shfl_sync(SSSD_FULL, bh, win), pkl = __shfl_sync(SSSD_FULL, bl, win);
    const int pos = __shfl_sync(SSSD_FULL, bp, win);  // live-list slot of the popped group
    const int gi = (int)(meta & 0x3fffffu);
    Group* gp = fr.cold(gi);
    const Group g = *gp;
    const uint32_t ghead = g.head & 0xffffffu, gnch = g.nch & 0x7fffffffu;
    const Child h = g.ch[ghead];
    const uint32_t D = g_depth(meta), rk = g_rank(meta);
    const double dsc = c.disc[rk * c.disc_stride + D];

    // draft insert: an existing (parent, token) keeps the first node (ref fusion.py:185-198)
    const int par = (int)(g.head >> 24);
    int nid = -1;
    if (d_fc[par] >= 0) {
      for (int i0 = 1; i0 < size; i0 += 32) {
        const int i = i0 + lane;
        const uint32_t hb = __ballot_sync(SSSD_FULL, i < size && d_par[i] == par && d_tok[i] == h.token);
        if (hb) {
          nid = i0 + __ffs(hb) - 1;
          break;
        }
      }
    }
    if (nid < 0) {
      nid = size++;
      if (lane == 0) {
        d_tok[nid] = h.token;
        d_par[nid] = (int16_t)par;
        d_fc[nid] = d_lc[nid] = -1;
        d_dep[nid] = (int16_t)(d_dep[par] + 1);
        d_ps[nid] = d_lc[par];
        if (d_lc[par] < 0) d_fc[par] = (int16_t)nid;
        d_lc[par] = (int16_t)nid;
      }
    }

    // advance the popped group's head
    {
      uint32_t nh = gnch, kh = 0xffffffffu, kl = 0xffffffffu;
      if (g.nch >> 31) {
        nh = ghead + 1;
        if (nh < gnch) prio_key(__dmul_rn(g.ch[nh].pp, dsc), kh, kl);
      } else {
        uint32_t bh2 = 0xffffffffu, bl2 = 0xffffffffu, bf2 = 0xffffffffu, bi2 = 0;
        bool bv2 = false;
        for (uint32_t k = lane; k < gnch; k += 32) {
          const Child ck = g.ch[k];
          uint32_t hh, ll;
          prio_key(__dmul_rn(ck.pp, dsc), hh, ll);
          if (key_less(pkh, pkl, h.first, hh, ll, ck.first) &&
              (!bv2 || key_less(hh, ll, ck.first, bh2, bl2, bf2))) {
            bh2 = hh;
            bl2 = ll;
            bf2 = ck.first;
            bi2 = k;
            bv2 = true;
          }
        }
        const int w2 = warp_argmin3(bv2, bh2, bl2, bf2);
        if (w2 >= 0) {
          nh = __shfl_sync(SSSD_FULL, bi2, w2);
          kh = __shfl_sync(SSSD_FULL, bh2, w2);
          kl = __shfl_sync(SSSD_FULL, bl2, w2);
        }
      }
      if (lane == 0) {
        gp->head = (g.head & 0xff000000u) | nh;
        if (nh < gnch) {
          fr.put(pos, kh, kl, meta);
        } else {  // exhausted: move the last live group into this slot
          uint32_t h2, l2, m2;
          fr.get(fr.A - 1, h2, l2, m2);
          fr.put(pos, h2, l2, m2);
        }
      }
      if (nh >= gnch) --fr.A;
    }
    __syncwarp();
    // push the popped source node's children (ref fusion.py:258-259)
    // (a node at its source's column depth has no children: skip the scan)
    if (D + 1 < (uint32_t)c.disc_stride && (int)D < sds[rk].depth)
      expand(sds[rk], rk, D + 1, h.a, h.b, false, h.pp, h.count, (uint32_t)nid,
             c.disc[rk * c.disc_stride + D + 1], fr, ar);
  }

  const long long t_popped = clock64();
  // DFS pre-order flatten, children in insertion order (ref draft.py:67-86),
  // level-parallel: subtree sizes bottom-up, then pre-order positions top-down
  // (a child's subtree ends where its next sibling's starts); each lane
  // owns the parents of one level and walks their child lists
  int16_t* sub = stk;  // subtree sizes
  int maxd = 0;
  for (int v = lane; v < size; v += 32) {
    sub[v] = 1;
    maxd = max(maxd, (int)d_dep[v]);
  }
  maxd = __reduce_max_sync(SSSD_FULL, maxd);
  __syncwarp();
  for (int dd = maxd - 1; dd >= 0; --dd) {
    for (int v = lane; v < size; v += 32) {
      if (d_dep[v] != dd) continue;
      int t = 1;
      for (int ch = d_lc[v]; ch >= 0; ch = d_ps[ch]) t += sub[ch];
      sub[v] = (int16_t)t;
    }
    __syncwarp();
  }
  if (lane == 0) n2p[0] = 0;
  __syncwarp();
  for (int dd = 0; dd < maxd; ++dd) {
    for (int v = lane; v < size; v += 32) {
      if (d_dep[v] != dd) continue;
      int end = n2p[v] + sub[v];  // children fill the subtree right to left
      for (int ch = d_lc[v]; ch >= 0; ch = d_ps[ch]) {
        end -= sub[ch];
        n2p[ch] = (int16_t)end;
      }
    }
    __syncwarp();
  }
  for (int v = lane; v < size; v += 32) pre[n2p[v]] = (int16_t)v;
  __syncwarp();
  uint32_t* o_tok = out.tokens + (size_t)b * S;
  int32_t* o_par = out.parents + (size_t)b * S;
  int32_t* o_dep = out.depths + (size_t)b * S;
  uint64_t* o_mask = out.mask + (size_t)b * S * W;
  for (int k = lane; k < S; k += 32) {
    if (k < size) {
      const int nid = pre[k];
      o_tok[k] = d_tok[nid];
      o_par[k] = nid == 0 ? -1 : (int32_t)n2p[d_par[nid]];
      o_dep[k] = d_dep[nid];
      // (the heap-order cross-check kernel keeps no per-node keys: priority
      // NaN and source -2 = unknown; position ids are exact)
      if (out.priority || out.source || out.pos)
        write_node_extra(out, c, b, k, nid == 0 ? __longlong_as_double(0x7ff0000000000000ll)
                                                : __longlong_as_double(0x7ff8000000000000ll),
                         nid == 0 ? -1 : -2, d_dep[nid]);
      uint64_t mw[SSSD_MAX_DRAFT / 64] = {0, 0, 0, 0};
      for (int x = nid; x >= 0; x = d_par[x]) {
        const int pk = n2p[x];
        mw[pk >> 6] |= 1ull << (pk & 63);
      }
      for (int w = 0; w < W; ++w) o_mask[(size_t)k * W + w] = mw[w];
    } else {
      o_tok[k] = 0;
      o_par[k] = -1;
      o_dep[k] = -1;
      for (int w = 0; w < W; ++w) o_mask[(size_t)k * W + w] = 0;
      if (out.priority || out.source || out.pos) write_node_extra(out, c, b, k, 0.0, -1, -1);
    }
  }
  if (lane == 0) {
    out.size[b] = size;
    if (cycles) {  // per-request profile (optional): see sssd_set_cycle_probe
      long long* st = cycles + (size_t)b * 8;
      const long long t_end = clock64();
      st[0] = t_end - t_start;
      st[1] = t_seeded - t_start;
      st[2] = t_popped - t_seeded;
      st[3] = t_end - t_popped;
      st[4] = pops;
      st[5] = ar.scanned;
      st[6] = max_live;
      st[7] = ar.spill;
    }
  }
}

// Longest-processing-time-first launch order for the fusion kernel: requests
// are bucketed by log2 of their element count (datastore elements + input
// occurrences x trees, a proxy for expansion work; propose_setup_kernel fills
// bucket[] and the 64-bin histogram) and emitted in descending bucket order,
// so long requests start in the first wave instead of forming the tail.
// Order within a bucket is arbitrary: requests are independent and every
// output is indexed by request.
__global__ void lpt_scatter_kernel(const uint8_t* bucket, const int32_t* hist, int32_t* fill, int b0, int b1,
                                   int32_t* order) {
  // requests [b0, b1) -> order[b0 ..] by bucket; positions inside a bucket are
  // reserved per block (one global atomic per bucket and block)
  __shared__ int start[64], cnt[64], base[64];
  if (threadIdx.x < 64) {
    int acc = 0;
    for (int i = 0; i < (int)threadIdx.x; ++i) acc += hist[i];
    start[threadIdx.x] = acc;
    cnt[threadIdx.x] = 0;
  }
  __syncthreads();
  const int b = b0 + blockIdx.x * blockDim.x + threadIdx.x;
  const int k = b < b1 ? bucket[b] : 0;
  const int local = b < b1 ? atomicAdd(&cnt[k], 1) : 0;
  __syncthreads();
  if (threadIdx.x < 64 && cnt[threadIdx.x]) base[threadIdx.x] = atomicAdd(&fill[threadIdx.x], cnt[threadIdx.x]);
  __syncthreads();
  if (b < b1) order[b0 + start[k] + base[k] + local] = b;
}

}  // namespace sssd
