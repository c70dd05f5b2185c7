// K5, all-nodes form: fusion + DFS flatten for SSSD drafts (sm_100a).
//
// Same output as the level-synchronous kernel (fusion_ls.cu) and the
// reference merge (ref fusion.py:209-261) + flatten (draft.py:67-86), bit for
// bit; tests/ane_elements.py states this exact algorithm over the kernel's
// element arrays and checks it against the oracle's heap merge.
//
// The reference pops source-trie nodes in the order G = (-priority, depth,
// rank, ticket); within one (depth, rank) class tickets follow
// ord(n) = (-priority(n), ord(parent(n)), first appearance(n)), and the draft
// is the first dec_len-1 distinct token paths in G order.  Instead of walking
// the tries level by level, one warp per request:
//
//  1. enumerates EVERY live node of every merge rank straight from the sorted
//     element arrays: element i starts a depth-d node iff len_i >= d and
//     lcp(i-1, i) < d; the node's run ends at the next element with lcp < d,
//     its count is a prefix-sum difference of the rank's weights, its parent
//     the depth-(d-1) node containing i (boundary bitmasks + popc), its path
//     probability pp(parent) * (count / count(parent)) (__ddiv_rn/__dmul_rn,
//     the reference's order), priority pp * discount; depth by depth, so a
//     parent is always computed first;
//  2. radix-selects a threshold T on k0 = ~bits(priority) holding at least C
//     nodes (C = dec_len-1, doubled if needed) -- every node that precedes the
//     last kept path in G has k0 <= its k0 <= T, so those candidates decide the
//     draft exactly;
//  3. sorts the candidates by (k0, depth, rank) (bitonic), orders ties by the
//     ord chain, dedupes paths (hash of the path, verified token by token),
//     and keeps the first dec_len-1 distinct paths;
//  4. flattens them as the level-synchronous kernel does.
//
// Requests whose node or element counts exceed the shared-memory tables (or
// whose candidates tie beyond them) are listed for the level-synchronous
// kernel, launched right after on the same stream over that list.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "propose.cuh"

namespace sssd {

namespace {

constexpr int kN = kAneNodes;   // live nodes per request
constexpr int kE = kAneElems;   // elements per merge rank
constexpr int kC = kAneCands;   // candidates
constexpr int kEW = kE / 32;    // bitmask words over elements
constexpr int kH = 2 * kC;      // path hash slots
constexpr uint32_t kRootPar = 0xffffu;
constexpr uint32_t kNone = 0xffffffffu;
constexpr int kTokStage = 8192;  // staged tokens (n * depth) per element array

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(a), "l"(src) : "memory");
}

struct AneSm {
  // live nodes (rank by rank, depth by depth)
  uint64_t k0[kN];     // ~bits(priority)
  double pp[kN];       // path probability
  uint32_t cnt[kN];
  uint32_t info[kN];   // parent (16) | depth << 16 | rank << 24
  uint32_t first[kN];  // first appearance: min position of the run's counted elements
  uint32_t tok[kN];    // token at the node's depth
  uint16_t cpos[kN];   // sorted candidate position
  // element scratch of the array being enumerated
  uint32_t W[kE + 1];  // prefix sums of the rank's weights
  uint32_t M[kE];      // staged meta words
  uint32_t O[kE];      // staged first-appearance positions
  uint32_t T[kTokStage];  // staged token columns (T[d * n + i]) when they fit
  uint32_t F[kE];      // run minimum of O over counted elements (run starts)
  uint16_t R[kE];      // run end (run starts)
  uint8_t lcp[kE];
  uint8_t len[kE];
  uint32_t bmask[kEW];   // depth-d run starts
  uint32_t omask[kEW];   // live depth-(d-1) node starts of the rank
  uint32_t opref[kEW];   // exclusive popc prefix of omask words
  uint32_t omask2[kEW];  // live depth-d node starts (being built)
  // candidates
  uint16_t cidx[kC];
  uint16_t cpid[kC];   // sorted position of the candidate's canonical path
  uint64_t ck0[kC];
  uint32_t csec[kC];   // depth << 24 | rank << 16 | node
  uint64_t hkey[kH];
  uint32_t hval[kH];
  uint32_t hist[256];
  // draft
  int32_t fpar[SSSD_MAX_DRAFT];
  int32_t fdep[SSSD_MAX_DRAFT];
  int32_t fpos[SSSD_MAX_DRAFT];
  int32_t ffc[SSSD_MAX_DRAFT];
  int32_t fns[SSSD_MAX_DRAFT];
  uint16_t dnode[SSSD_MAX_DRAFT];
  uint64_t kk[SSSD_MAX_DRAFT];
  SrcDesc sd[SSSD_MAX_P + 1];
};

__device__ __forceinline__ uint32_t inf_par(uint32_t x) { return x & 0xffffu; }
__device__ __forceinline__ uint32_t inf_dep(uint32_t x) { return (x >> 16) & 0xffu; }
__device__ __forceinline__ uint32_t inf_rank(uint32_t x) { return x >> 24; }

__device__ __forceinline__ uint64_t mix64(uint64_t h, uint32_t t) {
  h ^= (uint64_t)t + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h *= 0xff51afd7ed558ccdull;
  return h ^ (h >> 33);
}

// last set bit at or before i (-1 if none)
__device__ __forceinline__ int prev_bit(const uint32_t* m, int i) {
  int w = i >> 5;
  uint32_t x = m[w] & ((i & 31) == 31 ? 0xffffffffu : ((2u << (i & 31)) - 1u));
  while (!x) {
    if (--w < 0) return -1;
    x = m[w];
  }
  return (w << 5) + 31 - __clz(x);
}

// ord(a) vs ord(b) for two nodes of equal (k0, depth, rank): the k0 of the
// ancestors from the nodes up, then the first appearances of the shallowest
// differing ancestors (the ticket order of ref fusion.py:231-259)
__device__ int cmp_ord(const AneSm& s, int a, int b) {
  int x = a, y = b;
  uint32_t fa = 0, fb = 0;
  while (x != y) {
    if (s.k0[x] != s.k0[y]) return s.k0[x] < s.k0[y] ? -1 : 1;
    fa = s.first[x];
    fb = s.first[y];
    const uint32_t px = inf_par(s.info[x]), py = inf_par(s.info[y]);
    if (px == kRootPar || py == kRootPar) break;
    x = (int)px;
    y = (int)py;
  }
  return fa < fb ? -1 : (fa > fb ? 1 : 0);
}

}  // namespace

int ane_smem_bytes() { return (int)((sizeof(AneSm) + 15) / 16 * 16); }

__global__ void __launch_bounds__(32, 1)
    draft_ane_kernel(const SrcDesc* desc, const uint32_t* root_tok, KCfg c, sssd_draft_out out, int32_t* fb) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  AneSm& s = *reinterpret_cast<AneSm*>(smem_raw);
  const int b = c.b0 + blockIdx.x;  // (the grid spans the launch's requests)
  const int lane = lane_id();
  const uint32_t lt = lanemask_lt();
  const int S = c.S, K = S - 1;
  const int NR = c.P + 1;
  for (int r = lane; r < NR; r += 32) s.sd[r] = desc[(size_t)b * NR + r];
  __syncwarp();
  bool bail = false;
  int N = 0;

  // ---- 1. every live node, rank by rank, depth by depth --------------------
  const uint32_t* arr = nullptr;  // element array whose lcp / len / O are loaded
  int arr_n = -1;
  for (int rk = 0; rk < NR && K > 0 && !bail; ++rk) {
    const SrcDesc& sd = s.sd[rk];
    const int n = sd.n;
    if (n <= 0) continue;
    if (n > kE) {
      bail = true;
      break;
    }
    const int nw = (n + 31) >> 5;
    // the element array (meta, first positions, token columns) staged in
    // shared memory with asynchronous copies; the input ranks share one array
    const int D = min(sd.depth, c.disc_stride - 1);
    const bool staged = n * D <= kTokStage;
    if (sd.meta != arr || n != arr_n) {
      __syncwarp();
      arr = sd.meta;
      arr_n = n;
      for (int i = lane; i < n; i += 32) {
        cp_async4(&s.M[i], sd.meta + i);
        cp_async4(&s.O[i], sd.orig + i);
      }
      if (staged)
        for (int d = 0; d < D; ++d)
          for (int i = lane; i < n; i += 32) cp_async4(&s.T[d * n + i], sd.tok + (int64_t)d * sd.stride + i);
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncwarp();
      const uint32_t* tk = staged ? s.T : sd.tok;
      const int64_t ts = staged ? (int64_t)n : sd.stride;
      for (int i = lane; i < n; i += 32) {
        const int li = (int)el_len(s.M[i]);
        s.len[i] = (uint8_t)li;
        int l = 0;
        if (i > 0) {
          const int lim = min((int)el_len(s.M[i - 1]), li);
          while (l < lim && tk[l * ts + i - 1] == tk[l * ts + i]) ++l;
        }
        s.lcp[i] = (uint8_t)l;
      }
    }
    const uint32_t* tk = staged ? s.T : sd.tok;
    const int64_t ts = staged ? (int64_t)n : sd.stride;
    // weights (m >= threshold) and their prefix sums
    uint32_t root = 0;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      uint32_t w = 0;
      if (i < n) {
        const uint32_t mt = s.M[i];
        w = (int)el_m(mt) >= sd.thr ? el_wt(mt) : 0u;
      }
      uint32_t inc = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(SSSD_FULL, inc, o);
        if (lane >= o) inc += y;
      }
      if (i < n) s.W[i + 1] = root + inc;
      root += __shfl_sync(SSSD_FULL, inc, 31);
    }
    if (lane == 0) s.W[0] = 0;
    __syncwarp();
    if (root == 0) continue;
    int maxlen = 0;
    for (int i = lane; i < n; i += 32) maxlen = max(maxlen, (int)s.len[i]);
    maxlen = min(__reduce_max_sync(SSSD_FULL, maxlen), D);
    __syncwarp();
    int base_prev = 0;
    const double* drow = c.disc + (size_t)rk * c.disc_stride;
    for (int d = 1; d <= maxlen; ++d) {
      // run starts at depth d; run ends and run minima of the counted
      // positions (segmented suffix scans, chunks last to first)
      uint32_t c_min = kNone, c_end = (uint32_t)n;
      for (int w = nw - 1; w >= 0; --w) {
        const int i = (w << 5) + lane;
        const bool st = i < n && (i == 0 || (int)s.lcp[i] < d);
        const uint32_t m = __ballot_sync(SSSD_FULL, st);
        const uint32_t above = m & ~((2u << lane) - 1u);
        const int ns = above ? __ffs(above) - 1 : 32;
        uint32_t v = (i < n && s.W[i + 1] != s.W[i]) ? s.O[i] : kNone;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_down_sync(SSSD_FULL, v, o);
          if (lane + o < ns) v = min(v, y);
        }
        uint32_t e = ns < 32 ? (uint32_t)((w << 5) + ns) : c_end;
        if (ns == 32) v = min(v, c_min);
        if (i < n) {
          s.F[i] = v;
          s.R[i] = (uint16_t)min(e, (uint32_t)n);
        }
        if (lane == 0) s.bmask[w] = m;
        const uint32_t v0 = __shfl_sync(SSSD_FULL, v, 0);
        c_min = (m & 1u) ? kNone : v0;
        c_end = (m & 1u) ? (uint32_t)(w << 5) : __shfl_sync(SSSD_FULL, e, 0);
      }
      __syncwarp();
      const double disc_d = drow[d];
      const int base = N;
      int nlive = 0;
      for (int w = 0; w < nw; ++w) {
        const int i = (w << 5) + lane;
        bool live = false;
        uint32_t cntv = 0;
        if (i < n && ((s.bmask[w] >> lane) & 1u) && (int)s.len[i] >= d) {
          cntv = s.W[s.R[i]] - s.W[i];
          live = cntv > 0;
        }
        const uint32_t bal = __ballot_sync(SSSD_FULL, live);
        if (lane == 0) s.omask2[w] = bal;
        if (live) {
          const int id = base + nlive + __popc(bal & lt);
          if (id < kN) {
            double pp;
            uint32_t par = kRootPar;
            if (d == 1) {
              pp = cntv == root ? 1.0 : __ddiv_rn((double)cntv, (double)root);  // ref fusion.py:244
            } else {
              const int j = prev_bit(s.omask, i);  // the depth-(d-1) node containing i
              par = (uint32_t)(base_prev + s.opref[j >> 5] + __popc(s.omask[j >> 5] & ((1u << (j & 31)) - 1u)));
              const uint32_t pc = s.cnt[par];
              pp = __dmul_rn(s.pp[par], cntv == pc ? 1.0 : __ddiv_rn((double)cntv, (double)pc));  // :259
            }
            const double pr = __dmul_rn(pp, disc_d);  // ref fusion.py:246
            s.k0[id] = ~(uint64_t)__double_as_longlong(pr);
            s.pp[id] = pp;
            s.cnt[id] = cntv;
            s.info[id] = par | (uint32_t)d << 16 | (uint32_t)rk << 24;
            s.first[id] = s.F[i];
            s.tok[id] = tk[(d - 1) * ts + i];
            s.cpos[id] = 0xffff;
          }
        }
        nlive += __popc(bal);
      }
      __syncwarp();
      if (base + nlive > kN) {
        bail = true;
        break;
      }
      if (nlive == 0) break;
      // the depth-d starts become the parents of depth d + 1
      if (lane == 0) {
        uint32_t acc = 0;
        for (int w = 0; w < nw; ++w) {
          const uint32_t m = s.omask2[w];
          s.omask[w] = m;
          s.opref[w] = acc;
          acc += __popc(m);
        }
      }
      __syncwarp();
      base_prev = base;
      N = base + nlive;
    }
  }
  bail = __any_sync(SSSD_FULL, bail);

  // ---- 2-3. candidates: threshold, sort, dedupe ------------------------------
  int ndist = 0;  // distinct paths among the candidates
  int Cn = 0;
  if (!bail && K > 0 && N > 0) {
    uint64_t lo = ~0ull, hi = 0;
    for (int i = lane; i < N; i += 32) {
      lo = min(lo, s.k0[i]);
      hi = max(hi, s.k0[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, (uint64_t)__shfl_xor_sync(SSSD_FULL, (unsigned long long)lo, o));
      hi = max(hi, (uint64_t)__shfl_xor_sync(SSSD_FULL, (unsigned long long)hi, o));
    }
    const int sh0 = lo == hi ? -8 : ((63 - __clzll((long long)(lo ^ hi))) & ~7);
    int C = min(K, N);
    while (true) {
      // radix select: T with #{k0 <= T} >= C, at most `lim` candidates where a
      // whole digit bucket fits (the bytes above sh0 are common to all nodes)
      const int lim = min(kC, max(64, 2 * C));
      uint64_t pmask = sh0 + 8 >= 64 ? 0ull : ~((1ull << (sh0 + 8)) - 1ull);
      uint64_t prefix = lo & pmask;
      int need = C, below = 0;
      uint64_t T = 0;
      bool found = false;
      if (sh0 < 0 || N <= lim) {  // every node
        T = hi;
        found = N <= kC;
      }
      for (int sh = sh0; sh >= 0 && !found; sh -= 8) {
        for (int q = lane; q < 256; q += 32) s.hist[q] = 0;
        __syncwarp();
        for (int i0 = 0; i0 < N; i0 += 32) {
          const int i = i0 + lane;
          const uint64_t kv = i < N ? s.k0[i] : 0ull;
          const bool inb = i < N && (kv & pmask) == prefix;
          const uint32_t dg = inb ? (uint32_t)(kv >> sh) & 255u : 256u + (uint32_t)lane;
          const uint32_t mm = __match_any_sync(SSSD_FULL, dg);
          if (inb && lane == __ffs(mm) - 1) atomicAdd(&s.hist[dg], (uint32_t)__popc(mm));
        }
        __syncwarp();
        uint32_t part = 0;
        for (int q = 0; q < 8; ++q) part += s.hist[lane * 8 + q];
        uint32_t inc = part;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(SSSD_FULL, inc, o);
          if (lane >= o) inc += y;
        }
        const uint32_t hit = __ballot_sync(SSSD_FULL, inc >= (uint32_t)need);
        const int L = __ffs(hit) - 1;
        uint32_t cum = __shfl_sync(SSSD_FULL, inc - part, L);
        int dig = L * 8;
        for (; dig < L * 8 + 7; ++dig) {
          const uint32_t h = s.hist[dig];
          if (cum + h >= (uint32_t)need) break;
          cum += h;
        }
        const uint32_t hcnt = s.hist[dig];
        __syncwarp();
        prefix |= (uint64_t)dig << sh;
        pmask |= 255ull << sh;
        if (below + (int)cum + (int)hcnt <= lim || sh == 0) {  // the whole digit bucket
          T = prefix | (sh ? ((1ull << sh) - 1ull) : 0ull);
          found = below + (int)cum + (int)hcnt <= kC;
          break;
        }
        below += (int)cum;
        need -= (int)cum;
      }
      if (!found) {  // more than kC nodes tie on the C-th key
        bail = true;
        break;
      }
      // candidates (node order), then sorted
      Cn = 0;
      for (int i0 = 0; i0 < N; i0 += 32) {
        const int i = i0 + lane;
        const bool cand = i < N && s.k0[i] <= T;
        const uint32_t bal = __ballot_sync(SSSD_FULL, cand);
        if (cand) {
          const int q = Cn + __popc(bal & lt);
          s.ck0[q] = s.k0[i];
          s.csec[q] = (inf_dep(s.info[i]) << 24) | (inf_rank(s.info[i]) << 16) | (uint32_t)i;
        }
        Cn += __popc(bal);
      }
      int n2 = 32;
      while (n2 < Cn) n2 <<= 1;
      for (int q = Cn + lane; q < n2; q += 32) {
        s.ck0[q] = ~0ull;
        s.csec[q] = 0xffffffffu;
      }
      __syncwarp();
      // bitonic sort by (k0, depth, rank, node)
      for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int t = lane; t < (n2 >> 1); t += 32) {
            const int q = ((t & ~(j - 1)) << 1) | (t & (j - 1));  // lower index of the pair
            const int p = q | j;
            const uint64_t a0 = s.ck0[q], b0 = s.ck0[p];
            const uint32_t a1 = s.csec[q], b1 = s.csec[p];
            const bool gt = a0 > b0 || (a0 == b0 && a1 > b1);
            if (gt == ((q & k) == 0)) {
              s.ck0[q] = b0;
              s.ck0[p] = a0;
              s.csec[q] = b1;
              s.csec[p] = a1;
            }
          }
          __syncwarp();
        }
      }
      // equal (k0, depth, rank) runs: order by the ord chain (insertion sort by
      // one lane per run; such ties are rare and short)
      for (int q0 = 0; q0 < Cn; q0 += 32) {
        const int q = q0 + lane;
        bool head = false;
        if (q < Cn && q + 1 < Cn)
          head = (q == 0 || s.ck0[q - 1] != s.ck0[q] || (s.csec[q - 1] >> 16) != (s.csec[q] >> 16)) &&
                 s.ck0[q + 1] == s.ck0[q] && (s.csec[q + 1] >> 16) == (s.csec[q] >> 16);
        if (head) {
          int e = q + 1;
          while (e < Cn && s.ck0[e] == s.ck0[q] && (s.csec[e] >> 16) == (s.csec[q] >> 16)) ++e;
          for (int x = q + 1; x < e; ++x) {
            const uint32_t v = s.csec[x];
            int y = x - 1;
            while (y >= q && cmp_ord(s, (int)(s.csec[y] & 0xffffu), (int)(v & 0xffffu)) > 0) {
              s.csec[y + 1] = s.csec[y];
              --y;
            }
            s.csec[y + 1] = v;
          }
        }
      }
      for (int h = lane; h < kH; h += 32) {
        s.hkey[h] = ~0ull;
        s.hval[h] = kNone;
      }
      __syncwarp();
      for (int q = lane; q < Cn; q += 32) {
        const int i = (int)(s.csec[q] & 0xffffu);
        s.cidx[q] = (uint16_t)i;
        s.cpos[i] = (uint16_t)q;
      }
      // dedupe: canonical = the first candidate (sorted position) with the same
      // token path; paths are hashed, equal hashes verified token by token
      for (int q = lane; q < Cn; q += 32) {
        int x = s.cidx[q];
        uint64_t hsh = 0x243f6a8885a308d3ull ^ (uint64_t)inf_dep(s.info[x]);
        while (true) {
          hsh = mix64(hsh, s.tok[x]);
          const uint32_t px = inf_par(s.info[x]);
          if (px == kRootPar) break;
          x = (int)px;
        }
        if (hsh == ~0ull) hsh = 0;
        int slot = (int)(hsh & (uint64_t)(kH - 1));
        while (true) {
          const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(&s.hkey[slot]), ~0ull,
                                                    (unsigned long long)hsh);
          if (prev == ~0ull || prev == hsh) break;
          slot = (slot + 1) & (kH - 1);
        }
        atomicMin(&s.hval[slot], (uint32_t)q);
        s.ck0[q] = (uint64_t)slot;  // (sort keys no longer needed)
      }
      __syncwarp();
      bool collide = false;
      int nd = 0;
      for (int q0 = 0; q0 < Cn; q0 += 32) {
        const int q = q0 + lane;
        bool dist = false;
        if (q < Cn) {
          const int canon = (int)s.hval[s.ck0[q]];
          s.cpid[q] = (uint16_t)canon;
          dist = canon == q;
          if (!dist) {  // equal paths? (a 64-bit hash collision would not be)
            int x = s.cidx[q], y = s.cidx[canon];
            while (true) {
              if (s.tok[x] != s.tok[y] || inf_dep(s.info[x]) != inf_dep(s.info[y])) {
                collide = true;
                break;
              }
              const uint32_t px = inf_par(s.info[x]), py = inf_par(s.info[y]);
              if (px == kRootPar || py == kRootPar) break;
              x = (int)px;
              y = (int)py;
            }
          }
        }
        nd += __popc(__ballot_sync(SSSD_FULL, dist));
      }
      if (__any_sync(SSSD_FULL, collide)) {
        bail = true;
        break;
      }
      ndist = nd;
      if (ndist >= K || Cn == N) break;
      C = min(N, 2 * C);
      __syncwarp();
    }
  }
  bail = __any_sync(SSSD_FULL, bail);
  if (bail) {  // hand the request to the level-synchronous kernel
    if (lane == 0) fb[1 + atomicAdd(fb, 1)] = b;
    return;
  }

  // ---- 4. draft = root + the first K distinct paths (G order), flattened ----
  const int size = 1 + min(ndist, K);
  {
    int run = 0;
    for (int q0 = 0; q0 < Cn; q0 += 32) {
      const int q = q0 + lane;
      const bool dist = q < Cn && s.cpid[q] == q;
      const uint32_t bal = __ballot_sync(SSSD_FULL, dist);
      if (dist) {
        const int v = 1 + run + __popc(bal & lt);
        if (v < size) s.dnode[v] = s.cidx[q];
        s.hval[q] = (uint32_t)v;  // (hash values reused: candidate position -> draft index)
      }
      run += __popc(bal);
    }
  }
  __syncwarp();
  int maxd = 0;
  for (int v = lane; v < size; v += 32) {
    int pr = -1, dv = 0;
    if (v > 0) {
      const int i = s.dnode[v];
      const uint32_t par = inf_par(s.info[i]);
      pr = par == kRootPar ? 0 : (int)s.hval[s.cpid[s.cpos[par]]];
      dv = (int)inf_dep(s.info[i]);
    }
    s.fpar[v] = pr;
    s.fdep[v] = dv;
    maxd = max(maxd, dv);
  }
  __syncwarp();
  maxd = __reduce_max_sync(SSSD_FULL, maxd);
  uint32_t* o_tok = out.tokens + (size_t)b * S;
  int32_t* o_par = out.parents + (size_t)b * S;
  int32_t* o_dep = out.depths + (size_t)b * S;
  const bool extra = out.priority || out.source || out.pos;
  auto node_out = [&](int v, int k) {
    o_tok[k] = v == 0 ? root_tok[b] : s.tok[s.dnode[v]];
    o_par[k] = v == 0 ? -1 : s.fpos[s.fpar[v]];
    o_dep[k] = s.fdep[v];
    if (extra) {
      if (v == 0) {
        write_node_extra(out, c, b, k, __longlong_as_double(0x7ff0000000000000ll), -1, 0);
      } else {
        const int i = s.dnode[v];
        write_node_extra(out, c, b, k, __longlong_as_double((long long)~s.k0[i]), (int32_t)inf_rank(s.info[i]),
                         s.fdep[v]);
      }
    }
  };
  if (maxd <= 8 && size <= 127) {
    // pre-order position = rank of the node's ancestor-index path (7 bits per
    // depth; index order = sibling insertion order; a prefix sorts first)
    for (int v = lane; v < size; v += 32) {
      uint64_t key = 0;
      for (int u = v; u > 0; u = s.fpar[u]) key |= (uint64_t)u << (7 * (8 - s.fdep[u]));
      s.kk[v] = key;
    }
    __syncwarp();
    for (int v = lane; v < size; v += 32) {
      const uint64_t kv = s.kk[v];
      int r = 0;
      for (int q = 0; q < size; ++q) r += s.kk[q] < kv ? 1 : 0;
      s.fpos[v] = r;
    }
    __syncwarp();
    for (int v = lane; v < size; v += 32) node_out(v, s.fpos[v]);
  } else {
    // next sibling = the next index with the same parent (match_any inside a
    // chunk, a first-index-per-parent table across chunks), then a DFS walk
    for (int v = lane; v < size; v += 32) s.fpos[v] = -1;
    __syncwarp();
    for (int c0 = ((size - 1) >> 5) << 5; c0 >= 0; c0 -= 32) {
      const int v = c0 + lane;
      const bool ok = v >= 1 && v < size;
      const int p = ok ? s.fpar[v] : -2 - lane;
      const uint32_t mm = __match_any_sync(SSSD_FULL, p);
      const uint32_t above = mm & ~((2u << lane) - 1u);
      int ns = -1;
      if (ok) ns = above ? c0 + __ffs(above) - 1 : s.fpos[p];
      __syncwarp();
      if (ok) {
        s.fns[v] = ns;
        if (lane == __ffs(mm) - 1) s.fpos[p] = v;
      }
      __syncwarp();
    }
    for (int v = lane; v < size; v += 32) s.ffc[v] = s.fpos[v];
    __syncwarp();
    if (lane == 0) {
      int v = 0, k = 0;
      while (true) {
        s.fpos[v] = k;
        node_out(v, k);
        ++k;
        int nx = s.ffc[v];
        if (nx < 0) {
          int u = v;
          while (u > 0 && s.fns[u] < 0) u = s.fpar[u];
          if (u <= 0) break;
          nx = s.fns[u];
        }
        v = nx;
      }
    }
  }
  __syncwarp();
  const int Wd = (S + 63) >> 6;
  uint64_t* o_mask = out.mask + (size_t)b * S * Wd;
  for (int v = lane; v < size; v += 32) {  // mask row = ancestors-or-self (ref draft.py:80-84)
    const int k = s.fpos[v];
    for (int w = 0; w < Wd; ++w) {
      uint64_t m = 0;
      for (int x = v; x >= 0; x = s.fpar[x]) {
        const int pk = s.fpos[x];
        if ((pk >> 6) == w) m |= 1ull << (pk & 63);
      }
      o_mask[(size_t)k * Wd + w] = m;
    }
  }
  for (int k = size + lane; k < S; k += 32) {
    o_tok[k] = 0;
    o_par[k] = -1;
    o_dep[k] = -1;
    for (int w = 0; w < Wd; ++w) o_mask[(size_t)k * Wd + w] = 0;
    if (extra) write_node_extra(out, c, b, k, 0.0, -1, -1);
  }
  if (lane == 0) out.size[b] = size;
}

}  // namespace sssd
