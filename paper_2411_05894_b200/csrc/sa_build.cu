// K1: suffix array by prefix doubling with group refinement, on our own
// LSD radix sort (replaces ref datastore.py:81-109 build_suffix_array).
//
// The reference re-sorts every position by (rank[i], rank[i+k]) each round
// until all ranks are distinct (datastore.py:93-109).  The SA is unique
// (SURVEY A.1), so any correct order gives the same array; this build keeps
// the same doubling rounds but sorts only the ACTIVE positions -- those whose
// current group (equal k-prefix) is not yet a singleton.  Groups are
// contiguous slot ranges of the SA order, so sorting the active positions by
// (old group head, rank[i+k] + 1) and writing them back into the active slots
// in order refines every group in place.  On the phrase corpus the active
// fraction per round is 1.0, 0.90, 0.75, 0.52, 0.23, 0.04, 0.001 (10M tokens),
// 2.4 n sorted elements after the first round instead of 7 n.
//
// rank[p] = slot index of the head of p's group (ranks are group-start
// indices, as in the reference's cumsum re-rank up to a monotone relabeling).
//
// Radix sort: LSD, 8-bit digits, u64 keys (only the bits the round needs),
// u32 values; per pass an upsweep (per-tile digit histogram, warp-aggregated
// shared-memory atomics), a per-digit scan over tiles, and a stable scatter
// (each 4096-element tile in 16 striped rounds of 256: warp match_any gives
// the rank among equal digits in the warp, a per-round cross-warp prefix in
// shared memory the rank in the tile).  Scans and stream compaction: a
// three-phase block scan (tile reduce, scan of tile totals, tile scan).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace sssd {
int fail(int code, const char* fmt, ...);
int cuda_check(cudaError_t e, const char* what);

namespace {

constexpr int kT = 256;              // threads per tile
constexpr int kItems = 16;           // items per thread
constexpr int kTile = kT * kItems;   // 4096 elements per tile
constexpr int kDigits = 256;

inline unsigned tiles_of(uint64_t n) { return (unsigned)((n + kTile - 1) / kTile); }

// ---- radix sort ---------------------------------------------------------------

__global__ void __launch_bounds__(kT) rs_upsweep(const uint64_t* keys, uint64_t n, int shift, uint32_t* hist,
                                                unsigned nb, uint32_t* totals) {
  __shared__ uint32_t h[kDigits];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  uint32_t dig[kItems];
#pragma unroll
  for (int r = 0; r < kItems; ++r) {  // all loads first (independent)
    const uint64_t i = base + (uint64_t)r * kT + threadIdx.x;
    dig[r] = i < n ? (uint32_t)(keys[i] >> shift) & 255u : 256u + (threadIdx.x & 31);
  }
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const uint64_t i = base + (uint64_t)r * kT + threadIdx.x;
    const bool ok = i < n;
    const uint32_t d = dig[r];
    const uint32_t peers = __match_any_sync(SSSD_FULL, d);
    if (ok && (threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&h[d], (uint32_t)__popc(peers));
  }
  __syncthreads();
  hist[(size_t)threadIdx.x * nb + blockIdx.x] = h[threadIdx.x];  // digit-major
  if (h[threadIdx.x]) atomicAdd(totals + threadIdx.x, h[threadIdx.x]);
}


// One CTA per digit: exclusive scan of hist[d][0..nb) plus the digit's base
// (the counts of all smaller digits).
__global__ void __launch_bounds__(kT) rs_scan(const uint32_t* hist, unsigned nb, const uint32_t* totals,
                                             uint32_t* offs) {
  __shared__ uint32_t part[kT];
  __shared__ uint32_t s_base;
  const int d = blockIdx.x;
  // digit base: the totals of the smaller digits
  part[threadIdx.x] = (int)threadIdx.x < d ? totals[threadIdx.x] : 0u;
  __syncthreads();
  for (int o = kT / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) part[threadIdx.x] += part[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) s_base = part[0];
  __syncthreads();
  uint32_t run = s_base;
  const uint32_t* row = hist + (size_t)d * nb;
  uint32_t* orow = offs + (size_t)d * nb;
  for (unsigned b0 = 0; b0 < nb; b0 += kT) {
    const unsigned b = b0 + threadIdx.x;
    const uint32_t v = b < nb ? row[b] : 0u;
    // block exclusive scan of v
    uint32_t x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(SSSD_FULL, x, o);
      if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) part[w] = x;
    __syncthreads();
    uint32_t wsum = 0, tot = 0;
    for (int k = 0; k < kT / 32; ++k) {
      wsum += k < w ? part[k] : 0u;
      tot += part[k];
    }
    if (b < nb) orow[b] = run + wsum + x - v;
    run += tot;
  }
}

// Stable scatter of one tile: every thread loads its 16 (key, value) pairs
// up front (one burst of independent loads), then 16 striped rounds of 256
// assign output slots: warp match_any gives the rank among equal digits in
// the warp, a per-round cross-warp prefix per digit in shared memory the rank
// in the tile.  offs: digit-major [256][nb] global start of (digit, tile).
__global__ void __launch_bounds__(kT) rs_scatter(const uint64_t* kin, const uint32_t* vin, uint64_t n, int shift,
                                                const uint32_t* offs, unsigned nb, uint64_t* kout, uint32_t* vout) {
  __shared__ uint32_t base[kDigits];          // running output offset per digit in this tile
  __shared__ uint32_t wcnt[kT / 32][kDigits];  // (round << 8) | count of the digit in each warp this round
  __shared__ uint32_t woff[kT / 32][kDigits];  // exclusive offset of (warp, digit) this round
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  base[threadIdx.x] = offs[(size_t)threadIdx.x * nb + blockIdx.x];
  for (int k = 0; k < kT / 32; ++k) wcnt[k][threadIdx.x] = 0xffffff00u;  // no round has this stamp
  const uint64_t t0 = (uint64_t)blockIdx.x * kTile;
  uint64_t key[kItems];
  uint32_t val[kItems];
#pragma unroll
  for (int r = 0; r < kItems; ++r) {  // striped: element r*kT + t, so (round, thread) order = input order
    const uint64_t i = t0 + (uint64_t)r * kT + threadIdx.x;
    key[r] = i < n ? kin[i] : 0;
    val[r] = i < n ? vin[i] : 0;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const bool ok = t0 + (uint64_t)r * kT + threadIdx.x < n;
    const uint32_t d = ok ? (uint32_t)(key[r] >> shift) & 255u : 256u + lane;
    const uint32_t peers = __match_any_sync(SSSD_FULL, d);
    const uint32_t lr = __popc(peers & lanemask_lt());
    if (ok && lane == __ffs(peers) - 1) wcnt[w][d] = ((uint32_t)r << 8) | (uint32_t)__popc(peers);
    __syncthreads();
    {  // thread t owns digit t: exclusive prefix over the warps, advance the base
      const uint32_t dg = threadIdx.x;
      uint32_t run = base[dg];
#pragma unroll
      for (int k = 0; k < kT / 32; ++k) {
        const uint32_t e = wcnt[k][dg];
        woff[k][dg] = run;
        run += (e >> 8) == (uint32_t)r ? (e & 255u) : 0u;
      }
      base[dg] = run;
    }
    __syncthreads();
    if (ok) {
      const uint32_t pos = woff[w][d] + lr;
      kout[pos] = key[r];
      vout[pos] = val[r];
    }
  }
}


// ---- scans --------------------------------------------------------------------

// per-tile reduce (op: 0 = sum of u32 flags, 1 = max of u32)
template <int OP>
__device__ __forceinline__ uint32_t op2(uint32_t a, uint32_t b) {
  return OP == 0 ? a + b : (a > b ? a : b);
}

template <int OP>
__global__ void __launch_bounds__(kT) scan_reduce(const uint32_t* in, uint64_t n, uint32_t* tile_tot) {
  __shared__ uint32_t part[kT / 32];
  const uint64_t t0 = (uint64_t)blockIdx.x * kTile;
  uint32_t acc = 0;
  for (int r = 0; r < kItems; ++r) {
    const uint64_t i = t0 + (uint64_t)threadIdx.x * kItems + r;
    if (i < n) acc = op2<OP>(acc, in[i]);
  }
  for (int o = 16; o > 0; o >>= 1) acc = op2<OP>(acc, __shfl_down_sync(SSSD_FULL, acc, o));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int k = 0; k < kT / 32; ++k) t = op2<OP>(t, part[k]);
    tile_tot[blockIdx.x] = t;
  }
}

// exclusive scan of the tile totals (one CTA, sequential chunks)
template <int OP>
__global__ void __launch_bounds__(1024) scan_tiles(uint32_t* tot, unsigned nb, uint32_t* grand) {
  __shared__ uint32_t part[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t run = 0;
  for (unsigned b0 = 0; b0 < nb; b0 += 1024) {
    const unsigned b = b0 + threadIdx.x;
    const uint32_t v = b < nb ? tot[b] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(SSSD_FULL, x, o);
      if (lane >= o) x = op2<OP>(x, y);
    }
    __syncthreads();
    if (lane == 31) part[w] = x;
    __syncthreads();
    uint32_t pre = 0, all = 0;
    for (int k = 0; k < 32; ++k) {
      if (k < w) pre = op2<OP>(pre, part[k]);
      all = op2<OP>(all, part[k]);
    }
    // exclusive value for b: run (+) pre (+) (inclusive x without v)
    uint32_t excl_in_warp = __shfl_up_sync(SSSD_FULL, x, 1);
    if (lane == 0) excl_in_warp = 0;
    if (b < nb) tot[b] = op2<OP>(run, op2<OP>(pre, excl_in_warp));
    run = op2<OP>(run, all);
  }
  if (threadIdx.x == 0 && grand) *grand = run;
}

// inclusive (INCL) or exclusive scan of in -> out with the tile's carry-in
template <int OP, bool INCL>
__global__ void __launch_bounds__(kT) scan_tiles_apply(const uint32_t* in, uint64_t n, const uint32_t* carry,
                                                       uint32_t* out) {
  __shared__ uint32_t part[kT / 32];
  const uint64_t t0 = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kItems;
  uint32_t v[kItems];
  uint32_t acc = 0;
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    v[r] = t0 + r < n ? in[t0 + r] : 0u;
    acc = op2<OP>(acc, v[r]);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = acc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(SSSD_FULL, x, o);
    if (lane >= o) x = op2<OP>(x, y);
  }
  if (lane == 31) part[w] = x;
  __syncthreads();
  uint32_t pre = carry[blockIdx.x];
  for (int k = 0; k < w; ++k) pre = op2<OP>(pre, part[k]);
  uint32_t ex = __shfl_up_sync(SSSD_FULL, x, 1);
  if (lane == 0) ex = 0;
  uint32_t run = op2<OP>(pre, ex);  // exclusive prefix of this thread's first item
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    if (t0 + r < n) {
      const uint32_t inc = op2<OP>(run, v[r]);
      out[t0 + r] = INCL ? inc : run;
      run = inc;
    }
  }
}

// ---- suffix-array rounds -------------------------------------------------------

__global__ void sa_first_keys(const uint32_t* tokens, uint64_t n, uint64_t* key, uint32_t* val) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  key[i] = tokens[i];
  val[i] = (uint32_t)i;
}

// round 1 with m-gram keys: key[i] = (t[i]+1, .., t[i+m-1]+1) packed tb bits
// each, 0 past the corpus end (a shorter suffix sorts first, as in the
// reference's rank[i+k] + 1 / 0 keys, datastore.py:94-95)
__global__ void sa_mgram_keys(const uint32_t* tokens, uint64_t n, int m, int tb, uint64_t* key, uint32_t* val) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t k = 0;
  for (int j = 0; j < m; ++j) k = (k << tb) | (i + j < n ? (uint64_t)tokens[i + j] + 1 : 0ull);
  key[i] = k;
  val[i] = (uint32_t)i;
}

// keys of the active elements (slot order): (group head slot, rank[pos + k] + 1
// or 0 past the end) -- one random gather per element (the head and the
// position travel with the active list)
__global__ void sa_round_keys(const uint32_t* apos, const uint32_t* agrp, uint64_t A, const uint32_t* rank,
                              uint64_t n, uint64_t k, int rb, uint64_t* key, uint32_t* val) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A) return;
  const uint32_t pos = apos[i];
  const uint64_t r2 = (uint64_t)pos + k < n ? (uint64_t)rank[pos + k] + 1 : 0;
  key[i] = ((uint64_t)agrp[i] << rb) | r2;
  val[i] = pos;
}

// heads of the sorted active list: head slot (or 0) for the max-scan; the
// sorted positions go back into their (ascending) slots; with a token table,
// the first slot of every token
__global__ void sa_round_heads(const uint64_t* key, const uint32_t* val, uint64_t A, const uint32_t* aslot,
                               uint32_t* sa, uint32_t* head, uint32_t* first_slot) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A) return;
  const uint32_t slot = aslot ? aslot[i] : (uint32_t)i;
  sa[slot] = val[i];
  const bool h = i == 0 || key[i] != key[i - 1];
  head[i] = h ? slot : 0u;
  if (h && first_slot) first_slot[key[i]] = slot;
}

// rank update from the max-scanned heads (written only where the group head
// moved: a position keeps its rank while its group does not split before
// it; round 1 has no previous heads, rb < 0) and the next active flags (a
// singleton group = a head followed by a head or the end)
__global__ void sa_round_rank(const uint64_t* key, const uint32_t* val, uint64_t A, const uint32_t* grp, int rb,
                              uint32_t* rank, uint32_t* flag) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A) return;
  const uint64_t ki = key[i];
  if (rank && (rb < 0 || (uint32_t)(ki >> rb) != grp[i])) rank[val[i]] = grp[i];
  const bool h = i == 0 || ki != key[i - 1];
  const bool hn = i + 1 == A || key[i + 1] != ki;
  flag[i] = (h && hn) ? 0u : 1u;
}

// round 1 with a token table: rank[p] = first slot of tok[p] (coalesced)
__global__ void sa_rank_from_table(const uint32_t* tokens, uint64_t n, const uint32_t* first_slot, uint32_t* rank) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) rank[p] = first_slot[tokens[p]];
}

// the next active list: slots, positions and group heads of the flagged elements
__global__ void sa_compact(const uint32_t* flag, const uint32_t* idx, uint64_t A, const uint32_t* aslot,
                           const uint32_t* val, const uint32_t* grp, uint32_t* aslot_out, uint32_t* apos_out,
                           uint32_t* agrp_out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A || !flag[i]) return;
  const uint32_t o = idx[i];
  aslot_out[o] = aslot ? aslot[i] : (uint32_t)i;
  apos_out[o] = val[i];
  agrp_out[o] = grp[i];
}

int bits_of(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return b;
}

constexpr uint64_t kTableMinN = 1ull << 20;   // a first-slot token table pays from here
constexpr uint64_t kTableTokens = 1ull << 24; // tokens below this use it (64 MB)

struct SaWs2 {
  uint64_t *k0, *k1;
  uint32_t *v0, *v1;
  uint32_t *rank, *aslot, *aslot2, *apos, *apos2, *agrp, *agrp2, *tmp, *tmp2;
  uint32_t *hist, *offs;
  uint32_t* tiles;
  uint32_t* grand;
  uint32_t* totals;
  uint32_t* table;
  size_t total;
};

size_t al2(size_t x) { return (x + 255) / 256 * 256; }

SaWs2 carve2(uint8_t* base, uint64_t n) {
  SaWs2 w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    uint8_t* p = base ? base + off : nullptr;
    off += al2(bytes);
    return p;
  };
  const size_t nb = tiles_of(n);
  w.k0 = reinterpret_cast<uint64_t*>(take(8 * n));
  w.k1 = reinterpret_cast<uint64_t*>(take(8 * n));
  w.v0 = reinterpret_cast<uint32_t*>(take(4 * n));
  w.v1 = reinterpret_cast<uint32_t*>(take(4 * n));
  w.rank = reinterpret_cast<uint32_t*>(take(4 * n));
  w.aslot = reinterpret_cast<uint32_t*>(take(4 * n));
  w.aslot2 = reinterpret_cast<uint32_t*>(take(4 * n));
  w.apos = reinterpret_cast<uint32_t*>(take(4 * n));
  w.apos2 = reinterpret_cast<uint32_t*>(take(4 * n));
  w.agrp = reinterpret_cast<uint32_t*>(take(4 * n));
  w.agrp2 = reinterpret_cast<uint32_t*>(take(4 * n));
  w.tmp = reinterpret_cast<uint32_t*>(take(4 * n));
  w.tmp2 = reinterpret_cast<uint32_t*>(take(4 * n));
  w.hist = reinterpret_cast<uint32_t*>(take(4 * nb * kDigits));
  w.offs = reinterpret_cast<uint32_t*>(take(4 * nb * kDigits));
  w.tiles = reinterpret_cast<uint32_t*>(take(4 * nb));
  w.grand = reinterpret_cast<uint32_t*>(take(16));
  w.totals = reinterpret_cast<uint32_t*>(take(4 * kDigits));
  w.table = n >= kTableMinN ? reinterpret_cast<uint32_t*>(take(4 * kTableTokens)) : nullptr;
  w.total = off;
  return w;
}

// stable LSD sort of (key, val)[0..A) on the low `bits` bits; result in (k0, v0)
void radix_sort(SaWs2& w, uint64_t A, int bits, cudaStream_t st) {
  const unsigned nb = tiles_of(A);
  uint64_t *ka = w.k0, *kb = w.k1;
  uint32_t *va = w.v0, *vb = w.v1;
  for (int sh = 0; sh < bits; sh += 8) {
    cudaMemsetAsync(w.totals, 0, 4 * kDigits, st);
    rs_upsweep<<<nb, kT, 0, st>>>(ka, A, sh, w.hist, nb, w.totals);
    rs_scan<<<kDigits, kT, 0, st>>>(w.hist, nb, w.totals, w.offs);
    rs_scatter<<<nb, kT, 0, st>>>(ka, va, A, sh, w.offs, nb, kb, vb);
    uint64_t* tk = ka;
    ka = kb;
    kb = tk;
    uint32_t* tv = va;
    va = vb;
    vb = tv;
  }
  if (ka != w.k0) {  // odd pass count: the result is in the second buffers
    cudaMemcpyAsync(w.k0, ka, 8 * A, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(w.v0, va, 4 * A, cudaMemcpyDeviceToDevice, st);
  }
}

// scan of u32 in[0..A) -> out (OP 0 sum / 1 max), grand total to w.grand
template <int OP, bool INCL>
void scan(SaWs2& w, const uint32_t* in, uint64_t A, uint32_t* out, cudaStream_t st) {
  const unsigned nb = tiles_of(A);
  scan_reduce<OP><<<nb, kT, 0, st>>>(in, A, w.tiles);
  scan_tiles<OP><<<1, 1024, 0, st>>>(w.tiles, nb, w.grand);
  if (out) scan_tiles_apply<OP, INCL><<<nb, kT, 0, st>>>(in, A, w.tiles, out);
}

int read_grand(SaWs2& w, cudaStream_t st, uint32_t* v) {
  int rc = cuda_check(cudaMemcpyAsync(v, w.grand, 4, cudaMemcpyDeviceToHost, st), "sa count");
  if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "sa sync");
  return rc;
}

}  // namespace

size_t sa_build_workspace2(uint64_t n) { return carve2(nullptr, n ? n : 1).total; }

// tokens [n] -> sa_out [n]; synchronises once per doubling round (the active count)
int sa_build2(const uint32_t* tokens, uint64_t n, uint32_t* sa_out, void* workspace, size_t workspace_bytes,
              cudaStream_t st, int* rounds_out) {
  SaWs2 w = carve2(static_cast<uint8_t*>(workspace), n);
  if (!workspace || workspace_bytes < w.total)
    return fail(SSSD_E_WORKSPACE, "sa_build needs %zu workspace bytes, got %zu", w.total, workspace_bytes);
  if (n == 1) return cuda_check(cudaMemsetAsync(sa_out, 0, 4, st), "sa memset");
  int rc = 0;

  const int T = 256;
  auto grid = [](uint64_t m) { return (unsigned)((m + 255) / 256); };
  // round 1: sort by token (only the token bits: a max-reduce first)
  uint32_t maxtok = 0;
  scan<1, true>(w, tokens, n, nullptr, st);
  if ((rc = read_grand(w, st, &maxtok))) return rc;
  // Round 1 sorts by the first m tokens at once when m >= 2 of them fit a
  // 64-bit key (V = 32,000: 15 bits, m = 4): that replaces the reference's
  // k = 1 and k = 2 doubling rounds (which re-sort 90 % and 75 % of the
  // phrase corpus with 54-bit keys) by one 60-bit sort; the rounds below
  // continue at k = m.  Otherwise: by token, ranks from a token table.
  const int tb = bits_of((uint64_t)maxtok + 1);
  int m = 1;
  while (m < 4 && (m * 2) * tb <= 64) m *= 2;  // m in {1, 2, 4}: the doubling schedule stays k = m, 2m, ...
  const bool table = m == 1 && w.table && (uint64_t)maxtok < kTableTokens;
  if (m > 1) {
    sa_mgram_keys<<<grid(n), T, 0, st>>>(tokens, n, m, tb, w.k0, w.v0);
    radix_sort(w, n, m * tb, st);
  } else {
    sa_first_keys<<<grid(n), T, 0, st>>>(tokens, n, w.k0, w.v0);
    radix_sort(w, n, bits_of(maxtok) > 0 ? bits_of(maxtok) : 1, st);
  }
  sa_round_heads<<<grid(n), T, 0, st>>>(w.k0, w.v0, n, nullptr, sa_out, w.tmp, table ? w.table : nullptr);
  scan<1, true>(w, w.tmp, n, w.tmp2, st);
  if (table) sa_rank_from_table<<<grid(n), T, 0, st>>>(tokens, n, w.table, w.rank);
  sa_round_rank<<<grid(n), T, 0, st>>>(w.k0, w.v0, n, w.tmp2, -1, table ? nullptr : w.rank, w.tmp);
  scan<0, false>(w, w.tmp, n, w.v1, st);  // (v1, the sort's second buffer, is free here)
  sa_compact<<<grid(n), T, 0, st>>>(w.tmp, w.v1, n, nullptr, w.v0, w.tmp2, w.aslot, w.apos, w.agrp);
  uint32_t A32 = 0;
  if ((rc = read_grand(w, st, &A32))) return rc;
  uint64_t A = A32;
  const int rb = bits_of(n);  // heads < n and rank + 1 <= n
  // rounds reported as the reference's doubling rounds (datastore.py:93-109:
  // the initial token rank plus one per k = 1, 2, 4, ... up to the last k
  // this build processed), so the algorithmic-byte count does not depend on m
  int rounds = 1;
  for (int mm = m; mm > 1; mm >>= 1) ++rounds;
  for (uint64_t k = (uint64_t)m; A > 0; k *= 2) {
    if (k >= n) return fail(SSSD_E_ARG, "suffix doubling did not converge");
    ++rounds;
    sa_round_keys<<<grid(A), T, 0, st>>>(w.apos, w.agrp, A, w.rank, n, k, rb, w.k0, w.v0);
    radix_sort(w, A, 2 * rb, st);
    sa_round_heads<<<grid(A), T, 0, st>>>(w.k0, w.v0, A, w.aslot, sa_out, w.tmp, nullptr);
    scan<1, true>(w, w.tmp, A, w.tmp2, st);
    sa_round_rank<<<grid(A), T, 0, st>>>(w.k0, w.v0, A, w.tmp2, rb, w.rank, w.tmp);
    scan<0, false>(w, w.tmp, A, w.v1, st);
    sa_compact<<<grid(A), T, 0, st>>>(w.tmp, w.v1, A, w.aslot, w.v0, w.tmp2, w.aslot2, w.apos2, w.agrp2);
    uint32_t* t = w.aslot;
    w.aslot = w.aslot2;
    w.aslot2 = t;
    t = w.apos;
    w.apos = w.apos2;
    w.apos2 = t;
    t = w.agrp;
    w.agrp = w.agrp2;
    w.agrp2 = t;
    if ((rc = read_grand(w, st, &A32))) return rc;
    A = A32;
  }
  if (rounds_out) *rounds_out = rounds;
  return cuda_check(cudaGetLastError(), "sa_build launch");
}

}  // namespace sssd
