/* CPU oracle: suffix array by prefix doubling — TEST / BASELINE INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's build_suffix_array
 * (/root/reference/pkg/src/specdraft/datastore.py:81-109): rank positions by
 * their first token, then repeatedly order by (rank[i], rank[i+k] or "past the
 * end") and re-rank until every rank is distinct.  Positions stay sorted by
 * rank between rounds, so a round only re-sorts the members of each
 * still-tied rank group by the second key (singleton groups are final) — the
 * order the reference's full lexsort produces.  Any correct suffix array is
 * identical; tests/test_oracle_golden.py checks this against the
 * NumPy oracle and the reference-generated goldens.
 *
 * Used by bench.py --impl reference to build the 100M-token datastore on the
 * host; never by the product path.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint32_t key;
  uint32_t pos;
} kp;

static int cmp_kp(const void* a, const void* b) {
  const kp* x = (const kp*)a;
  const kp* y = (const kp*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->pos < y->pos ? -1 : (x->pos > y->pos ? 1 : 0);
}

/* stable LSD radix sort of (key, pos) pairs by key, 16-bit digits */
static void radix_kp(kp* a, kp* tmp, uint64_t n, uint32_t* cnt) {
  for (int pass = 0; pass < 2; ++pass) {
    const int sh = 16 * pass;
    memset(cnt, 0, sizeof(uint32_t) * 65537);
    for (uint64_t i = 0; i < n; ++i) cnt[((a[i].key >> sh) & 0xffff) + 1]++;
    for (int d = 0; d < 65536; ++d) cnt[d + 1] += cnt[d];
    for (uint64_t i = 0; i < n; ++i) tmp[cnt[(a[i].key >> sh) & 0xffff]++] = a[i];
    memcpy(a, tmp, sizeof(kp) * n);
  }
}

/* sa[n] = suffix array of tokens[0..n); returns 0 on success. */
int sa_oracle_build(const uint32_t* tokens, uint64_t n, uint32_t* sa) {
  if (n == 0) return -1;
  if (n == 1) {
    sa[0] = 0;
    return 0;
  }
  uint32_t* rank = malloc(sizeof(uint32_t) * n);
  uint32_t* newr = malloc(sizeof(uint32_t) * n);
  kp* a = malloc(sizeof(kp) * n);
  kp* tmp = malloc(sizeof(kp) * n);
  uint32_t* cnt = malloc(sizeof(uint32_t) * 65537);
  int rc = 0;
  if (!rank || !newr || !a || !tmp || !cnt) {
    rc = -2;
    goto out;
  }
  /* order by first token; rank = start index of the equal-token group */
  for (uint64_t i = 0; i < n; ++i) {
    a[i].key = tokens[i];
    a[i].pos = (uint32_t)i;
  }
  radix_kp(a, tmp, n, cnt);
  for (uint64_t j = 0; j < n; ++j) sa[j] = a[j].pos;
  rank[sa[0]] = 0;
  for (uint64_t j = 1; j < n; ++j) rank[sa[j]] = a[j].key == a[j - 1].key ? rank[sa[j - 1]] : (uint32_t)j;

  for (uint64_t k = 1;; k *= 2) {
    int pending = 0;
    memcpy(newr, rank, sizeof(uint32_t) * n);
    uint64_t g = 0;
    while (g < n) {
      const uint32_t rg = rank[sa[g]];
      uint64_t e = g + 1;
      while (e < n && rank[sa[e]] == rg) ++e;
      if (e - g > 1) {
        pending = 1;
        const uint64_t m = e - g;
        for (uint64_t j = 0; j < m; ++j) {
          const uint32_t i = sa[g + j];
          a[j].key = (uint64_t)i + k < n ? rank[i + k] + 1 : 0; /* shorter suffix first */
          a[j].pos = i;
        }
        if (m > 4096) radix_kp(a, tmp, m, cnt);
        else qsort(a, m, sizeof(kp), cmp_kp);
        uint32_t start = (uint32_t)g;
        for (uint64_t j = 0; j < m; ++j) {
          if (j > 0 && a[j].key != a[j - 1].key) start = (uint32_t)(g + j);
          sa[g + j] = a[j].pos;
          newr[a[j].pos] = start;
        }
      }
      g = e;
    }
    if (!pending) break;
    uint32_t* t = rank;
    rank = newr;
    newr = t;
  }
out:
  free(rank);
  free(newr);
  free(a);
  free(tmp);
  free(cnt);
  return rc;
}
