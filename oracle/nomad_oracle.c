/*
 * TEST INFRASTRUCTURE ONLY — the CPU restatement ("oracle") of the
 * reference's hot path, in plain C. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as the CHECKER; the
 * product (paper_2505_15511_b200/, libnomad_b200.so) never links or calls it.
 *
 * Each function cites the reference file:line it restates
 * (/root/reference/proj/include/nomad/...). The restatement is PINNED against
 * the reference itself: oracle/_ref/libnomad_ref.so (the unmodified
 * reference headers compiled by oracle/Makefile) and the golden fixtures in
 * tests/golden/ that tests/make_golden.py generated from it
 * (tests/test_oracle.py checks both).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off (no -march=native: SURVEY §2.5).
 * Error convention: 0 ok, else 1 + ErrorKind (error.hpp:25-36), message via
 * orc_last_error().
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum { K_IO = 0, K_DIMENSION, K_VALIDATION, K_SCHEMA, K_PARAMETER, K_CONFIG,
       K_DEGENERATE, K_DIVERGENCE, K_SIZE, K_INTERNAL };

static _Thread_local char g_err[512];

static int fail(int kind, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return 1 + kind;
}

const char* orc_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- rng.hpp */

/* rng.hpp:25-30 splitmix64 step */
uint64_t orc_mix_seed(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* rng.hpp:32-34 */
uint64_t orc_stream_seed(uint64_t base, uint64_t stream) {
  return orc_mix_seed(base ^ orc_mix_seed(stream));
}

/* std::mt19937_64 as fixed by [rand.predef] (the reference's Rng::gen_,
 * rng.hpp:81): w=64, n=312, m=156, r=31, a=0xB5026F5AA96619E9, u=29,
 * d=0x5555555555555555, s=17, b=0x71D67FFFEDA60000, t=37,
 * c=0xFFF7EEE000000000, l=43, f=6364136223846793005. */
typedef struct {
  uint64_t mt[312];
  int idx;
  double spare;
  int have_spare;
} orc_rng;

static void rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  r->idx = 312;
  r->spare = 0.0;
  r->have_spare = 0;
}

static void rng_twist(orc_rng* r) {
  const uint64_t hi = 0xFFFFFFFF80000000ull, lo = 0x7FFFFFFFull;
  for (int i = 0; i < 312; ++i) {
    uint64_t y = (r->mt[i] & hi) | (r->mt[(i + 1) % 312] & lo);
    uint64_t v = r->mt[(i + 156) % 312] ^ (y >> 1);
    if (y & 1ull) v ^= 0xB5026F5AA96619E9ull;
    r->mt[i] = v;
  }
  r->idx = 0;
}

static uint64_t rng_u64(orc_rng* r) {
  if (r->idx >= 312) rng_twist(r);
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}

/* rng.hpp:49-55 rejection on the top range */
static uint64_t rng_uniform_index(orc_rng* r, uint64_t n) {
  const uint64_t limit = n * (0xFFFFFFFFFFFFFFFFull / n);
  uint64_t draw = rng_u64(r);
  while (draw >= limit) draw = rng_u64(r);
  return draw % n;
}

/* rng.hpp:58-60 */
static double rng_uniform01(orc_rng* r) {
  return (double)(rng_u64(r) >> 11) * 0x1.0p-53;
}

/* rng.hpp:65-78 Box-Muller with one cached spare */
static double rng_gaussian(orc_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u = rng_uniform01(r);
  while (u == 0.0) u = rng_uniform01(r);
  const double v = rng_uniform01(r);
  const double radius = sqrt(-2.0 * log(u));
  const double angle = 6.283185307179586476925286766559 * v;
  r->spare = radius * sin(angle);
  r->have_spare = 1;
  return radius * cos(angle);
}

void orc_rng_u64(uint64_t seed, uint64_t count, uint64_t* out) {
  orc_rng r;
  rng_seed(&r, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng_u64(&r);
}
void orc_rng_gaussian(uint64_t seed, uint64_t count, double* out) {
  orc_rng r;
  rng_seed(&r, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng_gaussian(&r);
}
void orc_rng_uniform_index(uint64_t seed, uint64_t bound, uint64_t count,
                           uint64_t* out) {
  orc_rng r;
  rng_seed(&r, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng_uniform_index(&r, bound);
}

/* Synthetic Gaussian mixture (SURVEY §8(d) "Synthetic inputs"; not reference
 * code): centres c_b ~ N(0, spread^2 I), x_i = c_{i mod B} + N(0, I), all
 * drawn from one Rng(seed) stream, centres first (b-major), then points
 * (i-major), cast to f32. Shared by tests and the CPU baseline so GPU and
 * oracle see identical bytes. */
void orc_gaussian_mixture(uint64_t n, uint64_t d, uint64_t blobs, double spread,
                          uint64_t seed, float* out) {
  orc_rng r;
  rng_seed(&r, seed);
  double* centres = (double*)malloc(sizeof(double) * blobs * d);
  for (uint64_t i = 0; i < blobs * d; ++i) centres[i] = spread * rng_gaussian(&r);
  for (uint64_t i = 0; i < n; ++i) {
    const double* c = centres + (i % blobs) * d;
    for (uint64_t j = 0; j < d; ++j)
      out[i * d + j] = (float)(c[j] + rng_gaussian(&r));
  }
  free(centres);
}

/* --------------------------------------------------------- affinity.hpp */

/* affinity.hpp:32-42 */
int orc_inverse_rank_weights(uint64_t k, double* out) {
  if (k < 1) return fail(K_PARAMETER, "neighbor count must be >= 1");
  double total = 0.0;
  for (uint64_t t = 1; t <= k; ++t) {
    out[t - 1] = exp(1.0 / (double)t);
    total += out[t - 1];
  }
  for (uint64_t t = 0; t < k; ++t) out[t] /= total;
  return 0;
}

/* optimizer.hpp:85-91 */
double orc_lr_schedule(uint64_t epoch, uint64_t total, double lr0) {
  return lr0 * (1.0 - (double)epoch / (double)total);
}

/* ----------------------------------------------------------- kmeans.hpp */

/* kmeans.hpp:47-54: j-ascending fp64, no FMA */
static double sq_dist_fd(const float* a, const double* b, uint64_t d) {
  double acc = 0.0;
  for (uint64_t j = 0; j < d; ++j) {
    const double diff = (double)a[j] - b[j];
    acc += diff * diff;
  }
  return acc;
}

/* kmeans.hpp:56-68: strict '<' keeps the lowest centroid id on ties */
static uint32_t nearest_centroid(const double* cent, uint64_t C, uint64_t d,
                                 const float* x) {
  uint32_t best = 0;
  double best_d = sq_dist_fd(x, cent, d);
  for (uint64_t r = 1; r < C; ++r) {
    const double dd = sq_dist_fd(x, cent + r * d, d);
    if (dd < best_d) {
      best_d = dd;
      best = (uint32_t)r;
    }
  }
  return best;
}

static void recompute_sizes(uint64_t n, uint64_t C, const uint32_t* a,
                            uint32_t* sizes) {
  memset(sizes, 0, C * 4);
  for (uint64_t i = 0; i < n; ++i) ++sizes[a[i]];
}

/* kmeans.hpp:75-88: one cluster, ascending i, divide by count */
static void recompute_centroid(const float* x, uint64_t n, uint64_t d,
                               const uint32_t* a, double* cent, uint32_t r) {
  double* c = cent + (uint64_t)r * d;
  memset(c, 0, d * 8);
  uint64_t count = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (a[i] != r) continue;
    for (uint64_t j = 0; j < d; ++j) c[j] += (double)x[i * d + j];
    ++count;
  }
  if (count > 0)
    for (uint64_t j = 0; j < d; ++j) c[j] /= (double)count;
}

/* kmeans.hpp:90-104: all clusters in one ascending-i pass */
static void recompute_all(const float* x, uint64_t n, uint64_t d, uint64_t C,
                          const uint32_t* a, const uint32_t* sizes,
                          double* cent) {
  memset(cent, 0, C * d * 8);
  for (uint64_t i = 0; i < n; ++i) {
    double* c = cent + (uint64_t)a[i] * d;
    for (uint64_t j = 0; j < d; ++j) c[j] += (double)x[i * d + j];
  }
  for (uint64_t r = 0; r < C; ++r) {
    if (sizes[r] == 0) continue;
    for (uint64_t j = 0; j < d; ++j) cent[r * d + j] /= (double)sizes[r];
  }
}

/* kmeans.hpp:109-143: first empty cluster takes the farthest point (first
 * i on ties) of the first largest cluster; repeat until none is empty. */
static int repair_empty(const float* x, uint64_t n, uint64_t d, uint64_t C,
                        uint32_t* a, uint32_t* sizes, double* cent) {
  for (;;) {
    uint32_t empty = UINT32_MAX;
    for (uint64_t r = 0; r < C; ++r)
      if (sizes[r] == 0) { empty = (uint32_t)r; break; }
    if (empty == UINT32_MAX) return 0;
    uint32_t donor = 0;
    for (uint64_t r = 1; r < C; ++r)
      if (sizes[r] > sizes[donor]) donor = (uint32_t)r;
    if (sizes[donor] < 2)
      return fail(K_INTERNAL, "no donor cluster available for repair");
    uint64_t victim = UINT64_MAX;
    double worst = -1.0;
    for (uint64_t i = 0; i < n; ++i) {
      if (a[i] != donor) continue;
      const double dd = sq_dist_fd(x + i * d, cent + (uint64_t)donor * d, d);
      if (dd > worst) { worst = dd; victim = i; }
    }
    a[victim] = empty;
    --sizes[donor];
    ++sizes[empty];
    recompute_centroid(x, n, d, a, cent, donor);
    recompute_centroid(x, n, d, a, cent, empty);
  }
}

/* kmeans.hpp:148-154 */
double orc_quantization_error(const float* x, uint64_t n, uint64_t d,
                              const uint32_t* a, const double* cent) {
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i)
    acc += sq_dist_fd(x + i * d, cent + (uint64_t)a[i] * d, d);
  return acc / (double)n;
}

/* kmeans.hpp:157-161: storage-order sum of exact f32 squares */
double orc_default_kmeans_tol(const float* x, uint64_t n, uint64_t d) {
  double acc = 0.0;
  for (uint64_t i = 0; i < n * d; ++i) acc += (double)x[i] * x[i];
  return 1e-6 * (acc / (double)n);
}

typedef struct { uint64_t code; uint32_t i; } code_pt;
static int cmp_code_pt(const void* pa, const void* pb) {
  const code_pt* a = (const code_pt*)pa; const code_pt* b = (const code_pt*)pb;
  if (a->code != b->code) return a->code < b->code ? -1 : 1;
  return a->i < b->i ? -1 : (a->i > b->i);
}
typedef struct { uint64_t code; uint64_t start, size; } bucket_t;
/* std::stable_sort by size descending over buckets already in ascending code
 * order == sort by (size desc, code asc). */
static int cmp_bucket(const void* pa, const void* pb) {
  const bucket_t* a = (const bucket_t*)pa; const bucket_t* b = (const bucket_t*)pb;
  if (a->size != b->size) return a->size > b->size ? -1 : 1;
  return a->code < b->code ? -1 : (a->code > b->code);
}

/* kmeans.hpp:167-250 */
int orc_lsh_init(const float* x, uint64_t n, uint64_t d, uint64_t C,
                 uint64_t seed, uint32_t* a, double* cent, uint32_t* sizes) {
  if (C < 2 || C > n) {
    char m[128];
    snprintf(m, sizeof m, "cluster count must be in [2, n]; got %llu",
             (unsigned long long)C);
    return fail(K_PARAMETER, m);
  }
  orc_rng rng;
  rng_seed(&rng, orc_stream_seed(seed, 0x6c7368));
  double* mean = (double*)calloc(d, 8);
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t j = 0; j < d; ++j) mean[j] += (double)x[i * d + j];
  for (uint64_t j = 0; j < d; ++j) mean[j] /= (double)n;

  const uint64_t P = (uint64_t)ceil(log2(4.0 * (double)C));
  double* planes = (double*)malloc(P * d * 8);
  for (uint64_t t = 0; t < P * d; ++t) planes[t] = rng_gaussian(&rng);

  code_pt* cp = (code_pt*)malloc(n * sizeof(code_pt));
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t code = 0;
    for (uint64_t p = 0; p < P; ++p) {
      const double* w = planes + p * d;
      double proj = 0.0;
      for (uint64_t j = 0; j < d; ++j) proj += ((double)x[i * d + j] - mean[j]) * w[j];
      if (proj >= 0.0) code |= (1ull << p);
    }
    cp[i].code = code;
    cp[i].i = (uint32_t)i;
  }
  qsort(cp, n, sizeof(code_pt), cmp_code_pt);
  bucket_t* bk = (bucket_t*)malloc(n * sizeof(bucket_t));
  uint64_t nb = 0;
  for (uint64_t s = 0; s < n;) {
    uint64_t e = s;
    while (e < n && cp[e].code == cp[s].code) ++e;
    bk[nb].code = cp[s].code; bk[nb].start = s; bk[nb].size = e - s; ++nb;
    s = e;
  }
  qsort(bk, nb, sizeof(bucket_t), cmp_bucket);

  memset(cent, 0, C * d * 8);
  const uint64_t seeded = C < nb ? C : nb;
  for (uint64_t r = 0; r < seeded; ++r) {
    double* c = cent + r * d;
    for (uint64_t m = 0; m < bk[r].size; ++m) {
      const float* xi = x + (uint64_t)cp[bk[r].start + m].i * d;
      for (uint64_t j = 0; j < d; ++j) c[j] += (double)xi[j];
    }
    for (uint64_t j = 0; j < d; ++j) c[j] /= (double)bk[r].size;
  }
  if (seeded < C) {
    double scale = 0.0;
    for (uint64_t i = 0; i < n; ++i) scale += sq_dist_fd(x + i * d, mean, d);
    scale = sqrt(scale / (double)n) * 1e-3 + 1e-12;
    uint64_t source = 0;
    for (uint64_t r = seeded; r < C; ++r) {
      for (uint64_t j = 0; j < d; ++j)
        cent[r * d + j] = cent[source * d + j] + scale * rng_gaussian(&rng);
      source = (source + 1) % seeded;
    }
  }
  for (uint64_t i = 0; i < n; ++i) a[i] = nearest_centroid(cent, C, d, x + i * d);
  recompute_sizes(n, C, a, sizes);
  int rc = repair_empty(x, n, d, C, a, sizes, cent);
  free(mean); free(planes); free(cp); free(bk);
  return rc;
}

/* kmeans.hpp:257-296 */
int orc_kmeans_em(const float* x, uint64_t n, uint64_t d, uint64_t C,
                  uint32_t* a, double* cent, uint32_t* sizes, uint64_t max_iters,
                  double tol, double* qe_trace, uint64_t* n_trace) {
  double* prev = (double*)malloc(C * d * 8);
  uint64_t nt = 0;
  int rc = 0;
  for (uint64_t it = 0; it < max_iters; ++it) {
    uint64_t changes = 0;
    for (uint64_t i = 0; i < n; ++i) {
      const uint32_t b = nearest_centroid(cent, C, d, x + i * d);
      if (b != a[i]) { a[i] = b; ++changes; }
    }
    recompute_sizes(n, C, a, sizes);
    memcpy(prev, cent, C * d * 8);
    recompute_all(x, n, d, C, a, sizes, cent);
    if ((rc = repair_empty(x, n, d, C, a, sizes, cent))) break;
    double max_move = 0.0;
    for (uint64_t r = 0; r < C; ++r) {
      double mv = 0.0;
      for (uint64_t j = 0; j < d; ++j) {
        const double diff = cent[r * d + j] - prev[r * d + j];
        mv += diff * diff;
      }
      if (mv > max_move) max_move = mv; /* std::max(max_move, mv) */
    }
    if (qe_trace) qe_trace[nt] = orc_quantization_error(x, n, d, a, cent);
    ++nt;
    if (changes == 0 || max_move < tol) break;
  }
  if (n_trace) *n_trace = qe_trace ? nt : 0;
  free(prev);
  return rc;
}

/* -------------------------------------------------------------- knn.hpp */

/* knn.hpp:51-58 */
static double sq_dist_ff(const float* a, const float* b, uint64_t d) {
  double acc = 0.0;
  for (uint64_t j = 0; j < d; ++j) {
    const double diff = (double)a[j] - (double)b[j];
    acc += diff * diff;
  }
  return acc;
}

/* knn.hpp:65-109: per point, the min(k, size-1) smallest (dist, id) pairs
 * (std::partial_sort on pair<double,uint32_t>) among same-cluster points. */
int orc_build_knn(const float* x, uint64_t n, uint64_t d, uint64_t C,
                  const uint32_t* a, uint64_t k, uint32_t* offsets,
                  uint32_t* nbrs, double* dists) {
  if (k < 1) return fail(K_PARAMETER, "k must be >= 1");
  uint64_t* start = (uint64_t*)calloc(C + 1, 8);
  for (uint64_t i = 0; i < n; ++i) ++start[a[i] + 1];
  for (uint64_t r = 0; r < C; ++r) start[r + 1] += start[r];
  uint32_t* members = (uint32_t*)malloc(n * 4);
  uint64_t* fill = (uint64_t*)malloc(C * 8);
  memcpy(fill, start, C * 8);
  for (uint64_t i = 0; i < n; ++i) members[fill[a[i]]++] = (uint32_t)i;
  offsets[0] = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t size = start[a[i] + 1] - start[a[i]];
    const uint64_t want = k < size - 1 ? k : size - 1;
    offsets[i + 1] = offsets[i] + (uint32_t)want;
  }
  double* bd = (double*)malloc((k + 1) * 8);
  uint32_t* bi = (uint32_t*)malloc((k + 1) * 4);
  for (uint64_t r = 0; r < C; ++r) {
    const uint64_t s0 = start[r], s1 = start[r + 1];
    const uint64_t size = s1 - s0;
    const uint64_t want = k < size - 1 ? k : size - 1;
    if (size == 0 || want == 0) continue;
    for (uint64_t p = s0; p < s1; ++p) {
      const uint32_t i = members[p];
      uint64_t cnt = 0;
      for (uint64_t q = s0; q < s1; ++q) {
        const uint32_t j = members[q];
        if (j == i) continue;
        const double dd = sq_dist_ff(x + (uint64_t)i * d, x + (uint64_t)j * d, d);
        /* insertion into the sorted (dist, id) prefix of length <= want */
        if (cnt == want && !(dd < bd[want - 1] || (dd == bd[want - 1] && j < bi[want - 1])))
          continue;
        uint64_t pos = cnt < want ? cnt : want - 1;
        while (pos > 0 && (dd < bd[pos - 1] || (dd == bd[pos - 1] && j < bi[pos - 1]))) {
          bd[pos] = bd[pos - 1];
          bi[pos] = bi[pos - 1];
          --pos;
        }
        bd[pos] = dd;
        bi[pos] = j;
        if (cnt < want) ++cnt;
      }
      for (uint64_t t = 0; t < want; ++t) {
        nbrs[offsets[i] + t] = bi[t];
        dists[offsets[i] + t] = bd[t];
      }
    }
  }
  free(start); free(members); free(fill); free(bd); free(bi);
  return 0;
}

/* Per-row checkers (config B/C parity on a row sample). knn.hpp:88-106 for
 * the queries (indices into `members`, one cluster's rows in ascending id):
 * the min(k, m-1) smallest (sq_dist_ff, id) pairs over the other members.
 * Returns want. `threads` is ignored (single-threaded restatement). */
int orc_knn_rows(const float* members, const uint32_t* ids, uint64_t m, uint64_t d,
                 const uint64_t* queries, uint64_t nq, uint64_t k, uint32_t* out_ids,
                 double* out_dist, int32_t threads) {
  (void)threads;
  const uint64_t want = k < (m ? m - 1 : 0) ? k : (m ? m - 1 : 0);
  if (want == 0) return 0;
  double* bd = (double*)malloc((want + 1) * 8);
  uint32_t* bi = (uint32_t*)malloc((want + 1) * 4);
  for (uint64_t q = 0; q < nq; ++q) {
    const uint64_t qi = queries[q];
    uint64_t cnt = 0;
    for (uint64_t jj = 0; jj < m; ++jj) {
      if (jj == qi) continue;
      const uint32_t j = ids[jj];
      const double dd = sq_dist_ff(members + qi * d, members + jj * d, d);
      if (cnt == want && !(dd < bd[want - 1] || (dd == bd[want - 1] && j < bi[want - 1])))
        continue;
      uint64_t pos = cnt < want ? cnt : want - 1;
      while (pos > 0 && (dd < bd[pos - 1] || (dd == bd[pos - 1] && j < bi[pos - 1]))) {
        bd[pos] = bd[pos - 1];
        bi[pos] = bi[pos - 1];
        --pos;
      }
      bd[pos] = dd;
      bi[pos] = j;
      if (cnt < want) ++cnt;
    }
    for (uint64_t t = 0; t < want; ++t) {
      out_ids[q * k + t] = bi[t];
      out_dist[q * k + t] = bd[t];
    }
  }
  free(bd);
  free(bi);
  return (int)want;
}

/* kmeans.hpp:56-68 nearest_centroid for a set of rows (strict <). */
void orc_nearest_centroid_rows(const float* rows, uint64_t nr, uint64_t d,
                               const double* centroids, uint64_t C, uint32_t* out,
                               int32_t threads) {
  (void)threads;
  for (uint64_t i = 0; i < nr; ++i) out[i] = nearest_centroid(centroids, C, d, rows + i * d);
}

/* kmeans.hpp:75-88 one cluster's centroid from its member rows (ascending id). */
void orc_cluster_centroid(const float* members, uint64_t m, uint64_t d, double* out) {
  for (uint64_t j = 0; j < d; ++j) out[j] = 0.0;
  for (uint64_t i = 0; i < m; ++i)
    for (uint64_t j = 0; j < d; ++j) out[j] += (double)members[i * d + j];
  if (m)
    for (uint64_t j = 0; j < d; ++j) out[j] /= (double)m;
}

/* -------------------------------------------------------- optimizer.hpp */

static int cmp_cluster_order_sizes_ctx_dummy;
static const uint32_t* g_sizes_for_sort;
static int cmp_cluster_order(const void* pa, const void* pb) {
  const uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
  if (g_sizes_for_sort[a] != g_sizes_for_sort[b])
    return g_sizes_for_sort[a] > g_sizes_for_sort[b] ? -1 : 1;
  return a < b ? -1 : (a > b);
}

/* optimizer.hpp:106-144 greedy LPT. worker_points: n entries, worker-major,
 * ascending within each worker; worker_offsets: W+1. */
int orc_shard_clusters(uint64_t n, uint64_t C, const uint32_t* a, uint64_t W,
                       uint32_t* c2w, uint32_t* worker_points,
                       uint64_t* worker_offsets) {
  (void)cmp_cluster_order_sizes_ctx_dummy;
  if (W < 1) return fail(K_PARAMETER, "workers must be >= 1");
  if (C < W) {
    char m[128];
    snprintf(m, sizeof m, "clusters must be >= workers (%llu < %llu)",
             (unsigned long long)C, (unsigned long long)W);
    return fail(K_PARAMETER, m);
  }
  uint32_t* sizes = (uint32_t*)calloc(C, 4);
  for (uint64_t i = 0; i < n; ++i) ++sizes[a[i]];
  uint32_t* order = (uint32_t*)malloc(C * 4);
  for (uint64_t r = 0; r < C; ++r) order[r] = (uint32_t)r;
  g_sizes_for_sort = sizes;
  qsort(order, C, 4, cmp_cluster_order);
  uint64_t* load = (uint64_t*)calloc(W, 8);
  for (uint64_t t = 0; t < C; ++t) {
    const uint32_t c = order[t];
    uint64_t light = 0;
    for (uint64_t w = 1; w < W; ++w)
      if (load[w] < load[light]) light = w;
    c2w[c] = (uint32_t)light;
    load[light] += sizes[c];
  }
  if (worker_points && worker_offsets) {
    uint64_t off = 0;
    for (uint64_t w = 0; w < W; ++w) {
      worker_offsets[w] = off;
      for (uint64_t i = 0; i < n; ++i)
        if (c2w[a[i]] == w) worker_points[off++] = (uint32_t)i;
    }
    worker_offsets[W] = off;
  }
  free(sizes); free(order); free(load);
  return 0;
}

/* optimizer.hpp:149-176 */
int orc_gather_means(const double* layout, uint64_t n, uint64_t C,
                     const uint32_t* a, double* means) {
  uint32_t* counts = (uint32_t*)calloc(C, 4);
  for (uint64_t i = 0; i < n; ++i) ++counts[a[i]];
  memset(means, 0, C * 2 * 8);
  for (uint64_t i = 0; i < n; ++i) {
    means[2 * a[i]] += layout[2 * i];
    means[2 * a[i] + 1] += layout[2 * i + 1];
  }
  for (uint64_t r = 0; r < C; ++r) {
    if (counts[r] == 0) { free(counts); return fail(K_INTERNAL, "empty cluster in means gather"); }
    means[2 * r] /= (double)counts[r];
    means[2 * r + 1] /= (double)counts[r];
  }
  free(counts);
  return 0;
}

/* objective.hpp:36-41 */
static inline double cauchy(const double* a, const double* b) {
  const double dx = a[0] - b[0];
  const double dy = a[1] - b[1];
  const double sq = dx * dx + dy * dy;
  return 1.0 / (1.0 + sq);
}

/* objective.hpp:113-145 + 178-237 for one head. grads: 2*(1+nn+s). */
int orc_nomad_gradient(const double* layout, uint64_t n, uint32_t head,
                       const uint32_t* nb, const double* w, uint64_t nn,
                       const uint32_t* neg, uint64_t s, const uint32_t* remote,
                       const double* rprob, uint64_t nr, const double* means,
                       uint64_t C, double local_mass, uint64_t m_total,
                       double* loss_out, double* g) {
  (void)n; (void)C;
  if (s == 0 && local_mass != 0.0)
    return fail(K_CONFIG, "no local negative draws but local noise mass is non-zero");
  const double* h = layout + 2 * (uint64_t)head;
  double qneg_stack[64];
  double* qneg = s <= 64 ? qneg_stack : (double*)malloc(s * 8);
  double qrem_stack[256];
  double* qrem = nr <= 256 ? qrem_stack : (double*)malloc(nr * 8);
  double remote_sum = 0.0;
  for (uint64_t t = 0; t < nr; ++t) {
    const double q = cauchy(h, means + 2 * (uint64_t)remote[t]);
    qrem[t] = q;
    remote_sum += rprob[t] * q;
  }
  const double mean_field = (double)m_total * remote_sum;
  double sampled = 0.0, sf = 0.0;
  if (s > 0) {
    sf = (double)m_total * local_mass / (double)s;
    double qsum = 0.0;
    for (uint64_t t = 0; t < s; ++t) {
      const double q = cauchy(h, layout + 2 * (uint64_t)neg[t]);
      qneg[t] = q;
      qsum += q;
    }
    sampled = sf * qsum;
  }
  const double bg = mean_field + sampled;
  double loss = 0.0, gx = 0.0, gy = 0.0, bgs = 0.0;
  for (uint64_t t = 0; t < nn; ++t) {
    const double* o = layout + 2 * (uint64_t)nb[t];
    const double q = cauchy(h, o);
    const double wt = w[t];
    loss += wt * -log(q / (q + bg));
    bgs += wt / (q + bg);
    const double pull = 2.0 * wt * (1.0 / q - 1.0 / (q + bg)) * q * q;
    const double dx = h[0] - o[0];
    const double dy = h[1] - o[1];
    gx += pull * dx;
    gy += pull * dy;
    g[2 + 2 * t] = -pull * dx;
    g[3 + 2 * t] = -pull * dy;
  }
  for (uint64_t t = 0; t < s; ++t) {
    const double* o = layout + 2 * (uint64_t)neg[t];
    const double q = qneg[t];
    const double push = 2.0 * bgs * sf * q * q;
    const double dx = h[0] - o[0];
    const double dy = h[1] - o[1];
    gx -= push * dx;
    gy -= push * dy;
    g[2 + 2 * nn + 2 * t] = push * dx;
    g[3 + 2 * nn + 2 * t] = push * dy;
  }
  for (uint64_t t = 0; t < nr; ++t) {
    const double* mu = means + 2 * (uint64_t)remote[t];
    const double q = qrem[t];
    const double push = 2.0 * bgs * (double)m_total * rprob[t] * q * q;
    gx -= push * (h[0] - mu[0]);
    gy -= push * (h[1] - mu[1]);
  }
  g[0] = gx;
  g[1] = gy;
  *loss_out = loss;
  if (qneg != qneg_stack) free(qneg);
  if (qrem != qrem_stack) free(qrem);
  return 0;
}

/* optimizer.hpp:215-227 */
static int apply_update(double* layout, uint32_t p, double gx, double gy,
                        double step, uint64_t epoch, uint64_t draw) {
  double* q = layout + 2 * (uint64_t)p;
  q[0] -= step * gx;
  q[1] -= step * gy;
  if (!isfinite(q[0]) || !isfinite(q[1]) || fabs(q[0]) > 1e9 || fabs(q[1]) > 1e9) {
    char m[160];
    snprintf(m, sizeof m, "positions diverged at epoch %llu, head draw %llu (point %u)",
             (unsigned long long)epoch, (unsigned long long)draw, p);
    return fail(K_DIVERGENCE, m);
  }
  return 0;
}

typedef struct {
  uint64_t epochs, k, negatives, local_draws, batch_size, workers, n_clusters;
  uint64_t seed;
  double lr0;
  uint64_t kmeans_max_iters;
  double kmeans_tol;
  int32_t approx_all_but_own;
  int32_t head_only;
} orc_train_config;

typedef struct {
  uint32_t* points; uint64_t npoints;
  uint32_t* eligible; uint64_t neligible;
  uint32_t* remote; double* rprob; uint64_t nremote;
  double local_mass;
  orc_rng rng;
} worker_t;

/* The epoch loop of fit() (optimizer.hpp:355-470) from a given graph,
 * clusters and init layout; workers run one after another (their rows are
 * disjoint and the means snapshot is read-only, so the result equals the
 * reference's threaded run). Same signature as ref_train_epochs. */
int orc_train_epochs(uint64_t n, uint64_t C, const uint32_t* a,
                     const uint32_t* offsets, const uint32_t* nbrs, uint64_t k,
                     const orc_train_config* cfg, double* layout,
                     uint64_t first_epoch, uint64_t n_run, double* epoch_loss,
                     double* final_means, int32_t inline_workers,
                     double* seconds_out) {
  (void)inline_workers; (void)seconds_out;
  const uint64_t W = cfg->workers;
  if (W < 1) return fail(K_PARAMETER, "workers must be >= 1");
  if (k < 1) return fail(K_PARAMETER, "k must be >= 1");
  if (cfg->negatives < 1) return fail(K_PARAMETER, "negatives must be >= 1");
  if (cfg->local_draws < 1) return fail(K_PARAMETER, "local draws must be >= 1");
  if (cfg->batch_size < 1) return fail(K_PARAMETER, "batch size must be >= 1");
  int rc = 0;
  /* build_affinity (affinity.hpp:65-84): weight tables per neighbour count */
  double* wtab = (double*)calloc((k + 1) * k, 8);
  for (uint64_t c = 1; c <= k; ++c) orc_inverse_rank_weights(c, wtab + c * k);
  uint32_t* sizes = (uint32_t*)calloc(C, 4);
  for (uint64_t i = 0; i < n; ++i) ++sizes[a[i]];
  uint32_t* c2w = (uint32_t*)malloc(C * 4);
  uint32_t* wp = (uint32_t*)malloc(n * 4);
  uint64_t* woff = (uint64_t*)malloc((W + 1) * 8);
  if ((rc = orc_shard_clusters(n, C, a, W, c2w, wp, woff))) goto out0;
  worker_t* ws = (worker_t*)calloc(W, sizeof(worker_t));
  for (uint64_t w = 0; w < W; ++w) {
    worker_t* st = &ws[w];
    st->points = wp + woff[w];
    st->npoints = woff[w + 1] - woff[w];
    st->eligible = (uint32_t*)malloc((st->npoints + 1) * 4);
    for (uint64_t t = 0; t < st->npoints; ++t) {
      const uint32_t i = st->points[t];
      if (offsets[i + 1] > offsets[i]) st->eligible[st->neligible++] = i;
    }
    st->remote = (uint32_t*)malloc(C * 4);
    st->rprob = (double*)malloc(C * 8);
    uint64_t remote = 0;
    for (uint64_t r = 0; r < C; ++r) {
      if (c2w[r] == w) continue;
      st->remote[st->nremote] = (uint32_t)r;
      st->rprob[st->nremote++] = (double)sizes[r] / (double)n; /* affinity.hpp:104-105 */
      remote += sizes[r];
    }
    st->local_mass = (double)(n - remote) / (double)n;
    rng_seed(&st->rng, orc_stream_seed(cfg->seed, 0x776f726bull + w));
  }
  /* AllButOwnCluster pools: members per cluster (optimizer.hpp:374-380) */
  uint64_t* cstart = (uint64_t*)calloc(C + 1, 8);
  uint32_t* cmem = (uint32_t*)malloc(n * 4);
  for (uint64_t i = 0; i < n; ++i) ++cstart[a[i] + 1];
  for (uint64_t r = 0; r < C; ++r) cstart[r + 1] += cstart[r];
  {
    uint64_t* f = (uint64_t*)malloc(C * 8);
    memcpy(f, cstart, C * 8);
    for (uint64_t i = 0; i < n; ++i) cmem[f[a[i]]++] = (uint32_t)i;
    free(f);
  }
  const double lr0 = cfg->lr0 > 0.0 ? cfg->lr0 : (double)n / 10.0;
  double* means = (double*)malloc(C * 2 * 8);
  if ((rc = orc_gather_means(layout, n, C, a, means))) goto out1;
  const uint64_t S = cfg->local_draws;
  uint32_t* tails = (uint32_t*)malloc(S * 4);
  double* grads = (double*)malloc(2 * (1 + k + S) * 8);
  uint32_t* prem = (uint32_t*)malloc(C * 4);
  double* pprob = (double*)malloc(C * 8);
  for (uint64_t e = first_epoch; e < first_epoch + n_run && !rc; ++e) {
    if (e >= cfg->epochs) { rc = fail(K_PARAMETER, "epoch out of range for schedule"); break; }
    const double lr = orc_lr_schedule(e, cfg->epochs, lr0);
    const double step = lr / (double)cfg->batch_size;
    double loss_total = 0.0;
    uint64_t heads = 0;
    for (uint64_t w = 0; w < W && !rc; ++w) {
      worker_t* st = &ws[w];
      double loss_sum = 0.0;
      for (uint64_t t = 0; t < st->neligible && !rc; ++t) {
        const uint32_t head = st->eligible[rng_uniform_index(&st->rng, st->neligible)];
        const uint32_t* nb = nbrs + offsets[head];
        const uint64_t nn = offsets[head + 1] - offsets[head];
        const double* wt = wtab + nn * k;
        const uint32_t* pool = st->points;
        uint64_t pool_n = st->npoints;
        const uint32_t* rem = st->remote;
        const double* rp = st->rprob;
        uint64_t nr = st->nremote;
        double lm = st->local_mass;
        if (cfg->approx_all_but_own) { /* optimizer.hpp:264-277 */
          const uint32_t own = a[head];
          pool = cmem + cstart[own];
          pool_n = cstart[own + 1] - cstart[own];
          nr = 0;
          for (uint64_t r = 0; r < C; ++r) {
            if (r == own) continue;
            prem[nr] = (uint32_t)r;
            pprob[nr++] = (double)sizes[r] / (double)n;
          }
          rem = prem; rp = pprob;
          lm = (double)sizes[own] / (double)n;
        }
        for (uint64_t s = 0; s < S; ++s) tails[s] = pool[rng_uniform_index(&st->rng, pool_n)];
        double loss;
        if ((rc = orc_nomad_gradient(layout, n, head, nb, wt, nn, tails, S, rem, rp, nr,
                                     means, C, lm, cfg->negatives, &loss, grads)))
          break;
        loss_sum += loss;
        ++heads;
        if ((rc = apply_update(layout, head, grads[0], grads[1], step, e, t))) break;
        if (!cfg->head_only) {
          for (uint64_t j = 0; j < nn && !rc; ++j)
            rc = apply_update(layout, nb[j], grads[2 + 2 * j], grads[3 + 2 * j], step, e, t);
          for (uint64_t m = 0; m < S && !rc; ++m)
            rc = apply_update(layout, tails[m], grads[2 + 2 * nn + 2 * m],
                              grads[3 + 2 * nn + 2 * m], step, e, t);
        }
      }
      loss_total += loss_sum;
    }
    if (rc) break;
    if ((rc = orc_gather_means(layout, n, C, a, means))) break;
    if (epoch_loss) epoch_loss[e - first_epoch] = heads > 0 ? loss_total / (double)heads : 0.0;
  }
  if (!rc && final_means) memcpy(final_means, means, C * 2 * 8);
  free(tails); free(grads); free(prem); free(pprob);
out1:
  free(means); free(cstart); free(cmem);
  for (uint64_t w = 0; w < W; ++w) { free(ws[w].eligible); free(ws[w].remote); free(ws[w].rprob); }
  free(ws);
out0:
  free(wtab); free(sizes); free(c2w); free(wp); free(woff);
  return rc;
}

/* -------------------------------------------------------------- pca.hpp */

/* pca.hpp:34-55 */
static void cov_apply(const float* x, uint64_t n, uint64_t d, const double* mean,
                      const double* v, double* scratch, double* out) {
  for (uint64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (uint64_t j = 0; j < d; ++j) acc += ((double)x[i * d + j] - mean[j]) * v[j];
    scratch[i] = acc;
  }
  memset(out, 0, d * 8);
  for (uint64_t i = 0; i < n; ++i) {
    const double t = scratch[i];
    for (uint64_t j = 0; j < d; ++j) out[j] += ((double)x[i * d + j] - mean[j]) * t;
  }
  for (uint64_t j = 0; j < d; ++j) out[j] /= (double)n;
}
static double dotv(const double* a, const double* b, uint64_t d) {
  double acc = 0.0;
  for (uint64_t j = 0; j < d; ++j) acc += a[j] * b[j];
  return acc;
}
static double normalize(double* v, uint64_t d) {
  const double nrm = sqrt(dotv(v, v, d));
  if (nrm > 0.0)
    for (uint64_t j = 0; j < d; ++j) v[j] /= nrm;
  return nrm;
}

/* pca.hpp:79-218 */
int orc_pca_init(const float* x, uint64_t n, uint64_t d, uint64_t seed,
                 double* layout) {
  if (n < 2) return fail(K_PARAMETER, "need at least 2 rows");
  orc_rng rng;
  rng_seed(&rng, orc_stream_seed(seed, 0x706361));
  double* mean = (double*)calloc(d, 8);
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t j = 0; j < d; ++j) mean[j] += (double)x[i * d + j];
  for (uint64_t j = 0; j < d; ++j) mean[j] /= (double)n;
  double tv = 0.0, ts = 0.0;
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t j = 0; j < d; ++j) {
      const double c = (double)x[i * d + j] - mean[j];
      tv += c * c;
      ts += (double)x[i * d + j] * (double)x[i * d + j];
    }
  tv /= (double)n;
  ts /= (double)n;
  if (tv <= 1e-18 * (1.0 > ts ? 1.0 : ts)) { free(mean); return fail(K_DEGENERATE, "data has zero variance"); }
  double* scratch = (double*)malloc(n * 8);
  double* applied = (double*)malloc(d * 8);
  double* basis = (double*)calloc(2 * d, 8);
  double* prev = (double*)malloc(d * 8);
  double eig[2] = {0.0, 0.0};
  for (int comp = 0; comp < 2; ++comp) {
    double* v = basis + comp * d;
    for (uint64_t j = 0; j < d; ++j) v[j] = rng_gaussian(&rng);
    if (comp == 1) {
      const double ov = dotv(v, basis, d);
      for (uint64_t j = 0; j < d; ++j) v[j] -= ov * basis[j];
    }
    if (normalize(v, d) == 0.0) continue;
    for (uint64_t it = 0; it < 3000; ++it) {
      memcpy(prev, v, d * 8);
      cov_apply(x, n, d, mean, v, scratch, applied);
      if (comp == 1) {
        const double ov = dotv(applied, basis, d);
        for (uint64_t j = 0; j < d; ++j) applied[j] -= ov * basis[j];
      }
      memcpy(v, applied, d * 8);
      if (normalize(v, d) == 0.0) { memset(v, 0, d * 8); break; }
      double drift = 0.0;
      const double align = dotv(v, prev, d) < 0.0 ? -1.0 : 1.0;
      for (uint64_t j = 0; j < d; ++j) {
        const double diff = v[j] - align * prev[j];
        drift += diff * diff;
      }
      if (drift < 1e-30) break;
    }
    cov_apply(x, n, d, mean, v, scratch, applied);
    eig[comp] = dotv(v, applied, d);
  }
  double* b0 = basis;
  double* b1 = basis + d;
  if (dotv(b1, b1, d) > 0.0) {
    const double ov = dotv(b1, b0, d);
    for (uint64_t j = 0; j < d; ++j) b1[j] -= ov * b0[j];
    if (normalize(b1, d) > 0.0) {
      double* ca = (double*)malloc(d * 8);
      double* cb = (double*)malloc(d * 8);
      cov_apply(x, n, d, mean, b0, scratch, ca);
      cov_apply(x, n, d, mean, b1, scratch, cb);
      const double h00 = dotv(b0, ca, d), h01 = dotv(b0, cb, d), h11 = dotv(b1, cb, d);
      const double hg = 0.5 * (h00 - h11);
      const double root = sqrt(hg * hg + h01 * h01);
      eig[0] = 0.5 * (h00 + h11) + root;
      eig[1] = 0.5 * (h00 + h11) - root;
      double c = 1.0, s = 0.0;
      if (fabs(h01) > 1e-300) {
        const double t = eig[0] - h00;
        const double len = sqrt(h01 * h01 + t * t);
        c = h01 / len;
        s = t / len;
      } else if (h11 > h00) {
        c = 0.0;
        s = 1.0;
      }
      for (uint64_t j = 0; j < d; ++j) {
        const double f = c * b0[j] + s * b1[j];
        const double g = -s * b0[j] + c * b1[j];
        ca[j] = f;
        cb[j] = g;
      }
      memcpy(b0, ca, d * 8);
      memcpy(b1, cb, d * 8);
      free(ca); free(cb);
    }
  }
  for (int comp = 0; comp < 2; ++comp) {
    double* v = basis + comp * d;
    uint64_t arg = 0;
    for (uint64_t j = 1; j < d; ++j)
      if (fabs(v[j]) > fabs(v[arg])) arg = j;
    if (v[arg] < 0.0)
      for (uint64_t j = 0; j < d; ++j) v[j] = -v[j];
  }
  memset(layout, 0, n * 2 * 8);
  const int rank_def = eig[1] <= 1e-12 * (eig[0] > 0.0 ? eig[0] : 0.0);
  for (int comp = 0; comp < 2; ++comp) {
    if (comp == 1 && rank_def) {
      for (uint64_t i = 0; i < n; ++i)
        layout[2 * i + 1] = -1e-4 + (1e-4 - -1e-4) * rng_uniform01(&rng);
      break;
    }
    double cm = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (uint64_t j = 0; j < d; ++j) acc += ((double)x[i * d + j] - mean[j]) * basis[comp * d + j];
      layout[2 * i + comp] = acc;
      cm += acc;
    }
    cm /= (double)n;
    double var = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
      const double c = layout[2 * i + comp] - cm;
      var += c * c;
    }
    var /= (double)n;
    const double sd = sqrt(var);
    if (sd > 0.0)
      for (uint64_t i = 0; i < n; ++i) layout[2 * i + comp] /= sd;
  }
  free(mean); free(scratch); free(applied); free(basis); free(prev);
  return 0;
}
