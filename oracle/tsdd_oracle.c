/* TEST INFRASTRUCTURE — plain-C restatement of the reference's hot path.
 *
 * This is the CPU oracle ("port") the CUDA path is checked against.  It
 * restates, in this repo's own code, the algorithm of /root/reference/proj
 * (PhiDD / HOTSAX discord search); every function cites the reference
 * file:line it follows.  Parity is PINNED: tests/test_oracle_pin.py checks
 * every function here against the unmodified reference (oracle/_ref, built
 * from the reference sources by oracle/Makefile) and against the SPEC.md
 * known-answer examples, and
 * against tests/golden/workloads.json (reference outputs on the five seeded
 * BASELINE.json series).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product has no CPU fallback.
 *
 * All arithmetic is float64, as in the reference (series.hpp:15).  Positions
 * are 1-based at the C surface (discovery.hpp:21), rows 0-based inside.
 */
#define _POSIX_C_SOURCE 200809L
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_PARAMETER 2   /* tsdd::ParameterError        errors.hpp:10 */
#define ORC_VALIDATION 3  /* tsdd::ValidationError       errors.hpp:16 */
#define ORC_INFEASIBLE 4  /* tsdd::InfeasibleInputError  errors.hpp:22 */

static _Thread_local char g_err[256];

static int fail(int code, const char* fmt, unsigned long long a, unsigned long long b) {
  snprintf(g_err, sizeof g_err, fmt, a, b);
  return code;
}

const char* orc_last_error(void) { return g_err; }

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------------------ */
/* SAX breakpoints: equiprobable N(0,1) quantiles, lower half mirrored
 * (sax.cpp:14-46, tools/gen_breakpoints.py).  Regenerated with scipy
 * 1.18 norm.ppf by tools/gen_sax_breakpoints.py; identical to the
 * reference's literals to the last digit.                              */
static const double kBreaks[9][9] = {
    /* 2 */ {0},
    /* 3 */ {-0.43072729929545756, 0.43072729929545756},
    /* 4 */ {-0.67448975019608171, 0, 0.67448975019608171},
    /* 5 */ {-0.84162123357291418, -0.25334710313579972, 0.25334710313579972, 0.84162123357291418},
    /* 6 */ {-0.96742156610170105, -0.43072729929545756, 0, 0.43072729929545756, 0.96742156610170105},
    /* 7 */ {-1.0675705238781414, -0.56594882193286311, -0.1800123697927051, 0.1800123697927051,
             0.56594882193286311, 1.0675705238781414},
    /* 8 */ {-1.1503493803760079, -0.67448975019608171, -0.31863936396437514, 0, 0.31863936396437514,
             0.67448975019608171, 1.1503493803760079},
    /* 9 */ {-1.2206403488473501, -0.7647096737863871, -0.43072729929545756, -0.13971029888186212,
             0.13971029888186212, 0.43072729929545756, 0.7647096737863871, 1.2206403488473501},
    /* 10 */ {-1.2815515655446004, -0.84162123357291418, -0.52440051270804089, -0.25334710313579972, 0,
              0.25334710313579972, 0.52440051270804089, 0.84162123357291418, 1.2815515655446004},
};

static int check_alphabet(uint64_t a) {
  if (a < 2 || a > 10) /* sax.cpp:42-44 */
    return fail(ORC_PARAMETER, "alphabet cardinality %llu is outside the built-in range 2..10", a, 0);
  return ORC_OK;
}

/* symbol = 1 + #{breakpoints <= value}: lower-inclusive bins (sax.cpp:53-57) */
static uint32_t symbol_of(uint64_t a, double v) {
  const double* bp = kBreaks[a - 2];
  uint32_t s = 1;
  for (uint64_t k = 0; k + 1 < a; ++k) s += (bp[k] <= v);
  return s;
}

int orc_symbol_for(uint64_t alphabet, double value, uint32_t* symbol) {
  int rc = check_alphabet(alphabet);
  if (rc) return rc;
  *symbol = symbol_of(alphabet, value);
  return ORC_OK;
}

/* dict_size with the 2^24 guard (sax.cpp:134-145, sax.hpp:80) */
static int dict_size(uint64_t a, uint64_t w, uint64_t* out) {
  uint64_t size = 1;
  for (uint64_t j = 0; j < w; ++j) {
    size *= a;
    if (size > ((uint64_t)1 << 24))
      return fail(ORC_PARAMETER, "dictionary of |A|^word_len = %llu^%llu words exceeds the 2^24 guard", a, w);
  }
  *out = size;
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* z-normalisation with the population variance sum_sq/n - mu^2; sigma <
 * 1e-12 maps to zeros; multiply by 1/sigma (series.cpp:21-37).        */
static void znorm(double* d, size_t n) {
  double sum = 0.0, sq = 0.0;
  for (size_t i = 0; i < n; ++i) {
    sum += d[i];
    sq += d[i] * d[i];
  }
  const double mu = sum / (double)n;
  const double var = sq / (double)n - mu * mu;
  const double sigma = var > 0.0 ? sqrt(var) : 0.0;
  if (sigma < 1e-12) {
    memset(d, 0, n * sizeof(double));
    return;
  }
  const double inv = 1.0 / sigma;
  for (size_t i = 0; i < n; ++i) d[i] = (d[i] - mu) * inv;
}

int orc_z_normalize(double* data, uint64_t n) {
  if (n == 0) return fail(ORC_VALIDATION, "series is empty", 0, 0);
  znorm(data, n);
  return ORC_OK;
}

/* validate_series (series.cpp:10-19) */
static int validate(const double* x, uint64_t m) {
  if (m == 0) return fail(ORC_VALIDATION, "series is empty", 0, 0);
  for (uint64_t i = 0; i < m; ++i)
    if (!isfinite(x[i])) return fail(ORC_VALIDATION, "non-finite value at index %llu", i + 1, 0);
  return ORC_OK;
}

/* SubsequenceMatrix::build (series.cpp:46-74): N x stride row-major, each
 * window z-normalised on its own, right padding left at zero.          */
typedef struct {
  double* data;
  size_t rows, n, stride;
} Matrix;

static int matrix_build(const double* x, uint64_t m, uint64_t n, uint64_t vw, Matrix* out) {
  int rc = validate(x, m);
  if (rc) return rc;
  if (n < 1 || n > m)
    return fail(ORC_PARAMETER, "subsequence length n=%llu must satisfy 1 <= n <= m=%llu", n, m);
  if (vw < 1) return fail(ORC_PARAMETER, "vec_width must be >= 1", 0, 0);
  out->rows = m - n + 1;
  out->n = n;
  out->stride = n + (vw - n % vw) % vw;
  out->data = (double*)calloc(out->rows * out->stride, sizeof(double));
  if (!out->data) return fail(1, "out of memory", 0, 0);
#pragma omp parallel for schedule(static)
  for (ptrdiff_t i = 0; i < (ptrdiff_t)out->rows; ++i) {
    double* row = out->data + (size_t)i * out->stride;
    memcpy(row, x + i, n * sizeof(double));
    znorm(row, n);
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Distance: 8-wide blocks summed in the fixed tree ((s01+s23)+(s45+s67)),
 * blocks added to a running sum, abandon test `sum > threshold` every
 * `block` (>= 8) elements and once more after the zero-extended tail
 * (series.hpp:81-146).  Returns 1 when abandoned.                      */
static double block8(const double* a, const double* b, size_t len) {
  double d[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (size_t i = 0; i < len; ++i) d[i] = a[i] - b[i];
  const double s01 = d[0] * d[0] + d[1] * d[1];
  const double s23 = d[2] * d[2] + d[3] * d[3];
  const double s45 = d[4] * d[4] + d[5] * d[5];
  const double s67 = d[6] * d[6] + d[7] * d[7];
  return (s01 + s23) + (s45 + s67);
}

typedef struct {
  uint64_t calls, abandoned;
} Counters;

static int dist_ea(const double* a, const double* b, size_t len, double threshold, size_t block,
                   double* out, Counters* c) {
  ++c->calls;
  const size_t every = block < 8 ? 8 : block;
  double sum = 0.0;
  size_t i = 0, since = 0;
  for (; i + 8 <= len; i += 8) {
    sum += block8(a + i, b + i, 8);
    since += 8;
    if (since >= every) {
      since = 0;
      if (sum > threshold) {
        ++c->abandoned;
        return 1;
      }
    }
  }
  if (i < len) sum += block8(a + i, b + i, len - i);
  if (sum > threshold) {
    ++c->abandoned;
    return 1;
  }
  *out = sum;
  return 0;
}

int orc_distance(const double* a, const double* b, uint64_t len, double threshold, uint64_t block,
                 double* value, int* abandoned_flag) {
  Counters c = {0, 0};
  double v = 0.0;
  *abandoned_flag = dist_ea(a, b, len, threshold, block, &v, &c);
  *value = v;
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* PAA on an n*w unit grid: element t covers [t*w,(t+1)*w), segment k covers
 * [k*n,(k+1)*n); weighted sum / n (sax.cpp:63-80).                     */
static void paa_one(const double* v, size_t n, double* out, size_t w) {
  for (size_t k = 0; k < w; ++k) {
    const size_t lo = k * n, hi = (k + 1) * n;
    const size_t t0 = lo / w, t1 = (hi - 1) / w;
    double acc = 0.0;
    for (size_t t = t0; t <= t1; ++t) {
      const size_t el = t * w, eh = el + w;
      const size_t units = (eh < hi ? eh : hi) - (el > lo ? el : lo);
      acc += (double)units * v[t];
    }
    out[k] = acc / (double)n;
  }
}

int orc_paa_row(const double* values, uint64_t n, double* out, uint64_t w) {
  if (w < 1 || w > n)
    return fail(ORC_PARAMETER, "word_len=%llu must satisfy 1 <= word_len <= n=%llu", w, n);
  paa_one(values, n, out, w);
  return ORC_OK;
}

/* h = 1 + sum (a_j - 1) |A|^(w-j), big-endian (sax.cpp:121-132) */
int orc_word_hash(const uint32_t* word, uint64_t w, uint64_t alphabet, uint64_t* hash) {
  int rc = check_alphabet(alphabet);
  if (rc) return rc;
  uint64_t h = 0;
  for (uint64_t j = 0; j < w; ++j) {
    if (word[j] < 1 || word[j] > alphabet)
      return fail(ORC_PARAMETER, "symbol %llu is outside alphabet range 1..%llu", word[j], alphabet);
    h = h * alphabet + (word[j] - 1);
  }
  *hash = h + 1;
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* The index bundle (index.cpp:12-109): per-row hash, freq[i] = size of row
 * i's bucket, candidates = rows at the global minimum frequency (ascending,
 * 1-based), buckets as offsets into a position array filled by a stable
 * counting sort (ascending positions inside every bucket).             */
typedef struct {
  size_t rows;
  uint64_t dict;
  uint64_t* hash;     /* rows, 1-based hash values */
  uint32_t* freq;     /* rows */
  size_t* offsets;    /* dict + 1 */
  size_t* positions;  /* rows, 1-based */
  size_t* cand;       /* n_cand, 1-based */
  size_t n_cand;
} Index;

static void index_free(Index* ix) {
  free(ix->hash);
  free(ix->freq);
  free(ix->offsets);
  free(ix->positions);
  free(ix->cand);
  memset(ix, 0, sizeof *ix);
}

static int index_build(const Matrix* M, uint64_t w, uint64_t a, double* paa_out, uint32_t* sax_out,
                       Index* ix) {
  memset(ix, 0, sizeof *ix);
  int rc = check_alphabet(a);
  if (rc) return rc;
  if (w < 1 || w > M->n)
    return fail(ORC_PARAMETER, "word_len=%llu must satisfy 1 <= word_len <= n=%llu", w, M->n);
  rc = dict_size(a, w, &ix->dict);
  if (rc) return rc;
  const size_t N = M->rows;
  ix->rows = N;
  ix->hash = (uint64_t*)malloc(N * sizeof(uint64_t));
  ix->freq = (uint32_t*)malloc(N * sizeof(uint32_t));
  ix->offsets = (size_t*)calloc(ix->dict + 1, sizeof(size_t));
  ix->positions = (size_t*)malloc(N * sizeof(size_t));
  ix->cand = (size_t*)malloc(N * sizeof(size_t));
#pragma omp parallel for schedule(static)
  for (ptrdiff_t i = 0; i < (ptrdiff_t)N; ++i) {
    double seg[64];
    double* p = paa_out ? paa_out + (size_t)i * w : seg;
    if (!paa_out && w > 64) p = (double*)malloc(w * sizeof(double));
    paa_one(M->data + (size_t)i * M->stride, M->n, p, w); /* first n columns only, sax.cpp:97-98 */
    uint64_t h = 0;
    for (size_t k = 0; k < w; ++k) {
      const uint32_t s = symbol_of(a, p[k]);
      if (sax_out) sax_out[(size_t)i * w + k] = s;
      h = h * a + (s - 1);
    }
    ix->hash[i] = h + 1;
    if (!paa_out && w > 64) free(p);
  }
  /* histogram -> offsets (index.cpp:27-47, 85-90) */
  for (size_t i = 0; i < N; ++i) ++ix->offsets[ix->hash[i]]; /* slot h holds count of hash h */
  for (uint64_t h = 1; h <= ix->dict; ++h) ix->offsets[h] += ix->offsets[h - 1];
  /* now offsets[h] = end of bucket h = start of bucket h+1; offsets[h-1] = start of bucket h */
  uint32_t min_freq = UINT32_MAX;
  for (size_t i = 0; i < N; ++i) {
    const uint64_t h = ix->hash[i];
    ix->freq[i] = (uint32_t)(ix->offsets[h] - ix->offsets[h - 1]); /* index.cpp:51-64 */
    if (ix->freq[i] < min_freq) min_freq = ix->freq[i];
  }
  for (size_t i = 0; i < N; ++i)
    if (ix->freq[i] == min_freq) ix->cand[ix->n_cand++] = i + 1; /* index.cpp:66-79 */
  size_t* cursor = (size_t*)malloc((ix->dict + 1) * sizeof(size_t));
  memcpy(cursor, ix->offsets, (ix->dict + 1) * sizeof(size_t));
  for (size_t i = 0; i < N; ++i) ix->positions[cursor[ix->hash[i] - 1]++] = i + 1; /* index.cpp:92-97 */
  free(cursor);
  return ORC_OK;
}

int orc_prepare(const double* series, uint64_t m, uint64_t n, uint64_t word_len, uint64_t alphabet,
                double* rows, double* paa, uint32_t* sax, uint64_t* hashes, uint32_t* freq,
                uint64_t* candidates, uint64_t* n_candidates, uint64_t* bucket_positions) {
  Matrix M = {0};
  int rc = matrix_build(series, m, n, 8, &M);
  if (rc) return rc;
  if (rows)
    for (size_t i = 0; i < M.rows; ++i) memcpy(rows + i * n, M.data + i * M.stride, n * sizeof(double));
  Index ix;
  rc = index_build(&M, word_len, alphabet, paa, sax, &ix);
  if (rc == ORC_OK) {
    for (size_t i = 0; i < M.rows; ++i) {
      if (hashes) hashes[i] = ix.hash[i];
      if (freq) freq[i] = ix.freq[i];
      if (bucket_positions) bucket_positions[i] = ix.positions[i];
    }
    if (n_candidates) *n_candidates = ix.n_cand;
    if (candidates)
      for (size_t c = 0; c < ix.n_cand; ++c) candidates[c] = ix.cand[c];
  }
  index_free(&ix);
  free(M.data);
  return rc;
}

/* ------------------------------------------------------------------ */
/* Search.                                                             */

static size_t gap(size_t a, size_t b) { return a > b ? a - b : b - a; }

/* scan_position (discovery.cpp:41-77): bucket neighbours ascending, then all
 * other-word rows ascending; skip |i-j| < n; the in-row abandon threshold is
 * the running minimum; a completed distance strictly below the best-so-far
 * discards the position; strict `<` for the minimum update.  `bsf` is read
 * through a pointer so parallel callers see raises made by others.      */
static int scan_position(const Matrix* M, const Index* ix, size_t i, const volatile double* bsf,
                         int pruning, double* min_out, Counters* c) {
  const size_t n = M->n;
  const uint64_t hi = ix->hash[i];
  const double* ri = M->data + i * M->stride;
  double mn = INFINITY, d;
  for (size_t s = ix->offsets[hi - 1]; s < ix->offsets[hi]; ++s) {
    const size_t j = ix->positions[s] - 1;
    if (gap(i, j) < n) continue;
    if (dist_ea(ri, M->data + j * M->stride, M->stride, pruning ? mn : INFINITY, 8, &d, c)) continue;
    if (pruning && d < *bsf) return 1;
    if (d < mn) mn = d;
  }
  for (size_t j = 0; j < M->rows; ++j) {
    if (ix->hash[j] == hi || gap(i, j) < n) continue;
    if (dist_ea(ri, M->data + j * M->stride, M->stride, pruning ? mn : INFINITY, 8, &d, c)) continue;
    if (pruning && d < *bsf) return 1;
    if (d < mn) mn = d;
  }
  *min_out = mn;
  return 0;
}

typedef struct {
  double sq;
  size_t pos; /* 1-based, 0 = none */
} Best;

/* Exhaustive nn profile (discovery.cpp:123-173 with the profile kept). */
static void nn_profile(const Matrix* M, int threads, double* nn, uint64_t* calls) {
  uint64_t total = 0;
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads) reduction(+ : total)
  for (ptrdiff_t ii = 0; ii < (ptrdiff_t)M->rows; ++ii) {
    const size_t i = (size_t)ii;
    Counters c = {0, 0};
    double best = INFINITY, d;
    for (size_t j = 0; j < M->rows; ++j) {
      if (gap(i, j) < M->n) continue;
      dist_ea(M->data + i * M->stride, M->data + j * M->stride, M->stride, INFINITY, 8, &d, &c);
      if (d < best) best = d;
    }
    nn[i] = best;
    total += c.calls;
  }
  if (calls) *calls = total;
}

/* One exact search over the rows with allowed[i] != 0, in the reference's
 * two-stage order (Alg. 3 then Alg. 4, discovery.cpp:209-358):
 *   stage 1: the minimum-frequency candidates that are allowed, sequentially;
 *            bucket scan, then the other-word rows split over threads, each
 *            thread abandoning against its own running minimum; a neighbour
 *            below the best-so-far drops the candidate;
 *   stage 2: every other allowed row, dynamically scheduled, scan_position
 *            against the shared best-so-far, raised as rows complete; the
 *            stage winner is (greater distance, then smaller position) and
 *            replaces the stage-1 winner only when strictly greater.
 * engine: 1 = sequential hotsax order (discovery.cpp:175-207), 2 = phidd. */
static Best search_allowed(const Matrix* M, const Index* ix, const char* allowed, int engine,
                           int threads, int chunk, int pruning, Counters* total) {
  const size_t N = M->rows, n = M->n;
  char* is_cand = (char*)calloc(N, 1);
  for (size_t c = 0; c < ix->n_cand; ++c)
    if (allowed[ix->cand[c] - 1]) is_cand[ix->cand[c] - 1] = 1;
  volatile double bsf = 0.0;
  Best best = {0.0, 0};

  if (engine == 1) {
    for (int pass = 0; pass < 2; ++pass) {
      for (size_t i = 0; i < N; ++i) {
        if (!allowed[i] || is_cand[i] != (pass == 0)) continue;
        double mn;
        if (scan_position(M, ix, i, &bsf, pruning, &mn, total) || mn == INFINITY) continue;
        if (mn > best.sq) {
          best.sq = mn;
          best.pos = i + 1;
          bsf = mn;
        }
      }
    }
    free(is_cand);
    return best;
  }

  /* stage 1 */
  for (size_t c = 0; c < ix->n_cand; ++c) {
    const size_t i = ix->cand[c] - 1;
    if (!is_cand[i]) continue;
    const uint64_t hi = ix->hash[i];
    const double* ri = M->data + i * M->stride;
    double bucket_min = INFINITY, d;
    int dropped = 0;
    for (size_t s = ix->offsets[hi - 1]; s < ix->offsets[hi]; ++s) {
      const size_t j = ix->positions[s] - 1;
      if (gap(i, j) < n) continue;
      if (dist_ea(ri, M->data + j * M->stride, M->stride, pruning ? bucket_min : INFINITY, 8, &d, total)) continue;
      if (pruning && d < bsf) {
        dropped = 1;
        break;
      }
      if (d < bucket_min) bucket_min = d;
    }
    if (dropped) continue;
    double stage_min = bucket_min;
    int abort_flag = 0;
    uint64_t calls = 0, abandoned = 0;
#pragma omp parallel num_threads(threads)
    {
      Counters lc = {0, 0};
      double local_min = bucket_min, dd;
#pragma omp for schedule(dynamic, chunk) nowait
      for (ptrdiff_t jj = 0; jj < (ptrdiff_t)N; ++jj) {
        int stop;
#pragma omp atomic read
        stop = abort_flag;
        if (pruning && stop) continue;
        const size_t j = (size_t)jj;
        if (ix->hash[j] == hi || gap(i, j) < n) continue;
        if (dist_ea(ri, M->data + j * M->stride, M->stride, pruning ? local_min : INFINITY, 8, &dd, &lc)) continue;
        if (pruning && dd < bsf) {
#pragma omp atomic write
          abort_flag = 1;
          continue;
        }
        if (dd < local_min) local_min = dd;
      }
#pragma omp critical(orc_stage1)
      {
        if (local_min < stage_min) stage_min = local_min;
        calls += lc.calls;
        abandoned += lc.abandoned;
      }
    }
    total->calls += calls;
    total->abandoned += abandoned;
    if (abort_flag) continue;
    if (stage_min < INFINITY && stage_min > best.sq) { /* SharedBest::try_raise, discovery.hpp:43-52 */
      best.sq = stage_min;
      best.pos = i + 1;
      bsf = stage_min;
    }
  }

  /* stage 2 */
  Best s2 = {-1.0, 0};
  uint64_t calls = 0, abandoned = 0;
#pragma omp parallel num_threads(threads)
  {
    Counters lc = {0, 0};
    Best lb = {-1.0, 0};
#pragma omp for schedule(dynamic, chunk) nowait
    for (ptrdiff_t ii = 0; ii < (ptrdiff_t)N; ++ii) {
      const size_t i = (size_t)ii;
      if (!allowed[i] || is_cand[i]) continue;
      double mn;
      if (scan_position(M, ix, i, &bsf, pruning, &mn, &lc) || mn == INFINITY) continue;
      if (pruning) {
#pragma omp critical(orc_raise)
        if (mn > bsf) bsf = mn;
      }
      if (mn > lb.sq || (mn == lb.sq && i + 1 < lb.pos)) {
        lb.sq = mn;
        lb.pos = i + 1;
      }
    }
#pragma omp critical(orc_stage2)
    {
      if (lb.pos != 0 && (lb.sq > s2.sq || (lb.sq == s2.sq && lb.pos < s2.pos))) s2 = lb;
      calls += lc.calls;
      abandoned += lc.abandoned;
    }
  }
  total->calls += calls;
  total->abandoned += abandoned;
  if (s2.pos != 0 && s2.sq > best.sq) best = s2;
  free(is_cand);
  return best;
}

static int check_run(uint64_t m, uint64_t n, uint64_t w, uint64_t a, int threads, int chunk) {
  /* check_config order (pipeline.cpp:21-49) */
  if (n < 1 || n > m) return fail(ORC_PARAMETER, "n=%llu must satisfy 1 <= n <= m=%llu", n, m);
  if (w < 1 || w > n) return fail(ORC_PARAMETER, "word_len=%llu must satisfy 1 <= word_len <= n=%llu", w, n);
  if (threads < 1) return fail(ORC_PARAMETER, "threads must be >= 1, got %llu", (unsigned long long)threads, 0);
  if (chunk < 1) return fail(ORC_PARAMETER, "chunk must be >= 1, got %llu", (unsigned long long)chunk, 0);
  int rc = check_alphabet(a);
  if (rc) return rc;
  uint64_t dict;
  rc = dict_size(a, w, &dict);
  if (rc) return rc;
  const uint64_t rows = m - n + 1;
  if (rows < n + 1) /* require_feasible, discovery.cpp:114-121 */
    return fail(ORC_INFEASIBLE, "no subsequence has a non-self match: N=%llu <= n=%llu (need m >= 2n)", rows, n);
  return ORC_OK;
}

/* Top-k by exclusion zones: discord r is the arg-max of the
 * nn distance over rows at least n away from every earlier discord.  k = 1
 * is the reference's single search.  finalize (discovery.cpp:88-98): nothing
 * beat 0 -> position 1, distance 0; sqrt taken once.                     */
int orc_topk(const double* series, uint64_t m, uint64_t n, uint64_t word_len, uint64_t alphabet,
             int k, int threads, int chunk, uint64_t* positions, double* distances,
             uint64_t* calls, uint64_t* abandoned, double* prep_s, double* search_s) {
  int rc = validate(series, m);
  if (rc) return rc;
  rc = check_run(m, n, word_len, alphabet, threads, chunk);
  if (rc) return rc;
  if (k < 1) return fail(ORC_PARAMETER, "k must be >= 1", 0, 0);
  const double t0 = now_s();
  Matrix M = {0};
  rc = matrix_build(series, m, n, 8, &M);
  if (rc) return rc;
  Index ix;
  rc = index_build(&M, word_len, alphabet, NULL, NULL, &ix);
  if (rc) {
    free(M.data);
    return rc;
  }
  if (prep_s) *prep_s = now_s() - t0;
  const double t1 = now_s();
  char* allowed = (char*)malloc(M.rows);
  memset(allowed, 1, M.rows);
  Counters total = {0, 0};
  for (int r = 0; r < k; ++r) {
    Best b = search_allowed(&M, &ix, allowed, 2, threads, chunk, 1, &total);
    if (b.pos == 0) {
      b.pos = 1;
      b.sq = 0.0;
    }
    positions[r] = b.pos;
    distances[r] = sqrt(b.sq);
    const size_t p0 = b.pos - 1;
    const size_t lo = p0 >= n - 1 ? p0 - (n - 1) : 0;
    const size_t hi = p0 + (n - 1) < M.rows - 1 ? p0 + (n - 1) : M.rows - 1;
    for (size_t i = lo; i <= hi; ++i) allowed[i] = 0;
  }
  if (search_s) *search_s = now_s() - t1;
  if (calls) *calls = total.calls;
  if (abandoned) *abandoned = total.abandoned;
  free(allowed);
  index_free(&ix);
  free(M.data);
  return ORC_OK;
}

/* run_discovery (pipeline.cpp:53-93).  engine: 0 brute, 1 hotsax, 2 phidd. */
int orc_run_discovery(const double* series, uint64_t m, uint64_t n, uint64_t word_len,
                      uint64_t alphabet, int engine, int threads, int chunk, int disable_pruning,
                      uint64_t* position, double* distance, uint64_t* calls, uint64_t* abandoned,
                      double* prep_s, double* search_s) {
  int rc = validate(series, m);
  if (rc) return rc;
  rc = check_run(m, n, word_len, alphabet, threads, chunk);
  if (rc) return rc;
  const double t0 = now_s();
  Matrix M = {0};
  rc = matrix_build(series, m, n, 8, &M);
  if (rc) return rc;
  Index ix;
  rc = index_build(&M, word_len, alphabet, NULL, NULL, &ix);
  if (rc) {
    free(M.data);
    return rc;
  }
  if (prep_s) *prep_s = now_s() - t0;
  const double t1 = now_s();
  Counters total = {0, 0};
  Best b = {0.0, 0};
  if (engine == 0) {
    double* nn = (double*)malloc(M.rows * sizeof(double));
    nn_profile(&M, threads, nn, &total.calls);
    b.sq = -1.0;
    for (size_t i = 0; i < M.rows; ++i) { /* ties -> smallest position, discovery.cpp:158-165 */
      if (nn[i] == INFINITY) continue;
      if (nn[i] > b.sq) {
        b.sq = nn[i];
        b.pos = i + 1;
      }
    }
    free(nn);
  } else {
    char* allowed = (char*)malloc(M.rows);
    memset(allowed, 1, M.rows);
    b = search_allowed(&M, &ix, allowed, engine, threads, chunk, !disable_pruning, &total);
    free(allowed);
    if (b.pos == 0) {
      b.pos = 1;
      b.sq = 0.0;
    }
  }
  if (search_s) *search_s = now_s() - t1;
  if (position) *position = b.pos;
  if (distance) *distance = sqrt(b.sq);
  if (calls) *calls = total.calls;
  if (abandoned) *abandoned = total.abandoned;
  index_free(&ix);
  free(M.data);
  return ORC_OK;
}

int orc_nn_profile(const double* series, uint64_t m, uint64_t n, int threads, double* nn_sq) {
  Matrix M = {0};
  int rc = matrix_build(series, m, n, 8, &M);
  if (rc) return rc;
  nn_profile(&M, threads, nn_sq, NULL);
  free(M.data);
  return ORC_OK;
}
