/*
 * sb_oracle.c -- CPU restatement of the reference HyperBall hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity *checker*: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product path (paper_2604_08374_b200/, libsieveball_cuda.so)
 * never links, imports or calls anything under oracle/.
 *
 * Parity pinning: every register-level primitive below restates a shipped
 * reference function (hll.hpp / hll.cpp / kernels_scalar.cpp / leb128.hpp).
 * The loop (init / iterate_once / run) restates the SPEC contract and the
 * paper's Algorithm 1, because the reference ships no hyperball.cpp.  The
 * restatement is pinned against the compiled reference primitives
 * (oracle/_ref/libsbref.so, built from /root/reference/proj/src by
 * oracle/Makefile) and against the committed golden vectors in tests/golden/.
 *
 * Build: see oracle/Makefile (-O2 -ffp-contract=off, no FMA: the reference's
 * hll.cpp is compiled without -mfma, CMakeLists.txt:33-39).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SBO_OK 0
#define SBO_EINVAL 1   /* std::invalid_argument in the reference */
#define SBO_ERUNTIME 2 /* std::runtime_error in the reference */

/* ---- hll.hpp:13-20  SplitMix64 finalizer (no golden-gamma increment) ---- */
uint64_t sbo_splitmix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ULL;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBULL;
  x ^= x >> 31;
  return x;
}

/* ---- hll.cpp:9-19  HllParams ---- */
int sbo_params(unsigned p, uint32_t* m_out, double* alpha_out, uint32_t* row_bytes_out) {
  if (p < 4 || p > 16) return SBO_EINVAL;
  const uint32_t m = (uint32_t)1 << p;
  double alpha;
  switch (m) {
    case 16: alpha = 0.673; break;
    case 32: alpha = 0.697; break;
    case 64: alpha = 0.709; break;
    default: alpha = 0.7213 / (1.0 + 1.079 / m); break;
  }
  if (m_out) *m_out = m;
  if (alpha_out) *alpha_out = alpha;
  if (row_bytes_out) *row_bytes_out = m / 2;
  return SBO_OK;
}

/* ---- hll.hpp:50-60  packed register access (low nibble = even register) ---- */
static inline uint8_t get_reg(const uint8_t* row, uint32_t j) {
  const uint8_t b = row[j >> 1];
  return (j & 1) ? (uint8_t)(b >> 4) : (uint8_t)(b & 0x0F);
}
static inline void set_reg(uint8_t* row, uint32_t j, uint8_t value) {
  uint8_t* b = &row[j >> 1];
  if (j & 1)
    *b = (uint8_t)((*b & 0x0F) | (value << 4));
  else
    *b = (uint8_t)((*b & 0xF0) | (value & 0x0F));
}

/* ---- hll.cpp:21-29  hll_insert ---- */
void sbo_insert(uint8_t* row, uint64_t element, unsigned p) {
  const uint64_t h = sbo_splitmix64(element);
  const uint32_t index = (uint32_t)(h >> (64 - p));
  const uint64_t w = h << p;
  const unsigned lz = w == 0 ? (64 - p) : (unsigned)__builtin_clzll(w);
  const unsigned r = lz + 1 < 15u ? lz + 1 : 15u;
  const uint8_t rho = (uint8_t)r;
  if (get_reg(row, index) < rho) set_reg(row, index, rho);
}

/* ---- kernels_scalar.cpp:7-14  nibble_max_scalar ---- */
void sbo_nibble_max(uint8_t* dst, const uint8_t* src, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    const uint8_t a = dst[i], b = src[i];
    const uint8_t lo = (a & 0x0F) > (b & 0x0F) ? (a & 0x0F) : (b & 0x0F);
    const uint8_t hi = (a & 0xF0) > (b & 0xF0) ? (a & 0xF0) : (b & 0xF0);
    dst[i] = (uint8_t)(hi | lo);
  }
}

/* ---- kernels_scalar.cpp:16-25  harmonic_scalar ---- */
void sbo_harmonic(const uint8_t* regs, size_t n, uint64_t* numerator, uint32_t* zeros) {
  uint64_t num = 0;
  uint32_t z = 0;
  for (size_t i = 0; i < n; ++i) {
    const uint8_t lo = regs[i] & 0x0F;
    const uint8_t hi = regs[i] >> 4;
    num += ((uint64_t)1 << (15 - lo)) + ((uint64_t)1 << (15 - hi));
    z += (lo == 0) + (hi == 0);
  }
  *numerator = num;
  *zeros = z;
}

/* ---- hll.cpp:31-37  hll_estimate_from_sum (classic alpha_m + linear counting) ---- */
double sbo_estimate_from_sum(uint64_t numerator, uint32_t zeros, unsigned p) {
  uint32_t mm;
  double alpha;
  sbo_params(p, &mm, &alpha, NULL);
  const double m = (double)mm;
  const double harmonic = (double)numerator / 32768.0;
  const double raw = alpha * m * m / harmonic;
  if (raw <= 2.5 * m && zeros > 0) return m * log(m / (double)zeros);
  return raw;
}

/* ---- hll.cpp:39-41  hll_estimate ---- */
double sbo_estimate(const uint8_t* row, unsigned p) {
  uint64_t num;
  uint32_t z;
  sbo_harmonic(row, (size_t)1 << (p - 1), &num, &z);
  return sbo_estimate_from_sum(num, z, p);
}

/* ---- leb128.hpp:12-18  leb128_encode; returns bytes written (<= 10) ---- */
size_t sbo_leb128_encode(uint64_t value, uint8_t* out) {
  size_t k = 0;
  while (value >= 0x80) {
    out[k++] = (uint8_t)value | 0x80;
    value >>= 7;
  }
  out[k++] = (uint8_t)value;
  return k;
}

/* ---- leb128.hpp:28-39  leb128_decode (truncation / >10 bytes -> runtime error) ---- */
int sbo_leb128_decode(const uint8_t* bytes, size_t len, size_t* pos, uint64_t* out) {
  uint64_t value = 0;
  unsigned shift = 0;
  for (unsigned i = 0; i < 10; ++i) {
    if (*pos >= len) return SBO_ERUNTIME; /* "leb128: truncated varint" */
    const uint8_t b = bytes[(*pos)++];
    value |= (uint64_t)(b & 0x7F) << shift;
    if ((b & 0x80) == 0) {
      *out = value;
      return SBO_OK;
    }
    shift += 7;
  }
  return SBO_ERUNTIME; /* "leb128: varint exceeds 10 bytes" */
}

/* ---- HyperBall (Algorithm 1) ---- */

/* Init: zero both planes' rows, insert ORIGINAL id into its own
 * counter, estimate c_0. */
int sbo_hb_init(uint64_t n, const uint32_t* orig_id, unsigned p, uint8_t* cur, double* c0) {
  uint32_t rb;
  if (sbo_params(p, NULL, NULL, &rb) != SBO_OK) return SBO_EINVAL;
  if (n == 0) return SBO_EINVAL; /* "graph empty" */
  memset(cur, 0, (size_t)n * rb);
  for (uint64_t v = 0; v < n; ++v) {
    sbo_insert(cur + v * rb, orig_id ? (uint64_t)orig_id[v] : v, p);
    c0[v] = sbo_estimate(cur + v * rb, p);
  }
  return SBO_OK;
}

typedef struct {
  uint64_t n;
  const uint64_t* offsets;
  const uint32_t* degrees;
  const uint8_t* stream;
  uint64_t stream_len;
  unsigned p;
  uint32_t t;
  const uint8_t* cur;
  uint8_t* next;
  const double* c_prev;
  double* c_cur;
  double* sum_d;
  double* sum_d2;
  uint64_t begin, end;
  double max_inc;
  int status;
} sbo_work;

/* iterate_once body over [begin, end):
 *   next[v] <- cur[v]; next[v] <- max(next[v], cur[w]) for w in N(v);
 *   c_t[v] = estimate(next[v]); sum_d += t*(c_t - c_{t-1}); sum_d2 += t^2*(...). */
static void* sbo_iterate_range(void* arg) {
  sbo_work* w = (sbo_work*)arg;
  uint32_t rb;
  sbo_params(w->p, NULL, NULL, &rb);
  const double td = (double)w->t;
  const double tt = (double)((uint64_t)w->t * w->t);
  double mx = -INFINITY;
  for (uint64_t v = w->begin; v < w->end; ++v) {
    uint8_t* dst = w->next + v * rb;
    memcpy(dst, w->cur + v * rb, rb);
    /* NeighborCursor: first id absolute, then deltas */
    size_t pos = (size_t)w->offsets[v];
    const size_t row_end = (size_t)w->offsets[v + 1];
    uint64_t prev = 0;
    for (uint32_t k = 0; k < w->degrees[v]; ++k) {
      uint64_t x;
      if (sbo_leb128_decode(w->stream, row_end, &pos, &x) != SBO_OK) {
        w->status = SBO_ERUNTIME;
        return NULL;
      }
      const uint64_t id = k == 0 ? x : prev + x;
      if (id >= w->n || (k > 0 && x == 0)) {
        w->status = SBO_ERUNTIME;
        return NULL;
      }
      prev = id;
      sbo_nibble_max(dst, w->cur + id * rb, rb); /* hll_union_into, hll.hpp:74-76 */
    }
    const double c = sbo_estimate(dst, w->p);
    const double delta = c - w->c_prev[v];
    w->c_cur[v] = c;
    w->sum_d[v] = w->sum_d[v] + td * delta;
    w->sum_d2[v] = w->sum_d2[v] + tt * delta;
    if (delta > mx) mx = delta;
  }
  w->max_inc = mx;
  return NULL;
}

/* iterate_once over nodes [v0, v1) with a static contiguous partition over
 * `threads` workers (parallel.hpp:20-47 semantics: chunk = ceil(n/threads)).
 * Returns max_v (c_t - c_{t-1}) over [v0, v1) in *max_inc (-inf if empty). */
int sbo_hb_iterate(uint64_t n, const uint64_t* offsets, const uint32_t* degrees,
                   const uint8_t* stream, uint64_t stream_len, unsigned p, uint32_t t,
                   const uint8_t* cur, uint8_t* next, const double* c_prev, double* c_cur,
                   double* sum_d, double* sum_d2, uint64_t v0, uint64_t v1, unsigned threads,
                   double* max_inc) {
  if (sbo_params(p, NULL, NULL, NULL) != SBO_OK) return SBO_EINVAL;
  if (v1 > n || v0 > v1) return SBO_EINVAL;
  const uint64_t cnt = v1 - v0;
  if (threads == 0) threads = 1;
  if ((uint64_t)threads > (cnt ? cnt : 1)) threads = (unsigned)(cnt ? cnt : 1);
  sbo_work* ws = (sbo_work*)calloc(threads, sizeof(sbo_work));
  pthread_t* th = (pthread_t*)calloc(threads, sizeof(pthread_t));
  const uint64_t chunk = (cnt + threads - 1) / threads;
  for (unsigned i = 0; i < threads; ++i) {
    sbo_work* w = &ws[i];
    w->n = n; w->offsets = offsets; w->degrees = degrees; w->stream = stream;
    w->stream_len = stream_len; w->p = p; w->t = t; w->cur = cur; w->next = next;
    w->c_prev = c_prev; w->c_cur = c_cur; w->sum_d = sum_d; w->sum_d2 = sum_d2;
    uint64_t b = v0 + (uint64_t)i * chunk;
    if (b > v1) b = v1;
    uint64_t e = b + chunk;
    if (e > v1) e = v1;
    w->begin = b; w->end = e; w->max_inc = -INFINITY; w->status = SBO_OK;
  }
  if (threads == 1) {
    sbo_iterate_range(&ws[0]);
  } else {
    for (unsigned i = 0; i < threads; ++i) pthread_create(&th[i], NULL, sbo_iterate_range, &ws[i]);
    for (unsigned i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  }
  int st = SBO_OK;
  double mx = -INFINITY;
  for (unsigned i = 0; i < threads; ++i) {
    if (ws[i].status != SBO_OK && st == SBO_OK) st = ws[i].status;
    if (ws[i].max_inc > mx) mx = ws[i].max_inc;
  }
  free(ws);
  free(th);
  if (max_inc) *max_inc = mx;
  return st;
}

/* check_convergence: inclusive 0.5 threshold. */
int sbo_check_convergence(double max_increase) { return max_increase <= 0.5; }

/* run (PAPER.md:418-433 loop order):
 *   union -> estimate -> accumulate -> if max<=0.5 break -> if t==d stop -> swap.
 * depth_limit 0 = unlimited.  On return `final_regs` holds the registers after
 * the last executed iteration, c_final the matching estimates.
 * iterations = number of iterate_once calls executed. */
int sbo_hb_run(uint64_t n, const uint64_t* offsets, const uint32_t* degrees,
               const uint8_t* stream, uint64_t stream_len, const uint32_t* orig_id, unsigned p,
               uint32_t depth_limit, unsigned threads, uint8_t* final_regs, double* c_final,
               double* sum_d, double* sum_d2, uint32_t* iterations, int* converged) {
  uint32_t rb;
  if (sbo_params(p, NULL, NULL, &rb) != SBO_OK) return SBO_EINVAL;
  if (n == 0) return SBO_EINVAL;
  uint8_t* a = (uint8_t*)malloc((size_t)n * rb);
  uint8_t* b = (uint8_t*)malloc((size_t)n * rb);
  double* ca = (double*)malloc(n * sizeof(double));
  double* cb = (double*)malloc(n * sizeof(double));
  if (!a || !b || !ca || !cb) { free(a); free(b); free(ca); free(cb); return SBO_ERUNTIME; }
  memset(sum_d, 0, n * sizeof(double));
  memset(sum_d2, 0, n * sizeof(double));
  int st = sbo_hb_init(n, orig_id, p, a, ca);
  uint8_t *cur = a, *nxt = b;
  double *cp = ca, *cc = cb;
  uint32_t t = 0;
  int conv = 0;
  while (st == SBO_OK) {
    ++t;
    double mx;
    st = sbo_hb_iterate(n, offsets, degrees, stream, stream_len, p, t, cur, nxt, cp, cc, sum_d,
                        sum_d2, 0, n, threads, &mx);
    if (st != SBO_OK) break;
    if (sbo_check_convergence(mx)) { conv = 1; break; }
    if (depth_limit != 0 && t == depth_limit) break;
    uint8_t* tp = cur; cur = nxt; nxt = tp;
    double* tc = cp; cp = cc; cc = tc;
  }
  if (st == SBO_OK) {
    memcpy(final_regs, nxt, (size_t)n * rb);
    memcpy(c_final, cc, n * sizeof(double));
    *iterations = t;
    *converged = conv;
  }
  free(a); free(b); free(ca); free(cb);
  return st;
}

/* ---- metrics ---- */
/* D_k diamond value. */
static double diamond(double k) {
  return 2.0 * (k * (log2((k + 2.0) / 3.0) - 1.0) + 1.0) / ((k - 1.0) * (k - 2.0));
}

void sbo_metrics(uint64_t n, const double* sum_d, const double* sum_d2, const uint32_t* nv,
                 const uint32_t* deg, double* md, double* ihh, double* tekl, double* pv,
                 double* m1, double* m2) {
  for (uint64_t v = 0; v < n; ++v) {
    const double N = (double)nv[v];
    double MD = NAN, IHH = NAN, TK = NAN, PV = NAN, M1 = NAN, M2 = NAN;
    if (nv[v] >= 2) {
      MD = sum_d[v] / (N - 1.0);
      TK = log2((MD + 2.0) / 3.0);
      M1 = MD * (double)deg[v];
      M2 = sum_d2[v] / (N - 1.0);
      if (nv[v] >= 3) {
        const double RA = 2.0 * (MD - 1.0) / (N - 2.0);
        const double pvv = 1.0 - RA;
        PV = pvv > 0.0 ? (pvv < 1.0 ? pvv : 1.0) : 0.0; /* in [0, 1] */
        if (MD > 1.0) {                                 /* pre MD > 1, else NaN */
          const double RRA = RA / diamond(N);
          IHH = 1.0 / RRA;
        }
      }
    }
    md[v] = MD; ihh[v] = IHH; tekl[v] = TK; pv[v] = PV; m1[v] = M1; m2[v] = M2;
  }
}

/* ---- local metrics, brute force over decoded rows ----
 * control = sum_{w in N(v)} 1/deg(w) as the correctly rounded sum (exact
 * 128-bit fixed point with 96 fractional bits, then one rounding; the SPEC
 * does not pin a summation order, so the order-independent exact sum is the
 * contract); controllability = deg / |N2(v)| (N2 = nodes within 2 hops, v
 * excluded); clustering = edges among N(v) (directed) / (deg (deg - 1)). */
static int decode_rows(uint64_t n, const uint64_t* offsets, const uint32_t* degrees,
                       const uint8_t* stream, uint64_t** off_out, uint32_t** ids_out) {
  uint64_t* off = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  uint64_t tot = 0;
  for (uint64_t v = 0; v < n; ++v) { off[v] = tot; tot += degrees[v]; }
  off[n] = tot;
  uint32_t* ids = (uint32_t*)malloc((tot ? tot : 1) * sizeof(uint32_t));
  for (uint64_t v = 0; v < n; ++v) {
    size_t pos = (size_t)offsets[v];
    uint64_t prev = 0;
    for (uint32_t k = 0; k < degrees[v]; ++k) {
      uint64_t x;
      if (sbo_leb128_decode(stream, (size_t)offsets[v + 1], &pos, &x) != SBO_OK) {
        free(off); free(ids);
        return SBO_ERUNTIME;
      }
      prev = k == 0 ? x : prev + x;
      ids[off[v] + k] = (uint32_t)prev;
    }
  }
  *off_out = off;
  *ids_out = ids;
  return SBO_OK;
}

double sbo_exact_sum_recip(const uint32_t* degs, uint64_t count) {
  unsigned __int128 acc = 0;
  for (uint64_t k = 0; k < count; ++k) {
    if (degs[k] == 0) return INFINITY;
    int e;
    const double m = frexp(1.0 / (double)degs[k], &e); /* 1/d = m 2^e, m in [0.5, 1) */
    const uint64_t mant = (uint64_t)ldexp(m, 53);      /* exact, < 2^53 */
    acc += (unsigned __int128)mant << (96 + e - 53);
  }
  return ldexp((double)acc, -96); /* one round-to-nearest-even conversion */
}

int sbo_local_metrics(uint64_t n, const uint64_t* offsets, const uint32_t* degrees,
                      const uint8_t* stream, uint64_t v0, uint64_t v1, double* control,
                      double* controllability, double* clustering, uint64_t* among,
                      uint64_t* n2) {
  uint64_t* off;
  uint32_t* ids;
  if (v0 > v1 || v1 > n) return SBO_EINVAL;
  if (decode_rows(n, offsets, degrees, stream, &off, &ids) != SBO_OK) return SBO_ERUNTIME;
  uint64_t* mark = (uint64_t*)calloc(n ? n : 1, sizeof(uint64_t));
  uint64_t* mark2 = (uint64_t*)calloc(n ? n : 1, sizeof(uint64_t));
  uint32_t* dg = (uint32_t*)malloc((off[n] ? off[n] : 1) * sizeof(uint32_t));
  for (uint64_t v = v0; v < v1; ++v) {
    const uint64_t i = v - v0, stamp = v + 1;
    const uint32_t deg = degrees[v];
    const uint32_t* nv = ids + off[v];
    for (uint32_t k = 0; k < deg; ++k) dg[k] = degrees[nv[k]];
    control[i] = sbo_exact_sum_recip(dg, deg);
    for (uint32_t k = 0; k < deg; ++k) mark[nv[k]] = stamp;
    uint64_t tri = 0, cnt = 0;
    for (uint32_t k = 0; k < deg; ++k) {
      const uint32_t w = nv[k];
      if (w != v && mark2[w] != stamp) { mark2[w] = stamp; ++cnt; }
      for (uint64_t q = off[w]; q < off[w + 1]; ++q) {
        const uint32_t u = ids[q];
        if (mark[u] == stamp) ++tri;
        if (u != v && mark2[u] != stamp) { mark2[u] = stamp; ++cnt; }
      }
    }
    controllability[i] = cnt ? (double)deg / (double)cnt : NAN;
    clustering[i] = deg >= 2 ? (double)tri / ((double)deg * (double)(deg - 1)) : NAN;
    if (among) among[i] = tri;
    if (n2) n2[i] = cnt;
  }
  free(mark); free(mark2); free(dg); free(off); free(ids);
  return SBO_OK;
}

/* ---- exact BFS oracle: per-root BFS over the decoded rows ----
 * For every root v: sum_d[v] = sum of depths of every node reached within
 * depth_limit (0 = unlimited), sum_d2 = sum of squared depths, reach[v] = nodes
 * reached incl. v, hist[v * cap + t] = nodes at depth t (t < cap; deeper
 * levels are dropped and *max_depth tells the caller).  O(N |E|). */
int sbo_exact_bfs(uint64_t n, const uint64_t* offsets, const uint32_t* degrees,
                  const uint8_t* stream, uint32_t depth_limit, uint64_t* sum_d,
                  uint64_t* sum_d2, uint32_t* reach, uint32_t* hist, uint32_t cap,
                  uint32_t* max_depth) {
  uint64_t* off;
  uint32_t* ids;
  if (decode_rows(n, offsets, degrees, stream, &off, &ids) != SBO_OK) return SBO_ERUNTIME;
  uint32_t* dist = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  uint32_t* queue = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  uint32_t dmax = 0;
  if (hist) memset(hist, 0, n * cap * sizeof(uint32_t));
  for (uint64_t v = 0; v < n; ++v) {
    for (uint64_t u = 0; u < n; ++u) dist[u] = UINT32_MAX;
    uint64_t head = 0, tail = 0, s1 = 0, s2 = 0;
    dist[v] = 0;
    queue[tail++] = (uint32_t)v;
    while (head < tail) {
      const uint32_t u = queue[head++];
      const uint32_t du = dist[u];
      if (du) {
        s1 += du;
        s2 += (uint64_t)du * du;
        if (hist && du < cap) hist[v * cap + du] += 1;
        if (du > dmax) dmax = du;
      }
      if (depth_limit && du == depth_limit) continue;
      for (uint64_t q = off[u]; q < off[u + 1]; ++q) {
        const uint32_t w = ids[q];
        if (dist[w] == UINT32_MAX) {
          dist[w] = du + 1;
          queue[tail++] = w;
        }
      }
    }
    sum_d[v] = s1;
    sum_d2[v] = s2;
    reach[v] = (uint32_t)tail;
  }
  if (max_depth) *max_depth = dmax;
  free(dist); free(queue); free(off); free(ids);
  return SBO_OK;
}

/* Depth entropy (SPEC.md:531-535 exact mode): H = -sum_t p_t log2 p_t,
 * p_t = n_t / sum_{t>=1} n_t, increasing t; NaN when nothing is reached. */
void sbo_depth_entropy(uint64_t n, const uint32_t* hist, uint32_t cap, double* entropy) {
  for (uint64_t v = 0; v < n; ++v) {
    const uint32_t* h = hist + v * cap;
    uint64_t tot = 0;
    for (uint32_t t = 1; t < cap; ++t) tot += h[t];
    if (!tot) { entropy[v] = NAN; continue; }
    double H = 0.0;
    for (uint32_t t = 1; t < cap; ++t) {
      if (!h[t]) continue;
      const double p = (double)h[t] / (double)tot;
      H -= p * log2(p);
    }
    entropy[v] = H + 0.0;
  }
}
