/*
 * sb_synth.c -- the synthetic visibility-grid input of the benchmarks,
 * restated for the oracle (TEST INFRASTRUCTURE ONLY, see sb_oracle.c).
 *
 * The reference arm of bench.py (`--impl reference`) must not map the product
 * library at all, not even to build its input, so the CPU side generates the
 * same graph itself: bench.CONFIGS -> sbo_synth_grid -> (offsets, degrees,
 * stream) in the reference CSR layout (rows per SPEC.md
 * :202-210).  tests/test_oracle_synth.py checks it byte for byte against the
 * product generator (sb_csr_synth_grid) and against the stream hashes
 * committed in tests/golden/scale_reference.json.
 *
 * The graph:
 *   - obstacles: n_rects rectangles, sides in [rect_min, rect_max], drawn from
 *     a splitmix64 stream with the golden-gamma increment (h, w, row, col per
 *     rectangle, clipped to the grid);
 *   - nodes: the free cells in raster order;
 *   - edges: v -> w iff w != v is free, within the radius (radius2 = 0:
 *     unlimited; per grid row the column span is isqrt(radius2 - dr^2)) and
 *     the open segment between the cell centres crosses no obstacle cell's
 *     interior (exact integer walk; an exact corner crossing steps diagonally);
 *     an obstacle-free bounding box means visible;
 *   - rows list neighbours in raster order: first id absolute, then deltas,
 *     unsigned LEB128 (leb128.hpp:12-18).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint32_t rows, cols;
  uint64_t radius2;
  int64_t reach;         /* rows reachable above / below */
  uint8_t* blocked;      /* rows x cols */
  uint32_t* pref;        /* (rows+1) x (cols+1) blocked-cell prefix counts */
  uint32_t* node_of;     /* cell -> node id or UINT32_MAX */
  uint32_t* cell_of;     /* node -> cell */
  uint64_t n;
} synth_grid;

static uint64_t gamma_next(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static uint64_t int_sqrt(uint64_t v) { /* floor(sqrt(v)), bitwise */
  uint64_t r = 0, bit = 1ULL << 62;
  while (bit > v) bit >>= 2;
  while (bit) {
    if (v >= r + bit) {
      v -= r + bit;
      r = (r >> 1) + bit;
    } else {
      r >>= 1;
    }
    bit >>= 2;
  }
  return r;
}

static int box_clear(const synth_grid* g, int64_t ra, int64_t ca, int64_t rb, int64_t cb) {
  const int64_t r0 = ra < rb ? ra : rb, r1 = ra < rb ? rb : ra;
  const int64_t c0 = ca < cb ? ca : cb, c1 = ca < cb ? cb : ca;
  const uint64_t W = (uint64_t)g->cols + 1;
  const uint32_t* P = g->pref;
  const uint32_t s = P[(r1 + 1) * W + (c1 + 1)] - P[r0 * W + (c1 + 1)] - P[(r1 + 1) * W + c0] + P[r0 * W + c0];
  return s == 0;
}

/* Cells whose interior the open segment between the centres crosses: in units
 * where cell centres sit at odd coordinates, the segment leaves column-step k
 * at x = 2k+1 and row-step j at y = 2j+1; compare (2k+1)*|dy| with
 * (2j+1)*|dx| to know which boundary comes first (equal: a corner). */
static int sees(const synth_grid* g, int64_t r1, int64_t c1, int64_t r2, int64_t c2) {
  if (box_clear(g, r1, c1, r2, c2)) return 1;
  const int64_t dx = c2 - c1, dy = r2 - r1;
  const int64_t ax = dx < 0 ? -dx : dx, ay = dy < 0 ? -dy : dy;
  const int64_t sx = dx > 0 ? 1 : -1, sy = dy > 0 ? 1 : -1;
  int64_t x = c1, y = r1, k = 0, j = 0;
  while (k < ax || j < ay) {
    if (k < ax && j < ay) {
      const int64_t a = (2 * k + 1) * ay, b = (2 * j + 1) * ax;
      if (a <= b) { x += sx; ++k; }
      if (a >= b) { y += sy; ++j; }
    } else if (k < ax) {
      x += sx; ++k;
    } else {
      y += sy; ++j;
    }
    if (x == c2 && y == r2) return 1;
    if (g->blocked[(uint64_t)y * g->cols + (uint64_t)x]) return 0;
  }
  return 1;
}

static uint32_t varint_len(uint64_t v) {
  uint32_t k = 1;
  for (; v >= 0x80; v >>= 7) ++k;
  return k;
}

typedef struct {
  const synth_grid* g;
  uint32_t* degrees;
  uint64_t* row_bytes;     /* count pass */
  const uint64_t* offsets; /* write pass */
  uint8_t* stream;
  uint64_t v0, v1;
} synth_job;

/* One row: count (stream == NULL) or encode it. */
static void synth_row(const synth_grid* g, uint64_t v, uint32_t* deg_out, uint64_t* bytes_out, uint8_t* out) {
  const uint32_t cell = g->cell_of[v];
  const int64_t r = cell / g->cols, c = cell % g->cols;
  const int64_t rlo = r - g->reach < 0 ? 0 : r - g->reach;
  const int64_t rhi = r + g->reach > (int64_t)g->rows - 1 ? (int64_t)g->rows - 1 : r + g->reach;
  uint32_t deg = 0;
  uint64_t bytes = 0;
  int64_t prev = -1;
  for (int64_t r2 = rlo; r2 <= rhi; ++r2) {
    int64_t span = g->cols;
    if (g->radius2) span = (int64_t)int_sqrt(g->radius2 - (uint64_t)((r2 - r) * (r2 - r)));
    const int64_t clo = c - span < 0 ? 0 : c - span;
    const int64_t chi = c + span > (int64_t)g->cols - 1 ? (int64_t)g->cols - 1 : c + span;
    for (int64_t c2 = clo; c2 <= chi; ++c2) {
      if (r2 == r && c2 == c) continue;
      const uint32_t w = g->node_of[(uint64_t)r2 * g->cols + (uint64_t)c2];
      if (w == UINT32_MAX || !sees(g, r, c, r2, c2)) continue;
      uint64_t d = prev < 0 ? w : (uint64_t)(w - prev);
      prev = w;
      ++deg;
      if (out) {
        while (d >= 0x80) { *out++ = (uint8_t)(d | 0x80); d >>= 7; }
        *out++ = (uint8_t)d;
      } else {
        bytes += varint_len(d);
      }
    }
  }
  if (deg_out) *deg_out = deg;
  if (bytes_out) *bytes_out = bytes;
}

static void* synth_worker(void* arg) {
  synth_job* j = (synth_job*)arg;
  for (uint64_t v = j->v0; v < j->v1; ++v) {
    if (j->stream)
      synth_row(j->g, v, NULL, NULL, j->stream + j->offsets[v]);
    else
      synth_row(j->g, v, &j->degrees[v], &j->row_bytes[v], NULL);
  }
  return NULL;
}

static void run_jobs(synth_job* proto, uint64_t n, unsigned threads) {
  if (threads < 1) threads = 1;
  /* many small blocks, handed out round-robin: rows near obstacles cost more */
  const uint64_t blocks = (uint64_t)threads * 16;
  pthread_t* tid = (pthread_t*)calloc(threads, sizeof(pthread_t));
  synth_job* jobs = (synth_job*)calloc(blocks, sizeof(synth_job));
  for (uint64_t b = 0; b < blocks; ++b) {
    jobs[b] = *proto;
    jobs[b].v0 = n * b / blocks;
    jobs[b].v1 = n * (b + 1) / blocks;
  }
  for (uint64_t round = 0; round < 16; ++round) {
    for (unsigned t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, synth_worker, &jobs[round * threads + t]);
    for (unsigned t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  }
  free(jobs);
  free(tid);
}

/* Returns 0 and malloc'ed arrays (release with sbo_synth_free); 1 on bad
 * arguments, 2 if the grid has no free cell, 3 on allocation failure.
 * The stream gets 256 zero bytes of padding past *stream_len. */
int sbo_synth_grid(uint32_t rows, uint32_t cols, uint32_t n_rects, uint32_t rect_min, uint32_t rect_max,
                   uint64_t seed, uint64_t radius2, unsigned threads, uint64_t* n_out, uint64_t** offsets_out,
                   uint32_t** degrees_out, uint8_t** stream_out, uint64_t* stream_len_out) {
  if (!rows || !cols || (n_rects && (!rect_min || rect_max < rect_min))) return 1;
  synth_grid g;
  memset(&g, 0, sizeof(g));
  g.rows = rows;
  g.cols = cols;
  g.radius2 = radius2;
  const uint64_t cells = (uint64_t)rows * cols;
  g.blocked = (uint8_t*)calloc(cells, 1);
  g.pref = (uint32_t*)calloc(((uint64_t)rows + 1) * ((uint64_t)cols + 1), 4);
  g.node_of = (uint32_t*)malloc(cells * 4);
  g.cell_of = (uint32_t*)malloc(cells * 4);
  if (!g.blocked || !g.pref || !g.node_of || !g.cell_of) return 3;
  uint64_t s = seed;
  for (uint32_t i = 0; i < n_rects; ++i) {
    const uint32_t h = rect_min + (uint32_t)(gamma_next(&s) % (rect_max - rect_min + 1));
    const uint32_t w = rect_min + (uint32_t)(gamma_next(&s) % (rect_max - rect_min + 1));
    const uint32_t r0 = (uint32_t)(gamma_next(&s) % rows);
    const uint32_t c0 = (uint32_t)(gamma_next(&s) % cols);
    for (uint64_t r = r0; r < (uint64_t)r0 + h && r < rows; ++r)
      memset(g.blocked + r * cols + c0, 1, (c0 + w < cols ? c0 + w : cols) - c0);
  }
  const uint64_t W = (uint64_t)cols + 1;
  for (uint64_t r = 0; r < rows; ++r) {
    uint32_t run = 0; /* blocked cells in row r up to column c */
    for (uint64_t c = 0; c < cols; ++c) {
      run += g.blocked[r * cols + c];
      g.pref[(r + 1) * W + c + 1] = g.pref[r * W + c + 1] + run;
    }
  }
  for (uint64_t cell = 0; cell < cells; ++cell) {
    g.node_of[cell] = g.blocked[cell] ? UINT32_MAX : (uint32_t)g.n;
    if (!g.blocked[cell]) g.cell_of[g.n++] = (uint32_t)cell;
  }
  if (g.n == 0) return 2;
  g.reach = radius2 ? (int64_t)int_sqrt(radius2) : (int64_t)(rows > cols ? rows : cols);
  const uint64_t n = g.n;
  uint32_t* degrees = (uint32_t*)malloc(n * 4);
  uint64_t* rb = (uint64_t*)malloc(n * 8);
  uint64_t* offsets = (uint64_t*)malloc((n + 1) * 8);
  if (!degrees || !rb || !offsets) return 3;
  synth_job proto = {&g, degrees, rb, NULL, NULL, 0, 0};
  run_jobs(&proto, n, threads);
  offsets[0] = 0;
  for (uint64_t v = 0; v < n; ++v) offsets[v + 1] = offsets[v] + rb[v];
  free(rb);
  uint8_t* stream = (uint8_t*)malloc(offsets[n] + 256);
  if (!stream) return 3;
  memset(stream + offsets[n], 0, 256);
  synth_job wp = {&g, NULL, NULL, offsets, stream, 0, 0};
  run_jobs(&wp, n, threads);
  free(g.blocked);
  free(g.pref);
  free(g.node_of);
  free(g.cell_of);
  *n_out = n;
  *offsets_out = offsets;
  *degrees_out = degrees;
  *stream_out = stream;
  *stream_len_out = offsets[n];
  return 0;
}

void sbo_synth_free(void* p) { free(p); }
