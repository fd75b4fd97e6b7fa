// sb_csr.cpp -- host CompressedCsr: synthetic grid visibility graphs,
// delta-LEB128 encoding, UnionFind components
// (union_find.hpp semantics), VGACSR03 persistence,
// Hilbert renumbering and edge-balanced partitions.
#include <cuda_runtime_api.h>
#include <zlib.h>
#include <sys/stat.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sieveball_cuda.h"

#include "sb_error.h"

using sb::fail;
#define cfail sb::fail

struct sb_csr {
  uint64_t n = 0, edges = 0, stream_len = 0;
  std::vector<uint64_t> offsets;
  std::vector<uint32_t> degrees;
  uint8_t* stream = nullptr;  // stream_len + 64 zero padding
  std::vector<uint32_t> comp_id, comp_sizes, cell_of_node, hilbert_inverse;
  double ox = 0, oy = 0, spacing = 1;
  uint32_t rows = 0, cols = 0;
  bool pinned = false;
  ~sb_csr() {
    if (pinned) cudaHostUnregister(stream);
    free(stream);
  }
  bool alloc_stream(uint64_t len) {
    free(stream);
    stream = static_cast<uint8_t*>(malloc(len + 64));
    if (!stream) return false;
    memset(stream + len, 0, 64);
    stream_len = len;
    return true;
  }
};

namespace {

// Disjoint-set forest with path halving and union by rank; dense component
// ids by ascending first-node occurrence (union_find.hpp:10-52 semantics).
class UF {
 public:
  explicit UF(uint32_t n) : parent_(n), rank_(n, 0) { std::iota(parent_.begin(), parent_.end(), 0u); }
  uint32_t find(uint32_t v) {
    while (parent_[v] != v) {
      parent_[v] = parent_[parent_[v]];
      v = parent_[v];
    }
    return v;
  }
  void unite(uint32_t a, uint32_t b) {
    uint32_t ra = find(a), rb = find(b);
    if (ra == rb) return;
    if (rank_[ra] < rank_[rb]) std::swap(ra, rb);
    parent_[rb] = ra;
    if (rank_[ra] == rank_[rb]) ++rank_[ra];
  }
  void finalize(std::vector<uint32_t>& id, std::vector<uint32_t>& sizes) {
    const uint32_t n = static_cast<uint32_t>(parent_.size());
    id.assign(n, UINT32_MAX);
    sizes.clear();
    std::vector<uint32_t> root_to_id(n, UINT32_MAX);
    for (uint32_t v = 0; v < n; ++v) {
      const uint32_t r = find(v);
      if (root_to_id[r] == UINT32_MAX) {
        root_to_id[r] = static_cast<uint32_t>(sizes.size());
        sizes.push_back(0);
      }
      id[v] = root_to_id[r];
      ++sizes[id[v]];
    }
  }

 private:
  std::vector<uint32_t> parent_;
  std::vector<uint8_t> rank_;
};

inline int leb_len(uint64_t v) {
  int k = 1;
  while (v >= 0x80) {
    v >>= 7;
    ++k;
  }
  return k;
}
inline uint8_t* leb_put(uint8_t* o, uint64_t v) {  // leb128.hpp:12-18
  while (v >= 0x80) {
    *o++ = static_cast<uint8_t>(v) | 0x80;
    v >>= 7;
  }
  *o++ = static_cast<uint8_t>(v);
  return o;
}
inline bool leb_get(const uint8_t* s, uint64_t end, uint64_t& pos, uint64_t& out) {  // leb128.hpp:28-39
  uint64_t v = 0;
  unsigned shift = 0;
  for (int i = 0; i < 10; ++i) {
    if (pos >= end) return false;
    const uint8_t b = s[pos++];
    v |= uint64_t(b & 0x7f) << shift;
    if (!(b & 0x80)) {
      out = v;
      return true;
    }
    shift += 7;
  }
  return false;
}

template <class F>
void parallel_for(uint64_t n, unsigned threads, F&& fn) {
  if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
  if (threads <= 1 || n < 2) {
    fn(0, n);
    return;
  }
  std::atomic<uint64_t> next{0};
  const uint64_t blk = std::max<uint64_t>(64, n / (threads * 64ull) + 1);
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (;;) {
        const uint64_t b = next.fetch_add(blk);
        if (b >= n) break;
        fn(b, std::min(n, b + blk));
      }
    });
  for (auto& t : pool) t.join();
}

struct Grid {
  uint32_t rows, cols;
  std::vector<uint8_t> blocked;
  std::vector<uint32_t> pref;  // (rows+1) x (cols+1) prefix count of blocked cells
  bool any_blocked(int r0, int c0, int r1, int c1) const {  // inclusive box
    if (r0 > r1) std::swap(r0, r1);
    if (c0 > c1) std::swap(c0, c1);
    const uint64_t W = cols + 1;
    const uint32_t s = pref[(r1 + 1) * W + (c1 + 1)] - pref[r0 * W + (c1 + 1)] -
                       pref[(r1 + 1) * W + c0] + pref[r0 * W + c0];
    return s != 0;
  }
  bool is_blocked(int r, int c) const { return blocked[static_cast<uint64_t>(r) * cols + c] != 0; }
  // Exact integer line of sight between the centres of (r1,c1) and (r2,c2):
  // walk the cells whose interior the open segment crosses; at an exact
  // corner crossing step diagonally (the two side cells' interiors are not
  // touched).  Symmetric by construction.
  bool visible(int r1, int c1, int r2, int c2) const {
    if (!any_blocked(r1, c1, r2, c2)) return true;
    const int dx = c2 - c1, dy = r2 - r1;
    const int sx = dx > 0 ? 1 : -1, sy = dy > 0 ? 1 : -1;
    const int64_t ax = std::abs(dx), ay = std::abs(dy);
    int x = c1, y = r1;
    int64_t k = 0, j = 0;
    while (k < ax || j < ay) {
      if (k < ax && j < ay) {
        const int64_t lhs = (2 * k + 1) * ay, rhs = (2 * j + 1) * ax;
        if (lhs < rhs) {
          x += sx;
          ++k;
        } else if (lhs > rhs) {
          y += sy;
          ++j;
        } else {
          x += sx;
          y += sy;
          ++k;
          ++j;
        }
      } else if (k < ax) {
        x += sx;
        ++k;
      } else {
        y += sy;
        ++j;
      }
      if (x == c2 && y == r2) break;
      if (is_blocked(y, x)) return false;
    }
    return true;
  }
};

inline uint64_t isqrt64(uint64_t v) {
  uint64_t r = static_cast<uint64_t>(std::sqrt(static_cast<double>(v)));
  while (r * r > v) --r;
  while ((r + 1) * (r + 1) <= v) ++r;
  return r;
}

inline uint64_t rng_next(uint64_t& s) {  // splitmix64 stream (golden-gamma increment)
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Seeded rectangular obstacles (side in [rect_min, rect_max] cells).
void draw_rects(uint32_t rows, uint32_t cols, uint32_t n_rects, uint32_t rect_min, uint32_t rect_max, uint64_t seed,
                uint8_t* blocked) {
  uint64_t s = seed;
  for (uint32_t i = 0; i < n_rects; ++i) {
    const uint32_t h = rect_min + static_cast<uint32_t>(rng_next(s) % (rect_max - rect_min + 1));
    const uint32_t w = rect_min + static_cast<uint32_t>(rng_next(s) % (rect_max - rect_min + 1));
    const uint32_t r0 = static_cast<uint32_t>(rng_next(s) % rows);
    const uint32_t c0 = static_cast<uint32_t>(rng_next(s) % cols);
    for (uint32_t r = r0; r < std::min(rows, r0 + h); ++r)
      for (uint32_t c = c0; c < std::min(cols, c0 + w); ++c) blocked[static_cast<uint64_t>(r) * cols + c] = 1;
  }
}

void compute_components_from_stream(sb_csr* c) {
  UF uf(static_cast<uint32_t>(c->n));
  for (uint64_t v = 0; v < c->n; ++v) {
    uint64_t pos = c->offsets[v], prev = 0, x = 0;
    for (uint32_t k = 0; k < c->degrees[v]; ++k) {
      if (!leb_get(c->stream, c->offsets[v + 1], pos, x)) break;
      const uint64_t id = k ? prev + x : x;
      prev = id;
      if (id < c->n) uf.unite(static_cast<uint32_t>(v), static_cast<uint32_t>(id));
    }
  }
  uf.finalize(c->comp_id, c->comp_sizes);
}

}  // namespace

extern "C" {

int sb_grid_synth_mask(uint32_t rows, uint32_t cols, uint32_t n_rects, uint32_t rect_min, uint32_t rect_max,
                       uint64_t seed, uint8_t* blocked) {
  if (!blocked) return cfail(SB_EINVAL, "NULL mask");
  if (rows == 0 || cols == 0) return cfail(SB_EINVAL, "grid: rows and cols must be >= 1");
  if (n_rects && (rect_min == 0 || rect_max < rect_min)) return cfail(SB_EINVAL, "grid: bad rectangle size range");
  memset(blocked, 0, static_cast<uint64_t>(rows) * cols);
  draw_rects(rows, cols, n_rects, rect_min, rect_max, seed, blocked);
  return SB_OK;
}

int sb_csr_synth_grid(uint32_t rows, uint32_t cols, uint32_t n_rects, uint32_t rect_min,
                      uint32_t rect_max, uint64_t seed, uint64_t radius2, unsigned threads,
                      sb_csr** out) {
  if (!out) return cfail(SB_EINVAL, "out is NULL");
  *out = nullptr;
  if (rows == 0 || cols == 0) return cfail(SB_EINVAL, "grid: rows and cols must be >= 1");
  if (n_rects && (rect_min == 0 || rect_max < rect_min)) return cfail(SB_EINVAL, "grid: bad rectangle size range");
  Grid G;
  G.rows = rows;
  G.cols = cols;
  G.blocked.assign(static_cast<uint64_t>(rows) * cols, 0);
  draw_rects(rows, cols, n_rects, rect_min, rect_max, seed, G.blocked.data());
  const uint64_t W = cols + 1;
  G.pref.assign(static_cast<uint64_t>(rows + 1) * W, 0);
  for (uint32_t r = 0; r < rows; ++r)
    for (uint32_t c = 0; c < cols; ++c)
      G.pref[(r + 1) * W + (c + 1)] = G.blocked[static_cast<uint64_t>(r) * cols + c] + G.pref[r * W + (c + 1)] +
                                     G.pref[(r + 1) * W + c] - G.pref[r * W + c];
  auto c = std::make_unique<sb_csr>();
  c->rows = rows;
  c->cols = cols;
  std::vector<uint32_t> node_of_cell(static_cast<uint64_t>(rows) * cols, UINT32_MAX);
  for (uint64_t cell = 0; cell < node_of_cell.size(); ++cell)
    if (!G.blocked[cell]) {
      node_of_cell[cell] = static_cast<uint32_t>(c->cell_of_node.size());
      c->cell_of_node.push_back(static_cast<uint32_t>(cell));
    }
  const uint64_t n = c->cell_of_node.size();
  if (n == 0) return cfail(SB_ERUNTIME, "grid: zero active cells");
  c->n = n;
  const int64_t R = radius2 ? static_cast<int64_t>(isqrt64(radius2)) : std::max(rows, cols);
  // Visit v's visible cells in raster (= id) order.
  auto for_each_nb = [&](uint64_t v, auto&& emit) {
    const uint32_t cell = c->cell_of_node[v];
    const int r = static_cast<int>(cell / cols), cc = static_cast<int>(cell % cols);
    const int r_lo = static_cast<int>(std::max<int64_t>(0, r - R));
    const int r_hi = static_cast<int>(std::min<int64_t>(rows - 1, r + R));
    for (int r2 = r_lo; r2 <= r_hi; ++r2) {
      const int64_t dr = r2 - r;
      int64_t span = cols;
      if (radius2) span = static_cast<int64_t>(isqrt64(radius2 - static_cast<uint64_t>(dr * dr)));
      const int c_lo = static_cast<int>(std::max<int64_t>(0, cc - span));
      const int c_hi = static_cast<int>(std::min<int64_t>(cols - 1, cc + span));
      const uint64_t rowbase = static_cast<uint64_t>(r2) * cols;
      for (int c2 = c_lo; c2 <= c_hi; ++c2) {
        if (r2 == r && c2 == cc) continue;
        const uint32_t w = node_of_cell[rowbase + c2];
        if (w == UINT32_MAX) continue;
        if (G.visible(r, cc, r2, c2)) emit(w);
      }
    }
  };
  c->degrees.assign(n, 0);
  std::vector<uint64_t> rowbytes(n, 0);
  parallel_for(n, threads, [&](uint64_t b, uint64_t e) {
    for (uint64_t v = b; v < e; ++v) {
      uint32_t deg = 0;
      uint64_t bytes = 0;
      int64_t prev = -1;
      for_each_nb(v, [&](uint32_t w) {
        bytes += leb_len(prev < 0 ? w : static_cast<uint64_t>(w - prev));
        prev = w;
        ++deg;
      });
      c->degrees[v] = deg;
      rowbytes[v] = bytes;
    }
  });
  c->offsets.assign(n + 1, 0);
  for (uint64_t v = 0; v < n; ++v) {
    c->offsets[v + 1] = c->offsets[v] + rowbytes[v];
    c->edges += c->degrees[v];
  }
  if (!c->alloc_stream(c->offsets[n])) return cfail(SB_ENOMEM, "grid: cannot allocate %llu stream bytes", (unsigned long long)c->offsets[n]);
  parallel_for(n, threads, [&](uint64_t b, uint64_t e) {
    for (uint64_t v = b; v < e; ++v) {
      uint8_t* o = c->stream + c->offsets[v];
      int64_t prev = -1;
      for_each_nb(v, [&](uint32_t w) {
        o = leb_put(o, prev < 0 ? w : static_cast<uint64_t>(w - prev));
        prev = w;
      });
    }
  });
  // Components: every line of sight crosses a chain of free cells that are
  // edge- or corner-adjacent and mutually visible, so uniting the visibility
  // edges between 8-adjacent cells yields the same partition as uniting all
  // edges (what build_from_source does).
  UF uf(static_cast<uint32_t>(n));
  for (uint64_t v = 0; v < n; ++v) {
    const uint32_t cell = c->cell_of_node[v];
    const int r = static_cast<int>(cell / cols), cc = static_cast<int>(cell % cols);
    for (int dr = -1; dr <= 1; ++dr)
      for (int dc = -1; dc <= 1; ++dc) {
        if (!dr && !dc) continue;
        const int r2 = r + dr, c2 = cc + dc;
        if (r2 < 0 || c2 < 0 || r2 >= static_cast<int>(rows) || c2 >= static_cast<int>(cols)) continue;
        if (radius2 && static_cast<uint64_t>(dr * dr + dc * dc) > radius2) continue;
        const uint32_t w = node_of_cell[static_cast<uint64_t>(r2) * cols + c2];
        if (w == UINT32_MAX) continue;
        if (G.visible(r, cc, r2, c2)) uf.unite(static_cast<uint32_t>(v), w);
      }
  }
  uf.finalize(c->comp_id, c->comp_sizes);
  *out = c.release();
  return SB_OK;
}

}  // extern "C"

namespace {
// Delta-LEB128 encoding of a sorted adjacency, rows in
// parallel (byte counts -> offsets -> writes).  Components are left to the caller.
int encode_adjacency(sb_csr* c, uint64_t n, const uint64_t* adj_offsets, const uint32_t* adj_ids, unsigned threads) {
  c->n = n;
  c->degrees.assign(n, 0);
  c->offsets.assign(n + 1, 0);
  std::vector<uint64_t> rowbytes(n, 0);
  std::atomic<uint64_t> bad{UINT64_MAX};
  std::atomic<int> kind{0};
  parallel_for(n, threads, [&](uint64_t b, uint64_t e) {
    for (uint64_t v = b; v < e; ++v) {
      uint64_t bytes = 0;
      for (uint64_t k = adj_offsets[v]; k < adj_offsets[v + 1]; ++k) {
        const uint32_t w = adj_ids[k];
        int err = w >= n ? 1 : (k > adj_offsets[v] && w <= adj_ids[k - 1]) ? 2 : 0;
        if (err) {
          uint64_t cur = bad.load();
          while (v < cur && !bad.compare_exchange_weak(cur, v)) {
          }
          if (bad.load() == v) kind = err;
          break;
        }
        bytes += leb_len(k > adj_offsets[v] ? w - adj_ids[k - 1] : w);
      }
      c->degrees[v] = static_cast<uint32_t>(adj_offsets[v + 1] - adj_offsets[v]);
      rowbytes[v] = bytes;
    }
  });
  if (bad.load() != UINT64_MAX)
    return cfail(SB_EINVAL, kind == 1 ? "cgraph: neighbour id out of range at node %llu"
                                      : "cgraph: non-increasing neighbour list at node %llu",
                 (unsigned long long)bad.load());
  c->edges = 0;
  for (uint64_t v = 0; v < n; ++v) {
    c->offsets[v + 1] = c->offsets[v] + rowbytes[v];
    c->edges += c->degrees[v];
  }
  if (!c->alloc_stream(c->offsets[n])) return cfail(SB_ENOMEM, "cannot allocate stream");
  parallel_for(n, threads, [&](uint64_t b, uint64_t e) {
    for (uint64_t v = b; v < e; ++v) {
      uint8_t* o = c->stream + c->offsets[v];
      for (uint64_t k = adj_offsets[v]; k < adj_offsets[v + 1]; ++k)
        o = leb_put(o, k > adj_offsets[v] ? adj_ids[k] - adj_ids[k - 1] : adj_ids[k]);
    }
  });
  return SB_OK;
}
}  // namespace

extern "C" {

int sb_csr_from_adjacency(uint64_t n, const uint64_t* adj_offsets, const uint32_t* adj_ids, sb_csr** out) {
  if (!out) return cfail(SB_EINVAL, "out is NULL");
  *out = nullptr;
  if (n == 0) return cfail(SB_EINVAL, "graph empty");
  if (n > 0xffffffffull) return cfail(SB_EINVAL, "too many nodes");
  auto c = std::make_unique<sb_csr>();
  const int rc = encode_adjacency(c.get(), n, adj_offsets, adj_ids, 0);
  if (rc) return rc;
  UF uf(static_cast<uint32_t>(n));
  for (uint64_t v = 0; v < n; ++v)
    for (uint64_t k = adj_offsets[v]; k < adj_offsets[v + 1]; ++k) uf.unite(static_cast<uint32_t>(v), adj_ids[k]);
  uf.finalize(c->comp_id, c->comp_sizes);
  *out = c.release();
  return SB_OK;
}

int sb_csr_from_arrays(uint64_t n, const uint64_t* offsets, const uint32_t* degrees, const uint8_t* stream,
                       uint64_t stream_len, sb_csr** out) {
  if (!out) return cfail(SB_EINVAL, "out is NULL");
  *out = nullptr;
  if (n == 0) return cfail(SB_EINVAL, "graph empty");
  if (offsets[n] != stream_len) return cfail(SB_ERUNTIME, "cgraph: offsets[N] != stream length");
  auto c = std::make_unique<sb_csr>();
  c->n = n;
  c->offsets.assign(offsets, offsets + n + 1);
  c->degrees.assign(degrees, degrees + n);
  for (uint64_t v = 0; v < n; ++v) c->edges += degrees[v];
  if (!c->alloc_stream(stream_len)) return cfail(SB_ENOMEM, "cannot allocate stream");
  if (stream_len) memcpy(c->stream, stream, stream_len);
  compute_components_from_stream(c.get());
  *out = c.release();
  return SB_OK;
}

int sb_csr_describe(const sb_csr* c, sb_csr_desc* d) {
  if (!c || !d) return cfail(SB_EINVAL, "NULL argument");
  d->n = c->n;
  d->edges = c->edges;
  d->stream_len = c->stream_len;
  d->offsets = c->offsets.data();
  d->degrees = c->degrees.data();
  d->stream = c->stream;
  d->n_components = c->comp_sizes.size();
  d->component_id = c->comp_id.data();
  d->component_sizes = c->comp_sizes.data();
  d->cell_of_node = c->cell_of_node.empty() ? nullptr : c->cell_of_node.data();
  d->hilbert_inverse = c->hilbert_inverse.empty() ? nullptr : c->hilbert_inverse.data();
  d->origin_x = c->ox;
  d->origin_y = c->oy;
  d->spacing = c->spacing;
  d->rows = c->rows;
  d->cols = c->cols;
  return SB_OK;
}

int sb_csr_neighbors(const sb_csr* c, uint64_t v, uint32_t* ids) {
  if (!c || v >= c->n) return cfail(SB_EINVAL, "bad node");
  uint64_t pos = c->offsets[v], prev = 0, x = 0;
  for (uint32_t k = 0; k < c->degrees[v]; ++k) {
    if (!leb_get(c->stream, c->offsets[v + 1], pos, x)) return cfail(SB_ERUNTIME, "leb128: truncated varint");
    const uint64_t id = k ? prev + x : x;
    if (id >= c->n || (k && x == 0)) return cfail(SB_ERUNTIME, "cgraph: bad neighbour id");
    ids[k] = static_cast<uint32_t>(id);
    prev = id;
  }
  return SB_OK;
}

void sb_csr_destroy(sb_csr* c) { delete c; }

int sb_csr_pin(sb_csr* c, int pin) {
  if (!c) return cfail(SB_EINVAL, "NULL csr");
  if ((pin != 0) == c->pinned) return SB_OK;
  cudaError_t e = pin ? cudaHostRegister(c->stream, c->stream_len + 64, cudaHostRegisterDefault)
                      : cudaHostUnregister(c->stream);
  if (e != cudaSuccess) return cfail(SB_ECUDA, "cudaHostRegister: %s", cudaGetErrorString(e));
  c->pinned = pin != 0;
  return SB_OK;
}

// ---------------------------------------------------------------- Hilbert
// Canonical d2xy/xy2d (reflected Gray-code construction), order = ceil(log2(max(rows, cols))).
static uint64_t hilbert_xy2d(uint64_t order_n, uint64_t x, uint64_t y) {
  uint64_t d = 0;
  for (uint64_t s = order_n / 2; s > 0; s /= 2) {
    const uint64_t rx = (x & s) > 0, ry = (y & s) > 0;
    d += s * s * ((3 * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) {
        x = s - 1 - x;
        y = s - 1 - y;
      }
      std::swap(x, y);
    }
  }
  return d;
}

int sb_csr_hilbert_reorder(const sb_csr* c, sb_csr** out) {
  if (!c || !out) return cfail(SB_EINVAL, "NULL argument");
  *out = nullptr;
  if (c->cell_of_node.empty() || c->cols == 0) return cfail(SB_EINVAL, "hilbert: grid metadata absent");
  uint64_t side = 1;
  while (side < std::max(c->rows, c->cols)) side *= 2;
  const uint64_t n = c->n;
  std::vector<std::pair<uint64_t, uint32_t>> key(n);
  for (uint64_t v = 0; v < n; ++v) {
    const uint32_t cell = c->cell_of_node[v];
    key[v] = {hilbert_xy2d(side, cell % c->cols, cell / c->cols), static_cast<uint32_t>(v)};
  }
  std::sort(key.begin(), key.end());
  std::vector<uint32_t> inv(n), fwd(n);  // inv[new] = old, fwd[old] = new
  for (uint64_t i = 0; i < n; ++i) {
    inv[i] = key[i].second;
    fwd[key[i].second] = static_cast<uint32_t>(i);
  }
  std::vector<uint64_t> aoff(n + 1, 0);
  for (uint64_t i = 0; i < n; ++i) aoff[i + 1] = aoff[i] + c->degrees[inv[i]];
  std::vector<uint32_t> ids(aoff[n]);
  std::atomic<int> failed{0};
  parallel_for(n, 0, [&](uint64_t b, uint64_t e) {
    for (uint64_t i = b; i < e; ++i) {
      const uint32_t old = inv[i];
      uint32_t* row = ids.data() + aoff[i];
      if (sb_csr_neighbors(c, old, row) != SB_OK) {
        failed = 1;
        return;
      }
      for (uint64_t k = 0; k < c->degrees[old]; ++k) row[k] = fwd[row[k]];
      std::sort(row, row + c->degrees[old]);
    }
  });
  if (failed) return cfail(SB_ERUNTIME, "hilbert: malformed row in the source graph");
  auto rr = std::make_unique<sb_csr>();
  const int rc = encode_adjacency(rr.get(), n, aoff.data(), ids.data(), 0);
  if (rc) return rc;
  // Renumbering permutes components; dense ids by first occurrence in the new order.
  std::vector<uint32_t> remap(c->comp_sizes.size(), UINT32_MAX);
  rr->comp_id.resize(n);
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t oc = c->comp_id[inv[i]];
    if (remap[oc] == UINT32_MAX) {
      remap[oc] = static_cast<uint32_t>(rr->comp_sizes.size());
      rr->comp_sizes.push_back(c->comp_sizes[oc]);
    }
    rr->comp_id[i] = remap[oc];
  }
  sb_csr* r = rr.release();
  r->rows = c->rows;
  r->cols = c->cols;
  r->ox = c->ox;
  r->oy = c->oy;
  r->spacing = c->spacing;
  r->cell_of_node.resize(n);
  r->hilbert_inverse.resize(n);
  for (uint64_t i = 0; i < n; ++i) {
    r->cell_of_node[i] = c->cell_of_node[inv[i]];
    // original id (hash key); composes with an earlier reorder
    r->hilbert_inverse[i] = c->hilbert_inverse.empty() ? inv[i] : c->hilbert_inverse[inv[i]];
  }
  *out = r;
  return SB_OK;
}

// ---------------------------------------------------------------- VGACSR03
// Layout, little-endian: "VGACSR03" | u32 flags (bit0 hilbert) |
// u64 N | u64 |E| | u64 stream_len | f64 ox, oy, spacing | u32 rows, cols |
// u32 cell[N] | u64 offsets[N+1] | u32 degrees[N] | stream | u32 C |
// u32 comp_id[N] | u32 sizes[C] | [u32 hilbert_inverse[N]] | u32 CRC32(all before).
namespace {
struct Writer {
  FILE* f;
  uLong crc = crc32(0L, Z_NULL, 0);
  bool ok = true;
  void put(const void* p, uint64_t bytes) {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    while (bytes && ok) {
      const uint64_t k = std::min<uint64_t>(bytes, 1ull << 30);
      crc = crc32_z(crc, b, k);
      ok = fwrite(b, 1, k, f) == k;
      b += k;
      bytes -= k;
    }
  }
};
struct Reader {
  FILE* f;
  uLong crc = crc32(0L, Z_NULL, 0);
  bool get(void* p, uint64_t bytes) {
    uint8_t* b = static_cast<uint8_t*>(p);
    while (bytes) {
      const uint64_t k = std::min<uint64_t>(bytes, 1ull << 30);
      if (fread(b, 1, k, f) != k) return false;
      crc = crc32_z(crc, b, k);
      b += k;
      bytes -= k;
    }
    return true;
  }
};
}  // namespace

int sb_vgacsr_save(const sb_csr* c, const char* path) {
  if (!c || !path) return cfail(SB_EINVAL, "NULL argument");
  FILE* f = fopen(path, "wb");
  if (!f) return cfail(SB_ERUNTIME, "vgacsr: cannot open %s for writing", path);
  Writer w{f};
  const uint32_t flags = c->hilbert_inverse.empty() ? 0u : 1u;
  w.put("VGACSR03", 8);
  w.put(&flags, 4);
  w.put(&c->n, 8);
  w.put(&c->edges, 8);
  w.put(&c->stream_len, 8);
  w.put(&c->ox, 8);
  w.put(&c->oy, 8);
  w.put(&c->spacing, 8);
  w.put(&c->rows, 4);
  w.put(&c->cols, 4);
  std::vector<uint32_t> cells = c->cell_of_node;
  if (cells.empty()) {
    cells.resize(c->n);
    std::iota(cells.begin(), cells.end(), 0u);
  }
  w.put(cells.data(), c->n * 4);
  w.put(c->offsets.data(), (c->n + 1) * 8);
  w.put(c->degrees.data(), c->n * 4);
  w.put(c->stream, c->stream_len);
  const uint32_t C = static_cast<uint32_t>(c->comp_sizes.size());
  w.put(&C, 4);
  w.put(c->comp_id.data(), c->n * 4);
  w.put(c->comp_sizes.data(), static_cast<uint64_t>(C) * 4);
  if (flags & 1u) w.put(c->hilbert_inverse.data(), c->n * 4);
  const uint32_t crc = static_cast<uint32_t>(w.crc);
  const bool ok = w.ok && fwrite(&crc, 1, 4, f) == 4;
  if (fclose(f) != 0 || !ok) return cfail(SB_ERUNTIME, "vgacsr: write failed for %s", path);
  return SB_OK;
}

static int vgacsr_load(const char* path, sb_csr** out);

int sb_vgacsr_load(const char* path, sb_csr** out) {
  if (!path || !out) return cfail(SB_EINVAL, "NULL argument");
  *out = nullptr;
  try {  // no C++ exception crosses the C ABI
    return vgacsr_load(path, out);
  } catch (const std::bad_alloc&) {
    return cfail(SB_ENOMEM, "vgacsr: out of host memory loading %s", path);
  } catch (const std::exception& e) {
    return cfail(SB_ERUNTIME, "vgacsr: %s", e.what());
  }
}

static int vgacsr_load(const char* path, sb_csr** out) {
  FILE* f = fopen(path, "rb");
  if (!f) return cfail(SB_ERUNTIME, "vgacsr: cannot open %s", path);
  std::unique_ptr<FILE, int (*)(FILE*)> guard(f, fclose);
  Reader r{f};
  char magic[8];
  if (!r.get(magic, 8)) return cfail(SB_ERUNTIME, "vgacsr: truncated header");
  if (memcmp(magic, "VGACSR", 6) != 0) return cfail(SB_ERUNTIME, "vgacsr: bad magic");
  if (memcmp(magic + 6, "03", 2) != 0) return cfail(SB_ERUNTIME, "vgacsr: unsupported version %.2s", magic + 6);
  auto c = std::make_unique<sb_csr>();
  uint32_t flags = 0;
  uint64_t slen = 0;
  if (!r.get(&flags, 4) || !r.get(&c->n, 8) || !r.get(&c->edges, 8) || !r.get(&slen, 8) ||
      !r.get(&c->ox, 8) || !r.get(&c->oy, 8) || !r.get(&c->spacing, 8) || !r.get(&c->rows, 4) ||
      !r.get(&c->cols, 4))
    return cfail(SB_ERUNTIME, "vgacsr: truncated header");
  if (c->n == 0 || c->n > 0xffffffffull) return cfail(SB_ERUNTIME, "vgacsr: bad node count");
  const uint64_t n = c->n;
  // The header's sizes must fit the file before anything is allocated from them
  // (a truncated or corrupt header must not drive multi-GB allocations).
  struct stat sbuf;
  if (fstat(fileno(f), &sbuf) != 0) return cfail(SB_ERUNTIME, "vgacsr: cannot stat %s", path);
  const uint64_t fsize = static_cast<uint64_t>(sbuf.st_size);
  constexpr uint64_t kHeader = 8 + 4 + 8 + 8 + 8 + 24 + 8;
  const uint64_t fixed = kHeader + n * 4 + (n + 1) * 8 + n * 4 + 4 + n * 4 + ((flags & 1u) ? n * 4 : 0) + 4;
  if (slen > fsize || fixed > fsize || fixed + slen > fsize)
    return cfail(SB_ERUNTIME, "vgacsr: truncated file (header sizes exceed its %llu bytes)", (unsigned long long)fsize);
  const uint64_t comp_bytes = fsize - fixed - slen;  // what is left for sizes[C]
  c->cell_of_node.resize(n);
  c->offsets.resize(n + 1);
  c->degrees.resize(n);
  if (!r.get(c->cell_of_node.data(), n * 4) || !r.get(c->offsets.data(), (n + 1) * 8) ||
      !r.get(c->degrees.data(), n * 4))
    return cfail(SB_ERUNTIME, "vgacsr: truncated arrays");
  if (c->offsets[n] != slen) return cfail(SB_ERUNTIME, "vgacsr: offsets[N] != stream length");
  if (!c->alloc_stream(slen)) return cfail(SB_ENOMEM, "vgacsr: cannot allocate stream");
  if (!r.get(c->stream, slen)) return cfail(SB_ERUNTIME, "vgacsr: truncated stream");
  uint32_t C = 0;
  if (!r.get(&C, 4)) return cfail(SB_ERUNTIME, "vgacsr: truncated components");
  if (static_cast<uint64_t>(C) * 4 != comp_bytes || C == 0 || C > n)
    return cfail(SB_ERUNTIME, "vgacsr: component count %u does not match the file", C);
  c->comp_id.resize(n);
  c->comp_sizes.resize(C);
  if (!r.get(c->comp_id.data(), n * 4) || !r.get(c->comp_sizes.data(), static_cast<uint64_t>(C) * 4))
    return cfail(SB_ERUNTIME, "vgacsr: truncated components");
  if (flags & 1u) {
    c->hilbert_inverse.resize(n);
    if (!r.get(c->hilbert_inverse.data(), n * 4)) return cfail(SB_ERUNTIME, "vgacsr: truncated hilbert_inverse");
  }
  const uint32_t want = static_cast<uint32_t>(r.crc);
  uint32_t crc = 0;
  if (fread(&crc, 1, 4, f) != 4) return cfail(SB_ERUNTIME, "vgacsr: truncated checksum");
  if (crc != want) return cfail(SB_ERUNTIME, "vgacsr: checksum mismatch");
  uint64_t e = 0;
  for (uint64_t v = 0; v < n; ++v) e += c->degrees[v];
  if (e != c->edges) return cfail(SB_ERUNTIME, "vgacsr: edge count mismatch");
  std::vector<uint64_t> seen(C, 0);
  for (uint64_t v = 0; v < n; ++v) {
    if (c->comp_id[v] >= C) return cfail(SB_ERUNTIME, "vgacsr: component id out of range");
    ++seen[c->comp_id[v]];
  }
  for (uint32_t k = 0; k < C; ++k)
    if (seen[k] != c->comp_sizes[k]) return cfail(SB_ERUNTIME, "vgacsr: component sizes do not match the ids");
  *out = c.release();
  return SB_OK;
}

// ---------------------------------------------------------------- partition
// Contiguous ranges balanced on per-node work deg(v) + 1 (own-row copy), the
// weighted analogue of parallel_ranges (parallel.hpp:32-35).
int sb_partition_edges(uint64_t n, const uint64_t* offsets, const uint32_t* degrees, int parts, uint64_t* bounds) {
  (void)offsets;
  if (!degrees || !bounds || parts < 1) return cfail(SB_EINVAL, "bad partition arguments");
  uint64_t total = 0;
  for (uint64_t v = 0; v < n; ++v) total += static_cast<uint64_t>(degrees[v]) + 1;
  bounds[0] = 0;
  uint64_t acc = 0, v = 0;
  for (int k = 1; k < parts; ++k) {
    const unsigned __int128 goal = static_cast<unsigned __int128>(total) * k / parts;
    while (v < n && acc + degrees[v] + 1 <= goal) acc += static_cast<uint64_t>(degrees[v++]) + 1;
    bounds[k] = v;
  }
  bounds[parts] = n;
  return SB_OK;
}

// ---------------------------------------------------------------- depth entropy
// Exact-oracle-mode entropy: Shannon entropy in bits of the
// node's depth distribution, H = -sum_t p_t log2 p_t with p_t = n_t / S,
// S = sum_{t>=1} n_t, summed in increasing t (no FMA: -ffp-contract=off).
int sb_depth_entropy(uint64_t n, const uint32_t* hist, uint32_t hist_cap, double* entropy) {
  if (!hist || !entropy || hist_cap == 0) return cfail(SB_EINVAL, "sb_depth_entropy: bad arguments");
  for (uint64_t v = 0; v < n; ++v) {
    const uint32_t* h = hist + v * hist_cap;
    uint64_t tot = 0;
    for (uint32_t t = 1; t < hist_cap; ++t) tot += h[t];
    if (!tot) {
      entropy[v] = NAN;
      continue;
    }
    double H = 0.0;
    for (uint32_t t = 1; t < hist_cap; ++t) {
      if (!h[t]) continue;
      const double p = static_cast<double>(h[t]) / static_cast<double>(tot);
      H -= p * std::log2(p);
    }
    entropy[v] = H + 0.0;  // -0.0 -> 0.0 for a single depth bin
  }
  return SB_OK;
}

// ---------------------------------------------------------------- CSV writer
// cmd_analyze output: one row per node, NaN serialised "NaN",
// doubles with 17 significant digits (round-trip exact, byte-deterministic).
static void put_num(std::string& o, double x) {
  if (std::isnan(x)) {
    o += "NaN";
  } else if (std::isinf(x)) {
    o += x > 0 ? "inf" : "-inf";
  } else {
    char buf[32];
    o.append(buf, static_cast<size_t>(snprintf(buf, sizeof buf, "%.17g", x)));
  }
}

// Rows are formatted in parallel into per-block strings and written in order:
// the bytes do not depend on the thread count.
int sb_metrics_write_csv(const char* path, const sb_metric_table* t) {
  if (!path || !t) return cfail(SB_EINVAL, "sb_metrics_write_csv: NULL argument");
  FILE* f = fopen(path, "wb");
  if (!f) return cfail(SB_ERUNTIME, "cannot open %s for writing", path);
  fputs("x,y,node_id,component_id,node_count,connectivity,visual_mean_depth,integration_hh,integration_tekl,"
        "integration_pv,control,controllability,clustering,entropy,rel_entropy,first_moment,second_moment\n", f);
  auto col = [](const double* c, uint64_t i) { return c ? c[i] : NAN; };
  const double* cols[11] = {t->md, t->ihh, t->tekl, t->pv, t->control, t->controllability,
                            t->clustering, t->entropy, t->rel_entropy, t->m1, t->m2};
  const uint64_t blk = 256, nb = (t->n + blk - 1) / blk;  // parallel_for hands out >= 64 blocks per grab
  std::vector<std::string> parts(nb);
  parallel_for(nb, 0, [&](uint64_t b0, uint64_t b1) {
    for (uint64_t b = b0; b < b1; ++b) {
      std::string& o = parts[b];
      o.reserve(blk * 280);
      char buf[96];
      for (uint64_t i = b * blk; i < std::min<uint64_t>(t->n, (b + 1) * blk); ++i) {
        put_num(o, col(t->x, i));
        o += ',';
        put_num(o, col(t->y, i));
        o.append(buf, static_cast<size_t>(snprintf(
                          buf, sizeof buf, ",%llu,%u,%u,%u,",
                          static_cast<unsigned long long>(t->node_id ? t->node_id[i] : i),
                          t->component_id ? t->component_id[i] : 0u, t->node_count ? t->node_count[i] : 0u,
                          t->connectivity ? t->connectivity[i] : 0u)));
        for (int k = 0; k < 11; ++k) {
          put_num(o, col(cols[k], i));
          o += k == 10 ? '\n' : ',';
        }
      }
    }
  });
  bool bad = false;
  for (const auto& o : parts) bad |= fwrite(o.data(), 1, o.size(), f) != o.size();
  bad |= ferror(f) != 0;
  if (fclose(f) != 0 || bad) return cfail(SB_ERUNTIME, "write error on %s", path);
  return SB_OK;
}

}  // extern "C"
