// sb_vis.cu -- on-device construction of the grid visibility graph straight
// into the HBM-resident LEB128 delta-CSR (replaces the CPU build of
// cmd_build_graph: grid -> visibility -> compressed CSR, SPEC.md:100-219,
// PAPER.md:222-307), so the HyperBall path never round-trips the 4.8 GB
// stream through the host.
//
// Byte-identical to the host generator (sb_csr_synth_grid, sb_csr.cpp):
//   * same exact integer line of sight (cell centres at odd coordinates, the
//     open segment may not cross an obstacle cell's interior, exact corner
//     crossings step diagonally) behind the same blocked-box prefix-sum test;
//   * same candidate order (row by row, column ascending = raster id order);
//   * same delta-LEB128 rows (first id absolute);
//   * same component ids (UnionFind::finalize: dense ids by first node,
//     union_find.hpp:37-52) from the same 8-neighbour union.
//
//   vis_rows_kernel<false>  warp per node: degree and row bytes
//   vis_rows_kernel<true>   warp per node: writes the row at offsets[v]
//   Each warp step tests 32 consecutive candidate cells of one grid row (one
//   blocked-box test per grid row first: an obstacle-free box spanned by v and
//   the row's candidates makes the whole row visible); the visible ones are
//   ordered by a ballot, their deltas / varint lengths come
//   from the previous visible lane (or the carried previous id) and a warp
//   prefix sum of the lengths places every varint.
#include <cub/cub.cuh>

#include "sb_device.cuh"
#include "sb_internal.h"

namespace sb {

__device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint64_t isqrt64_dev(uint64_t v) {
  uint64_t r = static_cast<uint64_t>(sqrt(static_cast<double>(v)));
  while (r * r > v) --r;
  while ((r + 1) * (r + 1) <= v) ++r;
  return r;
}

__device__ __forceinline__ bool any_blocked(const VisArgs& a, int r0, int c0, int r1, int c1) {
  if (r0 > r1) {
    const int t = r0;
    r0 = r1;
    r1 = t;
  }
  if (c0 > c1) {
    const int t = c0;
    c0 = c1;
    c1 = t;
  }
  const uint64_t W = a.cols + 1;
  const uint32_t s = a.pref[(r1 + 1) * W + (c1 + 1)] - a.pref[r0 * W + (c1 + 1)] - a.pref[(r1 + 1) * W + c0] +
                     a.pref[r0 * W + c0];
  return s != 0;
}

// Exact integer line of sight between the centres of (r1,c1) and (r2,c2):
// walk the cells whose interior the open segment crosses, stepping in x when
// (2k+1)*ay < (2j+1)*ax, in y when greater, diagonally on an exact corner
// crossing -- the host generator's walk (sb_csr.cpp) with the two products
// kept as running 64-bit sums (2*ax*ay reaches 2^33 on a 2^32-cell grid).
__device__ bool visible(const VisArgs& a, int r1, int c1, int r2, int c2) {
  if (!any_blocked(a, r1, c1, r2, c2)) return true;
  const int dx = c2 - c1, dy = r2 - r1;
  const int sx = dx > 0 ? 1 : -1, sy = dy > 0 ? 1 : -1;
  const int ax = dx < 0 ? -dx : dx, ay = dy < 0 ? -dy : dy;
  int x = c1, y = r1, k = 0, j = 0;
  int64_t lhs = ay, rhs = ax;  // (2k+1)*ay and (2j+1)*ax
  const uint8_t* __restrict__ row = a.blocked + static_cast<uint64_t>(y) * a.cols;
  const int64_t rstep = sy * static_cast<int64_t>(a.cols);
  while (k < ax || j < ay) {
    const bool mx = k < ax && (j >= ay || lhs <= rhs);
    const bool my = j < ay && (k >= ax || lhs >= rhs);
    if (mx) {
      x += sx;
      ++k;
      lhs += 2 * static_cast<int64_t>(ay);
    }
    if (my) {
      y += sy;
      ++j;
      rhs += 2 * static_cast<int64_t>(ax);
      row += rstep;
    }
    if (x == c2 && y == r2) break;
    if (row[x]) return false;
  }
  return true;
}

__device__ __forceinline__ uint32_t leb_len32(uint32_t v) {
  return v < (1u << 7) ? 1u : v < (1u << 14) ? 2u : v < (1u << 21) ? 3u : v < (1u << 28) ? 4u : 5u;
}

template <bool WRITE>
__global__ void __launch_bounds__(256) vis_rows_kernel(VisArgs a) {
  const int lane = threadIdx.x & 31;
  const uint32_t ltm = (1u << lane) - 1u;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  for (uint64_t v = gw; v < a.n; v += nw) {
    const uint32_t cell = a.cell_of_node[v];
    const int r = static_cast<int>(cell / a.cols), cc = static_cast<int>(cell % a.cols);
    const int r_lo = static_cast<int>(imax64(0, r - a.R));
    const int r_hi = static_cast<int>(imin64(static_cast<int64_t>(a.rows) - 1, r + a.R));
    uint32_t deg = 0;
    uint64_t pos = WRITE ? a.offsets[v] : 0, bytes = 0;
    uint64_t step = a.masks ? a.step_off[v] : 0;  // visibility-mask word of the current warp step
    bool have_prev = false;
    uint32_t prev = 0;
    for (int r2 = r_lo; r2 <= r_hi; ++r2) {
      const int64_t dr = r2 - r;
      int64_t span = a.cols;
      if (a.radius2) span = static_cast<int64_t>(isqrt64_dev(a.radius2 - static_cast<uint64_t>(dr * dr)));
      const int c_lo = static_cast<int>(imax64(0, cc - span));
      const int c_hi = static_cast<int>(imin64(static_cast<int64_t>(a.cols) - 1, cc + span));
      const uint64_t rowbase = static_cast<uint64_t>(r2) * a.cols;
      // Every candidate segment of this grid row lies in the box spanned by
      // (r, cc) and the row's column range: no obstacle in it -> all visible.
      const bool clear = !any_blocked(a, r, min(cc, c_lo), r2, max(cc, c_hi));
      if (clear) {
        step += static_cast<uint64_t>(c_hi - c_lo + 32) / 32;  // no masks stored for clear rows
        // Obstacle-free row: its candidates are consecutive free cells, so their
        // node ids are consecutive (raster order) and every delta after the
        // row's first is 1 (2 across v itself): one varint + (count - 1) bytes.
        const bool self_row = r2 == r;
        const uint32_t span = static_cast<uint32_t>(c_hi - c_lo + 1);
        const uint32_t cnt = span - (self_row ? 1u : 0u);
        if (cnt == 0) continue;
        const uint32_t w0 = a.node_of_cell[rowbase + c_lo];
        const uint32_t first = w0 + ((self_row && c_lo == cc) ? 1u : 0u);
        const uint32_t last = w0 + span - 1u - ((self_row && c_hi == cc) ? 1u : 0u);
        const uint32_t d0 = have_prev ? first - prev : first;
        const uint32_t l0 = leb_len32(d0);
        if (WRITE) {
          if (lane == 0) {
            uint8_t* o = a.stream + pos;
            uint32_t x = d0;
            while (x >= 0x80u) {
              *o++ = static_cast<uint8_t>(x) | 0x80u;
              x >>= 7;
            }
            *o = static_cast<uint8_t>(x);
          }
          // bytes [pos + l0, pos + l0 + cnt - 1): delta 1 everywhere except 2 right
          // after v itself (when v has emitted cells on both sides); aligned words
          // of 0x01010101 in the middle, single bytes at the ends.
          const uint64_t b0 = pos + l0, len = cnt - 1u;
          const uint64_t two = (self_row && cc > c_lo && cc < c_hi) ? b0 + (cc - c_lo - 1) : ~0ull;
          const uint64_t mis = (4u - (b0 & 3u)) & 3u, head = len < mis ? len : mis;
          const uint64_t nw = (len - head) / 4u, tail0 = b0 + head + 4u * nw;
          if (lane < head) a.stream[b0 + lane] = (b0 + lane == two) ? 2u : 1u;
          for (uint64_t k = lane; k < nw; k += 32) {
            const uint64_t at = b0 + head + 4u * k;
            uint32_t word = 0x01010101u;
            if (two >= at && two < at + 4u) word += 1u << (8u * static_cast<uint32_t>(two - at));
            *reinterpret_cast<uint32_t*>(a.stream + at) = word;
          }
          if (lane < b0 + len - tail0) a.stream[tail0 + lane] = (tail0 + lane == two) ? 2u : 1u;
        }
        pos += l0 + cnt - 1;
        bytes += l0 + cnt - 1;
        deg += cnt;
        prev = last;
        have_prev = true;
        continue;
      }
      for (int base = c_lo; base <= c_hi; base += 32) {
        const int c2 = base + lane;
        bool emit = false;
        uint32_t w = 0;
        if (WRITE && a.masks) {  // the count pass stored this step's line-of-sight results
          emit = (a.masks[step] >> lane) & 1u;
          if (emit) w = a.node_of_cell[rowbase + c2];
        } else if (c2 <= c_hi && !(r2 == r && c2 == cc)) {
          w = a.node_of_cell[rowbase + c2];
          if (w != 0xffffffffu) emit = visible(a, r, cc, r2, c2);
        }
        const uint32_t mask = __ballot_sync(FULL, emit);
        if (!WRITE && a.masks && lane == 0) a.masks[step] = mask;
        ++step;
        if (!mask) continue;
        const uint32_t lower = mask & ltm;
        const uint32_t pw = __shfl_sync(FULL, w, lower ? 31 - __clz(lower) : 0);
        const uint32_t delta = lower ? w - pw : (have_prev ? w - prev : w);
        const uint32_t len = emit ? leb_len32(delta) : 0u;
        uint32_t incl = len;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(FULL, incl, d);
          if (lane >= d) incl += y;
        }
        if (WRITE && emit) {
          uint8_t* o = a.stream + pos + (incl - len);
          uint32_t x = delta;
          while (x >= 0x80u) {  // leb128.hpp:12-18
            *o++ = static_cast<uint8_t>(x) | 0x80u;
            x >>= 7;
          }
          *o = static_cast<uint8_t>(x);
        }
        const uint32_t total = __shfl_sync(FULL, incl, 31);
        pos += total;
        bytes += total;
        deg += __popc(mask);
        prev = __shfl_sync(FULL, w, 31 - __clz(mask));
        have_prev = true;
      }
    }
    if (!WRITE && lane == 0) {
      a.deg[v] = deg;
      a.bytes[v] = bytes;
    }
  }
}

// Warp steps (32 candidate columns of one grid row) per node: the count pass
// stores one visibility mask per step so the write pass need not re-walk lines
// of sight.
__global__ void vis_steps_kernel(VisArgs a, uint64_t* steps) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < a.n; v += gridDim.x * (uint64_t)blockDim.x) {
    const uint32_t cell = a.cell_of_node[v];
    const int r = static_cast<int>(cell / a.cols), cc = static_cast<int>(cell % a.cols);
    const int r_lo = static_cast<int>(imax64(0, r - a.R));
    const int r_hi = static_cast<int>(imin64(static_cast<int64_t>(a.rows) - 1, r + a.R));
    uint64_t n = 0;
    for (int r2 = r_lo; r2 <= r_hi; ++r2) {
      const int64_t dr = r2 - r;
      int64_t span = a.cols;
      if (a.radius2) span = static_cast<int64_t>(isqrt64_dev(a.radius2 - static_cast<uint64_t>(dr * dr)));
      const int c_lo = static_cast<int>(imax64(0, cc - span));
      const int c_hi = static_cast<int>(imin64(static_cast<int64_t>(a.cols) - 1, cc + span));
      n += static_cast<uint64_t>(c_hi - c_lo + 32) / 32;
    }
    steps[v] = n;
  }
}

cudaError_t launch_vis_steps(const VisArgs& a, uint64_t* steps, cudaStream_t s) {
  vis_steps_kernel<<<(a.n + 255) / 256 < 148 * 16 ? (a.n + 255) / 256 : 148 * 16, 256, 0, s>>>(a, steps);
  return cudaGetLastError();
}

// ---- grid preparation -------------------------------------------------------
__global__ void pref_rows_kernel(VisArgs a, uint32_t* pref) {
  const uint64_t W = a.cols + 1;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r <= a.rows; r += gridDim.x * blockDim.x) {
    uint32_t acc = 0;
    pref[r * W] = 0;
    for (uint32_t c = 0; c < a.cols; ++c) {
      if (r > 0) acc += a.blocked[static_cast<uint64_t>(r - 1) * a.cols + c];
      pref[r * W + c + 1] = acc;
    }
  }
}

__global__ void pref_cols_kernel(VisArgs a, uint32_t* pref) {
  const uint64_t W = a.cols + 1;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c <= a.cols; c += gridDim.x * blockDim.x)
    for (uint32_t r = 1; r <= a.rows; ++r) pref[r * W + c] += pref[(r - 1) * W + c];
}

__global__ void free_flags_kernel(const uint8_t* blocked, uint64_t cells, uint32_t* flag) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cells; i += gridDim.x * (uint64_t)blockDim.x)
    flag[i] = blocked[i] ? 0u : 1u;
}

__global__ void node_maps_kernel(const uint8_t* blocked, uint64_t cells, const uint32_t* scan, uint32_t* node_of_cell,
                                 uint32_t* cell_of_node) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cells;
       i += gridDim.x * (uint64_t)blockDim.x) {
    if (blocked[i]) {
      node_of_cell[i] = 0xffffffffu;
    } else {
      node_of_cell[i] = scan[i];
      cell_of_node[scan[i]] = static_cast<uint32_t>(i);
    }
  }
}

// ---- components (8-neighbour union, lock-free union-find) -------------------
__device__ __forceinline__ uint32_t uf_find(uint32_t* parent, uint32_t v) {
  uint32_t p = parent[v];
  while (p != v) {
    const uint32_t gp = parent[p];
    if (gp != p) parent[v] = gp;  // path halving (benign race)
    v = p;
    p = gp;
  }
  return v;
}

__global__ void cc_init_kernel(uint32_t* parent, uint64_t n) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += gridDim.x * (uint64_t)blockDim.x)
    parent[v] = static_cast<uint32_t>(v);
}

// Hooks the larger root under the smaller one, so every root is its
// component's smallest node id (= UnionFind's first-occurrence order).
__global__ void cc_hook_kernel(VisArgs a) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < a.n; v += gridDim.x * (uint64_t)blockDim.x) {
    const uint32_t cell = a.cell_of_node[v];
    const int r = static_cast<int>(cell / a.cols), cc = static_cast<int>(cell % a.cols);
    for (int dr = -1; dr <= 1; ++dr)
      for (int dc = -1; dc <= 1; ++dc) {
        if (!dr && !dc) continue;
        const int r2 = r + dr, c2 = cc + dc;
        if (r2 < 0 || c2 < 0 || r2 >= static_cast<int>(a.rows) || c2 >= static_cast<int>(a.cols)) continue;
        if (a.radius2 && static_cast<uint64_t>(dr * dr + dc * dc) > a.radius2) continue;
        const uint32_t w = a.node_of_cell[static_cast<uint64_t>(r2) * a.cols + c2];
        if (w == 0xffffffffu || !visible(a, r, cc, r2, c2)) continue;
        uint32_t u = static_cast<uint32_t>(v), x = w;
        for (;;) {
          u = uf_find(a.parent, u);
          x = uf_find(a.parent, x);
          if (u == x) break;
          if (u < x) {
            const uint32_t t = u;
            u = x;
            x = t;
          }
          if (atomicCAS(a.parent + u, u, x) == u) break;
        }
      }
  }
}

// root[v] goes to a separate array: a concurrent path-halving write may still
// move parent[v] to a non-root ancestor after v's own find returned.
__global__ void cc_flatten_kernel(uint32_t* parent, uint64_t n, uint32_t* root, uint32_t* is_root) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += gridDim.x * (uint64_t)blockDim.x) {
    const uint32_t r = uf_find(parent, static_cast<uint32_t>(v));
    root[v] = r;
    is_root[v] = r == v ? 1u : 0u;
  }
}

// comp[v] holds v's root on entry, its dense component id on exit.
__global__ void cc_label_kernel(const uint32_t* root_rank, uint64_t n, uint32_t* comp, uint32_t* sizes) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += gridDim.x * (uint64_t)blockDim.x) {
    const uint32_t c = root_rank[comp[v]];
    comp[v] = c;
    atomicAdd(sizes + c, 1u);
  }
}

static int sms() {
  int dev = 0, s = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
  return s;
}

cudaError_t launch_vis_prepare(VisArgs& a, uint32_t* pref, uint32_t* tmp_scan, uint64_t* n_out, cudaStream_t s) {
  const uint64_t cells = static_cast<uint64_t>(a.rows) * a.cols;
  pref_rows_kernel<<<(a.rows + 256) / 256, 256, 0, s>>>(a, pref);
  pref_cols_kernel<<<(a.cols + 256) / 256, 256, 0, s>>>(a, pref);
  uint32_t* flag = tmp_scan + cells;  // [scan cells | flags cells]
  free_flags_kernel<<<sms() * 8, 256, 0, s>>>(a.blocked, cells, flag);
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, tmp_scan, cells, s);
  if (e != cudaSuccess) return e;
  void* t = nullptr;
  e = cudaMallocAsync(&t, tb, s);
  if (e != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(t, tb, flag, tmp_scan, cells, s);
  cudaFreeAsync(t, s);
  if (e != cudaSuccess) return e;
  uint32_t last_scan = 0, last_flag = 0;
  cudaMemcpyAsync(&last_scan, tmp_scan + cells - 1, 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&last_flag, flag + cells - 1, 4, cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  *n_out = static_cast<uint64_t>(last_scan) + last_flag;
  return cudaGetLastError();
}

cudaError_t launch_vis_maps(const VisArgs& a, const uint32_t* scan, uint32_t* node_of_cell, uint32_t* cell_of_node,
                            cudaStream_t s) {
  const uint64_t cells = static_cast<uint64_t>(a.rows) * a.cols;
  node_maps_kernel<<<sms() * 8, 256, 0, s>>>(a.blocked, cells, scan, node_of_cell, cell_of_node);
  return cudaGetLastError();
}

cudaError_t launch_vis_rows(const VisArgs& a, bool write, cudaStream_t s) {
  if (write)
    vis_rows_kernel<true><<<sms() * 8, 256, 0, s>>>(a);
  else
    vis_rows_kernel<false><<<sms() * 8, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_scan_u64(const uint64_t* in, uint64_t* out, uint64_t count, cudaStream_t s) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, count, s);
  if (e != cudaSuccess) return e;
  void* t = nullptr;
  e = cudaMallocAsync(&t, tb, s);
  if (e != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(t, tb, in, out, count, s);
  cudaFreeAsync(t, s);
  return e;
}

// comp / sizes must hold n entries; returns the component count.
cudaError_t launch_vis_components(const VisArgs& a, uint32_t* comp, uint32_t* sizes, uint32_t* tmp2n,
                                  uint64_t* n_comp, cudaStream_t s) {
  const int g = sms() * 8;
  cc_init_kernel<<<g, 256, 0, s>>>(a.parent, a.n);
  cc_hook_kernel<<<g, 256, 0, s>>>(a);
  uint32_t* is_root = tmp2n;
  uint32_t* rank = tmp2n + a.n;
  cc_flatten_kernel<<<g, 256, 0, s>>>(a.parent, a.n, comp, is_root);
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tb, is_root, rank, a.n, s);
  if (e != cudaSuccess) return e;
  void* t = nullptr;
  e = cudaMallocAsync(&t, tb, s);
  if (e != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(t, tb, is_root, rank, a.n, s);
  cudaFreeAsync(t, s);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(sizes, 0, a.n * 4, s);
  cc_label_kernel<<<g, 256, 0, s>>>(rank, a.n, comp, sizes);
  uint32_t lr = 0, lf = 0;
  cudaMemcpyAsync(&lr, rank + a.n - 1, 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&lf, is_root + a.n - 1, 4, cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  *n_comp = static_cast<uint64_t>(lr) + lf;
  return cudaGetLastError();
}

}  // namespace sb
