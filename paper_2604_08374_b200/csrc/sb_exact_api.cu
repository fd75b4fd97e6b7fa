// sb_exact_api.cu -- C-ABI: exact bit-parallel BFS (oracle exact mode) and the
// exact local metrics built on it.
#include <algorithm>
#include <cstdio>
#include <memory>
#include <string>
#include <vector>

#include "sb_device.cuh"
#include "sb_handles.h"

extern "C" {

// ------------------------------------------------------------------ exact mode
// Exact neighbourhood function: bit-parallel BFS, the
// HyperBall loop with bitset rows and an OR union (see exact_* kernels).

static int exact_grow_hist(sb_exact* x, uint32_t need) {
  if (need < x->hist_cap) return SB_OK;
  uint32_t cap = std::max<uint32_t>(x->hist_cap * 2, 16);
  while (cap <= need) cap *= 2;
  const uint64_t n = x->g->n;
  uint32_t* nh = nullptr;
  CK(dalloc(&nh, n * cap * 4));
  CK(cudaMemsetAsync(nh, 0, n * cap * 4, x->stream));
  if (x->d_hist)
    CK(cudaMemcpy2DAsync(nh, cap * 4, x->d_hist, x->hist_cap * 4, x->hist_cap * 4, n, cudaMemcpyDeviceToDevice,
                         x->stream));
  CK(sync_stream(x->stream));
  dfree(x->d_hist);
  x->d_hist = nh;
  x->hist_cap = cap;
  return SB_OK;
}

int sb_exact_create(sb_graph* g, unsigned log2_block, uint32_t depth_limit, uint32_t flags, sb_exact** out) {
  if (!out) return fail(SB_EINVAL, "sb_exact_create: out is NULL");
  *out = nullptr;
  if (!g) return fail(SB_EINVAL, "sb_exact_create: NULL graph");
  if (g->v0 != 0 || g->v1 != g->n) return fail(SB_EINVAL, "sb_exact_create: needs the full graph on the device");
  if (log2_block < 12 || log2_block > 16) return fail(SB_EINVAL, "sb_exact_create: log2_block must be in [12, 16]");
  if (flags & ~(uint32_t)SB_HB_INTERVAL) return fail(SB_EINVAL, "sb_exact_create: only SB_HB_INTERVAL is supported");
  if (g->n == 0) return fail(SB_EINVAL, "sb_exact_create: graph empty");
  DeviceGuard dg(g->device);
  if (const int rc = graph_wait(g)) return rc;
  auto* x = new sb_exact();
  x->g = g;
  x->P = static_cast<int>(log2_block) - 2;
  x->row = 1ull << (x->P - 1);
  x->block = 1ull << log2_block;
  x->depth = depth_limit;
  x->flags = flags;
  x->slices = sb::union_slices(x->P);
  auto bail = [&](int rc) { delete x; return rc; };
#define XK(e)                                                 \
  do {                                                        \
    cudaError_t e_ = (e);                                     \
    if (e_ != cudaSuccess) return bail(cuda_fail(e_, #e));    \
  } while (0)
  XK(cudaStreamCreateWithFlags(&x->stream, cudaStreamNonBlocking));
  for (auto& e : x->ev) XK(cudaEventCreate(&e));
  const uint64_t n = g->n, plane = n * x->row;
  for (int i = 0; i < 2; ++i) XK(dalloc(&x->d_plane[i], plane + 64));
  XK(dalloc(&x->d_changed, n));
  XK(dalloc(&x->d_scratch, std::max<uint64_t>(g->n_items, 1) * x->slices * 512));
  XK(dalloc(&x->d_counter, n * x->slices * 4));
  XK(cudaMemset(x->d_counter, 0, n * x->slices * 4));
  XK(dalloc(&x->d_pop, n * 4));
  XK(dalloc(&x->d_reach, n * 4));
  XK(cudaMemset(x->d_reach, 0, n * 4));
  XK(dalloc(&x->d_sum, 2 * n * 8));
  XK(cudaMemset(x->d_sum, 0, 2 * n * 8));
  XK(dalloc(&x->d_misc, 2 * 8));
  if (flags & SB_HB_INTERVAL) {
    const int rc = build_run_index(g);  // sets max_run
    if (rc) return bail(rc);
    int K = 0;
    while (K < 10 && (2u << K) <= g->max_run) ++K;
    x->levels = K;
    if (K) XK(dalloc(&x->d_st, static_cast<uint64_t>(K) * plane + 64));
  }
#undef XK
  const int rc = exact_grow_hist(x, 15);
  if (rc) return bail(rc);
  *out = x;
  return SB_OK;
}

int sb_exact_run(sb_exact* x, uint64_t src_begin, uint64_t src_end, uint32_t* max_depth) {
  if (!x) return fail(SB_EINVAL, "NULL handle");
  sb_graph* g = x->g;
  if (src_begin > src_end || src_end > g->n) return fail(SB_EINVAL, "sb_exact_run: bad source range");
  DeviceGuard dg(g->device);
  const uint64_t n = g->n;
  sb::ExactArgs e{};
  e.n = n;
  e.pop = x->d_pop;
  e.reach = x->d_reach;
  e.sum_d = x->d_sum;
  e.sum_d2 = x->d_sum + n;
  e.changed_count = x->d_misc + 1;
  for (uint64_t s0 = src_begin; s0 < src_end; s0 += x->block) {
    const uint64_t s1 = std::min(s0 + x->block, src_end);
    int L = 0;
    e.plane = x->d_plane[L];
    e.s0 = s0;
    e.s1 = s1;
    CK(sb::launch_exact_init(x->P, e, x->stream));
    uint32_t t0 = 1;
    if (g->d_run_off) {
      // Depth 1 straight from the run index (the rows the first OR pass would
      // produce) -- one union pass fewer per block.
      int rc = exact_grow_hist(x, 1);
      if (rc) return rc;
      e.hist = x->d_hist;
      e.hist_cap = x->hist_cap;
      e.node_item = g->d_node_item;
      e.run_off = g->d_run_off;
      e.run_s = g->d_run_s;
      e.run_e = g->d_run_e;
      e.plane = x->d_plane[1];
      CK(cudaMemsetAsync(x->d_misc, 0, 16, x->stream));
      CK(cudaEventRecord(x->ev[0], x->stream));
      CK(sb::launch_exact_init1(x->P, e, x->stream));
      CK(cudaEventRecord(x->ev[1], x->stream));
      e.t = 1;
      CK(sb::launch_exact_count(x->P, e, x->stream));
      unsigned long long changed = 0;
      CK(cudaMemcpyAsync(&changed, x->d_misc + 1, 8, cudaMemcpyDeviceToHost, x->stream));
      CK(sync_stream(x->stream));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, x->ev[0], x->ev[1]);
      x->union_ms += ms;
      x->union_launches += 1;
      if (changed == 0 || (x->depth && x->depth == 1)) {
        if (changed) x->max_depth = std::max(x->max_depth, 1u);
        x->sources_done += s1 - s0;
        continue;
      }
      x->max_depth = std::max(x->max_depth, 1u);
      L = 1;
      t0 = 2;
    }
    for (uint32_t t = t0;; ++t) {
      int rc = exact_grow_hist(x, t);
      if (rc) return rc;
      e.hist = x->d_hist;
      e.hist_cap = x->hist_cap;
      CK(cudaMemsetAsync(x->d_misc, 0, 16, x->stream));
      sb::UnionArgs u{};
      graph_union_args(g, u);
      u.cur = x->d_plane[L];
      u.next = x->d_plane[1 - L];
      u.scratch = x->d_scratch;
      u.node_counter = x->d_counter;
      u.changed_out = x->d_changed;
      u.changed_in = x->d_changed;
      u.work = x->d_misc;
      CK(cudaEventRecord(x->ev[0], x->stream));
      if (x->flags & SB_HB_INTERVAL) {
        if (x->levels) CK(sb::launch_st_build(x->P, x->d_plane[L], x->d_st, n, x->levels, x->stream, true));
        sb::IntervalArgs ia{};
        ia.u = u;
        ia.st = x->d_st ? x->d_st : x->d_plane[L];
        ia.n_global = n;
        ia.levels = x->levels;
        ia.run_off = g->d_run_off;
        ia.run_s = g->d_run_s;
        ia.run_e = g->d_run_e;
        CK(sb::launch_union_interval(x->P, ia, x->stream, true));
      } else {
        CK(sb::launch_union_or(x->P, u, x->stream));
      }
      CK(cudaEventRecord(x->ev[1], x->stream));
      e.plane = x->d_plane[1 - L];
      e.t = t;
      CK(sb::launch_exact_count(x->P, e, x->stream));
      unsigned long long changed = 0;
      CK(cudaMemcpyAsync(&changed, x->d_misc + 1, 8, cudaMemcpyDeviceToHost, x->stream));
      CK(sync_stream(x->stream));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, x->ev[0], x->ev[1]);
      x->union_ms += ms;
      x->union_launches += 1;
      if (changed == 0) break;  // no row grew: every BFS of the block is complete
      x->max_depth = std::max(x->max_depth, t);
      if (x->depth && t == x->depth) break;
      L = 1 - L;
    }
    x->sources_done += s1 - s0;
  }
  if (max_depth) *max_depth = x->max_depth;
  return SB_OK;
}

int sb_exact_read(const sb_exact* x, uint64_t* sum_d, uint64_t* sum_d2, uint32_t* reach, uint32_t* hist,
                  uint32_t hist_cap) {
  if (!x) return fail(SB_EINVAL, "NULL handle");
  const uint64_t n = x->g->n;
  if (hist && hist_cap <= x->max_depth)
    return fail(SB_EINVAL, "sb_exact_read: hist_cap %u <= max depth %u", hist_cap, x->max_depth);
  DeviceGuard dg(x->g->device);
  if (sum_d) CK(cudaMemcpy(sum_d, x->d_sum, n * 8, cudaMemcpyDeviceToHost));
  if (sum_d2) CK(cudaMemcpy(sum_d2, x->d_sum + n, n * 8, cudaMemcpyDeviceToHost));
  if (reach) CK(cudaMemcpy(reach, x->d_reach, n * 4, cudaMemcpyDeviceToHost));
  if (hist) {
    const uint32_t w = std::min(hist_cap, x->hist_cap);
    memset(hist, 0, n * hist_cap * 4);
    CK(cudaMemcpy2D(hist, hist_cap * 4, x->d_hist, x->hist_cap * 4, w * 4, n, cudaMemcpyDeviceToHost));
  }
  return SB_OK;
}

int sb_exact_stats(const sb_exact* x, uint64_t* sources_done, uint32_t* max_depth, double* union_ms,
                   uint64_t* union_launches) {
  if (!x) return fail(SB_EINVAL, "NULL handle");
  if (sources_done) *sources_done = x->sources_done;
  if (max_depth) *max_depth = x->max_depth;
  if (union_ms) *union_ms = x->union_ms;
  if (union_launches) *union_launches = x->union_launches;
  return SB_OK;
}

void sb_exact_destroy(sb_exact* x) { delete x; }

// ------------------------------------------------------------------ local metrics
// Exact 1-/2-hop metrics over the device-resident run index;
// |N2(v)| = |B(v, 2)| - 1 from the exact bit-parallel BFS at depth 2.
int sb_local_metrics(sb_graph* g, uint64_t v0, uint64_t v1, double* control, double* controllability,
                     double* clustering, uint64_t* edges_among, uint64_t* n2) {
  if (!g) return fail(SB_EINVAL, "sb_local_metrics: NULL graph");
  if (g->v0 != 0 || g->v1 != g->n)
    return fail(SB_EINVAL, "sb_local_metrics: needs the full graph on the device (2-hop rows of any node)");
  if (v0 > v1 || v1 > g->n) return fail(SB_EINVAL, "sb_local_metrics: bad node range");
  DeviceGuard dg(g->device);
  int rc = graph_wait(g);
  if (rc) return rc;
  rc = build_run_index(g);
  if (rc) return rc;
  const uint64_t n = g->n, nl = v1 - v0;
  if (nl == 0) return SB_OK;
  // |N2(v)|: depth-2 exact BFS over every source block (cost ~ blocks x runs, best
  // for dense graphs) or per-node 2-hop bitmaps (cost ~ sum_w deg(w) runs(w),
  // best for large sparse graphs).  Crossover measured with the one-pass BFS
  // (depth-1 rows from the run index) on a 49,632-node grid, 13 blocks:
  // bitmap 6.3 vs BFS 8.2 ms at mean degree 898, 14.1 vs 11.5 ms at 1,536 ->
  // bitmaps win when avg degree < ~88 x blocks (C3, 350 x: BFS 2.2x faster;
  // city grid, 2.3 x: bitmap).
  const uint64_t blocks = (n + 4095) / 4096;
  bool n2_bitmap = static_cast<double>(g->edges_local) / static_cast<double>(n) < 88.0 * static_cast<double>(blocks);
  if (const char* e = getenv("SB_LOCAL_N2")) {  // test / A-B override: "bfs" or "bitmap"
    if (!strcmp(e, "bfs")) n2_bitmap = false;
    if (!strcmp(e, "bitmap")) n2_bitmap = true;
  }
  sb_exact* x = nullptr;
  std::unique_ptr<sb_exact, void (*)(sb_exact*)> xg(nullptr, sb_exact_destroy);
  if (!n2_bitmap) {
    rc = sb_exact_create(g, 12, 2, SB_HB_INTERVAL, &x);
    if (rc) return rc;
    xg.reset(x);
    rc = sb_exact_run(x, 0, n, nullptr);
    if (rc) return rc;
  }
  // [span_lo N | span_hi N | lo2 nl | hi2 nl | max 2] u32, [control | ctrl | clus] f64 nl, [among | n2 | work] u64
  const uint64_t u32_words = 2 * n + 2 * nl + 2;
  const uint64_t bytes = ((u32_words * 4 + 7) & ~7ull) + 5 * nl * 8 + 8;
  uint8_t* blk = nullptr;
  CK(dalloc(&blk, bytes));
  uint32_t* scratch = nullptr;
  struct Free {
    uint8_t*& p;
    uint32_t*& q;
    ~Free() {
      cudaStreamSynchronize(0);  // error paths: kernels on the legacy stream may still run
      dfree(p);
      dfree(q);
    }
  } fr{blk, scratch};
  sb::LocalArgs a{};
  a.n = n;
  a.v0 = v0;
  a.v1 = v1;
  a.degrees = g->d_deg;
  a.node_item = g->d_node_item;
  a.run_off = g->d_run_off;
  a.run_s = g->d_run_s;
  a.run_e = g->d_run_e;
  a.reach2 = n2_bitmap ? nullptr : x->d_reach;
  uint32_t* u = reinterpret_cast<uint32_t*>(blk);
  a.span_lo = u;
  a.span_hi = u + n;
  a.lo2 = n2_bitmap ? u + 2 * n : nullptr;
  a.hi2 = n2_bitmap ? u + 2 * n + nl : nullptr;
  a.max_words = u + 2 * n + 2 * nl;
  double* f = reinterpret_cast<double*>(blk + ((u32_words * 4 + 7) & ~7ull));
  a.control = f;
  a.controllability = f + nl;
  a.clustering = f + 2 * nl;
  a.edges_among = reinterpret_cast<unsigned long long*>(f + 3 * nl);
  a.n2 = a.edges_among + nl;
  a.work = a.n2 + nl;
  CK(cudaMemsetAsync(a.max_words, 0, 8, 0));
  CK(cudaMemsetAsync(a.work, 0, 8, 0));
  CK(sb::launch_local_spans(a, 0));
  unsigned int mw[2] = {0, 0};
  CK(cudaMemcpy(mw, a.max_words, 8, cudaMemcpyDeviceToHost));
  a.w1_words = std::max(mw[0], 1u);
  a.stride_words = 2ull * (a.w1_words + 1) + (n2_bitmap ? std::max(mw[1], 1u) : 0u);
  a.stride_words = (a.stride_words + 3) & ~3ull;  // 16-B aligned per-CTA regions (uint2 rank table)
  // SB_LOCAL_GLOBAL=1 forces the global-scratch bitmaps (test hook for wide windows)
  const char* force = getenv("SB_LOCAL_GLOBAL");
  const bool smem = a.stride_words * 4 <= sb::local_smem_limit() && !(force && atoi(force));
  if (!smem) {
    int grid = 0;
    CK(sb::launch_local(a, false, n2_bitmap, &grid, 0));
    CK(dalloc(&scratch, static_cast<uint64_t>(grid) * a.stride_words * 4));
    a.scratch = scratch;
  }
  CK(sb::launch_local(a, smem, n2_bitmap, nullptr, 0));
  CK(sync_stream(0));
  if (control) CK(cudaMemcpy(control, a.control, nl * 8, cudaMemcpyDeviceToHost));
  if (controllability) CK(cudaMemcpy(controllability, a.controllability, nl * 8, cudaMemcpyDeviceToHost));
  if (clustering) CK(cudaMemcpy(clustering, a.clustering, nl * 8, cudaMemcpyDeviceToHost));
  if (edges_among) CK(cudaMemcpy(edges_among, a.edges_among, nl * 8, cudaMemcpyDeviceToHost));
  if (n2) CK(cudaMemcpy(n2, a.n2, nl * 8, cudaMemcpyDeviceToHost));
  return SB_OK;
}

}  // extern "C"
