// sb_hb_api.cu -- C-ABI: HyperBall state, the Alg. 1 control loop, shard
// exchange (NCCL grouped broadcast / fused P2P peers / same-process copies), stats.
#include <algorithm>
#include <cstdio>
#include <memory>
#include <string>
#include <vector>

#include "sb_device.cuh"
#include "sb_handles.h"

static int hb_init(sb_hb* h) {
  sb_graph* g = h->g;
  const int L = h->latest = 0;
  h->t = 0;
  h->converged = h->finished = h->computed = false;
  h->stats.clear();
  CK(sb::launch_init(static_cast<int>(h->p), h->d_plane[L], g->n, g->d_orig, h->stream));
  CK(cudaMemsetAsync(h->d_changed[L], 1, g->n, h->stream));  // t=1 gathers every neighbour
  CK(cudaMemsetAsync(h->d_changed[1 - L], 0, g->n, h->stream));
  if (g->n_local) {
    CK(cudaMemsetAsync(h->d_sum_d, 0, g->n_local * 8, h->stream));
    CK(cudaMemsetAsync(h->d_sum_d2, 0, g->n_local * 8, h->stream));
    sb::EstArgs e{};
    e.plane = h->d_plane[L];
    e.node_begin = g->v0;
    e.n_local = g->n_local;
    e.lc = h->d_lc;
    e.alpha = h->alpha;
    e.m = static_cast<double>(1u << h->p);
    e.c_cur = h->d_c[L];
    e.t = 0;
    CK(sb::launch_estimate(static_cast<int>(h->p), 0, e, h->stream));
  }
  if (h->d_counter) CK(cudaMemsetAsync(h->d_counter, 0, std::max<uint64_t>(g->n_local, 1) * h->slices * 4, h->stream));
  // Everything that follows on this handle is ordered behind the stream; only
  // peers writing into this replica over P2P (and the caller's barrier after a
  // reset) need the initialisation complete before returning.
  if (h->npeers || h->comm) CK(sync_stream(h->stream));
  return SB_OK;
}

// Union arguments of this HyperBall: the graph's CSR / items / tiles / group
// path plus the handle's scratch, with the schedule rules applied.
static void hb_union_args(const sb_hb* h, sb::UnionArgs& u) {
  const sb_graph* g = h->g;
  graph_union_args(g, u);
  u.scratch = h->d_scratch;
  u.node_counter = h->d_counter;
  if (h->flags & SB_HB_SCHEDULE_WARP) u.n_tiles = 0;
  if (h->flags & SB_HB_SCHEDULE_GROUP) {  // every dense-enough group takes the group path
    u.node_lo = g->d_node_lo;
    u.shared_max_edges = ~0ull;
  } else if (h->p < 8 && g->edges_local < 6000ull * g->n_local) {
    // rows of <= 64 B on graphs of moderate degree: the gathers the group path
    // saves are cheap, and the per-node decode + fold is faster (C2, mean
    // degree 3,730: p=6 0.36 vs 0.81 ms, p=7 0.55 vs 1.02 ms; from p = 8 the
    // group path folds through the id ring: p=8 0.68 vs 0.96 ms); at C3 (mean
    // degree 20,278) the shared gathers win at every p (profiles/r02/group_threshold.json)
    u.node_lo = nullptr;
  }
  // Without the group path the per-warp item schedule balances better than
  // 8-node CTA tiles (C2 p=4 0.246 vs 0.260 ms, p=6 0.356 vs 0.379, C1 p=10
  // 0.140 vs 0.155; profiles/r02/group_threshold.json) -- except over a graph
  // still uploading, whose chunks are cut into tile ranges.
  if (!u.node_lo && !(h->flags & SB_HB_SCHEDULE_GROUP) && !g->pending) u.n_tiles = 0;
}

// Whether the first sb_hb_run over this handle's graph can be the wavefront of
// pipelined_run (a long asynchronous upload of one unsharded graph).
static bool wave_ok(const sb_hb* h) {
  const sb_graph* g = h->g;
  if (!g->pending || !g->d_chunk_rng || g->chunk_node.size() < 3) return false;
  if ((h->flags & (SB_HB_SKIP_UNCHANGED | SB_HB_SCHEDULE_WARP)) || h->npeers || h->comm) return false;
  if (g->v0 != 0 || g->n_local != g->n) return false;
  return g->stream_local >= (1ull << 30) || (h->flags & SB_HB_WAVEFRONT);
}

// Interval mode: the run index (built on first use; waits for an upload) and
// the sparse table, K = floor(log2(longest run)) levels, capped at 10 (longer
// runs peel 2^K blocks).
static int ensure_interval_ready(sb_hb* h) {
  if (!(h->flags & SB_HB_INTERVAL) || h->index_ready) return SB_OK;
  sb_graph* g = h->g;
  DeviceGuard dg(g->device);
  if (const int rc = build_run_index(g)) return rc;
  int K = 0;
  while (K < 10 && (2u << K) <= g->max_run) ++K;
  h->levels = K;
  dfree(h->d_st);
  if (K) CK(dalloc(&h->d_st, static_cast<uint64_t>(K) * g->n * h->row + 64));
  h->index_ready = true;
  return SB_OK;
}

extern "C" {

int sb_hb_create(sb_graph* g, unsigned p, uint32_t depth_limit, uint32_t flags, sb_hb** out) {
  if (!out) return fail(SB_EINVAL, "sb_hb_create: out is NULL");
  *out = nullptr;
  if (!g) return fail(SB_EINVAL, "sb_hb_create: NULL graph");
  if (p < 4 || p > 16) return fail(SB_EINVAL, "hll: precision must be in [4, 16]");
  if ((flags & SB_HB_INTERVAL) && (flags & SB_HB_SKIP_UNCHANGED))
    return fail(SB_EINVAL, "interval mode excludes SB_HB_SKIP_UNCHANGED");
  if ((flags & SB_HB_SCHEDULE_GROUP) && (flags & SB_HB_SCHEDULE_WARP))
    return fail(SB_EINVAL, "SB_HB_SCHEDULE_GROUP excludes SB_HB_SCHEDULE_WARP");
  if (flags & ~(SB_HB_SKIP_UNCHANGED | SB_HB_SCHEDULE_WARP | SB_HB_INTERVAL | SB_HB_SCHEDULE_GROUP | SB_HB_WAVEFRONT))
    return fail(SB_EINVAL, "sb_hb_create: unknown flags 0x%x", flags);
  DeviceGuard dg(g->device);
  auto* h = new sb_hb();
  h->g = g;
  h->p = p;
  h->depth = depth_limit;
  h->flags = flags;
  const uint32_t m = 1u << p;
  h->row = m / 2;
  h->slices = sb::union_slices(static_cast<int>(p));
  // alpha_m exactly as hll.cpp:13-18
  switch (m) {
    case 16: h->alpha = 0.673; break;
    case 32: h->alpha = 0.697; break;
    case 64: h->alpha = 0.709; break;
    default: h->alpha = 0.7213 / (1.0 + 1.079 / m); break;
  }
  auto bail = [&](int rc) { delete h; return rc; };
#define HK(x)                                                 \
  do {                                                        \
    cudaError_t e_ = (x);                                     \
    if (e_ != cudaSuccess) return bail(cuda_fail(e_, #x));    \
  } while (0)
  HK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  for (auto& e : h->ev) HK(cudaEventCreate(&e));
  const uint64_t plane = g->n * h->row;
  const uint64_t nl = std::max<uint64_t>(g->n_local, 1);
  for (int i = 0; i < 2; ++i) {
    HK(dalloc(&h->d_plane[i], plane + 64));
    HK(dalloc(&h->d_changed[i], g->n));
    HK(dalloc(&h->d_c[i], nl * 8));
  }
  HK(dalloc(&h->d_sum_d, nl * 8));
  HK(dalloc(&h->d_sum_d2, nl * 8));
  // Linear-counting table lc[z] = m * log(m / z) built with the host libm, so
  // the device never evaluates log (hll.cpp:35).
  std::vector<double> lc(m + 1, 0.0);
  const double md = static_cast<double>(m);
  for (uint32_t z = 1; z <= m; ++z) lc[z] = md * std::log(md / static_cast<double>(z));
  HK(dalloc(&h->d_lc, lc.size() * 8));
  HK(cudaMemcpy(h->d_lc, lc.data(), lc.size() * 8, cudaMemcpyHostToDevice));
  const uint64_t slice_bytes = std::min<uint64_t>(h->row, 512);
  HK(dalloc(&h->d_scratch, std::max<uint64_t>(g->n_items, 1) * h->slices * slice_bytes));
  HK(dalloc(&h->d_counter, nl * h->slices * 4));
  HK(dalloc(&h->d_misc, 4 * 8));
  if (flags & SB_HB_INTERVAL) {
    // over a long asynchronous upload the run index is built inside the first
    // run's wavefront (pipelined_run); otherwise now (waits for the upload)
    h->index_ready = false;
    if (!wave_ok(h)) {
      const int rc = ensure_interval_ready(h);
      if (rc) return bail(rc);
    }
  }
  HK(pinned_get(&h->h_misc, &h->h_misc_owned));
#undef HK
  const int rc = hb_init(h);
  if (rc != SB_OK) return bail(rc);
  *out = h;
  return SB_OK;
}

int sb_hb_reset(sb_hb* h) {
  if (!h) return fail(SB_EINVAL, "NULL handle");
  DeviceGuard dg(h->g->device);
  const int rc = hb_init(h);
  if (rc) return rc;
  // With fused P2P, a peer that already started iteration 1 stores rows and
  // changed flags into this replica: nobody may pass reset until every rank
  // has re-initialised its planes and flags (NCCL barrier on 8 bytes).
  if (h->npeers && h->comm && h->comm->nranks > 1) {
    NK(ncclAllReduce(h->d_misc + 3, h->d_misc + 3, 1, ncclUint64, ncclMax, h->comm->comm, h->stream));
    CK(sync_stream(h->stream));
  }
  return SB_OK;
}

void* sb_hb_stream(const sb_hb* h) { return h ? static_cast<void*>(h->stream) : nullptr; }

int sb_hb_step_compute(sb_hb* h, double* local_max) {
  if (!h) return fail(SB_EINVAL, "NULL handle");
  if (h->finished) return fail(SB_EINVAL, "hyperball: already finished (t=%u)", h->t);
  if (h->computed) return fail(SB_EINVAL, "hyperball: step_compute called twice without finish");
  sb_graph* g = h->g;
  DeviceGuard dg(g->device);
  if (g->broken) return fail(SB_ERUNTIME, "cgraph: the graph failed validation at upload");
  if (const int rc = ensure_interval_ready(h)) return rc;
  if (g->pending && (h->flags & SB_HB_SCHEDULE_WARP)) {  // the chunk pipeline needs the tile schedule
    const int rc = graph_wait(g);
    if (rc) return rc;
  }
  h->t += 1;
  const int L = h->latest, N = 1 - L;
  const bool skip_mode = (h->flags & SB_HB_SKIP_UNCHANGED) != 0;
  // Skip mode filters neighbours by last iteration's changed flags; while
  // nearly every row still changes the filter costs more than it saves (C3:
  // 96.5 vs 94.0 ms), so the plain kernel runs until fewer than 90 % of this
  // shard's rows changed.  Either kernel writes the same rows and flags.
  const uint64_t last_changed = h->stats.empty() ? g->n_local : h->stats.back().changed_nodes;
  const bool skip = skip_mode && last_changed * 10 < g->n_local * 9;
  h->cur_stats = sb_iter_stats{};
  h->cur_stats.t = h->t;
  CK(cudaMemsetAsync(h->d_misc, 0, 4 * 8, h->stream));
  CK(cudaEventRecord(h->ev[0], h->stream));
  if (g->n_local) {
    CK(cudaMemsetAsync(h->d_changed[N] + g->v0, 0, g->n_local, h->stream));
    sb::UnionArgs u{};
    hb_union_args(h, u);
    u.cur = h->d_plane[L];
    u.next = h->d_plane[N];
    u.changed_out = h->d_changed[N];
    u.changed_in = h->d_changed[L];
    u.work = h->d_misc;
    u.npeers = h->npeers;
    u.peer_next = h->d_peer_plane[N];
    u.peer_changed = h->d_peer_chg[N];
    CK(cudaEventRecord(h->ev[1], h->stream));
    if (h->flags & SB_HB_INTERVAL) {
      if (h->levels) CK(sb::launch_st_build(static_cast<int>(h->p), h->d_plane[L], h->d_st, g->n, h->levels, h->stream));
      sb::IntervalArgs ia{};
      ia.u = u;
      if (!ia.u.n_tiles) ia.u.n_tiles = g->n_tiles;  // interval kernel uses the tile schedule
      ia.st = h->d_st ? h->d_st : h->d_plane[L];
      ia.n_global = g->n;
      ia.levels = h->levels;
      ia.run_off = g->d_run_off;
      ia.run_s = g->d_run_s;
      ia.run_e = g->d_run_e;
      CK(sb::launch_union_interval(static_cast<int>(h->p), ia, h->stream));
    } else if (g->pending) {
      // First pass over a graph still streaming in: chunk k's tiles start as
      // soon as its bytes are copied and validated (overlaps PCIe with compute).
      // Consecutive chunks alternate between two streams (own work counters),
      // so chunk k+1's CTAs fill the SMs chunk k's last tiles leave idle.
      const size_t nk = g->chunk_node.size() - 1;
      if (!h->stream2) {
        CK(cudaStreamCreateWithFlags(&h->stream2, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
      }
      if (h->chunk_work_n < nk) {
        dfree(h->d_chunk_work);
        h->chunk_work_n = 0;
        CK(dalloc(&h->d_chunk_work, nk * 8));
        h->chunk_work_n = nk;
      }
      CK(cudaMemsetAsync(h->d_chunk_work, 0, nk * 8, h->stream));
      CK(cudaEventRecord(h->ev_fork, h->stream));
      CK(cudaStreamWaitEvent(h->stream2, h->ev_fork, 0));
      for (size_t k = 0; k < nk; ++k) {
        const uint64_t t0 = g->chunk_tile[k], t1 = g->chunk_tile[k + 1];
        if (t1 == t0) continue;
        cudaStream_t sk = (k & 1) ? h->stream2 : h->stream;
        CK(cudaStreamWaitEvent(sk, g->val_ev[k], 0));
        sb::UnionArgs uk = u;
        uk.err = g->d_err;  // stop at once if this or an earlier chunk failed validation
        uk.work = h->d_chunk_work + k;
        uk.tile_node0 = g->d_tile_node0 + t0;
        uk.tile_q = g->d_tile_q + t0;
        uk.n_tiles = t1 - t0;
        CK(sb::launch_union(static_cast<int>(h->p), skip, uk, sk));
      }
      CK(cudaEventRecord(h->ev_join, h->stream2));
      CK(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
    } else {
      CK(sb::launch_union(static_cast<int>(h->p), skip, u, h->stream));
    }
    CK(cudaEventRecord(h->ev[2], h->stream));
    sb::EstArgs e{};
    e.plane = h->d_plane[N];
    e.node_begin = g->v0;
    e.n_local = g->n_local;
    e.lc = h->d_lc;
    e.alpha = h->alpha;
    e.m = static_cast<double>(1u << h->p);
    e.c_prev = h->d_c[L];
    e.c_cur = h->d_c[N];
    e.sum_d = h->d_sum_d;
    e.sum_d2 = h->d_sum_d2;
    e.changed = h->d_changed[N];
    e.t = h->t;
    e.max_ord = h->d_misc + 1;
    e.changed_count = h->d_misc + 2;
    CK(sb::launch_estimate(static_cast<int>(h->p), skip_mode ? 2 : 1, e, h->stream));
  } else {
    CK(cudaEventRecord(h->ev[1], h->stream));
    CK(cudaEventRecord(h->ev[2], h->stream));
  }
  // The input flags are consumed: clear them now, so they can serve as next
  // iteration's output -- peers write into them only after the iteration
  // barrier (global max), never before this clear.
  CK(cudaMemsetAsync(h->d_changed[L], 0, g->n, h->stream));
  CK(cudaEventRecord(h->ev[3], h->stream));
  CK(cudaMemcpyAsync(h->h_misc, h->d_misc, 4 * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(sync_stream(h->stream));
  if (g->pending) {  // the upload finished inside this step: report a malformed stream now
    const int rc = graph_wait(g);
    if (rc) {
      h->t -= 1;
      return rc;
    }
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->ev[1], h->ev[2]);
  h->cur_stats.union_ms = ms;
  cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]);
  h->cur_stats.estimate_ms = ms;
  cudaEventElapsedTime(&ms, h->ev[0], h->ev[3]);
  h->cur_stats.step_ms = ms;
  h->cur_stats.changed_nodes = h->h_misc[2];
  h->computed = true;
  if (local_max) *local_max = decode_ord(h->h_misc[1]);
  return SB_OK;
}

int sb_hb_step_finish(sb_hb* h, double global_max, int* converged, int* finished) {
  if (!h) return fail(SB_EINVAL, "NULL handle");
  if (!h->computed) return fail(SB_EINVAL, "hyperball: step_finish without step_compute");
  h->computed = false;
  // Alg. 1: converged -> break (no swap); t == d -> stop.
  h->converged = sb_check_convergence(global_max) != 0;
  h->finished = h->converged || (h->depth != 0 && h->t == h->depth);
  h->latest = 1 - h->latest;  // registers / c of iteration t become "latest"
  h->cur_stats.max_increase = global_max;
  h->stats.push_back(h->cur_stats);
  if (converged) *converged = h->converged;
  if (finished) *finished = h->finished;
  return SB_OK;
}

int sb_hb_exchange_local(sb_hb* const* hs, int count) {
  if (!hs || count < 1) return fail(SB_EINVAL, "sb_hb_exchange_local: no handles");
  for (int i = 0; i < count; ++i) {
    if (!hs[i] || !hs[i]->computed) return fail(SB_EINVAL, "exchange: handle %d not computed", i);
    if (hs[i]->g->n != hs[0]->g->n || hs[i]->p != hs[0]->p) return fail(SB_EINVAL, "exchange: shape mismatch");
  }
  for (int i = 0; i < count; ++i) {
    const sb_hb* src = hs[i];
    const sb_graph* gs = src->g;
    if (!gs->n_local) continue;
    const int sN = 1 - src->latest;
    for (int j = 0; j < count; ++j) {
      if (j == i) continue;
      sb_hb* dst = hs[j];
      const int dN = 1 - dst->latest;
      DeviceGuard dg(dst->g->device);
      CK(cudaMemcpyPeerAsync(dst->d_plane[dN] + gs->v0 * src->row, dst->g->device,
                             src->d_plane[sN] + gs->v0 * src->row, gs->device,
                             gs->n_local * src->row, dst->stream));
      CK(cudaMemcpyPeerAsync(dst->d_changed[dN] + gs->v0, dst->g->device, src->d_changed[sN] + gs->v0,
                             gs->device, gs->n_local, dst->stream));
    }
  }
  for (int j = 0; j < count; ++j) {
    DeviceGuard dg(hs[j]->g->device);
    CK(sync_stream(hs[j]->stream));
  }
  return SB_OK;
}

static int exchange_nccl(sb_hb* h, double* gmax) {
  sb_comm* c = h->comm;
  sb_graph* g = h->g;
  const int N = 1 - h->latest;
  CK(cudaEventRecord(h->ev[0], h->stream));
  if (!h->npeers) {  // rows were not pushed by the kernel epilogue: broadcast the shards
    NK(ncclGroupStart());
    for (int r = 0; r < c->nranks; ++r) {
      const uint64_t a = h->bounds[r], b = h->bounds[r + 1];
      if (b == a) continue;
      uint8_t* rows = h->d_plane[N] + a * h->row;
      NK(ncclBroadcast(rows, rows, (b - a) * h->row, ncclUint8, r, c->comm, h->stream));
      uint8_t* ch = h->d_changed[N] + a;
      NK(ncclBroadcast(ch, ch, b - a, ncclUint8, r, c->comm, h->stream));
    }
    NK(ncclGroupEnd());
  }
  // 8-byte max; with fused P2P rows it is also the iteration barrier
  // (every rank's union kernel, and so its peer stores, has completed).
  NK(ncclAllReduce(h->d_misc + 1, h->d_misc + 1, 1, ncclUint64, ncclMax, c->comm, h->stream));
  CK(cudaEventRecord(h->ev[1], h->stream));
  CK(cudaMemcpyAsync(h->h_misc + 1, h->d_misc + 1, 8, cudaMemcpyDeviceToHost, h->stream));
  CK(sync_stream(h->stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]);
  h->cur_stats.exchange_ms = ms;
  *gmax = decode_ord(h->h_misc[1]);
  (void)g;
  return SB_OK;
}

int sb_hb_step(sb_hb* h, double* max_increase, int* converged, int* finished) {
  if (h && h->npeers && !(h->comm && h->comm->nranks > 1))
    return fail(SB_EINVAL, "peers attached without a communicator: use step_compute / step_finish "
                           "with an external barrier");
  double mx = 0.0;
  int rc = sb_hb_step_compute(h, &mx);
  if (rc) return rc;
  if (h->comm) {  // any attached communicator, a 1-rank one included: same code path at every N
    DeviceGuard dg(h->g->device);
    rc = exchange_nccl(h, &mx);
    if (rc) {
      h->computed = false;
      return rc;
    }
  }
  if (max_increase) *max_increase = mx;
  return sb_hb_step_finish(h, mx, converged, finished);
}

}  // extern "C"

// First run over a graph still uploading (sb_graph_create_async), dense mode,
// one unsharded graph: a wavefront over the upload chunks instead of one pass
// after another.  Pass p of chunk k reads pass p-1 of every chunk its rows
// reference -- the chunk's neighbour-id range, reduced at validation -- so
// passes 2, 3, ... start on the first chunks while later chunks still cross
// PCIe.  Every pass of the wavefront writes its own plane and changed flags
// (overlapping passes never overwrite what another still reads), on its own
// stream (higher priority for earlier passes), each chunk launch waiting on
// the events of the chunk-passes it reads.  Estimates run on h->stream in pass
// order once a pass is complete; a pass counts only if the previous one did
// not finish the run, and the state handed back is exactly the stepped run's
// (bit-identical: each row is the same max over the same rows).
// Sets *done when the run finished inside the wavefront; otherwise the caller
// continues with ordinary steps from the state left in d_plane[latest].
static int pipelined_run(sb_hb* h, bool* done) {
  *done = false;
  sb_graph* g = h->g;
  if (h->t != 0 || h->finished || h->computed || !wave_ok(h)) return SB_OK;
  const bool iv = (h->flags & SB_HB_INTERVAL) != 0;
  if (iv && (h->index_ready || g->d_run_off)) return SB_OK;  // interval: the index is built in here
  DeviceGuard dg(g->device);
  const int nk = static_cast<int>(g->chunk_node.size() - 1);
  const uint64_t plane = g->n * h->row;
  // interval mode: the sparse table of every pass, at the largest level count
  // (the longest run is only known once every chunk is counted)
  const int K = iv ? 10 : 0;
  const uint64_t per_pass = plane + 64 + g->n + (iv ? static_cast<uint64_t>(K) * plane + 64 : 0);
  // passes that may overlap the upload: a plane (+ table) each, within a quarter of free HBM
  int P = 12;
  if (h->depth) P = std::min<int>(P, static_cast<int>(h->depth));
  size_t fr = 0, tot = 0;
  CK(cudaMemGetInfo(&fr, &tot));
  while (P > 2 && static_cast<uint64_t>(P) * per_pass > fr / 4) --P;
  if (P < 2) return SB_OK;
  // resources (kept on the handle: the next first run reuses them).  The
  // planes of passes 2..5 up front -- a graph's first pool growth maps new
  // memory (slow, and stalls the wavefront if done inside it); passes beyond 5
  // only start on graphs whose rows reach few chunks, and get theirs on demand
  auto more_planes = [&](int count) -> int {
    while (static_cast<int>(h->d_xplane.size()) < count) {
      uint8_t* x = nullptr;
      uint8_t* c = nullptr;
      CK(dalloc(&x, plane + 64));
      h->d_xplane.push_back(x);
      CK(dalloc(&c, g->n));
      h->d_xchg.push_back(c);
    }
    return SB_OK;
  };
  auto more_tables = [&](int count) -> int {  // interval: tables of passes 0 .. count-1
    while (iv && static_cast<int>(h->d_xst.size()) < count) {
      uint8_t* x = nullptr;
      CK(dalloc(&x, static_cast<uint64_t>(K) * plane + 64));
      h->d_xst.push_back(x);
    }
    return SB_OK;
  };
  if (const int rc0 = more_planes(std::min(P - 1, 4))) return rc0;
  if (const int rc0 = more_tables(std::min(P, 5))) return rc0;
  while (static_cast<int>(h->pstream.size()) < P) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);  // hi is the numerically smaller, higher priority
    const int pr = std::max(hi, std::min(lo, hi + static_cast<int>(h->pstream.size())));
    cudaStream_t st = nullptr;
    CK(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, pr));
    h->pstream.push_back(st);
  }
  auto more_events = [&](std::vector<cudaEvent_t>& v, size_t count, unsigned flags) -> int {
    while (v.size() < count) {
      cudaEvent_t e = nullptr;
      CK(cudaEventCreateWithFlags(&e, flags));
      v.push_back(e);
    }
    return SB_OK;
  };
  if (const int rc0 = more_events(h->pev, static_cast<size_t>(P) * nk, cudaEventDisableTiming)) return rc0;
  if (const int rc0 = more_events(h->pev_t, 2 * static_cast<size_t>(P), cudaEventDefault)) return rc0;
  if (iv)
    if (const int rc0 = more_events(h->sev, static_cast<size_t>(P) * nk, cudaEventDisableTiming)) return rc0;
  if (h->pwork_n < static_cast<size_t>(P * nk)) {
    dfree(h->d_pwork);
    h->pwork_n = 0;
    CK(dalloc(&h->d_pwork, static_cast<size_t>(P * nk) * 8));
    h->pwork_n = static_cast<size_t>(P * nk);
  }
  // pass p's registers / changed flags: p = 0 the initialised plane, p = 1
  // the second plane, p >= 2 the extra ones; interval: table of pass p's plane
  auto pl = [&](int p) { return p == 0 ? h->d_plane[0] : p == 1 ? h->d_plane[1] : h->d_xplane[p - 2]; };
  auto cg = [&](int p) { return p == 0 ? h->d_changed[0] : p == 1 ? h->d_changed[1] : h->d_xchg[p - 2]; };
  auto stp = [&](int p) { return h->d_xst[p]; };
  RunIndexJob job;
  if (iv) {
    if (const int rc0 = rix_begin(g, job)) {
      rix_abort(g, job);
      return rc0;
    }
    CK(sb::launch_st_build(static_cast<int>(h->p), pl(0), stp(0), g->n, K, h->stream));  // the initial plane's table
  }
  CK(cudaMemsetAsync(h->d_pwork, 0, static_cast<size_t>(P * nk) * 8, h->stream));
  CK(cudaEventRecord(h->ev[0], h->stream));  // init + counters (+ table 0) done before any pass starts
  for (int p = 0; p < P; ++p) CK(cudaStreamWaitEvent(h->pstream[p], h->ev[0], 0));
  sb::UnionArgs base{};
  hb_union_args(h, base);
  base.err = g->d_err;    // every CTA stops if a chunk failed validation
  base.stop = nullptr;
  std::vector<int> dlo(nk, 0), dhi(nk, -1), next(P + 1, 0), next_st(P + 1, 0);
  auto chunk_of = [&](uint64_t id) {
    const int k = static_cast<int>(std::upper_bound(g->chunk_node.begin(), g->chunk_node.end(), id) -
                                   g->chunk_node.begin()) - 1;
    return std::min(std::max(k, 0), nk - 1);
  };
  // interval: the last chunk whose plane rows table (p, k) reads (2^K - 1 rows past k)
  auto kst = [&](int k) { return chunk_of(std::min<uint64_t>(g->n - 1, g->chunk_node[k + 1] + (1ull << K) - 2)); };
  auto launch = [&](int p, int k) -> int {  // pass p (1-based) of chunk k
    if (const int rc0 = more_planes(p - 1)) return rc0;
    cudaStream_t st = h->pstream[p - 1];
    if (k == 0) CK(cudaEventRecord(h->pev_t[2 * (p - 1)], st));
    if (p == 1) {
      CK(cudaStreamWaitEvent(st, iv ? job.ready[k] : g->val_ev[k], 0));
    } else {
      // the chunks its rows reference (interval: their table rows), and always
      // the chunk itself (its items' partial rows and arrival counters are reused)
      const std::vector<cudaEvent_t>& dep = iv ? h->sev : h->pev;
      CK(cudaStreamWaitEvent(st, h->pev[(p - 2) * nk + k], 0));
      if (iv) CK(cudaStreamWaitEvent(st, job.ready[k], 0));  // re-recorded if the run storage grew
      for (int j = dlo[k]; j <= dhi[k]; ++j) CK(cudaStreamWaitEvent(st, dep[(p - 2) * nk + j], 0));
    }
    const uint64_t n0 = g->chunk_node[k], n1 = g->chunk_node[k + 1];
    CK(cudaMemsetAsync(cg(p) + n0, 0, n1 - n0, st));
    const uint64_t t0 = g->chunk_tile[k], t1 = g->chunk_tile[k + 1];
    if (t1 > t0) {
      sb::UnionArgs u = base;
      u.cur = pl(p - 1);
      u.next = pl(p);
      u.changed_in = cg(p - 1);
      u.changed_out = cg(p);
      u.work = h->d_pwork + (p - 1) * nk + k;
      u.tile_node0 = g->d_tile_node0 + t0;
      u.tile_q = g->d_tile_q + t0;
      u.n_tiles = t1 - t0;
      if (iv) {
        sb::IntervalArgs ia{};
        ia.u = u;
        ia.st = stp(p - 1);
        ia.n_global = g->n;
        ia.levels = K;
        ia.run_off = g->d_run_off;
        ia.run_s = g->d_run_s;
        ia.run_e = g->d_run_e;
        ia.run_cap = job.cap;  // the index is filled with estimated storage
        CK(sb::launch_union_interval(static_cast<int>(h->p), ia, st));
      } else {
        CK(sb::launch_union(static_cast<int>(h->p), false, u, st));
      }
    }
    CK(cudaEventRecord(h->pev[(p - 1) * nk + k], st));
    if (k == nk - 1) CK(cudaEventRecord(h->pev_t[2 * (p - 1) + 1], st));
    return SB_OK;
  };
  auto launch_st = [&](int p, int k) -> int {  // table of pass p, rows of chunk k (after union(p) to kst(k))
    if (const int rc0 = more_tables(p + 1)) return rc0;
    cudaStream_t st = h->pstream[p - 1];
    CK(sb::launch_st_build_rows(static_cast<int>(h->p), pl(p), stp(p), g->n, K, g->chunk_node[k],
                                g->chunk_node[k + 1], st));
    CK(cudaEventRecord(h->sev[(p - 1) * nk + k], st));
    return SB_OK;
  };
  int P_enq = 1, known = 0;
  // enqueue every chunk-pass (and table) whose inputs are enqueued, in chunk
  // order per pass; `fresh`: passes may still start (the upload is in flight)
  auto pump = [&](bool fresh) -> int {
    for (bool progress = true; progress;) {
      progress = false;
      const int ready1 = iv ? static_cast<int>(job.filled) : nk;
      while (next[1] < ready1) {
        if (const int rc0 = launch(1, next[1]++)) return rc0;
        progress = true;
      }
      for (int p = 1; p <= P; ++p) {
        if (p >= 2) {
          const int* have = iv ? next_st.data() : next.data();
          while (next[p] < known && std::max(dhi[next[p]], next[p]) < have[p - 1] && (fresh || p <= P_enq)) {
            if (const int rc0 = launch(p, next[p]++)) return rc0;
            P_enq = std::max(P_enq, p);
            progress = true;
          }
        }
        if (iv && p < P && (fresh || p < P_enq)) {
          while (next_st[p] < nk && next[p] > kst(next_st[p]) && next[p] > 0) {
            if (const int rc0 = launch_st(p, next_st[p]++)) return rc0;
            progress = true;
          }
        }
      }
    }
    return SB_OK;
  };
  int rc = SB_OK;
  if (!iv) {  // pass 1 of every chunk waits only for its upload + validation
    for (int k = 0; k < nk && !rc; ++k) rc = launch(1, k);
    next[1] = nk;
  }
  // as each chunk lands: its neighbour range (interval: its runs), then --
  // while later chunks are still uploading -- every chunk-pass whose inputs
  // are all enqueued.  Passes are started only while the upload is in flight:
  // that work fills time the GPU would otherwise wait; once the last chunk is
  // in, the started passes are completed and the rest run one by one, so no
  // pass beyond the converging one is computed unless it overlapped the upload.
  for (int k = 0; k < nk && !rc; ++k) {
    CK(cudaEventSynchronize(g->val_ev[k]));
    uint32_t r[2] = {0u, 0u};
    CK(cudaMemcpy(r, g->d_chunk_rng + 2 * k, 8, cudaMemcpyDeviceToHost));
    if (r[0] <= r[1]) {
      dlo[k] = chunk_of(r[0]);
      dhi[k] = chunk_of(r[1]);
    }
    known = k + 1;
    if (iv) rc = rix_chunk(g, job, static_cast<size_t>(k));
    if (!rc) rc = pump(k < nk - 1);
  }
  auto drain = [&] {  // every launched chunk-pass done (scratch / counters are shared)
    for (int p = 0; p < P; ++p) cudaStreamSynchronize(h->pstream[p]);
  };
  if (!rc) rc = graph_wait(g);  // upload complete: a malformed stream is reported here
  bool overflow = false;
  if (iv && !rc) rc = rix_finish(g, job, &overflow);
  if (rc || overflow) {
    drain();
    if (iv) rix_abort(g, job);
    return rc;  // overflow: nothing was accounted; the caller runs the ordinary passes
  }
  rc = pump(false);  // complete the passes already started
  if (rc) {
    drain();
    return rc;
  }
  if (iv) {  // the handed-over state steps with the table the longest run needs
    if (const int rc0 = ensure_interval_ready(h)) {
      drain();
      return rc0;
    }
  }
  // estimates in pass order (Alg. 1: union -> estimate -> accumulate -> test)
  int last = 0;
  for (int p = 1; p <= P_enq; ++p) {
    h->t = static_cast<uint32_t>(p);
    h->cur_stats = sb_iter_stats{};
    h->cur_stats.t = h->t;
    CK(cudaMemsetAsync(h->d_misc, 0, 4 * 8, h->stream));
    CK(cudaStreamWaitEvent(h->stream, h->pev_t[2 * (p - 1) + 1], 0));
    CK(cudaEventRecord(h->ev[2], h->stream));
    sb::EstArgs e{};
    e.plane = pl(p);
    e.node_begin = g->v0;
    e.n_local = g->n_local;
    e.lc = h->d_lc;
    e.alpha = h->alpha;
    e.m = static_cast<double>(1u << h->p);
    e.c_prev = h->d_c[(p - 1) & 1];
    e.c_cur = h->d_c[p & 1];
    e.sum_d = h->d_sum_d;
    e.sum_d2 = h->d_sum_d2;
    e.changed = cg(p);
    e.t = h->t;
    e.max_ord = h->d_misc + 1;
    e.changed_count = h->d_misc + 2;
    CK(sb::launch_estimate(static_cast<int>(h->p), 1, e, h->stream));
    CK(cudaEventRecord(h->ev[3], h->stream));
    CK(cudaMemcpyAsync(h->h_misc, h->d_misc, 4 * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(sync_stream(h->stream));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->pev_t[2 * (p - 1)], h->pev_t[2 * (p - 1) + 1]);
    h->cur_stats.union_ms = ms;  // span of the pass's chunk launches (they overlap other passes)
    cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]);
    h->cur_stats.estimate_ms = ms;
    cudaEventElapsedTime(&ms, h->pev_t[2 * (p - 1)], h->ev[3]);
    h->cur_stats.step_ms = ms;
    h->cur_stats.changed_nodes = h->h_misc[2];
    const double mx = decode_ord(h->h_misc[1]);
    h->converged = sb_check_convergence(mx) != 0;
    h->finished = h->converged || (h->depth != 0 && h->t == h->depth);
    h->cur_stats.max_increase = mx;
    h->stats.push_back(h->cur_stats);
    last = p;
    if (h->finished) break;
  }
  // hand over to the two-plane stepping: d_plane[last & 1] holds pass `last`,
  // the other plane pass last - 1 (the "previous" registers), as after `last` steps
  for (int p = 0; p < P_enq; ++p) CK(cudaStreamWaitEvent(h->stream, h->pev_t[2 * p + 1], 0));
  for (int p = 0; p + 1 < P && iv; ++p)  // tables built for passes that did not start
    if (next_st[p + 1]) CK(cudaStreamWaitEvent(h->stream, h->sev[p * nk + next_st[p + 1] - 1], 0));
  for (int p = std::max(last - 1, 0); p <= last; ++p) {
    if (pl(p) != h->d_plane[p & 1]) CK(cudaMemcpyAsync(h->d_plane[p & 1], pl(p), plane, cudaMemcpyDeviceToDevice, h->stream));
    if (cg(p) != h->d_changed[p & 1]) CK(cudaMemcpyAsync(h->d_changed[p & 1], cg(p), g->n, cudaMemcpyDeviceToDevice, h->stream));
  }
  CK(sync_stream(h->stream));
  g->free_retired_runs();  // every launched pass is done
  h->latest = last & 1;
  *done = h->finished;
  return SB_OK;
}

// Back-to-back passes on one GPU (dense mode, no shards, graph resident): up
// to kBatch passes are enqueued at once and Alg. 1's test runs on the device
// after each (decide_kernel), turning the passes after the last one into
// no-ops -- one host round trip per batch instead of per pass.  Same kernels,
// same order of operations, bit-identical state and statistics.
static constexpr int kBatch = 8;
static int batched_run(sb_hb* h) {
  sb_graph* g = h->g;
  DeviceGuard dg(g->device);
  static_assert((kBatch * 2 + 2) * 8 <= sb::rt::kPinnedSlot, "batch records fit the pinned read-back slot");
  if (!h->d_bflags) {
    CK(dalloc(&h->d_bflags, 4 * 4));
    CK(dalloc(&h->d_brec, kBatch * 2 * 8));
  }
  unsigned long long* rec = h->h_misc;  // the handle's pinned slot
  while (static_cast<int>(h->bev.size()) < 2 * kBatch + 1) {
    cudaEvent_t e = nullptr;
    CK(cudaEventCreate(&e));
    h->bev.push_back(e);
  }
  sb::UnionArgs base{};
  hb_union_args(h, base);
  base.stop = h->d_bflags;
  while (!h->finished) {
    int K = kBatch;
    if (h->depth) K = std::min<int>(K, static_cast<int>(h->depth - h->t));
    CK(cudaMemsetAsync(h->d_bflags, 0, 4 * 4, h->stream));
    CK(cudaMemsetAsync(h->d_misc, 0, 4 * 8, h->stream));
    CK(cudaEventRecord(h->bev[2 * kBatch], h->stream));
    int L = h->latest;
    for (int i = 0; i < K; ++i) {
      const int N = 1 - L;
      const uint32_t t = h->t + 1 + i;
      CK(sb::launch_clear_flags(h->d_bflags, h->d_changed[N] + g->v0, g->n_local, h->stream));
      CK(cudaEventRecord(h->bev[2 * i], h->stream));
      if (g->n_local) {
        sb::UnionArgs u = base;
        u.cur = h->d_plane[L];
        u.next = h->d_plane[N];
        u.changed_out = h->d_changed[N];
        u.changed_in = h->d_changed[L];
        u.work = h->d_misc;
        CK(sb::launch_union(static_cast<int>(h->p), false, u, h->stream));
      }
      CK(cudaEventRecord(h->bev[2 * i + 1], h->stream));
      if (g->n_local) {
        sb::EstArgs e{};
        e.plane = h->d_plane[N];
        e.node_begin = g->v0;
        e.n_local = g->n_local;
        e.lc = h->d_lc;
        e.alpha = h->alpha;
        e.m = static_cast<double>(1u << h->p);
        e.c_prev = h->d_c[L];
        e.c_cur = h->d_c[N];
        e.sum_d = h->d_sum_d;
        e.sum_d2 = h->d_sum_d2;
        e.changed = h->d_changed[N];
        e.t = t;
        e.max_ord = h->d_misc + 1;
        e.changed_count = h->d_misc + 2;
        e.stop = h->d_bflags;
        CK(sb::launch_estimate(static_cast<int>(h->p), 1, e, h->stream));
      }
      CK(sb::launch_clear_flags(h->d_bflags, h->d_changed[L], g->n, h->stream));  // consumed flags
      CK(sb::launch_decide(h->d_misc, h->d_bflags, h->d_brec + 2 * i, t, h->depth, h->stream));
      L = N;
    }
    CK(cudaMemcpyAsync(rec, h->d_brec, K * 2 * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(rec + 2 * kBatch, h->d_bflags, 4 * 4, cudaMemcpyDeviceToHost, h->stream));
    CK(sync_stream(h->stream));
    const unsigned int* fl = reinterpret_cast<const unsigned int*>(rec + 2 * kBatch);
    const int ran = fl[0] ? static_cast<int>(fl[1] - h->t) : K;
    for (int i = 0; i < ran; ++i) {
      sb_iter_stats st{};
      st.t = h->t + 1 + i;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, h->bev[2 * i], h->bev[2 * i + 1]);
      st.union_ms = ms;
      if (i + 1 < K) {
        cudaEventElapsedTime(&ms, h->bev[2 * i + 1], h->bev[2 * i + 2]);
        st.estimate_ms = ms;
      }
      cudaEventElapsedTime(&ms, i ? h->bev[2 * i - 1] : h->bev[2 * kBatch], h->bev[2 * i + 1]);
      st.step_ms = ms;
      st.changed_nodes = rec[2 * i + 1];
      st.max_increase = decode_ord(rec[2 * i]);
      h->stats.push_back(st);
    }
    h->t += static_cast<uint32_t>(ran);
    h->latest = (h->latest + ran) & 1;
    h->converged = fl[0] && fl[2];
    h->finished = fl[0] != 0;
  }
  return SB_OK;
}

extern "C" {

int sb_hb_run(sb_hb* h, uint32_t* iterations, int* converged) {
  if (!h) return fail(SB_EINVAL, "NULL handle");
  bool done = false;
  if (const int rc = pipelined_run(h, &done)) return rc;
  if (const int rc = ensure_interval_ready(h)) return rc;
  if (!h->finished && !h->computed && !h->comm && !h->npeers && !h->g->pending && !h->g->broken &&
      !(h->flags & (SB_HB_INTERVAL | SB_HB_SKIP_UNCHANGED))) {
    if (const int rc = batched_run(h)) return rc;
  }
  int conv = 0, fin = h->finished ? 1 : 0;
  while (!fin) {
    const int rc = sb_hb_step(h, nullptr, &conv, &fin);
    if (rc) return rc;
  }
  if (iterations) *iterations = h->t;
  if (converged) *converged = h->converged;
  return SB_OK;
}

static int ensure_tmp(sb_hb* h, uint64_t bytes) {
  if (h->tmp_bytes >= bytes) return SB_OK;
  dfree(h->d_tmp);
  h->tmp_bytes = 0;
  CK(dalloc(&h->d_tmp, bytes));
  h->tmp_bytes = bytes;
  return SB_OK;
}

int sb_hb_read_registers(const sb_hb* hc, int which, uint64_t v0, uint64_t v1, uint8_t* dst) {
  sb_hb* h = const_cast<sb_hb*>(hc);
  if (!h || !dst) return fail(SB_EINVAL, "NULL argument");
  if (v0 > v1 || v1 > h->g->n) return fail(SB_EINVAL, "bad row range");
  if (which != SB_REGS_LATEST && which != SB_REGS_PREVIOUS) return fail(SB_EINVAL, "bad plane selector");
  if (v0 == v1) return SB_OK;
  DeviceGuard dg(h->g->device);
  const int idx = which == SB_REGS_LATEST ? h->latest : 1 - h->latest;
  const uint64_t bytes = (v1 - v0) * h->row;
  int rc = ensure_tmp(h, bytes);
  if (rc) return rc;
  CK(sb::launch_to_packed(static_cast<int>(h->p), h->d_plane[idx] + v0 * h->row, h->d_tmp, v1 - v0, h->stream));
  CK(cudaMemcpyAsync(dst, h->d_tmp, bytes, cudaMemcpyDeviceToHost, h->stream));
  CK(sync_stream(h->stream));
  return SB_OK;
}

int sb_hb_set_registers(sb_hb* h, const uint8_t* packed) {
  if (!h || !packed) return fail(SB_EINVAL, "NULL argument");
  if (h->computed) return fail(SB_EINVAL, "set_registers during a step");
  sb_graph* g = h->g;
  DeviceGuard dg(g->device);
  const uint64_t bytes = g->n * h->row;
  int rc = ensure_tmp(h, bytes);
  if (rc) return rc;
  const int L = h->latest;
  CK(cudaMemcpyAsync(h->d_tmp, packed, bytes, cudaMemcpyHostToDevice, h->stream));
  CK(sb::launch_from_packed(static_cast<int>(h->p), h->d_tmp, h->d_plane[L], g->n, h->stream));
  CK(cudaMemsetAsync(h->d_changed[L], 1, g->n, h->stream));
  if (g->n_local) {
    sb::EstArgs e{};
    e.plane = h->d_plane[L];
    e.node_begin = g->v0;
    e.n_local = g->n_local;
    e.lc = h->d_lc;
    e.alpha = h->alpha;
    e.m = static_cast<double>(1u << h->p);
    e.c_cur = h->d_c[L];
    CK(sb::launch_estimate(static_cast<int>(h->p), 0, e, h->stream));
  }
  CK(sync_stream(h->stream));
  h->finished = h->converged = false;
  return SB_OK;
}

int sb_hb_read_state(const sb_hb* h, double* c_latest, double* c_previous, double* sum_d,
                     double* sum_d2, uint8_t* changed, uint32_t* t, int* converged, int* finished) {
  if (!h) return fail(SB_EINVAL, "NULL handle");
  const sb_graph* g = h->g;
  DeviceGuard dg(g->device);
  CK(sync_stream(h->stream));  // work still queued on the handle (e.g. a reset)
  const uint64_t nb = g->n_local * 8;
  if (g->n_local) {
    if (c_latest) CK(cudaMemcpy(c_latest, h->d_c[h->latest], nb, cudaMemcpyDeviceToHost));
    if (c_previous) CK(cudaMemcpy(c_previous, h->d_c[1 - h->latest], nb, cudaMemcpyDeviceToHost));
    if (sum_d) CK(cudaMemcpy(sum_d, h->d_sum_d, nb, cudaMemcpyDeviceToHost));
    if (sum_d2) CK(cudaMemcpy(sum_d2, h->d_sum_d2, nb, cudaMemcpyDeviceToHost));
    if (changed) CK(cudaMemcpy(changed, h->d_changed[h->latest] + g->v0, g->n_local, cudaMemcpyDeviceToHost));
  }
  if (t) *t = h->t;
  if (converged) *converged = h->converged;
  if (finished) *finished = h->finished;
  return SB_OK;
}

int sb_hb_metrics(const sb_hb* hc, const uint32_t* nv, const uint32_t* deg, double* md, double* ihh,
                  double* tekl, double* pv, double* m1, double* m2) {
  sb_hb* h = const_cast<sb_hb*>(hc);
  if (!h || !nv || !deg) return fail(SB_EINVAL, "NULL argument");
  const uint64_t n = h->g->n_local;
  if (!n) return SB_OK;
  DeviceGuard dg(h->g->device);
  // one device block: [nv u32 | deg u32 | 6 x f64 outputs]
  const uint64_t bytes = n * 8 + 6 * n * 8;
  int rc = ensure_tmp(h, bytes);
  if (rc) return rc;
  uint32_t* d_nv = reinterpret_cast<uint32_t*>(h->d_tmp);
  uint32_t* d_deg = d_nv + n;
  double* o = reinterpret_cast<double*>(h->d_tmp + n * 8);
  CK(cudaMemcpyAsync(d_nv, nv, n * 4, cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(d_deg, deg, n * 4, cudaMemcpyHostToDevice, h->stream));
  sb::MetricArgs a{};
  a.n = n;
  a.sum_d = h->d_sum_d;
  a.sum_d2 = h->d_sum_d2;
  a.nv = d_nv;
  a.deg = d_deg;
  a.md = o;
  a.ihh = o + n;
  a.tekl = o + 2 * n;
  a.pv = o + 3 * n;
  a.m1 = o + 4 * n;
  a.m2 = o + 5 * n;
  CK(sb::launch_metrics(a, h->stream));
  double* outs[6] = {md, ihh, tekl, pv, m1, m2};
  for (int i = 0; i < 6; ++i)
    if (outs[i]) CK(cudaMemcpyAsync(outs[i], o + i * n, n * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(sync_stream(h->stream));
  return SB_OK;
}

int sb_hb_stats(const sb_hb* h, sb_iter_stats* out, uint32_t cap, uint32_t* count) {
  if (!h) return fail(SB_EINVAL, "NULL handle");
  const uint32_t n = static_cast<uint32_t>(h->stats.size());
  if (out)
    for (uint32_t i = 0; i < n && i < cap; ++i) out[i] = h->stats[i];
  if (count) *count = n;
  return SB_OK;
}

void sb_hb_destroy(sb_hb* h) { delete h; }

// ------------------------------------------------------------------ NCCL
int sb_comm_unique_id(void* id_out) {
  if (!id_out) return fail(SB_EINVAL, "NULL id");
  static_assert(sizeof(ncclUniqueId) == SB_COMM_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  NK(ncclGetUniqueId(&id));
  memcpy(id_out, &id, sizeof(id));
  return SB_OK;
}

int sb_comm_create(int nranks, int rank, const void* id, int device, sb_comm** out) {
  if (!out || !id) return fail(SB_EINVAL, "NULL argument");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SB_EINVAL, "bad rank/nranks");
  DeviceGuard dg(device);
  auto* c = new sb_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  const ncclResult_t r = ncclCommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    c->comm = nullptr;
    delete c;
    return fail(SB_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  *out = c;
  return SB_OK;
}

int sb_hb_attach_comm(sb_hb* h, sb_comm* c, const uint64_t* bounds) {
  if (!h || !c || !bounds) return fail(SB_EINVAL, "NULL argument");
  if (bounds[0] != 0 || bounds[c->nranks] != h->g->n) return fail(SB_EINVAL, "bounds must cover [0, N)");
  for (int r = 0; r < c->nranks; ++r)
    if (bounds[r + 1] < bounds[r]) return fail(SB_EINVAL, "bounds not monotone");
  if (bounds[c->rank] != h->g->v0 || bounds[c->rank + 1] != h->g->v1)
    return fail(SB_EINVAL, "graph range does not match this rank's bounds");
  if (c->device != h->g->device) return fail(SB_EINVAL, "communicator device != graph device");
  h->comm = c;
  h->bounds.assign(bounds, bounds + c->nranks + 1);
  return SB_OK;
}

void sb_comm_destroy(sb_comm* c) { delete c; }

// ------------------------------------------------------------------ fused P2P exchange
// Pool memory cannot be exported with cudaIpcGetMemHandle: on first export the
// planes and changed flags move to cudaMalloc blocks (contents copied).
static int make_planes_ipc(sb_hb* h) {
  if (h->planes_ipc) return SB_OK;
  const uint64_t sizes[2] = {h->g->n * h->row + 64, h->g->n};
  uint8_t** bufs[4] = {&h->d_plane[0], &h->d_plane[1], &h->d_changed[0], &h->d_changed[1]};
  uint8_t* fresh[4] = {nullptr, nullptr, nullptr, nullptr};
  for (int k = 0; k < 4; ++k) {
    const cudaError_t e = dalloc_ipc(&fresh[k], sizes[k / 2]);
    if (e != cudaSuccess) {
      for (auto& f : fresh) dfree_ipc(f);
      return cuda_fail(e, "cudaMalloc (IPC-exportable planes)");
    }
  }
  for (int k = 0; k < 4; ++k) CK(cudaMemcpyAsync(fresh[k], *bufs[k], sizes[k / 2], cudaMemcpyDeviceToDevice, h->stream));
  CK(sync_stream(h->stream));
  for (int k = 0; k < 4; ++k) {
    dfree(*bufs[k]);
    *bufs[k] = fresh[k];
  }
  h->planes_ipc = true;
  return SB_OK;
}

int sb_hb_ipc_handles(const sb_hb* hc, void* out, size_t cap) {
  sb_hb* h = const_cast<sb_hb*>(hc);
  if (!h || !out) return fail(SB_EINVAL, "NULL argument");
  if (cap < SB_IPC_HANDLE_BYTES) return fail(SB_EINVAL, "handle buffer too small (%d bytes needed)", SB_IPC_HANDLE_BYTES);
  static_assert(sizeof(cudaIpcMemHandle_t) * 4 == SB_IPC_HANDLE_BYTES, "ipc handle size");
  DeviceGuard dg(h->g->device);
  if (h->computed) return fail(SB_EINVAL, "ipc_handles during a step");
  if (const int rc = make_planes_ipc(h)) return rc;
  cudaIpcMemHandle_t hs[4];
  CK(cudaIpcGetMemHandle(&hs[0], h->d_plane[0]));
  CK(cudaIpcGetMemHandle(&hs[1], h->d_plane[1]));
  CK(cudaIpcGetMemHandle(&hs[2], h->d_changed[0]));
  CK(cudaIpcGetMemHandle(&hs[3], h->d_changed[1]));
  memcpy(out, hs, sizeof(hs));
  return SB_OK;
}

int sb_hb_attach_peers(sb_hb* h, int nranks, int rank, const void* handles, const uint64_t* bounds) {
  if (!h || !handles || !bounds) return fail(SB_EINVAL, "NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SB_EINVAL, "bad rank/nranks");
  if (h->npeers) return fail(SB_EINVAL, "peers already attached");
  if (bounds[0] != 0 || bounds[nranks] != h->g->n) return fail(SB_EINVAL, "bounds must cover [0, N)");
  if (bounds[rank] != h->g->v0 || bounds[rank + 1] != h->g->v1)
    return fail(SB_EINVAL, "graph range does not match this rank's bounds");
  DeviceGuard dg(h->g->device);
  std::vector<uint8_t*> pl[2], ch[2];
  const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
  for (int r = 0; r < nranks; ++r) {
    if (r == rank) continue;
    void* q[4];
    for (int k = 0; k < 4; ++k) {
      CK(cudaIpcOpenMemHandle(&q[k], hs[4 * r + k], cudaIpcMemLazyEnablePeerAccess));
      h->ipc_opened.push_back(q[k]);
    }
    pl[0].push_back(static_cast<uint8_t*>(q[0]));
    pl[1].push_back(static_cast<uint8_t*>(q[1]));
    ch[0].push_back(static_cast<uint8_t*>(q[2]));
    ch[1].push_back(static_cast<uint8_t*>(q[3]));
  }
  const int np = nranks - 1;
  for (int i = 0; i < 2; ++i) {
    CK(dalloc(&h->d_peer_plane[i], std::max(np, 1) * sizeof(uint8_t*)));
    CK(dalloc(&h->d_peer_chg[i], std::max(np, 1) * sizeof(uint8_t*)));
    if (np) {
      CK(cudaMemcpy(h->d_peer_plane[i], pl[i].data(), np * sizeof(uint8_t*), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(h->d_peer_chg[i], ch[i].data(), np * sizeof(uint8_t*), cudaMemcpyHostToDevice));
    }
  }
  h->npeers = np;
  h->bounds.assign(bounds, bounds + nranks + 1);
  return SB_OK;
}


}  // extern "C"
