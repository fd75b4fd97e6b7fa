// sb_graph_api.cu -- C-ABI: device graphs (upload, asynchronous chunked upload,
// on-device grid build), their validation, work items and run index.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "sb_device.cuh"
#include "sb_handles.h"

// ------------------------------------------------------------------ run index
// Runs of consecutive ids per work item (interval mode, exact mode, local
// metrics), decoded once from the device-resident stream: count pass, device
// scan of offsets, fill pass.  Also sets g->max_run (longest run within a work
// item; sizes the interval mode's sparse table).
static void rix_free(RunIndexJob& j) {
  dfree(j.d_cnt);
  dfree(j.d_aux);
  for (cudaEvent_t e : j.ready) cudaEventDestroy(e);
  j.ready.clear();
  if (j.s) {
    cudaStreamSynchronize(j.s);
    cudaStreamDestroy(j.s);
    j.s = nullptr;
  }
}

void rix_abort(sb_graph* g, RunIndexJob& j) {
  rix_free(j);
  g->free_retired_runs();
  dfree(g->d_run_off);
  dfree(g->d_run_s);
  dfree(g->d_run_e);
  g->n_runs = 0;
}

static int rix_setup(sb_graph* g, RunIndexJob& j) {
  if (reinterpret_cast<uintptr_t>(g->d_stream) & 15) return fail(SB_ERUNTIME, "internal: stream not 16-B aligned");
  sb::RunIndexArgs& a = j.a;
  a = sb::RunIndexArgs{};
  a.stream = g->d_stream;
  a.stream_len = g->stream_local;
  a.item_off = g->d_item_off;
  a.item_base = g->d_item_base;
  a.item_count = g->d_item_count;
  a.n_items = g->n_items;
  a.item_begin = 0;
  a.item_end = g->n_items;
  a.range_end_byte = g->stream_local;
  CK(dalloc(&j.d_cnt, g->n_items * 8 + 8));
  CK(dalloc(&j.d_aux, 2 * 8));
  CK(dalloc(&g->d_run_off, (g->n_items + 1) * 8));
  a.run_count = j.d_cnt;
  a.max_run = reinterpret_cast<unsigned int*>(j.d_cnt + g->n_items);
  CK(cudaMemsetAsync(a.max_run, 0, 4, 0));
  CK(cudaMemsetAsync(j.d_aux, 0, 16, 0));
  CK(sync_stream(0));
  return SB_OK;
}

int rix_begin(sb_graph* g, RunIndexJob& j) {
  if (const int rc = rix_setup(g, j)) return rc;
  CK(cudaStreamCreateWithFlags(&j.s, cudaStreamNonBlocking));
  j.a.err = g->d_err;
  const size_t nk = g->chunk_item.size() - 1;
  j.probe = std::min<size_t>(1, nk - 1);  // chunk 0 is the small 1/64 one
  j.ready.assign(nk, nullptr);
  for (auto& e : j.ready) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return SB_OK;
}

static int rix_fill(sb_graph* g, RunIndexJob& j, size_t k_end) {  // fills chunks [filled, k_end)
  if (k_end <= j.filled) return SB_OK;
  sb::RunIndexArgs f = j.a;
  f.item_begin = g->chunk_item[j.filled];
  f.item_end = g->chunk_item[k_end];
  f.range_end_byte = g->chunk_byte[k_end];  // the next chunk's items are not cut yet
  f.run_off = g->d_run_off;
  f.run_s = g->d_run_s;
  f.run_e = g->d_run_e;
  f.run_cap = j.cap;
  f.overflow = reinterpret_cast<unsigned int*>(j.d_aux + 1);
  if (f.item_end > f.item_begin) CK(sb::launch_run_index(f, true, j.s));
  for (size_t k = j.filled; k < k_end; ++k) CK(cudaEventRecord(j.ready[k], j.s));
  j.filled = k_end;
  return SB_OK;
}

// Chunk k (after its validation): count + offsets, then the run total so far
// is read back (the count of one chunk is short; the host is waiting for the
// next chunk's copy anyway).  The first full-size chunk sizes the run storage
// from the runs per stream byte so far (x 1.25 + slack) and the chunks so far
// are written; a later chunk that would not fit grows it (runs written so far
// are copied over on j.s, and the chunks' ready events re-recorded after the
// copy, so a pass launched later reads the new storage only once it holds
// them; the old storage stays alive for the passes already launched on it).
int rix_chunk(sb_graph* g, RunIndexJob& j, size_t k) {
  sb::RunIndexArgs& a = j.a;
  const size_t nk = g->chunk_item.size() - 1;
  a.item_begin = g->chunk_item[k];
  a.item_end = g->chunk_item[k + 1];
  a.range_end_byte = g->chunk_byte[k + 1];
  CK(cudaStreamWaitEvent(j.s, g->val_ev[k], 0));
  if (a.item_end > a.item_begin) {
    CK(sb::launch_run_index(a, false, j.s));
    CK(sb::launch_run_offsets(j.d_cnt, g->d_run_off, a.item_begin, a.item_end, j.d_aux, j.s));
  }
  if (j.failed || (!j.cap && k < j.probe && k + 1 < nk)) return SB_OK;
  unsigned long long tot = 0, err = 0;
  CK(cudaMemcpyAsync(&tot, j.d_aux, 8, cudaMemcpyDeviceToHost, j.s));
  CK(cudaMemcpyAsync(&err, g->d_err, 8, cudaMemcpyDeviceToHost, j.s));  // validation of chunks <= k is done
  CK(sync_stream(j.s));
  // a malformed chunk: the count pass stopped early, so the totals are garbage;
  // write nothing more (the upload reports the error, the index is discarded).
  // A valid stream never holds more runs than bytes.
  if (err != ~0ull || tot > g->stream_local + g->n_items) {
    j.failed = true;
    return SB_OK;
  }
  if (tot > j.cap) {
    const uint64_t bytes = std::max<uint64_t>(g->chunk_byte[k + 1], 1);
    uint64_t cap = static_cast<uint64_t>(static_cast<double>(tot) / static_cast<double>(bytes) *
                                         static_cast<double>(g->stream_local) * 1.25) + g->n_items + 1024;
    if (j.cap) cap = std::max<uint64_t>(cap, 2 * j.cap);
    uint32_t* s = nullptr;
    uint32_t* e = nullptr;
    CK(dalloc(&s, cap * 4));
    if (const cudaError_t ce = dalloc(&e, cap * 4)) {
      dfree(s);
      CK(ce);
    }
    if (j.cap) {  // a grown store: the runs written so far move over
      CK(cudaMemcpyAsync(s, g->d_run_s, j.cap * 4, cudaMemcpyDeviceToDevice, j.s));
      CK(cudaMemcpyAsync(e, g->d_run_e, j.cap * 4, cudaMemcpyDeviceToDevice, j.s));
      for (size_t kk = 0; kk < j.filled; ++kk) CK(cudaEventRecord(j.ready[kk], j.s));
      g->retired_runs.push_back(g->d_run_s);
      g->retired_runs.push_back(g->d_run_e);
      ++j.grown;
    }
    g->d_run_s = s;
    g->d_run_e = e;
    j.cap = cap;
  }
  return rix_fill(g, j, k + 1);
}

int rix_finish(sb_graph* g, RunIndexJob& j, bool* overflow) {
  *overflow = false;
  CK(sync_stream(j.s));
  unsigned long long aux[2] = {0, 0};
  CK(cudaMemcpy(aux, j.d_aux, 16, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&g->max_run, j.a.max_run, 4, cudaMemcpyDeviceToHost));
  g->n_runs = aux[0];
  CK(cudaMemcpy(g->d_run_off + g->n_items, &aux[0], 8, cudaMemcpyHostToDevice));
  *overflow = aux[1] != 0 || j.filled + 1 < g->chunk_item.size();
  rix_free(j);
  return SB_OK;
}

int build_run_index(sb_graph* g) {
  if (g->d_run_off || g->n_items == 0) return SB_OK;
  if (g->broken) return fail(SB_ERUNTIME, "cgraph: the graph failed validation at upload");
  RunIndexJob j;
  if (g->pending && g->chunk_item.size() > 2) {
    // still uploading: the index is built chunk by chunk under the PCIe copies
    int rc = rix_begin(g, j);
    for (size_t k = 0; k + 1 < g->chunk_item.size() && !rc; ++k) rc = rix_chunk(g, j, k);
    if (!rc) rc = graph_wait(g);
    bool overflow = false;
    if (!rc) rc = rix_finish(g, j, &overflow);
    if (rc) {
      rix_abort(g, j);
      return rc;
    }
    if (!overflow) {
      g->free_retired_runs();  // no pass reads the outgrown storage here
      return SB_OK;
    }
    rix_abort(g, j);  // storage estimate too small: rebuild with exact storage
  }
  if (const int rc = graph_wait(g)) return rc;
  int rc = rix_setup(g, j);
  sb::RunIndexArgs& a = j.a;
  auto done = [&](int r) {
    if (r) rix_abort(g, j);
    else rix_free(j);
    return r;
  };
  if (rc) return done(rc);
  cudaError_t e = sb::launch_run_index(a, false, 0);
  if (e == cudaSuccess) e = sb::launch_run_offsets(j.d_cnt, g->d_run_off, 0, g->n_items, j.d_aux, 0);
  unsigned long long tot = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&tot, j.d_aux, 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(&g->max_run, a.max_run, 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return done(cuda_fail(e, "run index count"));
  g->n_runs = tot;
  e = cudaMemcpy(g->d_run_off + g->n_items, &tot, 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = dalloc(&g->d_run_s, std::max<uint64_t>(g->n_runs, 1) * 4);
  if (e == cudaSuccess) e = dalloc(&g->d_run_e, std::max<uint64_t>(g->n_runs, 1) * 4);
  if (e != cudaSuccess) return done(cuda_fail(e, "run index storage"));
  a.run_off = g->d_run_off;
  a.run_s = g->d_run_s;
  a.run_e = g->d_run_e;
  e = sb::launch_run_index(a, true, 0);
  if (e == cudaSuccess) e = cudaStreamSynchronize(0);
  if (e != cudaSuccess) return done(cuda_fail(e, "run index fill"));
  return done(SB_OK);
}


extern "C" {

const char* sb_last_error(void) { return sb::last_error(); }
const char* sb_version(void) { return "sieveball-b200 0.1 (sm_100a)"; }

int sb_device_count(int* n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *n = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  *n = c;
  return SB_OK;
}

int sb_release_cached_memory(int device) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail(SB_EINVAL, "bad device %d", device);
  DeviceGuard dg(device);
  CK(cudaDeviceSynchronize());
  cudaMemPool_t pool;
  CK(cudaDeviceGetDefaultMemPool(&pool, device));
  CK(cudaMemPoolTrimTo(pool, 0));
  return SB_OK;
}

int sb_check_convergence(double max_increase) { return max_increase <= 0.5 ? 1 : 0; }

}  // extern "C"

// ------------------------------------------------------------------ graph
// Work items, CTA tiles and the upload-time validation of the device-resident
// stream slice (shared by sb_graph_create and the on-device grid builder).
static int graph_setup_host(sb_graph* g, const uint32_t* deg_local) {
  // Work items: <= chunk neighbours each, sized so the edge work splits into
  // ~4 items per resident warp (load balance) but stays >= 512 ids (decode
  // and merge amortisation; 128 measured no faster on C1).
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
  const uint64_t target = g->edges_local / (static_cast<uint64_t>(sms) * 64 * 4);
  g->chunk = static_cast<uint32_t>(std::min<uint64_t>(8192, std::max<uint64_t>(512, target)));
  std::vector<uint32_t> node_item(g->n_local + 1);
  uint64_t items = 0;
  for (uint64_t i = 0; i < g->n_local; ++i) {
    node_item[i] = static_cast<uint32_t>(items);
    const uint32_t d = deg_local[i];
    items += d ? (d + g->chunk - 1) / g->chunk : 1;
  }
  if (items > 0xffffffffull) return fail(SB_EINVAL, "too many work items");
  node_item[g->n_local] = static_cast<uint32_t>(items);
  g->n_items = items;
  // Tiles for the CTA schedule: group k = local nodes [8k, 8k+8), one tile per
  // chunk index up to the group's largest item count.
  std::vector<uint32_t> tn0, tq;
  for (uint64_t k = 0; k < g->n_local; k += 8) {
    uint32_t mx = 0;
    for (uint64_t i = k; i < std::min<uint64_t>(k + 8, g->n_local); ++i) mx = std::max(mx, node_item[i + 1] - node_item[i]);
    for (uint32_t q = 0; q < mx; ++q) {
      tn0.push_back(static_cast<uint32_t>(k));
      tq.push_back(q);
    }
  }
  g->n_tiles = tn0.size();
  CK(dalloc(&g->d_tile_node0, std::max<size_t>(tn0.size(), 1) * 4));
  CK(dalloc(&g->d_tile_q, std::max<size_t>(tq.size(), 1) * 4));
  if (!tn0.empty()) {
    CK(cudaMemcpy(g->d_tile_node0, tn0.data(), tn0.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(g->d_tile_q, tq.data(), tq.size() * 4, cudaMemcpyHostToDevice));
  }
  CK(dalloc(&g->d_node_item, node_item.size() * 4));
  CK(cudaMemcpy(g->d_node_item, node_item.data(), node_item.size() * 4, cudaMemcpyHostToDevice));
  g->h_node_item = std::move(node_item);
  const uint64_t ni = std::max<uint64_t>(items, 1);
  CK(dalloc(&g->d_item_off, ni * 8));
  CK(dalloc(&g->d_item_base, ni * 4));
  CK(dalloc(&g->d_item_count, ni * 4));
  CK(dalloc(&g->d_item_node, ni * 4));
  CK(dalloc(&g->d_node_lo, std::max<uint64_t>(g->n_local, 1) * 4));
  CK(dalloc(&g->d_node_hi, std::max<uint64_t>(g->n_local, 1) * 4));
  CK(dalloc(&g->d_err, 16));
  CK(cudaMemset(g->d_err, 0xff, 8));
  CK(cudaMemset(reinterpret_cast<uint8_t*>(g->d_err) + 8, 0, 8));
  return SB_OK;
}

// Upload-time validation of local nodes [n0, n1) (LEB128 well-formed, strictly
// increasing ids < n, exactly degrees[v] ids) + work items; errors land in d_err.
static cudaError_t launch_validate(sb_graph* g, uint64_t n0, uint64_t n1, cudaStream_t s) {
  if (n1 <= n0) return cudaSuccess;
  if (reinterpret_cast<uintptr_t>(g->d_stream) & 15) return cudaErrorMisalignedAddress;  // 16-B window loads
  sb::BuildArgs a{};
  a.stream = g->d_stream;
  a.row_off = g->d_rowoff;
  a.degrees = g->d_deg;
  a.n_local = g->n_local;
  a.n_global = g->n;
  a.node_begin = n0;
  a.node_end = n1;
  a.chunk = g->chunk;
  a.node_item = g->d_node_item;
  a.item_off = g->d_item_off;
  a.item_base = g->d_item_base;
  a.item_count = g->d_item_count;
  a.item_node = g->d_item_node;
  a.node_lo = g->d_node_lo;
  a.node_hi = g->d_node_hi;
  a.err_node = g->d_err;
  return sb::launch_build_items(a, s);
}

void graph_union_args(const sb_graph* g, sb::UnionArgs& u) {
  u.stream = g->d_stream;
  u.item_off = g->d_item_off;
  u.item_base = g->d_item_base;
  u.item_count = g->d_item_count;
  u.item_node = g->d_item_node;
  u.node_item = g->d_node_item;
  u.n_items = g->n_items;
  u.node_begin = g->v0;
  u.n_local = g->n_local;
  u.n_tiles = g->n_tiles;
  u.tile_node0 = g->d_tile_node0;
  u.tile_q = g->d_tile_q;
  u.row_off = g->d_rowoff;
  u.degrees = g->d_deg;
  u.node_lo = g->d_node_lo;
  u.node_hi = g->d_node_hi;
  // A group tile is one CTA's work: above half a resident CTA's fair share of
  // the slice's edges (SMs x 4 CTAs) it would stretch the launch's tail, so
  // such groups -- and every group of a small graph, where the per-node items
  // are what fills the machine -- take the per-node items.
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
  u.shared_max_edges = g->edges_local / (2ull * 4ull * static_cast<uint64_t>(sms));
  // fewer 16-node groups than resident CTAs: no group can qualify, so launch
  // the kernel without the group path (no per-tile group test; C1)
  if (g->n_local < 16ull * 4ull * static_cast<uint64_t>(sms)) u.node_lo = nullptr;
}

static int graph_check(sb_graph* g) {
  unsigned long long err = 0;
  CK(cudaMemcpy(&err, g->d_err, 8, cudaMemcpyDeviceToHost));
  if (err != ~0ull) {
    g->broken = 1;
    return fail(SB_ERUNTIME, "cgraph: malformed compressed row at node %llu (bad varint, "
                             "non-increasing or out-of-range id, or degree mismatch)",
                (unsigned long long)(err + g->v0));
  }
  return SB_OK;
}

// Work items, CTA tiles and the upload-time validation of the device-resident
// stream slice (shared by sb_graph_create and the on-device grid builder).
int graph_setup(sb_graph* g, const uint32_t* deg_local) {
  int rc = graph_setup_host(g, deg_local);
  if (rc) return rc;
  CK(launch_validate(g, 0, g->n_local, 0));
  CK(sync_stream(0));
  return graph_check(g);
}

// Completes an asynchronous upload (sb_graph_create_async): waits for every
// chunk's copy + validation and reports a malformed stream (sticky).
int graph_wait(sb_graph* g) {
  if (g->broken) return fail(SB_ERUNTIME, "cgraph: the graph failed validation at upload");
  if (!g->pending) return SB_OK;
  DeviceGuard dg(g->device);
  CK(sync_stream(g->up_stream));
  CK(sync_stream(g->val_stream));
  g->pending = false;
  return graph_check(g);
}

static int graph_create(uint64_t n, const uint64_t* offsets, const uint32_t* degrees, const uint8_t* stream,
                        uint64_t stream_len, const uint32_t* orig_id, uint64_t node_begin, uint64_t node_end,
                        int device, bool async, sb_graph** out) {
  if (!out) return fail(SB_EINVAL, "sb_graph_create: out is NULL");
  *out = nullptr;
  if (n == 0) return fail(SB_EINVAL, "hyperball: graph empty");
  if (n > 0xffffffffull) return fail(SB_EINVAL, "graph has more than 2^32 nodes");
  if (!offsets || !degrees || (stream_len && !stream))
    return fail(SB_EINVAL, "sb_graph_create: NULL array");
  if (node_begin > node_end || node_end > n) return fail(SB_EINVAL, "sb_graph_create: bad node range");
  if (offsets[n] != stream_len) return fail(SB_ERUNTIME, "cgraph: offsets[N] != stream length");
  for (uint64_t v = node_begin; v < node_end; ++v)
    if (offsets[v + 1] < offsets[v]) return fail(SB_ERUNTIME, "cgraph: offsets decrease at node %llu", (unsigned long long)v);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(SB_ECUDA, "no CUDA device: the HyperBall path has no CPU fallback");
  if (device < 0 || device >= ndev) return fail(SB_EINVAL, "bad device %d", device);
  DeviceGuard dg(device);
  auto* g = new sb_graph();
  g->device = device;
  g->n = n;
  g->v0 = node_begin;
  g->v1 = node_end;
  g->n_local = node_end - node_begin;
  const uint64_t b0 = offsets[node_begin], b1 = offsets[node_end];
  g->stream_local = b1 - b0;
  uint64_t edges = 0;
  for (uint64_t v = node_begin; v < node_end; ++v) edges += degrees[v];
  g->edges_local = edges;
  auto bail = [&](int rc) { delete g; return rc; };
#define GK(x)                                                 \
  do {                                                        \
    cudaError_t e_ = (x);                                     \
    if (e_ != cudaSuccess) return bail(cuda_fail(e_, #x));    \
  } while (0)
  // zero padding: the decoders read whole windows past a row's end (512-byte
  // steps + the next lane's word + alignment)
  GK(dalloc(&g->d_stream, g->stream_local + sb::kStreamPad));
  GK(cudaMemset(g->d_stream + g->stream_local, 0, sb::kStreamPad));
  if (g->stream_local && !async)
    GK(cudaMemcpy(g->d_stream, stream + b0, g->stream_local, cudaMemcpyHostToDevice));
  std::vector<uint64_t> ro(g->n_local + 1);
  for (uint64_t i = 0; i <= g->n_local; ++i) ro[i] = offsets[node_begin + i] - b0;
  GK(dalloc(&g->d_rowoff, ro.size() * 8));
  GK(cudaMemcpy(g->d_rowoff, ro.data(), ro.size() * 8, cudaMemcpyHostToDevice));
  GK(dalloc(&g->d_deg, std::max<uint64_t>(g->n_local, 1) * 4));
  if (g->n_local) GK(cudaMemcpy(g->d_deg, degrees + node_begin, g->n_local * 4, cudaMemcpyHostToDevice));
  if (orig_id) {
    GK(dalloc(&g->d_orig, n * 4));
    GK(cudaMemcpy(g->d_orig, orig_id, n * 4, cudaMemcpyHostToDevice));
  }
  if (!async) {
    const int rc = graph_setup(g, degrees + node_begin);
    if (rc) return bail(rc);
    *out = g;
    return SB_OK;
  }
  // Asynchronous: a small first chunk (1/64 of the bytes, so the first union
  // tiles start early) then K-1 chunks of ~equal stream bytes, on 16-node
  // (group path) boundaries; copy k on up_stream, validation k on val_stream after copy k.
  const int rc = graph_setup_host(g, degrees + node_begin);
  if (rc) return bail(rc);
  GK(cudaStreamCreateWithFlags(&g->up_stream, cudaStreamNonBlocking));
  GK(cudaStreamCreateWithFlags(&g->val_stream, cudaStreamNonBlocking));
  uint64_t kmax = 16;  // 16 / 24 / 32 / 48 / 64 measured: 16 is fastest at C3
#ifdef SB_AB_UPLOAD_CHUNKS  // A-B builds only (make -B NVEXTRA=-DSB_AB_UPLOAD_CHUNKS): no switch in the product .so
  if (const char* e = getenv("SB_UPLOAD_CHUNKS")) kmax = std::max(1, std::min(256, atoi(e)));
#endif
  const int K = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(kmax, g->n_local / 64)));
  const uint64_t first = K > 1 ? g->stream_local / 64 : 0;
  g->chunk_node.assign(1, 0);
  for (int k = 1; k < K; ++k) {
    const uint64_t goal = b0 + first + (g->stream_local - first) * (k - 1) / (K - 1);
    uint64_t v = std::lower_bound(offsets + node_begin, offsets + node_end, goal) - (offsets + node_begin);
    v = std::min<uint64_t>(v & ~15ull, g->n_local);  // whole 16-node groups per chunk
    if (v > g->chunk_node.back()) g->chunk_node.push_back(v);
  }
  if (g->chunk_node.back() != g->n_local) g->chunk_node.push_back(g->n_local);
  // tile ranges: tiles are ordered by 8-node group (chunks hold whole 16-node groups)
  std::vector<uint32_t> tn0(g->n_tiles);
  if (g->n_tiles) GK(cudaMemcpy(tn0.data(), g->d_tile_node0, g->n_tiles * 4, cudaMemcpyDeviceToHost));
  g->chunk_tile.clear();
  for (uint64_t cn : g->chunk_node)
    g->chunk_tile.push_back(std::lower_bound(tn0.begin(), tn0.end(), static_cast<uint32_t>(std::min<uint64_t>(cn, 0xffffffffull))) - tn0.begin());
  g->chunk_tile.back() = g->n_tiles;
  g->chunk_item.clear();
  g->chunk_byte.clear();
  for (uint64_t cn : g->chunk_node) {
    g->chunk_item.push_back(g->h_node_item[cn]);
    g->chunk_byte.push_back(offsets[node_begin + cn] - b0);  // slice-relative start of the chunk's bytes
  }
  const size_t nk = g->chunk_node.size() - 1;
  GK(dalloc(&g->d_chunk_rng, nk * 2 * 4));
  g->val_ev.resize(nk, nullptr);
  for (size_t k = 0; k < nk; ++k) {
    cudaEvent_t copied = nullptr;
    GK(cudaEventCreateWithFlags(&g->val_ev[k], cudaEventDisableTiming));
    GK(cudaEventCreateWithFlags(&copied, cudaEventDisableTiming));
    const uint64_t s0 = ro[g->chunk_node[k]], s1 = ro[g->chunk_node[k + 1]];
    if (s1 > s0) GK(cudaMemcpyAsync(g->d_stream + s0, stream + b0 + s0, s1 - s0, cudaMemcpyHostToDevice, g->up_stream));
    GK(cudaEventRecord(copied, g->up_stream));
    GK(cudaStreamWaitEvent(g->val_stream, copied, 0));
    cudaEventDestroy(copied);  // released once the wait is enqueued
    GK(launch_validate(g, g->chunk_node[k], g->chunk_node[k + 1], g->val_stream));
    GK(sb::launch_chunk_range(g->d_node_lo, g->d_node_hi, g->chunk_node[k], g->chunk_node[k + 1],
                              g->d_chunk_rng + 2 * k, g->val_stream));
    GK(cudaEventRecord(g->val_ev[k], g->val_stream));
  }
  g->pending = true;
#undef GK
  *out = g;
  return SB_OK;
}

extern "C" {

int sb_graph_create(uint64_t n, const uint64_t* offsets, const uint32_t* degrees, const uint8_t* stream,
                    uint64_t stream_len, const uint32_t* orig_id, uint64_t node_begin, uint64_t node_end,
                    int device, sb_graph** out) {
  return graph_create(n, offsets, degrees, stream, stream_len, orig_id, node_begin, node_end, device, false, out);
}

int sb_graph_create_async(uint64_t n, const uint64_t* offsets, const uint32_t* degrees, const uint8_t* stream,
                          uint64_t stream_len, const uint32_t* orig_id, uint64_t node_begin, uint64_t node_end,
                          int device, sb_graph** out) {
  return graph_create(n, offsets, degrees, stream, stream_len, orig_id, node_begin, node_end, device, true, out);
}

int sb_graph_wait(sb_graph* g) {
  if (!g) return fail(SB_EINVAL, "NULL graph");
  return graph_wait(g);
}

// ------------------------------------------------------------------ on-device graph build
// Grid -> visibility -> delta-LEB128 CSR entirely in HBM (sb_vis.cu), then the
// same work-item setup and validation as an uploaded graph.
int sb_graph_build_grid(uint32_t rows, uint32_t cols, const uint8_t* blocked, uint64_t radius2, int device,
                        sb_graph** out) {
  if (!out) return fail(SB_EINVAL, "sb_graph_build_grid: out is NULL");
  *out = nullptr;
  if (rows == 0 || cols == 0) return fail(SB_EINVAL, "grid: rows and cols must be >= 1");
  if (!blocked) return fail(SB_EINVAL, "sb_graph_build_grid: NULL mask");
  const uint64_t cells = static_cast<uint64_t>(rows) * cols;
  if (cells >= 0xffffffffull) return fail(SB_EINVAL, "grid: more than 2^32 - 1 cells");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(SB_ECUDA, "no CUDA device: the HyperBall path has no CPU fallback");
  if (device < 0 || device >= ndev) return fail(SB_EINVAL, "bad device %d", device);
  DeviceGuard dg(device);
  auto* g = new sb_graph();
  g->device = device;
  g->rows = rows;
  g->cols = cols;
  uint8_t* d_mask = nullptr;
  uint32_t *d_pref = nullptr, *d_scan = nullptr, *d_noc = nullptr, *d_tmp = nullptr;
  uint64_t *d_bytes = nullptr, *d_steps = nullptr, *d_stepoff = nullptr;
  uint32_t* d_masks = nullptr;
  auto cleanup = [&] {
    dfree(d_mask); dfree(d_pref); dfree(d_scan); dfree(d_noc); dfree(d_tmp); dfree(d_bytes);
    dfree(d_steps); dfree(d_stepoff); dfree(d_masks);
  };
  auto bail = [&](int rc) { cleanup(); delete g; return rc; };
#define BK(x)                                                 \
  do {                                                        \
    cudaError_t e_ = (x);                                     \
    if (e_ != cudaSuccess) return bail(cuda_fail(e_, #x));    \
  } while (0)
  cudaStream_t s = 0;
  BK(dalloc(&d_mask, cells));
  BK(cudaMemcpy(d_mask, blocked, cells, cudaMemcpyHostToDevice));
  BK(dalloc(&d_pref, static_cast<uint64_t>(rows + 1) * (cols + 1) * 4));
  BK(dalloc(&d_scan, 2 * cells * 4));
  sb::VisArgs a{};
  a.rows = rows;
  a.cols = cols;
  a.radius2 = radius2;
  a.blocked = d_mask;
  a.pref = d_pref;
  uint64_t n = 0;
  BK(sb::launch_vis_prepare(a, d_pref, d_scan, &n, s));
  if (n == 0) return bail(fail(SB_ERUNTIME, "grid: zero active cells"));
  g->n = n;
  g->v0 = 0;
  g->v1 = n;
  g->n_local = n;
  BK(dalloc(&d_noc, cells * 4));
  BK(dalloc(&g->d_cell, n * 4));
  BK(sb::launch_vis_maps(a, d_scan, d_noc, g->d_cell, s));
  a.node_of_cell = d_noc;
  a.cell_of_node = g->d_cell;
  a.n = n;
  if (radius2) {  // isqrt64 as the host generator
    uint64_t r = static_cast<uint64_t>(std::sqrt(static_cast<double>(radius2)));
    while (r * r > radius2) --r;
    while ((r + 1) * (r + 1) <= radius2) ++r;
    a.R = static_cast<int64_t>(r);
  } else {
    a.R = std::max(rows, cols);
  }
  // Line-of-sight results of the count pass are kept (one mask word per warp
  // step) so the write pass does not walk them again; skipped if HBM is short.
  if (dalloc(&d_steps, (n + 1) * 8) == cudaSuccess && dalloc(&d_stepoff, (n + 1) * 8) == cudaSuccess) {
    BK(cudaMemsetAsync(d_steps + n, 0, 8, s));
    BK(sb::launch_vis_steps(a, d_steps, s));
    BK(sb::launch_scan_u64(d_steps, d_stepoff, n + 1, s));
    uint64_t words = 0;
    BK(cudaMemcpy(&words, d_stepoff + n, 8, cudaMemcpyDeviceToHost));
    if (dalloc(&d_masks, std::max<uint64_t>(words, 1) * 4) == cudaSuccess) {
      a.masks = d_masks;
      a.step_off = d_stepoff;
    } else {
      cudaGetLastError();  // clear the allocation failure; the write pass recomputes instead
    }
  } else {
    cudaGetLastError();
  }
  auto free_masks = [&] { dfree(d_masks); dfree(d_steps); dfree(d_stepoff); a.masks = nullptr; a.step_off = nullptr; };
  BK(dalloc(&g->d_deg, n * 4));
  BK(dalloc(&d_bytes, (n + 1) * 8));
  BK(cudaMemsetAsync(d_bytes + n, 0, 8, s));
  a.deg = g->d_deg;
  a.bytes = d_bytes;
  BK(sb::launch_vis_rows(a, false, s));
  BK(dalloc(&g->d_rowoff, (n + 1) * 8));
  BK(sb::launch_scan_u64(d_bytes, g->d_rowoff, n + 1, s));
  uint64_t total = 0;
  BK(cudaMemcpy(&total, g->d_rowoff + n, 8, cudaMemcpyDeviceToHost));
  g->stream_local = total;
  BK(dalloc(&g->d_stream, total + sb::kStreamPad));
  BK(cudaMemsetAsync(g->d_stream + total, 0, sb::kStreamPad, s));
  a.offsets = g->d_rowoff;
  a.stream = g->d_stream;
  BK(sb::launch_vis_rows(a, true, s));
  BK(cudaStreamSynchronize(s));
  free_masks();
  // components (the 2n scratch doubles as the union-find parent array + ranks)
  BK(dalloc(&d_tmp, 3 * n * 4));
  BK(dalloc(&g->d_comp, n * 4));
  BK(dalloc(&g->d_comp_sizes, n * 4));
  a.parent = d_tmp;
  BK(sb::launch_vis_components(a, g->d_comp, g->d_comp_sizes, d_tmp + n, &g->n_comp, s));
  std::vector<uint32_t> deg(n);
  BK(cudaMemcpy(deg.data(), g->d_deg, n * 4, cudaMemcpyDeviceToHost));
  uint64_t edges = 0;
  for (uint64_t v = 0; v < n; ++v) edges += deg[v];
  g->edges_local = edges;
  cleanup();
  const int rc = graph_setup(g, deg.data());
  if (rc) {
    delete g;
    return rc;
  }
#undef BK
  *out = g;
  return SB_OK;
}

int sb_graph_grid_info(const sb_graph* g, uint32_t* rows, uint32_t* cols, uint32_t* cell_of_node,
                       uint32_t* component_id, uint32_t* component_sizes, uint64_t* n_components) {
  if (!g) return fail(SB_EINVAL, "NULL graph");
  if (!g->d_cell) return fail(SB_EINVAL, "sb_graph_grid_info: graph was not built from a grid");
  DeviceGuard dg(g->device);
  if (rows) *rows = g->rows;
  if (cols) *cols = g->cols;
  if (n_components) *n_components = g->n_comp;
  if (cell_of_node) CK(cudaMemcpy(cell_of_node, g->d_cell, g->n * 4, cudaMemcpyDeviceToHost));
  if (component_id) CK(cudaMemcpy(component_id, g->d_comp, g->n * 4, cudaMemcpyDeviceToHost));
  if (component_sizes) CK(cudaMemcpy(component_sizes, g->d_comp_sizes, g->n_comp * 4, cudaMemcpyDeviceToHost));
  return SB_OK;
}

int sb_graph_download(const sb_graph* g, uint64_t* offsets, uint32_t* degrees, uint8_t* stream) {
  if (!g) return fail(SB_EINVAL, "NULL graph");
  DeviceGuard dg(g->device);
  if (const int rc = graph_wait(const_cast<sb_graph*>(g))) return rc;
  if (offsets) CK(cudaMemcpy(offsets, g->d_rowoff, (g->n_local + 1) * 8, cudaMemcpyDeviceToHost));
  if (degrees) CK(cudaMemcpy(degrees, g->d_deg, g->n_local * 4, cudaMemcpyDeviceToHost));
  if (stream && g->stream_local) CK(cudaMemcpy(stream, g->d_stream, g->stream_local, cudaMemcpyDeviceToHost));
  return SB_OK;
}

int sb_graph_stats(const sb_graph* g, uint64_t* n_local, uint64_t* edges_local,
                   uint64_t* stream_bytes_local, uint64_t* n_items, uint32_t* chunk) {
  if (!g) return fail(SB_EINVAL, "NULL graph");
  if (n_local) *n_local = g->n_local;
  if (edges_local) *edges_local = g->edges_local;
  if (stream_bytes_local) *stream_bytes_local = g->stream_local;
  if (n_items) *n_items = g->n_items;
  if (chunk) *chunk = g->chunk;
  return SB_OK;
}

void sb_graph_destroy(sb_graph* g) { delete g; }

}  // extern "C"
