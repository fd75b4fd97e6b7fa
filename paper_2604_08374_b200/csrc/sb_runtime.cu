// sb_runtime.cu -- host side of the C-ABI: device graph, HyperBall state,
// Alg. 1 control loop, shard exchange (NCCL / same-process copies), stats.
#include <nccl.h>

#include <algorithm>
#include <memory>
#include <chrono>
#include <cstdlib>
#include <thread>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sieveball_cuda.h"
#include "sb_device.cuh"
#include "sb_error.h"
#include "sb_internal.h"

using sb::fail;

namespace {
int cuda_fail(cudaError_t e, const char* what) {
  return fail(e == cudaErrorMemoryAllocation ? SB_ENOMEM : SB_ECUDA, "%s: %s", what,
              cudaGetErrorString(e));
}

#define CK(x)                                          \
  do {                                                 \
    cudaError_t e_ = (x);                              \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x);   \
  } while (0)

#define NK(x)                                                               \
  do {                                                                      \
    ncclResult_t r_ = (x);                                                  \
    if (r_ != ncclSuccess) return fail(SB_ENCCL, "%s: %s", #x, ncclGetErrorString(r_)); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

template <class T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

// Stream sync with an optional watchdog: SB_SYNC_TIMEOUT_S=<seconds> turns a
// device hang into an SB_ECUDA error instead of a blocked host thread.
cudaError_t sync_stream(cudaStream_t s) {
  static const double limit = [] {
    const char* e = getenv("SB_SYNC_TIMEOUT_S");
    return e ? atof(e) : 0.0;
  }();
  if (limit <= 0.0) return cudaStreamSynchronize(s);
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e != cudaErrorNotReady) return e;
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit)
      return cudaErrorLaunchTimeout;
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

double decode_ord(unsigned long long e) {
  if (e == 0ull) return -INFINITY;  // no node contributed
  unsigned long long u = (e >> 63) ? (e & 0x7fffffffffffffffull) : ~e;
  double x;
  memcpy(&x, &u, 8);
  return x;
}
}  // namespace

struct sb_graph {
  int device = 0;
  uint64_t n = 0, v0 = 0, v1 = 0, n_local = 0, edges_local = 0, stream_local = 0;
  uint8_t* d_stream = nullptr;
  uint64_t* d_rowoff = nullptr;
  uint32_t* d_deg = nullptr;
  uint32_t* d_orig = nullptr;
  uint32_t chunk = 0;
  uint64_t n_items = 0;
  uint32_t* d_node_item = nullptr;
  uint64_t* d_item_off = nullptr;
  uint32_t* d_item_base = nullptr;
  uint32_t* d_item_count = nullptr;
  uint32_t* d_item_node = nullptr;
  uint32_t max_run = 0;               // longest run of consecutive neighbour ids
  uint64_t n_runs = 0;                // interval-mode run index (built on first use)
  uint64_t* d_run_off = nullptr;
  uint32_t* d_run_s = nullptr;
  uint32_t* d_run_e = nullptr;
  uint64_t n_tiles = 0;               // CTA tiles: (8-node group, chunk index)
  uint32_t* d_tile_node0 = nullptr;
  uint32_t* d_tile_q = nullptr;
  // built on the device from a grid (sb_graph_build_grid)
  uint32_t rows = 0, cols = 0;
  uint64_t n_comp = 0;
  uint32_t* d_cell = nullptr;         // cell_of_node
  uint32_t* d_comp = nullptr;         // component id per node
  uint32_t* d_comp_sizes = nullptr;   // n_comp sizes
  // asynchronous chunked upload (sb_graph_create_async): chunk k's stream
  // bytes are copied on up_stream and validated on val_stream; val_ev[k]
  // fires when chunk k (nodes [chunk_node[k], chunk_node[k+1])) is usable.
  bool pending = false;
  int broken = 0;                     // validation failed (sticky SB_ERUNTIME)
  unsigned long long* d_err = nullptr;  // [0] min bad node, [1] max run
  cudaStream_t up_stream = nullptr, val_stream = nullptr;
  std::vector<cudaEvent_t> val_ev;
  std::vector<uint64_t> chunk_node, chunk_tile;
  ~sb_graph() {
    DeviceGuard dg(device);
    dfree(d_stream); dfree(d_rowoff); dfree(d_deg); dfree(d_orig); dfree(d_node_item);
    dfree(d_item_off); dfree(d_item_base); dfree(d_item_count); dfree(d_item_node);
    dfree(d_tile_node0); dfree(d_tile_q);
    dfree(d_run_off); dfree(d_run_s); dfree(d_run_e);
    dfree(d_cell); dfree(d_comp); dfree(d_comp_sizes);
    if (up_stream) cudaStreamSynchronize(up_stream);
    if (val_stream) cudaStreamSynchronize(val_stream);
    for (auto e : val_ev) cudaEventDestroy(e);
    if (up_stream) cudaStreamDestroy(up_stream);
    if (val_stream) cudaStreamDestroy(val_stream);
    dfree(d_err);
  }
};

struct sb_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
  ~sb_comm() {
    if (comm) ncclCommDestroy(comm);
  }
};

struct sb_hb {
  sb_graph* g = nullptr;
  unsigned p = 10;
  uint32_t depth = 0, flags = 0;
  uint64_t row = 0;
  int slices = 1;
  uint8_t* d_plane[2] = {nullptr, nullptr};
  uint8_t* d_changed[2] = {nullptr, nullptr};
  double* d_c[2] = {nullptr, nullptr};
  double* d_sum_d = nullptr;
  double* d_sum_d2 = nullptr;
  double* d_lc = nullptr;
  uint8_t* d_scratch = nullptr;
  uint32_t* d_counter = nullptr;
  unsigned long long* d_misc = nullptr;  // [0] work, [1] max_ord, [2] changed count
  unsigned long long* h_misc = nullptr;  // pinned
  uint8_t* d_tmp = nullptr;              // packed export buffer
  uint8_t* d_st = nullptr;               // interval mode: sparse-table levels 1..levels
  int levels = 0;
  uint64_t tmp_bytes = 0;
  int latest = 0;     // plane / c / changed index holding iteration t
  uint32_t t = 0;
  bool converged = false, finished = false, computed = false;
  double alpha = 0.0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<sb_iter_stats> stats;
  sb_iter_stats cur_stats{};
  sb_comm* comm = nullptr;
  std::vector<uint64_t> bounds;
  // fused P2P exchange (CUDA IPC): peers' planes / changed flags by parity
  int npeers = 0;
  std::vector<void*> ipc_opened;
  uint8_t** d_peer_plane[2] = {nullptr, nullptr};
  uint8_t** d_peer_chg[2] = {nullptr, nullptr};
  ~sb_hb() {
    DeviceGuard dg(g ? g->device : 0);
    for (void* q : ipc_opened) cudaIpcCloseMemHandle(q);
    for (int i = 0; i < 2; ++i) { dfree(d_peer_plane[i]); dfree(d_peer_chg[i]); }
    for (int i = 0; i < 2; ++i) { dfree(d_plane[i]); dfree(d_changed[i]); dfree(d_c[i]); }
    dfree(d_sum_d); dfree(d_sum_d2); dfree(d_lc); dfree(d_scratch); dfree(d_counter);
    dfree(d_misc); dfree(d_tmp); dfree(d_st);
    if (h_misc) cudaFreeHost(h_misc);
    for (auto& e : ev) if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
  }
};

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

int sb_check_convergence(double max_increase) { return max_increase <= 0.5 ? 1 : 0; }

// ------------------------------------------------------------------ graph
// Work items, CTA tiles and the upload-time validation of the device-resident
// stream slice (shared by sb_graph_create and the on-device grid builder).
static int graph_setup_host(sb_graph* g, const uint32_t* deg_local) {
  // Work items: <= chunk neighbours each, sized so the edge work splits into
  // ~4 items per resident warp (load balance) but stays >= 512 ids (decode
  // and merge amortisation).
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
  CK(cudaMalloc(&g->d_tile_node0, std::max<size_t>(tn0.size(), 1) * 4));
  CK(cudaMalloc(&g->d_tile_q, std::max<size_t>(tq.size(), 1) * 4));
  if (!tn0.empty()) {
    CK(cudaMemcpy(g->d_tile_node0, tn0.data(), tn0.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(g->d_tile_q, tq.data(), tq.size() * 4, cudaMemcpyHostToDevice));
  }
  CK(cudaMalloc(&g->d_node_item, node_item.size() * 4));
  CK(cudaMemcpy(g->d_node_item, node_item.data(), node_item.size() * 4, cudaMemcpyHostToDevice));
  const uint64_t ni = std::max<uint64_t>(items, 1);
  CK(cudaMalloc(&g->d_item_off, ni * 8));
  CK(cudaMalloc(&g->d_item_base, ni * 4));
  CK(cudaMalloc(&g->d_item_count, ni * 4));
  CK(cudaMalloc(&g->d_item_node, ni * 4));
  CK(cudaMalloc(&g->d_err, 16));
  CK(cudaMemset(g->d_err, 0xff, 8));
  CK(cudaMemset(reinterpret_cast<uint8_t*>(g->d_err) + 8, 0, 8));
  return SB_OK;
}

// Upload-time validation of local nodes [n0, n1) (LEB128 well-formed, strictly
// increasing ids < n, exactly degrees[v] ids) + work items; errors land in d_err.
static cudaError_t launch_validate(sb_graph* g, uint64_t n0, uint64_t n1, cudaStream_t s) {
  if (n1 <= n0) return cudaSuccess;
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
  a.err_node = g->d_err;
  a.max_run = reinterpret_cast<unsigned int*>(g->d_err + 1);
  return sb::launch_build_items(a, s);
}

static int graph_check(sb_graph* g) {
  unsigned long long err = 0;
  CK(cudaMemcpy(&err, g->d_err, 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&g->max_run, g->d_err + 1, 4, cudaMemcpyDeviceToHost));
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
static int graph_setup(sb_graph* g, const uint32_t* deg_local) {
  int rc = graph_setup_host(g, deg_local);
  if (rc) return rc;
  CK(launch_validate(g, 0, g->n_local, 0));
  CK(sync_stream(0));
  return graph_check(g);
}

// Completes an asynchronous upload (sb_graph_create_async): waits for every
// chunk's copy + validation and reports a malformed stream (sticky).
static int graph_wait(sb_graph* g) {
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
  // 256 B of zero padding: the decoder reads whole 128-byte windows (+8 for alignment).
  GK(cudaMalloc(&g->d_stream, g->stream_local + 256));
  GK(cudaMemset(g->d_stream + g->stream_local, 0, 256));
  if (g->stream_local && !async)
    GK(cudaMemcpy(g->d_stream, stream + b0, g->stream_local, cudaMemcpyHostToDevice));
  std::vector<uint64_t> ro(g->n_local + 1);
  for (uint64_t i = 0; i <= g->n_local; ++i) ro[i] = offsets[node_begin + i] - b0;
  GK(cudaMalloc(&g->d_rowoff, ro.size() * 8));
  GK(cudaMemcpy(g->d_rowoff, ro.data(), ro.size() * 8, cudaMemcpyHostToDevice));
  GK(cudaMalloc(&g->d_deg, std::max<uint64_t>(g->n_local, 1) * 4));
  if (g->n_local) GK(cudaMemcpy(g->d_deg, degrees + node_begin, g->n_local * 4, cudaMemcpyHostToDevice));
  if (orig_id) {
    GK(cudaMalloc(&g->d_orig, n * 4));
    GK(cudaMemcpy(g->d_orig, orig_id, n * 4, cudaMemcpyHostToDevice));
  }
  if (!async) {
    const int rc = graph_setup(g, degrees + node_begin);
    if (rc) return bail(rc);
    *out = g;
    return SB_OK;
  }
  // Asynchronous: K chunks of ~equal stream bytes on 8-node (tile group)
  // boundaries; copy k on up_stream, validation k on val_stream after copy k.
  const int rc = graph_setup_host(g, degrees + node_begin);
  if (rc) return bail(rc);
  GK(cudaStreamCreateWithFlags(&g->up_stream, cudaStreamNonBlocking));
  GK(cudaStreamCreateWithFlags(&g->val_stream, cudaStreamNonBlocking));
  const int K = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(16, g->n_local / 64)));
  g->chunk_node.assign(1, 0);
  for (int k = 1; k < K; ++k) {
    const uint64_t goal = b0 + g->stream_local * k / K;
    uint64_t v = std::lower_bound(offsets + node_begin, offsets + node_end, goal) - (offsets + node_begin);
    v = std::min<uint64_t>(v & ~7ull, g->n_local);
    if (v > g->chunk_node.back()) g->chunk_node.push_back(v);
  }
  if (g->chunk_node.back() != g->n_local) g->chunk_node.push_back(g->n_local);
  // tile ranges: tiles are ordered by 8-node group
  std::vector<uint32_t> tn0(g->n_tiles);
  if (g->n_tiles) GK(cudaMemcpy(tn0.data(), g->d_tile_node0, g->n_tiles * 4, cudaMemcpyDeviceToHost));
  g->chunk_tile.clear();
  for (uint64_t cn : g->chunk_node)
    g->chunk_tile.push_back(std::lower_bound(tn0.begin(), tn0.end(), static_cast<uint32_t>(std::min<uint64_t>(cn, 0xffffffffull))) - tn0.begin());
  g->chunk_tile.back() = g->n_tiles;
  const size_t nk = g->chunk_node.size() - 1;
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
    GK(cudaEventRecord(g->val_ev[k], g->val_stream));
  }
  g->pending = true;
#undef GK
  *out = g;
  return SB_OK;
}

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
  uint64_t* d_bytes = nullptr;
  auto cleanup = [&] { dfree(d_mask); dfree(d_pref); dfree(d_scan); dfree(d_noc); dfree(d_tmp); dfree(d_bytes); };
  auto bail = [&](int rc) { cleanup(); delete g; return rc; };
#define BK(x)                                                 \
  do {                                                        \
    cudaError_t e_ = (x);                                     \
    if (e_ != cudaSuccess) return bail(cuda_fail(e_, #x));    \
  } while (0)
  cudaStream_t s = 0;
  BK(cudaMalloc(&d_mask, cells));
  BK(cudaMemcpy(d_mask, blocked, cells, cudaMemcpyHostToDevice));
  BK(cudaMalloc(&d_pref, static_cast<uint64_t>(rows + 1) * (cols + 1) * 4));
  BK(cudaMalloc(&d_scan, 2 * cells * 4));
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
  BK(cudaMalloc(&d_noc, cells * 4));
  BK(cudaMalloc(&g->d_cell, n * 4));
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
  BK(cudaMalloc(&g->d_deg, n * 4));
  BK(cudaMalloc(&d_bytes, (n + 1) * 8));
  BK(cudaMemsetAsync(d_bytes + n, 0, 8, s));
  a.deg = g->d_deg;
  a.bytes = d_bytes;
  BK(sb::launch_vis_rows(a, false, s));
  BK(cudaMalloc(&g->d_rowoff, (n + 1) * 8));
  BK(sb::launch_scan_u64(d_bytes, g->d_rowoff, n + 1, s));
  uint64_t total = 0;
  BK(cudaMemcpy(&total, g->d_rowoff + n, 8, cudaMemcpyDeviceToHost));
  g->stream_local = total;
  BK(cudaMalloc(&g->d_stream, total + 256));
  BK(cudaMemsetAsync(g->d_stream + total, 0, 256, s));
  a.offsets = g->d_rowoff;
  a.stream = g->d_stream;
  BK(sb::launch_vis_rows(a, true, s));
  // components (the 2n scratch doubles as the union-find parent array + ranks)
  BK(cudaMalloc(&d_tmp, 3 * n * 4));
  BK(cudaMalloc(&g->d_comp, n * 4));
  BK(cudaMalloc(&g->d_comp_sizes, n * 4));
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

// ------------------------------------------------------------------ HyperBall
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
  CK(sync_stream(h->stream));
  return SB_OK;
}

// Interval mode: runs of consecutive ids per work item, decoded once from the
// device-resident LEB128 stream (count pass, host scan, fill pass).
static int build_run_index(sb_graph* g) {
  if (g->d_run_off || g->n_items == 0) return SB_OK;
  sb::RunIndexArgs a{};
  a.stream = g->d_stream;
  a.item_off = g->d_item_off;
  a.item_base = g->d_item_base;
  a.item_count = g->d_item_count;
  a.n_items = g->n_items;
  uint64_t* d_cnt = nullptr;
  CK(cudaMalloc(&d_cnt, g->n_items * 8));
  a.run_count = d_cnt;
  CK(sb::launch_run_index(a, false, 0));
  CK(sync_stream(0));
  std::vector<uint64_t> off(g->n_items + 1, 0);
  CK(cudaMemcpy(off.data() + 1, d_cnt, g->n_items * 8, cudaMemcpyDeviceToHost));
  cudaFree(d_cnt);
  for (uint64_t i = 0; i < g->n_items; ++i) off[i + 1] += off[i];
  g->n_runs = off[g->n_items];
  CK(cudaMalloc(&g->d_run_off, off.size() * 8));
  CK(cudaMemcpy(g->d_run_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&g->d_run_s, std::max<uint64_t>(g->n_runs, 1) * 4));
  CK(cudaMalloc(&g->d_run_e, std::max<uint64_t>(g->n_runs, 1) * 4));
  a.run_off = g->d_run_off;
  a.run_s = g->d_run_s;
  a.run_e = g->d_run_e;
  CK(sb::launch_run_index(a, true, 0));
  CK(sync_stream(0));
  return SB_OK;
}

int sb_hb_create(sb_graph* g, unsigned p, uint32_t depth_limit, uint32_t flags, sb_hb** out) {
  if (!out) return fail(SB_EINVAL, "sb_hb_create: out is NULL");
  *out = nullptr;
  if (!g) return fail(SB_EINVAL, "sb_hb_create: NULL graph");
  if (p < 4 || p > 16) return fail(SB_EINVAL, "hll: precision must be in [4, 16]");
  if ((flags & SB_HB_INTERVAL) && (p < 10 || (flags & SB_HB_SKIP_UNCHANGED)))
    return fail(SB_EINVAL, "interval mode needs p >= 10 and excludes SB_HB_SKIP_UNCHANGED");
  DeviceGuard dg(g->device);
  auto* h = new sb_hb();
  h->g = g;
  h->p = p;
  h->depth = depth_limit;
  h->flags = flags;
  if (const char* e = getenv("SB_UNION_SCHEDULE")) {  // A/B override for benchmarking
    if (!strcmp(e, "warp")) h->flags |= SB_HB_SCHEDULE_WARP;
    if (!strcmp(e, "tile")) h->flags &= ~SB_HB_SCHEDULE_WARP;
  }
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
    HK(cudaMalloc(&h->d_plane[i], plane + 64));
    HK(cudaMalloc(&h->d_changed[i], g->n));
    HK(cudaMalloc(&h->d_c[i], nl * 8));
  }
  HK(cudaMalloc(&h->d_sum_d, nl * 8));
  HK(cudaMalloc(&h->d_sum_d2, nl * 8));
  // Linear-counting table lc[z] = m * log(m / z) built with the host libm, so
  // the device never evaluates log (hll.cpp:35).
  std::vector<double> lc(m + 1, 0.0);
  const double md = static_cast<double>(m);
  for (uint32_t z = 1; z <= m; ++z) lc[z] = md * std::log(md / static_cast<double>(z));
  HK(cudaMalloc(&h->d_lc, lc.size() * 8));
  HK(cudaMemcpy(h->d_lc, lc.data(), lc.size() * 8, cudaMemcpyHostToDevice));
  const uint64_t slice_bytes = std::min<uint64_t>(h->row, 512);
  HK(cudaMalloc(&h->d_scratch, std::max<uint64_t>(g->n_items, 1) * h->slices * slice_bytes));
  HK(cudaMalloc(&h->d_counter, nl * h->slices * 4));
  HK(cudaMalloc(&h->d_misc, 4 * 8));
  if (flags & SB_HB_INTERVAL) {
    if (const int rc = graph_wait(g)) return bail(rc);  // max_run comes from the validation pass
    // levels K = floor(log2(longest run)), capped at 10 (longer runs peel 2^K blocks)
    int K = 0;
    while (K < 10 && (2u << K) <= g->max_run) ++K;
    h->levels = K;
    if (K) HK(cudaMalloc(&h->d_st, static_cast<uint64_t>(K) * plane + 64));
    const int rc = build_run_index(g);
    if (rc) return bail(rc);
  }
  HK(cudaMallocHost(&h->h_misc, 4 * 8));
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
  if (g->pending && (h->flags & SB_HB_SCHEDULE_WARP)) {  // the chunk pipeline needs the tile schedule
    const int rc = graph_wait(g);
    if (rc) return rc;
  }
  h->t += 1;
  const int L = h->latest, N = 1 - L;
  const bool skip = (h->flags & SB_HB_SKIP_UNCHANGED) != 0;
  h->cur_stats = sb_iter_stats{};
  h->cur_stats.t = h->t;
  CK(cudaMemsetAsync(h->d_misc, 0, 4 * 8, h->stream));
  CK(cudaEventRecord(h->ev[0], h->stream));
  if (g->n_local) {
    CK(cudaMemsetAsync(h->d_changed[N] + g->v0, 0, g->n_local, h->stream));
    sb::UnionArgs u{};
    u.stream = g->d_stream;
    u.item_off = g->d_item_off;
    u.item_base = g->d_item_base;
    u.item_count = g->d_item_count;
    u.item_node = g->d_item_node;
    u.node_item = g->d_node_item;
    u.n_items = g->n_items;
    u.node_begin = g->v0;
    u.cur = h->d_plane[L];
    u.next = h->d_plane[N];
    u.scratch = h->d_scratch;
    u.node_counter = h->d_counter;
    u.changed_out = h->d_changed[N];
    u.changed_in = h->d_changed[L];
    u.work = h->d_misc;
    u.n_local = g->n_local;
    u.n_tiles = (h->flags & SB_HB_SCHEDULE_WARP) ? 0 : g->n_tiles;
    u.tile_node0 = g->d_tile_node0;
    u.tile_q = g->d_tile_q;
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
      for (size_t k = 0; k + 1 < g->chunk_node.size(); ++k) {
        const uint64_t t0 = g->chunk_tile[k], t1 = g->chunk_tile[k + 1];
        if (t1 == t0) continue;
        CK(cudaStreamWaitEvent(h->stream, g->val_ev[k], 0));
        CK(cudaMemsetAsync(h->d_misc, 0, 8, h->stream));  // work counter
        sb::UnionArgs uk = u;
        uk.tile_node0 = g->d_tile_node0 + t0;
        uk.tile_q = g->d_tile_q + t0;
        uk.n_tiles = t1 - t0;
        CK(sb::launch_union(static_cast<int>(h->p), skip, uk, h->stream));
      }
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
    CK(sb::launch_estimate(static_cast<int>(h->p), skip ? 2 : 1, e, h->stream));
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
  if (h->comm && h->comm->nranks > 1) {
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

int sb_hb_run(sb_hb* h, uint32_t* iterations, int* converged) {
  if (!h) return fail(SB_EINVAL, "NULL handle");
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
  CK(cudaMalloc(&h->d_tmp, bytes));
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

// ------------------------------------------------------------------ exact mode
// Exact neighbourhood function: bit-parallel BFS, the
// HyperBall loop with bitset rows and an OR union (see exact_* kernels).
struct sb_exact {
  sb_graph* g = nullptr;
  int P = 10;                       // row geometry: 2^(P-1) bytes = 2^(P+2) sources
  uint64_t row = 0, block = 0;
  uint32_t depth = 0, flags = 0;
  int slices = 1, levels = 0;
  uint8_t* d_plane[2] = {nullptr, nullptr};
  uint8_t* d_changed = nullptr;     // union epilogue flags (unused by the count)
  uint8_t* d_scratch = nullptr;
  uint32_t* d_counter = nullptr;
  uint8_t* d_st = nullptr;
  uint32_t* d_pop = nullptr;
  uint32_t* d_reach = nullptr;
  unsigned long long* d_sum = nullptr;   // [sum_d n | sum_d2 n]
  uint32_t* d_hist = nullptr;
  uint32_t hist_cap = 0;
  unsigned long long* d_misc = nullptr;  // [0] work, [1] changed count
  uint32_t max_depth = 0;
  uint64_t sources_done = 0;
  double union_ms = 0.0;
  uint64_t union_launches = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~sb_exact() {
    DeviceGuard dg(g ? g->device : 0);
    for (int i = 0; i < 2; ++i) dfree(d_plane[i]);
    dfree(d_changed); dfree(d_scratch); dfree(d_counter); dfree(d_st); dfree(d_pop);
    dfree(d_reach); dfree(d_sum); dfree(d_hist); dfree(d_misc);
    for (auto e : ev) if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
  }
};

static int exact_grow_hist(sb_exact* x, uint32_t need) {
  if (need < x->hist_cap) return SB_OK;
  uint32_t cap = std::max<uint32_t>(x->hist_cap * 2, 16);
  while (cap <= need) cap *= 2;
  const uint64_t n = x->g->n;
  uint32_t* nh = nullptr;
  CK(cudaMalloc(&nh, n * cap * 4));
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
  for (int i = 0; i < 2; ++i) XK(cudaMalloc(&x->d_plane[i], plane + 64));
  XK(cudaMalloc(&x->d_changed, n));
  XK(cudaMalloc(&x->d_scratch, std::max<uint64_t>(g->n_items, 1) * x->slices * 512));
  XK(cudaMalloc(&x->d_counter, n * x->slices * 4));
  XK(cudaMemset(x->d_counter, 0, n * x->slices * 4));
  XK(cudaMalloc(&x->d_pop, n * 4));
  XK(cudaMalloc(&x->d_reach, n * 4));
  XK(cudaMemset(x->d_reach, 0, n * 4));
  XK(cudaMalloc(&x->d_sum, 2 * n * 8));
  XK(cudaMemset(x->d_sum, 0, 2 * n * 8));
  XK(cudaMalloc(&x->d_misc, 2 * 8));
  if (flags & SB_HB_INTERVAL) {
    int K = 0;
    while (K < 10 && (2u << K) <= g->max_run) ++K;
    x->levels = K;
    if (K) XK(cudaMalloc(&x->d_st, static_cast<uint64_t>(K) * plane + 64));
    const int rc = build_run_index(g);
    if (rc) return bail(rc);
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
    for (uint32_t t = 1;; ++t) {
      int rc = exact_grow_hist(x, t);
      if (rc) return rc;
      e.hist = x->d_hist;
      e.hist_cap = x->hist_cap;
      CK(cudaMemsetAsync(x->d_misc, 0, 16, x->stream));
      sb::UnionArgs u{};
      u.stream = g->d_stream;
      u.item_off = g->d_item_off;
      u.item_base = g->d_item_base;
      u.item_count = g->d_item_count;
      u.item_node = g->d_item_node;
      u.node_item = g->d_node_item;
      u.n_items = g->n_items;
      u.node_begin = 0;
      u.cur = x->d_plane[L];
      u.next = x->d_plane[1 - L];
      u.scratch = x->d_scratch;
      u.node_counter = x->d_counter;
      u.changed_out = x->d_changed;
      u.changed_in = x->d_changed;
      u.work = x->d_misc;
      u.n_local = n;
      u.n_tiles = g->n_tiles;
      u.tile_node0 = g->d_tile_node0;
      u.tile_q = g->d_tile_q;
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
  // |B(v, 2)| for every node: two OR-union iterations per 4096-source block
  sb_exact* x = nullptr;
  rc = sb_exact_create(g, 12, 2, SB_HB_INTERVAL, &x);
  if (rc) return rc;
  std::unique_ptr<sb_exact, void (*)(sb_exact*)> xg(x, sb_exact_destroy);
  rc = sb_exact_run(x, 0, n, nullptr);
  if (rc) return rc;
  // [span_lo N | span_hi N | max 1] u32, [control | ctrl | clus] f64 nl, [among | n2 | work] u64
  const uint64_t u32_words = 2 * n + 1;
  const uint64_t bytes = ((u32_words * 4 + 7) & ~7ull) + 5 * nl * 8 + 8;
  uint8_t* blk = nullptr;
  CK(cudaMalloc(&blk, bytes));
  uint32_t* scratch = nullptr;
  struct Free {
    uint8_t*& p;
    uint32_t*& q;
    ~Free() { if (p) cudaFree(p); if (q) cudaFree(q); }
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
  a.reach2 = x->d_reach;
  uint32_t* u = reinterpret_cast<uint32_t*>(blk);
  a.span_lo = u;
  a.span_hi = u + n;
  a.max_words = u + 2 * n;
  double* f = reinterpret_cast<double*>(blk + ((u32_words * 4 + 7) & ~7ull));
  a.control = f;
  a.controllability = f + nl;
  a.clustering = f + 2 * nl;
  a.edges_among = reinterpret_cast<unsigned long long*>(f + 3 * nl);
  a.n2 = a.edges_among + nl;
  a.work = a.n2 + nl;
  CK(cudaMemsetAsync(a.max_words, 0, 4, 0));
  CK(cudaMemsetAsync(a.work, 0, 8, 0));
  CK(sb::launch_local_spans(a, 0));
  unsigned int mw = 0;
  CK(cudaMemcpy(&mw, a.max_words, 4, cudaMemcpyDeviceToHost));
  a.w1_words = std::max(mw, 1u);
  a.stride_words = 2ull * (a.w1_words + 1);
  // SB_LOCAL_GLOBAL=1 forces the global-scratch bitmaps (test hook for wide windows)
  const char* force = getenv("SB_LOCAL_GLOBAL");
  const bool smem = a.stride_words * 4 <= sb::local_smem_limit() && !(force && atoi(force));
  if (!smem) {
    int grid = 0;
    CK(sb::launch_local(a, false, &grid, 0));
    CK(cudaMalloc(&scratch, static_cast<uint64_t>(grid) * a.stride_words * 4));
    a.scratch = scratch;
  }
  CK(sb::launch_local(a, smem, nullptr, 0));
  CK(sync_stream(0));
  if (control) CK(cudaMemcpy(control, a.control, nl * 8, cudaMemcpyDeviceToHost));
  if (controllability) CK(cudaMemcpy(controllability, a.controllability, nl * 8, cudaMemcpyDeviceToHost));
  if (clustering) CK(cudaMemcpy(clustering, a.clustering, nl * 8, cudaMemcpyDeviceToHost));
  if (edges_among) CK(cudaMemcpy(edges_among, a.edges_among, nl * 8, cudaMemcpyDeviceToHost));
  if (n2) CK(cudaMemcpy(n2, a.n2, nl * 8, cudaMemcpyDeviceToHost));
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
int sb_hb_ipc_handles(const sb_hb* h, void* out, size_t cap) {
  if (!h || !out) return fail(SB_EINVAL, "NULL argument");
  if (cap < SB_IPC_HANDLE_BYTES) return fail(SB_EINVAL, "handle buffer too small (%d bytes needed)", SB_IPC_HANDLE_BYTES);
  static_assert(sizeof(cudaIpcMemHandle_t) * 4 == SB_IPC_HANDLE_BYTES, "ipc handle size");
  DeviceGuard dg(h->g->device);
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
    CK(cudaMalloc(&h->d_peer_plane[i], std::max(np, 1) * sizeof(uint8_t*)));
    CK(cudaMalloc(&h->d_peer_chg[i], std::max(np, 1) * sizeof(uint8_t*)));
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
