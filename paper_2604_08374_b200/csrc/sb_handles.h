// sb_handles.h -- PRIVATE: the C-ABI handle types (sb_graph, sb_hb, sb_comm,
// sb_exact), the runtime utilities shared by the host translation units, and
// the internal graph helpers.  Not installed; include/sieveball_cuda.h is the API.
#pragma once
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/sieveball_cuda.h"
#include "sb_error.h"
#include "sb_internal.h"

namespace sb {
namespace rt {
inline int cuda_fail(cudaError_t e, const char* what) {
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

// Device memory comes from the device's default stream-ordered pool, told to
// keep what is freed (release threshold = all): repeated create / destroy
// cycles -- a service analysing many grids, the end-to-end bench -- then reuse
// the multi-GB stream and plane buffers instead of paying the driver's
// map / unmap (and cudaFree's device-wide sync) every time, the way torch's
// caching allocator does.  sb_release_cached_memory() hands it back.  Owners
// synchronise their streams before dfree.  Buffers shared with peer processes
// over CUDA IPC (HyperBall planes and changed flags) stay on cudaMalloc.
inline cudaError_t keep_pool(int dev) {
  static std::once_flag once[128];
  if (dev < 0 || dev >= 128) return cudaErrorInvalidDevice;
  cudaError_t e = cudaSuccess;
  std::call_once(once[dev], [&] {
    cudaMemPool_t pool;
    e = cudaDeviceGetDefaultMemPool(&pool, dev);
    uint64_t keep = ~0ull;
    if (e == cudaSuccess) e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  });
  return e;
}

template <class T>
inline cudaError_t dalloc(T** p, size_t bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = keep_pool(dev);
  if (e != cudaSuccess) return e;
  void* q = nullptr;
  e = cudaMallocAsync(&q, bytes, cudaStreamPerThread);
  if (e == cudaErrorMemoryAllocation) {  // return cached blocks to the driver once, then retry
    cudaGetLastError();
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, dev);
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(&q, bytes, cudaStreamPerThread);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamPerThread);
  if (e == cudaSuccess) *p = static_cast<T*>(q);
  return e;
}

template <class T>
inline void dfree(T*& p) {
  if (p) cudaFreeAsync(p, cudaStreamPerThread);
  p = nullptr;
}

template <class T>
inline cudaError_t dalloc_ipc(T** p, size_t bytes) {
  return cudaMalloc(p, bytes);
}

template <class T>
inline void dfree_ipc(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

// 32-byte page-locked host slots (each HyperBall handle's per-iteration
// read-back) carved from one process-wide slab: cudaMallocHost / cudaFreeHost
// per handle cost milliseconds, more than a whole small-graph run.
constexpr int kPinnedSlot = 256, kPinnedSlots = 4096;  // per handle: step read-back / batched-run records
struct PinnedSlab {
  std::mutex mu;
  uint8_t* base = nullptr;
  std::vector<int> free_slots;
  bool failed = false;
};
inline PinnedSlab& pinned_slab() {
  static PinnedSlab* s = new PinnedSlab();  // never destroyed: slots may outlive static teardown
  return *s;
}
// Returns a slot, or a private cudaMallocHost block when the slab is exhausted
// (*owned = true: release with cudaFreeHost).
inline cudaError_t pinned_get(unsigned long long** out, bool* owned) {
  PinnedSlab& s = pinned_slab();
  {
    std::lock_guard<std::mutex> lk(s.mu);
    if (!s.base && !s.failed) {
      void* p = nullptr;
      if (cudaHostAlloc(&p, static_cast<size_t>(kPinnedSlot) * kPinnedSlots, cudaHostAllocPortable) == cudaSuccess) {
        s.base = static_cast<uint8_t*>(p);
        for (int i = kPinnedSlots - 1; i >= 0; --i) s.free_slots.push_back(i);
      } else {
        cudaGetLastError();
        s.failed = true;
      }
    }
    if (!s.free_slots.empty()) {
      const int i = s.free_slots.back();
      s.free_slots.pop_back();
      *out = reinterpret_cast<unsigned long long*>(s.base + static_cast<size_t>(i) * kPinnedSlot);
      *owned = false;
      return cudaSuccess;
    }
  }
  *owned = true;
  return cudaMallocHost(reinterpret_cast<void**>(out), kPinnedSlot);
}
inline void pinned_put(unsigned long long* p, bool owned) {
  if (!p) return;
  if (owned) {
    cudaFreeHost(p);
    return;
  }
  PinnedSlab& s = pinned_slab();
  std::lock_guard<std::mutex> lk(s.mu);
  s.free_slots.push_back(static_cast<int>((reinterpret_cast<uint8_t*>(p) - s.base) / kPinnedSlot));
}

// Stream sync with an optional watchdog: SB_SYNC_TIMEOUT_S=<seconds> turns a
// device hang into an SB_ECUDA error instead of a blocked host thread.
inline cudaError_t sync_stream(cudaStream_t s) {
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

inline double decode_ord(unsigned long long e) {
  if (e == 0ull) return -INFINITY;  // no node contributed
  unsigned long long u = (e >> 63) ? (e & 0x7fffffffffffffffull) : ~e;
  double x;
  memcpy(&x, &u, 8);
  return x;
}
}  // namespace rt
}  // namespace sb

using sb::fail;
using sb::rt::cuda_fail;
using sb::rt::DeviceGuard;
using sb::rt::decode_ord;
using sb::rt::dalloc;
using sb::rt::dalloc_ipc;
using sb::rt::dfree;
using sb::rt::dfree_ipc;
using sb::rt::pinned_get;
using sb::rt::pinned_put;
using sb::rt::sync_stream;

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
  uint32_t* d_node_lo = nullptr;      // first / last neighbour id per local node (validation pass)
  uint32_t* d_node_hi = nullptr;
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
  uint32_t* d_chunk_rng = nullptr;      // per chunk: min first / max last neighbour id (after val_ev[k])
  std::vector<uint64_t> chunk_node, chunk_tile, chunk_item, chunk_byte;
  std::vector<uint32_t> h_node_item;  // local node -> first work item (host copy)
  // run storage outgrown while a wavefront still reads it (freed once its passes are done)
  std::vector<uint32_t*> retired_runs;
  void free_retired_runs() {
    for (uint32_t*& r : retired_runs) dfree(r);
    retired_runs.clear();
  }
  ~sb_graph() {
    DeviceGuard dg(device);
    if (up_stream) cudaStreamSynchronize(up_stream);
    if (val_stream) cudaStreamSynchronize(val_stream);
    dfree(d_stream); dfree(d_rowoff); dfree(d_deg); dfree(d_orig); dfree(d_node_item);
    dfree(d_item_off); dfree(d_item_base); dfree(d_item_count); dfree(d_item_node);
    dfree(d_node_lo); dfree(d_node_hi); dfree(d_chunk_rng);
    dfree(d_tile_node0); dfree(d_tile_q);
    dfree(d_run_off); dfree(d_run_s); dfree(d_run_e);
    free_retired_runs();
    dfree(d_cell); dfree(d_comp); dfree(d_comp_sizes);
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
  unsigned long long* h_misc = nullptr;  // pinned (slab slot unless h_misc_owned)
  bool h_misc_owned = false;
  bool planes_ipc = false;               // planes / changed flags re-allocated for CUDA IPC export
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
  // first pass over a graph still uploading: second stream + per-chunk work counters
  cudaStream_t stream2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  unsigned long long* d_chunk_work = nullptr;
  size_t chunk_work_n = 0;
  // wavefront first run (pipelined_run): a plane + changed flags per pass >= 2,
  // a stream per pass, an event per (pass, chunk), pass start / end events
  std::vector<uint8_t*> d_xplane, d_xchg;
  std::vector<uint8_t*> d_xst;            // interval mode: a sparse table per wavefront pass
  std::vector<cudaEvent_t> sev;            // interval mode: sparse-table rows of (pass, chunk) ready
  bool index_ready = true;                 // interval mode: run index + sparse table allocated
  std::vector<cudaStream_t> pstream;
  std::vector<cudaEvent_t> pev, pev_t;
  // back-to-back passes (batched_run): device flags [stop, last pass, converged],
  // per-pass [max increase, changed count], pinned read-back, timing events
  unsigned int* d_bflags = nullptr;
  unsigned long long* d_brec = nullptr;
  std::vector<cudaEvent_t> bev;
  unsigned long long* d_pwork = nullptr;
  size_t pwork_n = 0;
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
    if (stream) cudaStreamSynchronize(stream);
    if (stream2) cudaStreamSynchronize(stream2);
    for (void* q : ipc_opened) cudaIpcCloseMemHandle(q);
    for (int i = 0; i < 2; ++i) { dfree(d_peer_plane[i]); dfree(d_peer_chg[i]); }
    for (int i = 0; i < 2; ++i) {
      if (planes_ipc) {
        dfree_ipc(d_plane[i]);
        dfree_ipc(d_changed[i]);
      } else {
        dfree(d_plane[i]);
        dfree(d_changed[i]);
      }
      dfree(d_c[i]);
    }
    dfree(d_sum_d); dfree(d_sum_d2); dfree(d_lc); dfree(d_scratch); dfree(d_counter);
    for (cudaStream_t ps : pstream) cudaStreamSynchronize(ps);
    dfree(d_misc); dfree(d_tmp); dfree(d_st); dfree(d_chunk_work); dfree(d_pwork);
    for (uint8_t* x : d_xplane) dfree(x);
    for (uint8_t* x : d_xchg) dfree(x);
    for (uint8_t* x : d_xst) dfree(x);
    for (cudaEvent_t e : sev) cudaEventDestroy(e);
    for (cudaEvent_t e : pev) cudaEventDestroy(e);
    for (cudaEvent_t e : pev_t) cudaEventDestroy(e);
    for (cudaEvent_t e : bev) cudaEventDestroy(e);
    dfree(d_bflags); dfree(d_brec);
    for (cudaStream_t ps : pstream) cudaStreamDestroy(ps);
    pinned_put(h_misc, h_misc_owned);
    for (auto& e : ev) if (e) cudaEventDestroy(e);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (stream) cudaStreamDestroy(stream);
    if (stream2) cudaStreamDestroy(stream2);
  }
};

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
    if (stream) cudaStreamSynchronize(stream);
    for (int i = 0; i < 2; ++i) dfree(d_plane[i]);
    dfree(d_changed); dfree(d_scratch); dfree(d_counter); dfree(d_st); dfree(d_pop);
    dfree(d_reach); dfree(d_sum); dfree(d_hist); dfree(d_misc);
    for (auto e : ev) if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
  }
};

// Internal graph helpers (sb_graph_api.cu).
int graph_setup(sb_graph* g, const uint32_t* deg_local);
// Union arguments shared by HyperBall and exact mode: CSR slice, work items,
// CTA tiles and the group path of union_kernel.
void graph_union_args(const sb_graph* g, sb::UnionArgs& u);
int graph_wait(sb_graph* g);
int build_run_index(sb_graph* g);
// The run index built incrementally over an asynchronous upload: chunk k is
// counted, offset and (once the storage is sized) written after its
// validation; ready[k] fires when chunk k's runs are in place.
struct RunIndexJob {
  sb::RunIndexArgs a{};
  uint64_t* d_cnt = nullptr;
  unsigned long long* d_aux = nullptr;  // [0] run total, [1] overflow flag
  uint64_t cap = 0;                     // run storage entries (0: not yet allocated)
  size_t probe = 0, filled = 0;         // chunks [0, filled) have their fill enqueued
  int grown = 0;                        // times the run storage grew
  bool failed = false;                  // a chunk failed validation: nothing more is written
  cudaStream_t s = nullptr;
  std::vector<cudaEvent_t> ready;
};
int rix_begin(sb_graph* g, RunIndexJob& j);
int rix_chunk(sb_graph* g, RunIndexJob& j, size_t k);
// After the upload: totals, last offset, max run; *overflow: the run storage
// could not be allocated (the index must be rebuilt: rix_abort + build_run_index).
int rix_finish(sb_graph* g, RunIndexJob& j, bool* overflow);
void rix_abort(sb_graph* g, RunIndexJob& j);
