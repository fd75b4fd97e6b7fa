// sb_internal.h -- argument blocks and launchers shared by the runtime and kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sb {

struct BuildArgs {
  const uint8_t* stream;       // local stream slice (padded)
  const uint64_t* row_off;     // local byte offsets, n_local + 1
  const uint32_t* degrees;     // local degrees
  uint64_t n_local;
  uint64_t n_global;
  uint64_t node_begin, node_end;  // local nodes to validate (node_end 0 = n_local)
  uint32_t chunk;              // neighbours per work item
  const uint32_t* node_item;   // local node -> first item (n_local + 1)
  uint64_t* item_off;
  uint32_t* item_base;
  uint32_t* item_count;
  uint32_t* item_node;
  uint32_t* node_lo;           // first / last neighbour id per local node (empty row: ~0 / 0)
  uint32_t* node_hi;
  unsigned long long* err_node;  // min local node with a malformed row (~0 = none)
};

// Zero bytes after every device stream slice: the decoders read whole windows
// past a row's end (decode16_to_bitmap: 512 bytes + 4 + alignment).
constexpr uint64_t kStreamPad = 1024;

struct UnionArgs {
  const uint8_t* stream;
  const uint64_t* item_off;
  const uint32_t* item_base;
  const uint32_t* item_count;
  const uint32_t* item_node;   // local node index
  const uint32_t* node_item;   // local node -> first item (n_local + 1)
  uint64_t n_items;
  uint64_t node_begin;         // global id of local node 0
  const uint8_t* cur;          // full replica, global rows
  uint8_t* next;               // global rows (own range written)
  uint8_t* scratch;            // per work unit partial rows
  uint32_t* node_counter;      // n_local * slices arrival counters (self-resetting)
  uint8_t* changed_out;        // global-indexed, 1 = registers changed this iteration
  const uint8_t* changed_in;   // global-indexed, previous iteration (skip mode)
  unsigned long long* work;    // dynamic work counter (zeroed per launch)
  // Upload-time validation verdict (min bad local node, ~0 = clean; NULL once
  // the upload is complete).  During the pipelined first pass a chunk's union
  // starts right after its validation: CTAs stop fetching work once it is set,
  // so ids from a malformed row are never used as row addresses.
  const unsigned long long* err;
  // CTA tile schedule (n_tiles == 0 -> per-warp item schedule)
  uint64_t n_tiles;
  uint64_t n_local;
  const uint32_t* tile_node0;  // first local node of the 8-node group
  const uint32_t* tile_q;      // chunk index within each node of the group
  // Tile-shared gathers (union_kernel's group path): whole rows of the group's
  // 8 nodes, decoded from their row offsets; the group takes the path when its
  // id span is dense in edges and it holds <= shared_max_edges (else per-node items).
  const uint64_t* row_off;     // local byte offsets (n_local + 1)
  const uint32_t* degrees;     // local degrees
  const uint32_t* node_lo;     // first / last neighbour id per local node (NULL: path off)
  const uint32_t* node_hi;
  uint64_t shared_max_edges;
  // Back-to-back passes (sb_hb_run without a per-pass host test): every CTA
  // returns at once when the run already finished on the device (NULL: off)
  const unsigned int* stop;
  // Fused shard exchange: every finished row (and its changed flag) is also
  // stored straight into each peer GPU's replica (CUDA IPC / NVLink P2P).
  uint8_t* const* peer_next;     // [npeers] peers' `next` planes
  uint8_t* const* peer_changed;  // [npeers] peers' `changed_out` flags
  int npeers;
};

// Interval mode: runs of consecutive neighbour ids [s, e] are folded with two
// sparse-table rows max(ST_k[s], ST_k[e - 2^k + 1]), k = floor(log2(e - s + 1)).
struct IntervalArgs {
  UnionArgs u;                 // work items / tiles / planes as in the dense kernel
  const uint8_t* st;           // levels 1..K, level k at st + (k-1) * n_global * ROW
  uint64_t n_global;
  int levels;                  // K
  const uint64_t* run_off;     // per item: first run (n_items + 1)
  const uint32_t* run_s;       // run start ids
  const uint32_t* run_e;       // run end ids (inclusive)
  uint64_t run_cap;            // != 0: runs stored below this (an index still being filled
                               // with estimated storage: items past it were not written)
};

// Run index, derived once per graph from the LEB128 stream (run_index_kernel).
struct RunIndexArgs {
  const uint8_t* stream;
  uint64_t stream_len;         // bytes (prefetch bound)
  const uint64_t* item_off;
  const uint32_t* item_base;
  const uint32_t* item_count;
  uint64_t n_items;
  uint64_t item_begin, item_end;  // items this launch covers (an upload chunk, or all)
  uint64_t range_end_byte;        // end of item_end - 1 (the next item may not exist yet)
  const unsigned long long* err;  // upload validation verdict (~0 = clean; NULL: validated)
  uint64_t* run_count;         // count pass: runs per item
  unsigned int* max_run;       // count pass: longest run within an item
  const uint64_t* run_off;     // fill pass: offsets (n_items + 1)
  uint32_t* run_s;
  uint32_t* run_e;
  uint64_t run_cap;            // fill pass: entries of run_s / run_e; an item past it is
  unsigned int* overflow;      // skipped and flags *overflow (NULL: exact allocation)
};

struct EstArgs {
  const uint8_t* plane;        // registers to estimate (global rows)
  uint64_t node_begin;
  uint64_t n_local;
  const double* lc;            // lc[z] = m * log(m / z), host-built (hll.cpp:35)
  double alpha;
  double m;
  const double* c_prev;        // local
  double* c_cur;               // local
  double* sum_d;               // local
  double* sum_d2;              // local
  const uint8_t* changed;      // global-indexed
  uint32_t t;
  unsigned long long* max_ord; // ordered-encoded max increase
  unsigned long long* changed_count;
  const unsigned int* stop;    // NULL, or the device-side "run finished" flag (the pass is a no-op)
};

// Exact mode (bit-parallel BFS over blocks of 2^(P+2) sources).
struct ExactArgs {
  uint8_t* plane;              // init target / count source (global rows)
  uint64_t n;
  uint64_t s0, s1;             // source block
  uint32_t* pop;               // per node popcount after the previous iteration
  unsigned long long* sum_d;   // exact sum of depths
  unsigned long long* sum_d2;  // exact sum of squared depths
  uint32_t* reach;             // nodes reached (incl. itself), accumulated over blocks
  uint32_t* hist;              // hist[v * hist_cap + t] = # sources at depth t
  uint32_t hist_cap;
  uint32_t t;
  unsigned long long* changed_count;
  // exact_init1 (rows at depth 1 straight from the run index)
  const uint32_t* node_item;
  const uint64_t* run_off;
  const uint32_t* run_s;
  const uint32_t* run_e;
};

// On-device grid visibility graph construction (sb_vis.cu).
struct VisArgs {
  uint32_t rows, cols;
  uint64_t radius2;            // 0 = unlimited
  int64_t R;                   // row reach: isqrt(radius2) or max(rows, cols)
  const uint8_t* blocked;      // rows * cols, 1 = obstacle cell
  const uint32_t* pref;        // (rows + 1) * (cols + 1) prefix counts of blocked cells
  const uint32_t* node_of_cell;
  const uint32_t* cell_of_node;
  uint64_t n;
  uint32_t* deg;               // pass 1
  uint64_t* bytes;             // pass 1
  const uint64_t* offsets;     // pass 2
  uint8_t* stream;             // pass 2
  uint32_t* parent;            // components
  uint32_t* masks;             // per-warp-step visibility masks (NULL: recompute in the write pass)
  const uint64_t* step_off;    // first mask word per node (n + 1)
};

cudaError_t launch_vis_prepare(VisArgs& a, uint32_t* pref, uint32_t* tmp_scan, uint64_t* n_out, cudaStream_t s);
cudaError_t launch_vis_maps(const VisArgs& a, const uint32_t* scan, uint32_t* node_of_cell, uint32_t* cell_of_node,
                            cudaStream_t s);
cudaError_t launch_vis_rows(const VisArgs& a, bool write, cudaStream_t s);
cudaError_t launch_vis_steps(const VisArgs& a, uint64_t* steps, cudaStream_t s);
cudaError_t launch_scan_u64(const uint64_t* in, uint64_t* out, uint64_t count, cudaStream_t s);
cudaError_t launch_vis_components(const VisArgs& a, uint32_t* comp, uint32_t* sizes, uint32_t* tmp2n,
                                  uint64_t* n_comp, cudaStream_t s);

struct MetricArgs {
  uint64_t n;
  const double* sum_d;
  const double* sum_d2;
  const uint32_t* nv;
  const uint32_t* deg;
  double *md, *ihh, *tekl, *pv, *m1, *m2;
};

// Exact local metrics (sb_local.cu).  Requires the full graph on the device.
struct LocalArgs {
  uint64_t n;                  // nodes of the graph
  uint64_t v0, v1;             // nodes to compute
  const uint32_t* degrees;     // N
  const uint32_t* node_item;   // N + 1
  const uint64_t* run_off;     // per item (n_items + 1)
  const uint32_t* run_s;
  const uint32_t* run_e;
  uint32_t* span_lo;           // N: first neighbour id (0xffffffff if none)
  uint32_t* span_hi;           // N: last neighbour id
  const uint32_t* reach2;      // N: |B(v, 2)| from the exact BFS at depth 2 (BFS mode)
  uint32_t* lo2;               // [v1 - v0]: 2-hop id window (bitmap mode; NULL in BFS mode)
  uint32_t* hi2;
  unsigned int* max_words;     // [0] max 1-hop window words, [1] max 2-hop window words
  double* control;             // [v1 - v0]
  double* controllability;
  double* clustering;
  unsigned long long* edges_among;  // optional
  unsigned long long* n2;           // optional
  uint32_t* scratch;           // global bitmaps (non-smem path): grid * stride_words
  uint64_t stride_words;       // 2 * (w1_words + 1) [+ w2_words in bitmap mode]
  uint32_t w1_words;
  unsigned long long* work;
};

cudaError_t launch_local_spans(const LocalArgs& a, cudaStream_t s);
// grid_out != NULL: only returns the grid the launch would use.
cudaError_t launch_local(const LocalArgs& a, bool smem, bool n2_bitmap, int* grid_out, cudaStream_t s);
size_t local_smem_limit();

cudaError_t launch_build_items(const BuildArgs& a, cudaStream_t s);
cudaError_t launch_chunk_range(const uint32_t* lo, const uint32_t* hi, uint64_t n0, uint64_t n1, uint32_t* out,
                               cudaStream_t s);
cudaError_t launch_init(int p, uint8_t* plane, uint64_t n, const uint32_t* orig, cudaStream_t s);
cudaError_t launch_union(int p, bool skip, const UnionArgs& a, cudaStream_t s);
cudaError_t launch_st_build(int p, const uint8_t* cur, uint8_t* st, uint64_t n, int levels, cudaStream_t s,
                            bool orop = false);
cudaError_t launch_union_interval(int p, const IntervalArgs& a, cudaStream_t s, bool orop = false);
// Sparse-table levels 1..levels for rows [r0, r1) (each level over the rows the next one reads).
cudaError_t launch_st_build_rows(int p, const uint8_t* cur, uint8_t* st, uint64_t n, int levels, uint64_t r0,
                                 uint64_t r1, cudaStream_t s);
cudaError_t launch_union_or(int p, const UnionArgs& a, cudaStream_t s);
cudaError_t launch_exact_init(int p, const ExactArgs& a, cudaStream_t s);
cudaError_t launch_exact_init1(int p, const ExactArgs& a, cudaStream_t s);
cudaError_t launch_exact_count(int p, const ExactArgs& a, cudaStream_t s);
cudaError_t launch_run_index(const RunIndexArgs& a, bool fill, cudaStream_t s);
// run_off[i] = *total + exclusive prefix of run_count over items [i0, i1], i.e. run_off[i1] is the
// end of item i1 - 1; *total += their sum.
cudaError_t launch_run_offsets(const uint64_t* run_count, uint64_t* run_off, uint64_t i0, uint64_t i1,
                               unsigned long long* total, cudaStream_t s);
cudaError_t launch_estimate(int p, int mode, const EstArgs& a, cudaStream_t s);
cudaError_t launch_to_packed(int p, const uint8_t* bits, uint8_t* packed, uint64_t rows, cudaStream_t s);
cudaError_t launch_from_packed(int p, const uint8_t* packed, uint8_t* bits, uint64_t rows, cudaStream_t s);
cudaError_t launch_metrics(const MetricArgs& a, cudaStream_t s);
// Device-side Alg. 1 test after pass t (flags[0] = stop, [1] = last pass, [2] = converged)
// and a flag clear that is skipped once the run stopped.
cudaError_t launch_decide(unsigned long long* misc, unsigned int* flags, unsigned long long* rec, uint32_t t,
                          uint32_t depth, cudaStream_t s);
cudaError_t launch_clear_flags(const unsigned int* flags, uint8_t* bytes, uint64_t n, cudaStream_t s);
int union_slices(int p);

}  // namespace sb
