/*
 * sieveball_cuda.h -- C-ABI of the B200 HyperBall library (libsieveball_cuda.so).
 *
 * Drop-in boundary for the reference's HyperBall path.  The
 * reference exposes it as C++ (SPEC.md signatures; hyperball.cpp / cgraph.cpp
 * are unshipped, CMakeLists.txt:20,25); this header is the plain-C seam a
 * host in any language binds, and include/sieveball/hyperball_cuda.hpp wraps
 * it back into the reference's C++ shapes and exceptions.
 *
 *   reference interface                                   replaced by
 *   -----------------------------------------------------  ---------------------------
 *   CompressedCsr arrays + load_vgacsr   sb_csr_* / sb_vgacsr_* (host)
 *     (layout :253)                       sb_graph_create (-> HBM)
 *   hyperball::run(graph, HllParams, depth)  sb_hb_create + sb_hb_run
 *   hyperball::iterate_once              sb_hb_step
 *   hyperball::check_convergence         sb_check_convergence
 *   HllParams(p) (hll.cpp:9-19), invalid_argument          SB_EINVAL from sb_hb_create
 *   kernels::Ops nibble_max_inplace / harmonic_sum         fused into the device kernels
 *     (kernels.hpp:21-37)                                  (bit-exact by contract)
 *   metrics: mean_depth, integration_* , moments           sb_hb_metrics
 *
 *   metrics::local_metrics               sb_local_metrics
 *   oracle exact BFS / neighbourhood function sb_exact_* (bit-parallel, on device)
 *   cli cmd_analyze CSV                      sb_metrics_write_csv
 *   cmd_build_graph grid/visibility/CSR  sb_graph_build_grid (on device), sb_grid_synth_mask
 *   parallel_ranges (parallel.hpp:20-47)                   sb_partition_edges + sb_comm
 *
 * Conventions: every function returns SB_OK (0) or an error code; the message
 * of the last error on the calling thread is in sb_last_error().  Host arrays
 * are owned by the caller and copied; handles own all device memory.  One host
 * thread per handle at a time.  No CPU fallback: without a CUDA device every
 * device entry point fails with SB_ECUDA.
 */
#ifndef SIEVEBALL_CUDA_H
#define SIEVEBALL_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SB_OK = 0,
  SB_EINVAL = 1,   /* std::invalid_argument (hll.cpp:10) */
  SB_ERUNTIME = 2, /* std::runtime_error (leb128.hpp:32,38) */
  SB_ECUDA = 3,
  SB_ENCCL = 4,
  SB_ENOMEM = 5
};

/* sb_hb_create flags */
#define SB_HB_SKIP_UNCHANGED 1u /* gather only neighbours whose registers changed last iteration (bit-exact) */
#define SB_HB_SCHEDULE_WARP 2u  /* per-warp work-item schedule instead of the default 8-node CTA tiles */
#define SB_HB_INTERVAL 4u       /* variant: fold runs of consecutive ids via a per-iteration sparse table
                                   (bit-exact; any p; not combinable with SKIP_UNCHANGED) */
#define SB_HB_SCHEDULE_GROUP 8u /* 16-node shared-gather groups wherever the rows overlap densely, at every p and
                                   also on graphs too small to fill the device (default: p >= 9 or mean degree
                                   >= 6000, >= 16 x 4 x SMs nodes, groups within half a resident CTA's share of
                                   the edges); not combinable with SCHEDULE_WARP */

#define SB_HB_WAVEFRONT 16u     /* first sb_hb_run over an sb_graph_create_async graph: run the wavefront
                                   over the upload chunks whatever the stream size (default: streams
                                   >= 1 GB; dense mode, one shard; bit-identical either way) */

/* sb_hb_read_registers `which` */
#define SB_REGS_LATEST 0   /* registers after the last executed iteration (c_t) */
#define SB_REGS_PREVIOUS 1 /* registers before it (c_{t-1}) */

typedef struct sb_csr sb_csr;     /* host CompressedCsr */
typedef struct sb_graph sb_graph; /* device-resident CSR slice on one GPU */
typedef struct sb_hb sb_hb;       /* HyperBallState on one GPU */
typedef struct sb_comm sb_comm;   /* NCCL communicator for node-range sharding */

const char* sb_last_error(void);
const char* sb_version(void);
int sb_device_count(int* n);
/* Device buffers come from the device's default stream-ordered memory pool,
 * which keeps freed blocks so repeated graph / HyperBall create-destroy cycles
 * reuse them (buffers shared over CUDA IPC excepted).  This returns the cached
 * blocks of `device` to the driver (after a device synchronise). */
int sb_release_cached_memory(int device);

/* ---------------- host CompressedCsr ---------------- */
typedef struct {
  uint64_t n;            /* node count N */
  uint64_t edges;        /* |E| = sum of degrees (directed) */
  uint64_t stream_len;   /* offsets[N] */
  const uint64_t* offsets;        /* N+1 byte offsets */
  const uint32_t* degrees;        /* N */
  const uint8_t* stream;          /* stream_len bytes (+64 zero bytes of padding) */
  uint64_t n_components;
  const uint32_t* component_id;   /* N */
  const uint32_t* component_sizes;/* n_components */
  const uint32_t* cell_of_node;   /* N (grid cell index), may be NULL */
  const uint32_t* hilbert_inverse;/* N original id per node, NULL if not reordered */
  double origin_x, origin_y, spacing;
  uint32_t rows, cols;
} sb_csr_desc;

/* Synthetic grid visibility graph: rows x cols cells, n_rects random
 * axis-aligned rectangular obstacles with side in [rect_min, rect_max] cells
 * (seeded), visibility radius^2 in cells^2 (0 = unlimited).  Line of sight is
 * exact in integer arithmetic: the open centre-to-centre segment may not
 * intersect the interior of an obstacle cell.  Ids are raster order. */
int sb_csr_synth_grid(uint32_t rows, uint32_t cols, uint32_t n_rects, uint32_t rect_min,
                      uint32_t rect_max, uint64_t seed, uint64_t radius2, unsigned threads,
                      sb_csr** out);
/* The obstacle mask sb_csr_synth_grid draws (rows * cols bytes, 1 = blocked). */
int sb_grid_synth_mask(uint32_t rows, uint32_t cols, uint32_t n_rects, uint32_t rect_min, uint32_t rect_max,
                       uint64_t seed, uint8_t* blocked);
/* Builds from an uncompressed sorted adjacency (adj_offsets[n+1], adj_ids);
 * rows must be strictly increasing ("non-increasing input -> error"). */
int sb_csr_from_adjacency(uint64_t n, const uint64_t* adj_offsets, const uint32_t* adj_ids,
                          sb_csr** out);
/* Wraps caller arrays (copied); components computed with UnionFind if NULL. */
int sb_csr_from_arrays(uint64_t n, const uint64_t* offsets, const uint32_t* degrees,
                       const uint8_t* stream, uint64_t stream_len, sb_csr** out);
int sb_csr_describe(const sb_csr* c, sb_csr_desc* out);
/* Decodes row v into ids (capacity >= degrees[v]); returns SB_ERUNTIME on a malformed row. */
int sb_csr_neighbors(const sb_csr* c, uint64_t v, uint32_t* ids);
/* Hilbert renumbering: new graph, hilbert_inverse set. */
int sb_csr_hilbert_reorder(const sb_csr* c, sb_csr** out);
int sb_vgacsr_save(const sb_csr* c, const char* path);
int sb_vgacsr_load(const char* path, sb_csr** out);
void sb_csr_destroy(sb_csr* c);
/* Page-locks (pin=1) or releases the stream buffer for full-speed H2D upload. */
int sb_csr_pin(sb_csr* c, int pin);

/* Edge-balanced contiguous node ranges: bounds[0]=0 <= ... <= bounds[parts]=n. */
int sb_partition_edges(uint64_t n, const uint64_t* offsets, const uint32_t* degrees, int parts,
                       uint64_t* bounds);

/* ---------------- device graph + HyperBall ---------------- */
/* Uploads rows [node_begin, node_end) of the CSR (stream slice, offsets,
 * degrees) to HBM of `device`, validates every row (LEB128 well-formed,
 * strictly increasing ids < n, exactly degrees[v] ids) and cuts rows into work
 * items.  orig_id (N entries, NULL = identity) is the hash key per node
 * (SPEC.md:454).  Errors: SB_EINVAL (bad range / empty graph), SB_ERUNTIME
 * (malformed stream), SB_ECUDA / SB_ENOMEM. */
int sb_graph_create(uint64_t n, const uint64_t* offsets, const uint32_t* degrees,
                    const uint8_t* stream, uint64_t stream_len, const uint32_t* orig_id,
                    uint64_t node_begin, uint64_t node_end, int device, sb_graph** out);
/* On-device graph construction (cmd_build_graph's grid -> visibility -> CSR
 * phases, SPEC.md:100-219 / PAPER.md:222-307, run in HBM): rows x cols grid,
 * blocked[r * cols + c] = 1 for obstacle cells, visibility radius^2 in cells^2
 * (0 = unlimited).  Produces the full graph on `device` -- stream, offsets,
 * degrees, UnionFind components and cell map -- byte-identical to
 * sb_csr_synth_grid on the same mask (same exact integer line of sight).
 * Errors: SB_EINVAL (bad sizes), SB_ERUNTIME (no free cell). */
int sb_graph_build_grid(uint32_t rows, uint32_t cols, const uint8_t* blocked, uint64_t radius2, int device,
                        sb_graph** out);
/* Grid metadata of a device-built graph (NULL outputs skipped). */
int sb_graph_grid_info(const sb_graph* g, uint32_t* rows, uint32_t* cols, uint32_t* cell_of_node,
                       uint32_t* component_id, uint32_t* component_sizes, uint64_t* n_components);
/* Copies the device CSR slice back: offsets (n_local + 1, slice-relative), degrees, stream bytes. */
int sb_graph_download(const sb_graph* g, uint64_t* offsets, uint32_t* degrees, uint8_t* stream);
/* Same as sb_graph_create, but the stream bytes are copied in ~16 chunks on a
 * copy stream and validated chunk by chunk on a second stream; the call
 * returns once the copies are enqueued.  The first sb_hb_step starts each
 * chunk's tiles as soon as that chunk is validated, so the PCIe upload
 * overlaps the first iteration.  The host stream buffer must stay valid and
 * unmodified (pinned for full speed) until sb_graph_wait or the first step
 * returns; a malformed stream is reported there (SB_ERUNTIME, sticky). */
int sb_graph_create_async(uint64_t n, const uint64_t* offsets, const uint32_t* degrees,
                          const uint8_t* stream, uint64_t stream_len, const uint32_t* orig_id,
                          uint64_t node_begin, uint64_t node_end, int device, sb_graph** out);
/* Waits for an asynchronous upload and reports its validation result. */
int sb_graph_wait(sb_graph* g);
int sb_graph_stats(const sb_graph* g, uint64_t* n_local, uint64_t* edges_local,
                   uint64_t* stream_bytes_local, uint64_t* n_items, uint32_t* chunk);
void sb_graph_destroy(sb_graph* g);

/* HyperBallState on the device; init (insert orig_id, estimate c_0).
 * p in [4,16] else SB_EINVAL; depth_limit 0 = unlimited. */
int sb_hb_create(sb_graph* g, unsigned p, uint32_t depth_limit, uint32_t flags, sb_hb** out);
/* iterate_once + check_convergence + (if not finished) swap, exactly Alg. 1
 * order.  With an attached communicator the shard exchange
 * and the global max run inside.  *finished = converged || t == depth_limit. */
int sb_hb_step(sb_hb* h, double* max_increase, int* converged, int* finished);
/* Loops sb_hb_step until finished (== hyperball::run). */
int sb_hb_run(sb_hb* h, uint32_t* iterations, int* converged);
/* Split step for same-process shards (tests / single-GPU logical sharding):
 * compute -> exchange_local(all shards) -> finish(global max). */
int sb_hb_step_compute(sb_hb* h, double* local_max_increase);
int sb_hb_exchange_local(sb_hb* const* hs, int count);
int sb_hb_step_finish(sb_hb* h, double global_max_increase, int* converged, int* finished);

/* Registers in the REFERENCE packed layout (m/2 bytes per row, low nibble =
 * even register, hll.hpp:31-32), rows [v0, v1) of the replica. */
int sb_hb_read_registers(const sb_hb* h, int which, uint64_t v0, uint64_t v1, uint8_t* dst);
/* Overwrites the latest registers of ALL rows (packed layout) and re-estimates
 * c for the local range (treated as c_t; t unchanged).  Test hook. */
int sb_hb_set_registers(sb_hb* h, const uint8_t* packed_all_rows);
/* Local-range state (any pointer may be NULL).  c_latest = c_t, c_previous = c_{t-1}. */
int sb_hb_read_state(const sb_hb* h, double* c_latest, double* c_previous, double* sum_d,
                     double* sum_d2, uint8_t* changed, uint32_t* t, int* converged,
                     int* finished);
/* Metrics for the local range: nv = component size per local
 * node, deg = degree per local node.  Outputs may be NULL. */
int sb_hb_metrics(const sb_hb* h, const uint32_t* nv, const uint32_t* deg, double* md,
                  double* ihh, double* tekl, double* pv, double* m1, double* m2);

/* ---------------- exact neighbourhood function ----------------
 * The reference's exact oracle mode (per-source BFS, true neighbourhood
 * function, Eq. 1 identity) as a bit-parallel BFS on the device: the
 * HyperBall loop with every HLL row replaced by a reachability bitset over a
 * block of 2^log2_block sources (log2_block in [12, 16]) and the register max
 * replaced by OR.  Needs the full graph on the device.  depth_limit 0 =
 * unlimited; flags: SB_HB_INTERVAL folds runs of consecutive ids through a
 * sparse table (same result).  sb_exact_run accumulates over the sources
 * [src_begin, src_end) -- shard sources across GPUs and sum the outputs. */
typedef struct sb_exact sb_exact;
int sb_exact_create(sb_graph* g, unsigned log2_block, uint32_t depth_limit, uint32_t flags, sb_exact** out);
int sb_exact_run(sb_exact* x, uint64_t src_begin, uint64_t src_end, uint32_t* max_depth);
/* Per node (N entries): sum_d = sum of BFS depths to every reached source,
 * sum_d2 = sum of squared depths, reach = sources reached incl. itself (the
 * component size N_v when all sources ran, unlimited depth); hist (N x
 * hist_cap, row-major, hist_cap > max depth) = # sources at each depth. */
int sb_exact_read(const sb_exact* x, uint64_t* sum_d, uint64_t* sum_d2, uint32_t* reach, uint32_t* hist,
                  uint32_t hist_cap);
int sb_exact_stats(const sb_exact* x, uint64_t* sources_done, uint32_t* max_depth, double* union_ms,
                   uint64_t* union_launches);
void sb_exact_destroy(sb_exact* x);
/* Shannon entropy (bits) of each node's depth distribution (SPEC.md:531-535,
 * exact-oracle mode): H = -sum_t p_t log2 p_t, p_t = hist[t] / sum_{t>=1} hist[t];
 * NaN for a node that reaches nothing.  Host computation (libm log2). */
int sb_depth_entropy(uint64_t n, const uint32_t* hist, uint32_t hist_cap, double* entropy);

/* ---------------- exact local metrics ----------------
 * For nodes [v0, v1) of a device graph that holds the FULL graph (created with
 * node range [0, N); the 2-hop rows of any node are read):
 *   control         = sum_{w in N(v)} 1/deg(w), the correctly rounded sum
 *                     (128-bit fixed point; order independent); 0 if deg 0
 *   controllability = deg(v) / |N2(v)|, N2 = nodes within 2 hops except v; NaN if empty
 *   clustering      = edges_among(v) / (deg(v) (deg(v) - 1)), NaN if deg < 2
 *   edges_among     = sum_{w in N(v)} |N(w) & N(v)| (directed count), n2 = |N2(v)|
 * connectivity is deg(v).  Outputs have v1 - v0 entries; any may be NULL.
 * Shard by node range across GPUs: no exchange is needed. */
int sb_local_metrics(sb_graph* g, uint64_t v0, uint64_t v1, double* control, double* controllability,
                     double* clustering, uint64_t* edges_among, uint64_t* n2);

/* ---------------- metric table + CSV ----------------
 * One row per node; NULL columns are written as NaN (0 for the counts). */
typedef struct {
  uint64_t n;
  const uint32_t* node_id;          /* NULL: 0..n-1 */
  const double *x, *y;              /* world coordinates of the cell centre */
  const uint32_t* component_id;
  const uint32_t* node_count;       /* N_v */
  const uint32_t* connectivity;     /* deg */
  const double *md, *ihh, *tekl, *pv, *control, *controllability, *clustering, *entropy, *rel_entropy,
      *m1, *m2;
} sb_metric_table;
int sb_metrics_write_csv(const char* path, const sb_metric_table* t);

typedef struct {
  uint32_t t;              /* iteration number */
  float union_ms;          /* fused decode-union kernel (CUDA events) */
  float estimate_ms;       /* estimate + accumulate kernel */
  float exchange_ms;       /* shard exchange (NCCL / local copies) */
  float step_ms;           /* device time from the step's first to its last enqueued operation */
  double max_increase;
  uint64_t changed_nodes;  /* local nodes whose registers changed */
} sb_iter_stats;
/* Copies up to `cap` per-iteration records since create/reset; *count = total. */
int sb_hb_stats(const sb_hb* h, sb_iter_stats* out, uint32_t cap, uint32_t* count);
/* Re-initialises the state (t = 0, registers from orig_id, sums zeroed).
 * Collective with fused P2P peers: with a communicator attached it ends in a
 * barrier; with an external barrier the caller must synchronise all ranks
 * after sb_hb_reset and before the next step. */
int sb_hb_reset(sb_hb* h);
/* Raw CUDA stream the handle launches on (cudaStream_t as void*). */
void* sb_hb_stream(const sb_hb* h);
void sb_hb_destroy(sb_hb* h);

int sb_check_convergence(double max_increase); /* 1 iff max_increase <= 0.5 */

/* ---------------- multi-GPU (one process per GPU) ---------------- */
#define SB_COMM_ID_BYTES 128
int sb_comm_unique_id(void* id_out /* SB_COMM_ID_BYTES */);
int sb_comm_create(int nranks, int rank, const void* id, int device, sb_comm** out);
/* Attaches the communicator; bounds[nranks+1] = node ranges of all ranks
 * (this rank's graph must cover [bounds[rank], bounds[rank+1])). */
int sb_hb_attach_comm(sb_hb* h, sb_comm* c, const uint64_t* bounds);
void sb_comm_destroy(sb_comm* c);

/* Fused shard exchange over peer memory (CUDA IPC -> NVLink P2P): the union
 * kernel's epilogue stores every finished row and changed flag straight into
 * each peer's replica, so no separate row collective runs.  Export this rank's
 * handles, gather all ranks' (any transport), attach.  Iterations are then
 * ordered by the 8-byte max reduction: NCCL all-reduce inside sb_hb_step when
 * a communicator is attached, otherwise the caller's barrier between
 * sb_hb_step_compute and sb_hb_step_finish. */
#define SB_IPC_HANDLE_BYTES 256
int sb_hb_ipc_handles(const sb_hb* h, void* out, size_t cap);
int sb_hb_attach_peers(sb_hb* h, int nranks, int rank, const void* handles /* nranks * SB_IPC_HANDLE_BYTES */,
                       const uint64_t* bounds);

#ifdef __cplusplus
}
#endif
#endif /* SIEVEBALL_CUDA_H */
