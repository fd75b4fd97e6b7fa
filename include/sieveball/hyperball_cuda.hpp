// hyperball_cuda.hpp -- C++ facade over the C-ABI (include/sieveball_cuda.h)
// that restores the reference's C++ API shapes and exception behaviour:
//   HllParams(p)                      hll.hpp:22-29 / hll.cpp:9-19 (invalid_argument)
//   CompressedCsr, neighbors(), load_vgacsr/save_vgacsr, hilbert_reorder
//                                     SPEC.md:174-257
//   hyperball::run / iterate_once / check_convergence
//                                     SPEC.md:418-444
//   metrics::mean_depth / integration_* / moments
//                                     SPEC.md:485-529
//   DeviceGraph::local_metrics        SPEC.md:530-537 (exact, on device)
//   DeviceGraph::from_grid            cmd_build_graph grid -> visibility -> CSR, in HBM
//   ExactBfs                          oracle exact_bfs_all, bit-parallel on device
//   analyze(...)                      cmd_analyze -> metric CSV
// SB_EINVAL -> std::invalid_argument, everything else -> std::runtime_error.
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../sieveball_cuda.h"

namespace sieveball::cuda {

inline void check(int rc) {
  if (rc == SB_OK) return;
  const std::string msg = sb_last_error();
  if (rc == SB_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct HllParams {
  explicit HllParams(unsigned precision) : p(precision) {
    if (p < 4 || p > 16) throw std::invalid_argument("hll: precision must be in [4, 16]");
    m = uint32_t{1} << p;
    row_bytes = m / 2;
    switch (m) {
      case 16: alpha_m = 0.673; break;
      case 32: alpha_m = 0.697; break;
      case 64: alpha_m = 0.709; break;
      default: alpha_m = 0.7213 / (1.0 + 1.079 / m); break;
    }
  }
  unsigned p;
  uint32_t m;
  double alpha_m;
  uint32_t row_bytes;
};

class CompressedCsr {
 public:
  static CompressedCsr synth_grid(uint32_t rows, uint32_t cols, uint32_t n_rects, uint32_t rect_min,
                                  uint32_t rect_max, uint64_t seed, uint64_t radius2, unsigned threads = 0) {
    sb_csr* c = nullptr;
    check(sb_csr_synth_grid(rows, cols, n_rects, rect_min, rect_max, seed, radius2, threads, &c));
    return CompressedCsr(c);
  }
  static CompressedCsr from_adjacency(const std::vector<uint64_t>& off, const std::vector<uint32_t>& ids) {
    sb_csr* c = nullptr;
    check(sb_csr_from_adjacency(off.size() - 1, off.data(), ids.data(), &c));
    return CompressedCsr(c);
  }
  static CompressedCsr load_vgacsr(const std::string& path) {
    sb_csr* c = nullptr;
    check(sb_vgacsr_load(path.c_str(), &c));
    return CompressedCsr(c);
  }
  void save_vgacsr(const std::string& path) const { check(sb_vgacsr_save(c_.get(), path.c_str())); }
  CompressedCsr hilbert_reorder() const {
    sb_csr* c = nullptr;
    check(sb_csr_hilbert_reorder(c_.get(), &c));
    return CompressedCsr(c);
  }
  std::vector<uint32_t> neighbors(uint64_t v) const {
    std::vector<uint32_t> ids(d_.degrees[v]);
    check(sb_csr_neighbors(c_.get(), v, ids.data()));
    return ids;
  }
  const sb_csr_desc& desc() const { return d_; }
  uint64_t node_count() const { return d_.n; }
  uint64_t edge_count() const { return d_.edges; }

 private:
  explicit CompressedCsr(sb_csr* c) : c_(c, sb_csr_destroy) { check(sb_csr_describe(c, &d_)); }
  std::shared_ptr<sb_csr> c_;
  sb_csr_desc d_{};
};

// A graph resident in HBM: uploaded from a CompressedCsr (rows [v0, v1)) or
// built on the device from a raster obstacle mask.
class DeviceGraph {
 public:
  // async_upload: chunked upload overlapped with the first HyperBall pass
  // (sb_graph_create_async); `g` must outlive the upload (wait() / first step).
  explicit DeviceGraph(const CompressedCsr& g, int device = 0, uint64_t v0 = 0, uint64_t v1 = UINT64_MAX,
                       bool async_upload = false) {
    const sb_csr_desc& d = g.desc();
    if (v1 == UINT64_MAX) v1 = d.n;
    sb_graph* gr = nullptr;
    auto create = async_upload ? sb_graph_create_async : sb_graph_create;
    check(create(d.n, d.offsets, d.degrees, d.stream, d.stream_len, d.hilbert_inverse, v0, v1, device, &gr));
    init(gr, d.n, v0, v1);
  }
  void wait() const { check(sb_graph_wait(g_.get())); }
  static DeviceGraph from_grid(uint32_t rows, uint32_t cols, const std::vector<uint8_t>& blocked, uint64_t radius2,
                               int device = 0) {
    if (blocked.size() != static_cast<size_t>(rows) * cols) throw std::invalid_argument("mask size != rows * cols");
    sb_graph* gr = nullptr;
    check(sb_graph_build_grid(rows, cols, blocked.data(), radius2, device, &gr));
    uint64_t n = 0;
    check(sb_graph_stats(gr, &n, nullptr, nullptr, nullptr, nullptr));
    DeviceGraph g;
    g.init(gr, n, 0, n);
    return g;
  }
  struct Local {
    std::vector<double> control, controllability, clustering;
    std::vector<uint64_t> edges_among, n2;
  };
  // Exact local metrics for nodes [v0, v1) (full-graph handle required).
  Local local_metrics(uint64_t v0 = 0, uint64_t v1 = UINT64_MAX) const {
    if (v1 == UINT64_MAX) v1 = n_;
    Local L;
    const uint64_t k = v1 > v0 ? v1 - v0 : 0;
    L.control.resize(k);
    L.controllability.resize(k);
    L.clustering.resize(k);
    L.edges_among.resize(k);
    L.n2.resize(k);
    check(sb_local_metrics(g_.get(), v0, v1, L.control.data(), L.controllability.data(), L.clustering.data(),
                           L.edges_among.data(), L.n2.data()));
    return L;
  }
  struct GridInfo {
    uint32_t rows = 0, cols = 0;
    std::vector<uint32_t> cell_of_node, component_id, component_sizes;
  };
  GridInfo grid_info() const {
    GridInfo gi;
    uint64_t nc = 0;
    check(sb_graph_grid_info(g_.get(), &gi.rows, &gi.cols, nullptr, nullptr, nullptr, &nc));
    gi.cell_of_node.resize(n_);
    gi.component_id.resize(n_);
    gi.component_sizes.resize(nc);
    check(sb_graph_grid_info(g_.get(), nullptr, nullptr, gi.cell_of_node.data(), gi.component_id.data(),
                             gi.component_sizes.data(), nullptr));
    return gi;
  }
  std::vector<uint32_t> degrees() const {
    std::vector<uint32_t> d(nl_);
    check(sb_graph_download(g_.get(), nullptr, d.data(), nullptr));
    return d;
  }
  sb_graph* handle() const { return g_.get(); }
  uint64_t node_count() const { return n_; }
  uint64_t local_count() const { return nl_; }

 private:
  DeviceGraph() = default;
  void init(sb_graph* gr, uint64_t n, uint64_t v0, uint64_t v1) {
    g_.reset(gr, sb_graph_destroy);
    n_ = n;
    nl_ = v1 - v0;
  }
  std::shared_ptr<sb_graph> g_;
  uint64_t n_ = 0, nl_ = 0;
};

struct HyperBallState {
  std::vector<uint8_t> registers;  // latest plane, reference packed layout
  std::vector<double> c_prev, c_curr, sum_d, sum_d2;
  uint32_t t = 0;
  bool converged = false;
};

inline bool check_convergence(double max_increase) { return sb_check_convergence(max_increase) != 0; }

// One GPU's HyperBall over rows [v0, v1) of the graph (whole graph by default).
class HyperBall {
 public:
  HyperBall(const CompressedCsr& g, const HllParams& P, std::optional<uint32_t> depth_limit,
            int device = 0, bool skip_unchanged = false, uint64_t v0 = 0, uint64_t v1 = UINT64_MAX)
      : P_(P) {
    const sb_csr_desc& d = g.desc();
    if (v1 == UINT64_MAX) v1 = d.n;
    sb_graph* gr = nullptr;
    check(sb_graph_create(d.n, d.offsets, d.degrees, d.stream, d.stream_len, d.hilbert_inverse, v0, v1,
                          device, &gr));
    g_.reset(gr, sb_graph_destroy);
    sb_hb* h = nullptr;
    check(sb_hb_create(gr, P.p, depth_limit.value_or(0), skip_unchanged ? SB_HB_SKIP_UNCHANGED : 0u, &h));
    h_.reset(h, sb_hb_destroy);
    n_ = d.n;
    nl_ = v1 - v0;
  }
  HyperBall(const DeviceGraph& g, const HllParams& P, std::optional<uint32_t> depth_limit, uint32_t flags = 0)
      : P_(P) {
    g_ = std::shared_ptr<sb_graph>(g.handle(), [keep = std::make_shared<DeviceGraph>(g)](sb_graph*) {});
    sb_hb* h = nullptr;
    check(sb_hb_create(g.handle(), P.p, depth_limit.value_or(0), flags, &h));
    h_.reset(h, sb_hb_destroy);
    n_ = g.node_count();
    nl_ = g.local_count();
  }
  struct Metrics {
    std::vector<double> md, ihh, tekl, pv, m1, m2;
  };
  // MD / IHH / Tekl / PV / moments for the local range, on device.
  Metrics metrics(const std::vector<uint32_t>& nv, const std::vector<uint32_t>& deg) const {
    Metrics m;
    for (auto* v : {&m.md, &m.ihh, &m.tekl, &m.pv, &m.m1, &m.m2}) v->resize(nl_);
    check(sb_hb_metrics(h_.get(), nv.data(), deg.data(), m.md.data(), m.ihh.data(), m.tekl.data(), m.pv.data(),
                        m.m1.data(), m.m2.data()));
    return m;
  }
  // iterate_once + check_convergence; returns the max cardinality increase.
  double iterate_once() {
    double mx = 0;
    int conv = 0, fin = 0;
    check(sb_hb_step(h_.get(), &mx, &conv, &fin));
    return mx;
  }
  uint32_t run() {
    uint32_t it = 0;
    int conv = 0;
    check(sb_hb_run(h_.get(), &it, &conv));
    return it;
  }
  bool finished() const {
    int fin = 0;
    check(sb_hb_read_state(h_.get(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &fin));
    return fin != 0;
  }
  HyperBallState state(bool with_registers = true) const {
    HyperBallState s;
    s.c_curr.resize(nl_);
    s.c_prev.resize(nl_);
    s.sum_d.resize(nl_);
    s.sum_d2.resize(nl_);
    int conv = 0;
    check(sb_hb_read_state(h_.get(), s.c_curr.data(), s.c_prev.data(), s.sum_d.data(), s.sum_d2.data(),
                           nullptr, &s.t, &conv, nullptr));
    s.converged = conv != 0;
    if (with_registers) {
      s.registers.resize(n_ * P_.row_bytes);
      check(sb_hb_read_registers(h_.get(), SB_REGS_LATEST, 0, n_, s.registers.data()));
    }
    return s;
  }
  std::vector<sb_iter_stats> stats() const {
    uint32_t n = 0;
    check(sb_hb_stats(h_.get(), nullptr, 0, &n));
    std::vector<sb_iter_stats> v(n);
    check(sb_hb_stats(h_.get(), v.data(), n, &n));
    return v;
  }
  void reset() { check(sb_hb_reset(h_.get())); }
  sb_hb* handle() const { return h_.get(); }

 private:
  HllParams P_;
  std::shared_ptr<sb_graph> g_;
  std::shared_ptr<sb_hb> h_;
  uint64_t n_ = 0, nl_ = 0;
};

// Exact neighbourhood function (oracle exact_bfs_all) on the device.
class ExactBfs {
 public:
  ExactBfs(const DeviceGraph& g, std::optional<uint32_t> depth_limit, unsigned log2_block = 12,
           bool interval = false)
      : keep_(std::make_shared<DeviceGraph>(g)), n_(g.node_count()) {
    sb_exact* x = nullptr;
    check(sb_exact_create(g.handle(), log2_block, depth_limit.value_or(0), interval ? SB_HB_INTERVAL : 0u, &x));
    x_.reset(x, sb_exact_destroy);
  }
  uint32_t run(uint64_t src_begin = 0, uint64_t src_end = UINT64_MAX) {
    uint32_t md = 0;
    check(sb_exact_run(x_.get(), src_begin, src_end == UINT64_MAX ? n_ : src_end, &md));
    return md;
  }
  struct Result {
    std::vector<uint64_t> sum_d, sum_d2;
    std::vector<uint32_t> reach, hist;  // hist: n x cap
    uint32_t cap = 0;
    std::vector<double> entropy;
  };
  Result result() const {
    Result r;
    uint32_t md = 0;
    check(sb_exact_stats(x_.get(), nullptr, &md, nullptr, nullptr));
    r.cap = md + 1;
    r.sum_d.resize(n_);
    r.sum_d2.resize(n_);
    r.reach.resize(n_);
    r.hist.resize(n_ * r.cap);
    r.entropy.resize(n_);
    check(sb_exact_read(x_.get(), r.sum_d.data(), r.sum_d2.data(), r.reach.data(), r.hist.data(), r.cap));
    check(sb_depth_entropy(n_, r.hist.data(), r.cap, r.entropy.data()));
    return r;
  }

 private:
  std::shared_ptr<DeviceGraph> keep_;
  std::shared_ptr<sb_exact> x_;
  uint64_t n_ = 0;
};

// hyperball::run on one GPU.
inline HyperBallState run(const CompressedCsr& g, const HllParams& P, std::optional<uint32_t> depth_limit,
                          int device = 0) {
  HyperBall hb(g, P, depth_limit, device);
  hb.run();
  return hb.state(true);
}

namespace metrics {  // SPEC.md:485-529 (per node, closed form)
inline double mean_depth(double sum_d, uint32_t nv) { return nv < 2 ? NAN : sum_d / (nv - 1.0); }
inline double integration_tekl(double md) { return std::log2((md + 2.0) / 3.0); }
inline double relative_asymmetry(double md, uint32_t nv) { return 2.0 * (md - 1.0) / (nv - 2.0); }
inline double diamond(double k) {
  return 2.0 * (k * (std::log2((k + 2.0) / 3.0) - 1.0) + 1.0) / ((k - 1.0) * (k - 2.0));
}
inline double integration_hh(double md, uint32_t nv) {
  if (nv < 3 || std::isnan(md) || !(md > 1.0)) return NAN;  // pre: MD > 1
  return 1.0 / (relative_asymmetry(md, nv) / diamond(nv));
}
inline double integration_pv(double md, uint32_t nv) {
  if (nv < 3 || std::isnan(md)) return NAN;
  const double x = 1.0 - relative_asymmetry(md, nv);
  return x > 0.0 ? (x < 1.0 ? x : 1.0) : 0.0;  // in [0, 1]
}
}  // namespace metrics

// cmd_analyze on one GPU: HyperBall (or exact) BFS metrics +
// exact local metrics -> CSV.  nv / deg / coordinates come from the caller's
// graph description (component sizes per node, degrees, cell centres).
struct AnalyzeInput {
  std::vector<uint32_t> nv, deg, component_id;
  std::vector<double> x, y;
};

inline uint32_t analyze(const DeviceGraph& g, const AnalyzeInput& in, const HllParams& P,
                        std::optional<uint32_t> depth, bool exact, bool interval, const std::string& csv_path) {
  const uint64_t n = g.node_count();
  std::vector<double> md, ihh, tekl, pv, m1, m2, ent(n, NAN), rel(n, NAN);
  uint32_t iterations = 0;
  if (!exact) {
    HyperBall hb(g, P, depth, interval ? SB_HB_INTERVAL : 0u);
    iterations = hb.run();
    auto m = hb.metrics(in.nv, in.deg);
    md = std::move(m.md); ihh = std::move(m.ihh); tekl = std::move(m.tekl);
    pv = std::move(m.pv); m1 = std::move(m.m1); m2 = std::move(m.m2);
  } else {
    ExactBfs x(g, depth, 12, interval);
    iterations = x.run();
    auto r = x.result();
    md.resize(n); ihh.resize(n); tekl.resize(n); pv.resize(n); m1.resize(n); m2.resize(n);
    for (uint64_t v = 0; v < n; ++v) {
      const uint32_t N = in.nv[v];
      md[v] = metrics::mean_depth(static_cast<double>(r.sum_d[v]), N);
      ihh[v] = metrics::integration_hh(md[v], N);
      tekl[v] = N >= 2 ? metrics::integration_tekl(md[v]) : NAN;
      pv[v] = metrics::integration_pv(md[v], N);
      m1[v] = N >= 2 ? md[v] * in.deg[v] : NAN;
      m2[v] = N >= 2 ? static_cast<double>(r.sum_d2[v]) / (N - 1.0) : NAN;
    }
    ent = std::move(r.entropy);
  }
  const auto L = g.local_metrics();
  sb_metric_table t{};
  t.n = n;
  t.x = in.x.empty() ? nullptr : in.x.data();
  t.y = in.y.empty() ? nullptr : in.y.data();
  t.component_id = in.component_id.data();
  t.node_count = in.nv.data();
  t.connectivity = in.deg.data();
  t.md = md.data(); t.ihh = ihh.data(); t.tekl = tekl.data(); t.pv = pv.data();
  t.control = L.control.data(); t.controllability = L.controllability.data(); t.clustering = L.clustering.data();
  t.entropy = ent.data(); t.rel_entropy = rel.data(); t.m1 = m1.data(); t.m2 = m2.data();
  check(sb_metrics_write_csv(csv_path.c_str(), &t));
  return iterations;
}

}  // namespace sieveball::cuda
