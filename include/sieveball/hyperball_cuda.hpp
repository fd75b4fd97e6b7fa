// hyperball_cuda.hpp -- C++ facade over the C-ABI (include/sieveball_cuda.h)
// that restores the reference's C++ API shapes and exception behaviour:
//   HllParams(p)                      hll.hpp:22-29 / hll.cpp:9-19 (invalid_argument)
//   CompressedCsr, neighbors(), load_vgacsr/save_vgacsr, hilbert_reorder
//                                     SPEC.md:174-257
//   hyperball::run / iterate_once / check_convergence
//                                     SPEC.md:418-444
//   metrics::mean_depth / integration_* / moments
//                                     SPEC.md:485-529
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
  if (nv < 3 || std::isnan(md) || md == 1.0) return NAN;
  return 1.0 / (relative_asymmetry(md, nv) / diamond(nv));
}
inline double integration_pv(double md, uint32_t nv) {
  if (nv < 3 || std::isnan(md)) return NAN;
  const double x = 1.0 - relative_asymmetry(md, nv);
  return x > 0.0 ? x : 0.0;
}
}  // namespace metrics

}  // namespace sieveball::cuda
