// sb_hyperball -- C++ host driver over the facade (the reference's analyze /
// bench shapes): builds or loads a graph, runs HyperBall on
// one GPU, prints per-iteration timings and a metrics summary.
//
//   sb_hyperball synth ROWS COLS RECTS RMIN RMAX SEED RADIUS2 P DEPTH [--skip]
//   sb_hyperball load  FILE.vgacsr P DEPTH [--skip]
//   sb_hyperball analyze ROWS COLS RECTS RMIN RMAX SEED RADIUS2 P DEPTH hyperball|exact OUT.csv [--interval]
//       cmd_build_graph + cmd_analyze on one GPU: the visibility graph is built
//       in HBM from the obstacle mask, then BFS + local metrics -> CSV
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sieveball/hyperball_cuda.hpp"

using namespace sieveball::cuda;

static int cmd_analyze(int argc, char** argv) {
  if (argc < 13) {
    std::fprintf(stderr, "usage: %s analyze ROWS COLS RECTS RMIN RMAX SEED RADIUS2 P DEPTH hyperball|exact OUT.csv "
                         "[--interval]\n", argv[0]);
    return 2;
  }
  const uint32_t rows = std::atoi(argv[2]), cols = std::atoi(argv[3]);
  const uint64_t radius2 = std::strtoull(argv[8], nullptr, 10);
  const HllParams P(std::atoi(argv[9]));
  const uint32_t depth = std::atoi(argv[10]);
  const std::string mode = argv[11];
  if (mode != "hyperball" && mode != "exact") throw std::invalid_argument("mode must be hyperball or exact");
  const bool interval = std::strcmp(argv[argc - 1], "--interval") == 0;
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  auto tc = std::chrono::steady_clock::now();
  DeviceGraph::from_grid(1, 1, std::vector<uint8_t>{0}, 0);  // CUDA context + module load, timed apart
  auto t0 = std::chrono::steady_clock::now();
  std::printf("CUDA context + module load: %.1f ms\n", ms(tc, t0));
  std::vector<uint8_t> mask(static_cast<size_t>(rows) * cols);
  check(sb_grid_synth_mask(rows, cols, std::atoi(argv[4]), std::atoi(argv[5]), std::atoi(argv[6]),
                           std::strtoull(argv[7], nullptr, 10), mask.data()));
  const DeviceGraph g = DeviceGraph::from_grid(rows, cols, mask, radius2);
  auto t1 = std::chrono::steady_clock::now();
  const auto gi = g.grid_info();
  AnalyzeInput in;
  in.deg = g.degrees();
  in.component_id = gi.component_id;
  const uint64_t n = g.node_count();
  in.nv.resize(n);
  in.x.resize(n);
  in.y.resize(n);
  for (uint64_t v = 0; v < n; ++v) {
    in.nv[v] = gi.component_sizes[gi.component_id[v]];
    in.x[v] = (gi.cell_of_node[v] % cols) + 0.5;  // cell centre, unit spacing
    in.y[v] = (gi.cell_of_node[v] / cols) + 0.5;
  }
  const uint32_t it = analyze(g, in, P, depth ? std::optional<uint32_t>(depth) : std::nullopt, mode == "exact",
                              interval, argv[12]);
  auto t2 = std::chrono::steady_clock::now();
  std::printf("graph built on device: N=%llu (%.1f ms); %s BFS + local metrics + CSV: %.1f ms; iterations=%u\n",
              (unsigned long long)n, ms(t0, t1), mode.c_str(), ms(t1, t2), it);
  return 0;
}

int main(int argc, char** argv) {
  try {
    if (argc >= 2 && std::strcmp(argv[1], "analyze") == 0) return cmd_analyze(argc, argv);
    if (argc < 2) {
      std::fprintf(stderr, "usage: %s synth ROWS COLS RECTS RMIN RMAX SEED RADIUS2 P DEPTH [--skip]\n"
                           "       %s load FILE P DEPTH [--skip]\n", argv[0], argv[0]);
      return 2;
    }
    const std::string mode = argv[1];
    bool skip = std::strcmp(argv[argc - 1], "--skip") == 0;
    auto t0 = std::chrono::steady_clock::now();
    std::optional<CompressedCsr> g;
    unsigned p = 10;
    uint32_t depth = 0;
    if (mode == "synth" && argc >= 11) {
      g = CompressedCsr::synth_grid(std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4]), std::atoi(argv[5]),
                                    std::atoi(argv[6]), std::strtoull(argv[7], nullptr, 10),
                                    std::strtoull(argv[8], nullptr, 10));
      p = std::atoi(argv[9]);
      depth = std::atoi(argv[10]);
    } else if (mode == "load" && argc >= 5) {
      g = CompressedCsr::load_vgacsr(argv[2]);
      p = std::atoi(argv[3]);
      depth = std::atoi(argv[4]);
    } else {
      std::fprintf(stderr, "bad arguments\n");
      return 2;
    }
    auto t1 = std::chrono::steady_clock::now();
    HllParams P(p);
    HyperBall hb(*g, P, depth ? std::optional<uint32_t>(depth) : std::nullopt, 0, skip);
    auto t2 = std::chrono::steady_clock::now();
    const uint32_t it = hb.run();
    auto t3 = std::chrono::steady_clock::now();
    const auto st = hb.stats();
    const double ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); }(t2, t3);
    std::printf("graph: N=%llu |E|=%llu stream=%llu B (build %.1f ms, upload+init %.1f ms)\n",
                (unsigned long long)g->node_count(), (unsigned long long)g->edge_count(),
                (unsigned long long)g->desc().stream_len,
                std::chrono::duration<double, std::milli>(t1 - t0).count(),
                std::chrono::duration<double, std::milli>(t2 - t1).count());
    for (const auto& s : st)
      std::printf("t=%u union=%.3f ms estimate=%.3f ms changed=%llu max_inc=%.4f\n", s.t, s.union_ms, s.estimate_ms,
                  (unsigned long long)s.changed_nodes, s.max_increase);
    const double upd = static_cast<double>(g->edge_count()) * P.m * it;
    std::printf("iterations=%u hyperball=%.3f ms  edge-register updates/s=%.3e\n", it, ms, upd / (ms * 1e-3));
    const HyperBallState s = hb.state(false);
    const auto& d = g->desc();
    double md_sum = 0;
    uint64_t cnt = 0;
    for (uint64_t v = 0; v < d.n; ++v) {
      const double md = metrics::mean_depth(s.sum_d[v], d.component_sizes[d.component_id[v]]);
      if (!std::isnan(md)) {
        md_sum += md;
        ++cnt;
      }
    }
    std::printf("mean MD over %llu nodes = %.6f\n", (unsigned long long)cnt, cnt ? md_sum / cnt : NAN);
    return 0;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "invalid argument: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
