// ref_shim.cpp -- C entry points over the COMPILED reference primitives.
//
// TEST INFRASTRUCTURE ONLY (see oracle/sb_oracle.c header).  Built by
// oracle/Makefile together with /root/reference/proj/src/{hll,kernels,
// kernels_scalar,kernels_avx2}.cpp into oracle/_ref/libsbref.so (git-ignored).
// No reference source is copied into this repository; the Makefile compiles
// the files where they lie.
//
// The reference ships no hyperball.cpp, so the loop below restates SPEC.md
// :407-472 / PAPER.md:406-436 exactly like oracle/sb_oracle.c, but every
// register operation goes through the reference's own code:
//   sieveball::hll_insert        (hll.cpp:21-29)
//   sieveball::hll_union_into    (hll.hpp:74-76 -> kernels::ops(), AVX2 when available)
//   sieveball::hll_estimate      (hll.cpp:39-41 -> ops().harmonic_sum + hll.cpp:31-37)
//   sieveball::leb128_decode     (leb128.hpp:28-39)
//   sieveball::parallel_ranges   (parallel.hpp:20-47)
#include <cmath>
#include <cstring>
#include <limits>
#include <span>
#include <stdexcept>
#include <vector>

#include "sieveball/hll.hpp"
#include "sieveball/kernels.hpp"
#include "sieveball/leb128.hpp"
#include "sieveball/parallel.hpp"

using namespace sieveball;

namespace {
int code_of(const std::exception_ptr& e) {
  try {
    std::rethrow_exception(e);
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (...) {
    return 2;
  }
}
}  // namespace

extern "C" {

const char* sbref_ops_name() { return kernels::ops().name; }

uint64_t sbref_splitmix64(uint64_t x) { return splitmix64(x); }

int sbref_params(unsigned p, uint32_t* m, double* alpha, uint32_t* row_bytes) {
  try {
    HllParams P(p);
    *m = P.m;
    *alpha = P.alpha_m;
    *row_bytes = P.row_bytes;
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// Insert `element` into a single counter row (row_bytes = m/2).
int sbref_insert(uint8_t* row, uint64_t element, unsigned p) {
  try {
    HllParams P(p);
    HllRegisterPlane plane(1, P);
    std::memcpy(plane.row(0), row, P.row_bytes);
    hll_insert(plane, 0, element, P);
    std::memcpy(row, plane.row(0), P.row_bytes);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

void sbref_nibble_max(uint8_t* dst, const uint8_t* src, size_t n, int scalar) {
  (scalar ? kernels::scalar_ops() : kernels::ops()).nibble_max_inplace(dst, src, n);
}

void sbref_harmonic(const uint8_t* regs, size_t n, int scalar, uint64_t* num, uint32_t* zeros) {
  const kernels::HarmonicSum s = (scalar ? kernels::scalar_ops() : kernels::ops()).harmonic_sum(regs, n);
  *num = s.numerator;
  *zeros = s.zeros;
}

double sbref_estimate_from_sum(uint64_t num, uint32_t zeros, unsigned p) {
  HllParams P(p);
  kernels::HarmonicSum s;
  s.numerator = num;
  s.zeros = zeros;
  return hll_estimate_from_sum(s, P);
}

double sbref_estimate(const uint8_t* row, unsigned p) { return hll_estimate(row, HllParams(p)); }

// Returns bytes written.
size_t sbref_leb128_encode(uint64_t value, uint8_t* out) {
  std::vector<uint8_t> v = leb128_encode(value);
  std::memcpy(out, v.data(), v.size());
  return v.size();
}

int sbref_leb128_decode(const uint8_t* bytes, size_t len, size_t* pos, uint64_t* out) {
  try {
    *out = leb128_decode(std::span<const uint8_t>(bytes, len), *pos);
    return 0;
  } catch (...) {
    return 2;
  }
}

int sbref_hb_init(uint64_t n, const uint32_t* orig_id, unsigned p, uint8_t* cur, double* c0) {
  try {
    HllParams P(p);
    if (n == 0) throw std::invalid_argument("graph empty");
    HllRegisterPlane plane(n, P);
    for (uint64_t v = 0; v < n; ++v) hll_insert(plane, v, orig_id ? orig_id[v] : v, P);
    std::memcpy(cur, plane.bytes().data(), n * P.row_bytes);
    for (uint64_t v = 0; v < n; ++v) c0[v] = hll_estimate(plane.row(v), P);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// iterate_once over [v0, v1) with parallel_ranges over `threads`.
int sbref_hb_iterate(uint64_t n, const uint64_t* offsets, const uint32_t* degrees,
                     const uint8_t* stream, uint64_t stream_len, unsigned p, uint32_t t,
                     const uint8_t* cur, uint8_t* next, const double* c_prev, double* c_cur,
                     double* sum_d, double* sum_d2, uint64_t v0, uint64_t v1, unsigned threads,
                     double* max_inc) {
  try {
    HllParams P(p);
    const uint32_t rb = P.row_bytes;
    if (v1 > n || v0 > v1) throw std::invalid_argument("node range");
    const double td = static_cast<double>(t);
    const double tt = static_cast<double>(uint64_t{t} * t);
    const unsigned nthreads = threads ? threads : default_thread_count();
    std::vector<double> local(nthreads + 1, -std::numeric_limits<double>::infinity());
    const std::span<const uint8_t> all(stream, stream_len);
    parallel_ranges(v1 - v0, nthreads, [&](uint64_t b, uint64_t e, unsigned w) {
      double mx = -std::numeric_limits<double>::infinity();
      for (uint64_t v = v0 + b; v < v0 + e; ++v) {
        uint8_t* dst = next + v * rb;
        std::memcpy(dst, cur + v * rb, rb);  // next[v] <- cur[v]
        const std::span<const uint8_t> row = all.subspan(0, offsets[v + 1]);
        size_t pos = offsets[v];
        uint64_t prev = 0;
        for (uint32_t k = 0; k < degrees[v]; ++k) {
          const uint64_t x = leb128_decode(row, pos);
          const uint64_t id = k == 0 ? x : prev + x;
          if (id >= n || (k > 0 && x == 0)) throw std::runtime_error("cgraph: bad neighbour id");
          prev = id;
          hll_union_into(dst, cur + id * rb, rb);
        }
        const double c = hll_estimate(dst, P);
        const double delta = c - c_prev[v];
        c_cur[v] = c;
        sum_d[v] = sum_d[v] + td * delta;
        sum_d2[v] = sum_d2[v] + tt * delta;
        if (delta > mx) mx = delta;
      }
      local[w] = mx;
    });
    double mx = -std::numeric_limits<double>::infinity();
    for (double x : local) mx = x > mx ? x : mx;
    if (max_inc) *max_inc = mx;
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

}  // extern "C"
