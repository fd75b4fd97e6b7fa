// sb_local.cu -- exact local VGA metrics on the device:
//   connectivity    = deg(v)
//   control         = sum_{w in N(v)} 1/deg(w)          (exactly rounded sum)
//   controllability = deg(v) / |N2(v)|,  N2(v) = nodes within two hops, v excluded
//   clustering      = (directed edges among N(v)) / (deg(v) (deg(v) - 1))
// These are "computed exactly from the 1-hop neighbourhood and are unaffected
// by the HLL approximation" (§3.3) and must bit-equal the oracle
// (acceptance criterion 9).
//
// The passes read the device-resident run index (runs of consecutive
// neighbour ids, built once from the LEB128 stream by run_index_kernel), so
// the per-edge work is proportional to the number of RUNS of the neighbour's
// row, not its degree (~175 runs vs ~20k ids per row on C3):
//   span_kernel   thread per node: first / last neighbour id
//   ctrl_kernel   warp per node: control, summed in 128-bit fixed point
//                 (2^-96 units) so the result is the correctly rounded sum,
//                 independent of summation order
//   local_kernel  CTA per node: bitmap of N(v) over [lo1, hi1] interleaved with
//                 word prefix popcounts; for every w in N(v) and every run of
//                 N(w): |run & N(v)| by two rank queries (clustering).  The
//                 runs of all w in one run [s, e] of N(v) are one contiguous
//                 range of the run index, strided over by the whole CTA.  The
//                 bitmap lives in shared memory when the widest window fits
//                 (1024-thread CTAs for windows > 56 KB), else in a per-CTA
//                 global scratch (L2-resident).
// |N2(v)| (controllability), two methods chosen by the caller on cost:
//   BFS mode    |B(v, 2)| - 1 from the exact bit-parallel BFS at depth 2
//               (sb_exact_*, the fused decode-union kernels with OR); the
//               kernel only divides
//   bitmap mode local_kernel<., true, .> range-ORs every run of every N(w)
//               into a per-node 2-hop bitmap over [lo2, hi2] (from
//               ctrl_kernel) and popcounts it
#include <cmath>

#include "sb_device.cuh"
#include "sb_internal.h"

namespace sb {

// ---- 128-bit fixed point (96 fractional bits) ------------------------------
struct U128 {
  unsigned long long lo, hi;
};

__device__ __forceinline__ void u128_add(U128& a, const U128& b) {
  const unsigned long long lo = a.lo + b.lo;
  a.hi += b.hi + (lo < a.lo ? 1ull : 0ull);
  a.lo = lo;
}

// x in [2^-32, 1] (x = 1/deg, deg < 2^32) as an exact multiple of 2^-96.
__device__ __forceinline__ U128 to_fixed96(double x) {
  const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(x));
  const int e = static_cast<int>((bits >> 52) & 0x7ff);
  const unsigned long long mant = (bits & ((1ull << 52) - 1)) | (1ull << 52);
  const int sh = e - 979;  // x = mant * 2^(e - 1075); fixed = mant << (96 + e - 1075)
  U128 r;
  r.lo = mant << sh;                      // sh in [12, 44]
  r.hi = mant >> (64 - sh);
  return r;
}

__device__ __forceinline__ double pow2(int k) {  // exact 2^k, |k| < 1000
  return __longlong_as_double(static_cast<long long>(1023 + k) << 52);
}

// Correctly rounded (nearest-even) value of a * 2^-96.
__device__ __forceinline__ double fixed96_to_double(const U128& a) {
  if (a.hi == 0) return __dmul_rn(__ull2double_rn(a.lo), pow2(-96));
  const int lz = __clzll(static_cast<long long>(a.hi));
  unsigned long long top = lz ? (a.hi << lz) | (a.lo >> (64 - lz)) : a.hi;
  const unsigned long long rest = lz ? a.lo << lz : a.lo;
  top |= rest != 0 ? 1ull : 0ull;  // sticky below the 64-bit window
  return __dmul_rn(__ull2double_rn(top), pow2(64 - lz - 96));
}

__device__ __forceinline__ U128 warp_sum128(U128 a) {
#pragma unroll
  for (int d = 16; d; d >>= 1) {
    U128 b;
    b.lo = __shfl_xor_sync(FULL, a.lo, d);
    b.hi = __shfl_xor_sync(FULL, a.hi, d);
    u128_add(a, b);
  }
  return a;
}

// ---- runs of a node --------------------------------------------------------
__device__ __forceinline__ void node_runs(const LocalArgs& a, uint64_t v, uint64_t& r0, uint64_t& r1) {
  r0 = a.run_off[a.node_item[v]];
  r1 = a.run_off[a.node_item[v + 1]];
}

__global__ void __launch_bounds__(256) span_kernel(LocalArgs a) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < a.n; v += gridDim.x * (uint64_t)blockDim.x) {
    uint64_t r0, r1;
    node_runs(a, v, r0, r1);
    a.span_lo[v] = r1 > r0 ? a.run_s[r0] : 0xffffffffu;
    a.span_hi[v] = r1 > r0 ? a.run_e[r1 - 1] : 0u;
  }
}

// Warp per node of [v0, v1): control and the widest 1-hop id window.
__global__ void __launch_bounds__(256) ctrl_kernel(LocalArgs a) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  for (uint64_t v = a.v0 + gw; v < a.v1; v += nw) {
    uint64_t r0, r1;
    node_runs(a, v, r0, r1);
    U128 acc{0ull, 0ull};
    bool zero_deg = false;
    uint32_t lo = a.span_lo[v], hi = a.span_hi[v];  // 2-hop window (bitmap mode)
    for (uint64_t r = r0; r < r1; ++r) {
      const uint32_t s = a.run_s[r], e = a.run_e[r];
      for (uint64_t w = s + lane; w <= e; w += 32) {
        const uint32_t dw = a.degrees[w];
        if (a.lo2) {
          lo = min(lo, a.span_lo[w]);
          hi = max(hi, a.span_hi[w]);
        }
        if (dw == 0) {
          zero_deg = true;  // only in an asymmetric graph: 1/0 = +inf
        } else {
          u128_add(acc, to_fixed96(__ddiv_rn(1.0, static_cast<double>(dw))));
        }
      }
    }
    acc = warp_sum128(acc);
    zero_deg = __any_sync(FULL, zero_deg);
    if (a.lo2) {
#pragma unroll
      for (int d = 16; d; d >>= 1) {
        lo = min(lo, __shfl_xor_sync(FULL, lo, d));
        hi = max(hi, __shfl_xor_sync(FULL, hi, d));
      }
    }
    if (lane == 0) {
      a.control[v - a.v0] = zero_deg ? INFINITY : fixed96_to_double(acc);
      if (r1 > r0) {
        atomicMax(a.max_words, (a.span_hi[v] - a.span_lo[v]) / 32 + 1);
        if (a.lo2) {
          a.lo2[v - a.v0] = lo;
          a.hi2[v - a.v0] = hi;
          atomicMax(a.max_words + 1, (hi - lo) / 32 + 1);
        }
      }
    }
  }
}

// Sets bits [s, e] (relative to the window) of bm.  Interior words are plain
// all-ones stores (any concurrent OR of a subset leaves them all-ones).
__device__ __forceinline__ void range_set(uint32_t* bm, uint32_t s, uint32_t e) {
  const uint32_t ws = s >> 5, we = e >> 5;
  const uint32_t ms = 0xffffffffu << (s & 31), me = 0xffffffffu >> (31 - (e & 31));
  if (ws == we) {
    atomicOr(bm + ws, ms & me);
  } else {
    atomicOr(bm + ws, ms);
    for (uint32_t w = ws + 1; w < we; ++w) bm[w] = 0xffffffffu;
    atomicOr(bm + we, me);
  }
}

// rk[k] = {# set bits in words < k, word k} of the N(v) bitmap: one 8-byte
// shared load per rank query.  rank(i) = # set bits at relative positions < i.
__device__ __forceinline__ uint32_t rank1(const uint2* rk, uint32_t i) {
  const uint2 x = rk[i >> 5];
  return x.x + __popc(x.y & ((1u << (i & 31)) - 1u));
}

// N2BM: |N2(v)| from a per-node 2-hop bitmap (range-OR of every run of every
// N(w) over the 2-hop window) instead of the depth-2 BFS counts in reach2 --
// linear in sum_w deg(w) runs(w), the cheaper choice for large, low-degree graphs.
// BS threads per CTA: 1024 when the per-node windows are so large (wide grids
// in raster id space) that only one or two CTAs fit an SM, so a node's slice
// loop still has 32 warps to hide latency with.
template <bool SMEM, bool N2BM, int BS>
__global__ void __launch_bounds__(BS) local_kernel(LocalArgs a) {
  constexpr int NW = BS / 32;
  extern __shared__ uint2 dyn_s[];
  __shared__ unsigned long long s_node;
  __shared__ unsigned long long s_red[NW], s_reach[NW];
  __shared__ uint32_t s_scan[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint2* rk = SMEM ? dyn_s : reinterpret_cast<uint2*>(a.scratch + blockIdx.x * a.stride_words);  // w1 + 1
  uint32_t* bm2 = reinterpret_cast<uint32_t*>(rk + a.w1_words + 1);  // N2BM: w2 words
  for (;;) {
    if (threadIdx.x == 0) s_node = atomicAdd(a.work, 1ull);
    __syncthreads();
    const uint64_t v = a.v0 + s_node;
    if (v >= a.v1) break;
    const uint64_t i = v - a.v0;
    uint64_t r0, r1;
    node_runs(a, v, r0, r1);
    const uint32_t deg = a.degrees[v];
    if (r1 == r0) {  // isolated node
      if (threadIdx.x == 0) {
        a.controllability[i] = NAN;
        a.clustering[i] = NAN;
        if (a.edges_among) a.edges_among[i] = 0;
        if (a.n2) a.n2[i] = 0;
      }
      __syncthreads();
      continue;
    }
    const uint32_t lo1 = a.span_lo[v], hi1 = a.span_hi[v];
    const uint32_t n1w = (hi1 - lo1) / 32 + 1;
    const uint32_t lo2 = N2BM ? a.lo2[i] : 0u, hi2 = N2BM ? a.hi2[i] : 0u;
    const uint32_t n2w = N2BM ? (hi2 - lo2) / 32 + 1 : 0u;
    for (uint32_t k = threadIdx.x; k <= n1w; k += blockDim.x) rk[k] = make_uint2(0u, 0u);
    if (N2BM)
      for (uint32_t k = threadIdx.x; k < n2w; k += blockDim.x) bm2[k] = 0u;
    __syncthreads();
    for (uint64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {  // runs of N(v) are disjoint
      const uint32_t s = a.run_s[r] - lo1, e = a.run_e[r] - lo1;
      const uint32_t ws = s >> 5, we = e >> 5;
      const uint32_t ms = 0xffffffffu << (s & 31), me = 0xffffffffu >> (31 - (e & 31));
      if (ws == we) {
        atomicOr(&rk[ws].y, ms & me);
      } else {
        atomicOr(&rk[ws].y, ms);
        for (uint32_t w = ws + 1; w < we; ++w) rk[w].y = 0xffffffffu;  // all-ones is OR-stable
        atomicOr(&rk[we].y, me);
      }
      if (N2BM) range_set(bm2, s + lo1 - lo2, e + lo1 - lo2);  // N(v) itself is in N2(v)
    }
    __syncthreads();
    // exclusive prefix popcount of the words [0, n1w]
    {
      const uint32_t per = (n1w + 1 + blockDim.x - 1) / blockDim.x;
      const uint32_t k0 = threadIdx.x * per, k1 = min(k0 + per, n1w + 1);
      uint32_t sum = 0;
      for (uint32_t k = k0; k < k1; ++k) sum += __popc(rk[k].y);
      uint32_t incl = sum;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += y;
      }
      if (lane == 31) s_scan[warp] = incl;
      __syncthreads();
      uint32_t off = 0;
      for (int q = 0; q < warp; ++q) off += s_scan[q];
      uint32_t run = off + incl - sum;
      for (uint32_t k = k0; k < k1; ++k) {
        rk[k].x = run;
        run += __popc(rk[k].y);
      }
    }
    __syncthreads();
    // For a run [s, e] of N(v) the runs of N(s), ..., N(e) are ONE contiguous
    // range of the (node-ordered) run index: the whole CTA strides over it.
    unsigned long long among = 0;
    for (uint64_t r = r0; r < r1; ++r) {
      const uint32_t s = a.run_s[r], e = a.run_e[r];
      const uint64_t q0 = a.run_off[a.node_item[s]], q1 = a.run_off[a.node_item[e + 1]];
      const uint32_t* __restrict__ qs = a.run_s + q0;
      const uint32_t* __restrict__ qe = a.run_e + q0;
      const uint32_t cnt = static_cast<uint32_t>(q1 - q0);
      uint32_t part = 0;  // < 2^32: at most the window size per slice
      for (uint32_t k = threadIdx.x; k < cnt; k += BS) {
        const uint32_t qsk = qs[k], qek = qe[k];
        const uint32_t cs = max(qsk, lo1), ce = min(qek, hi1);
        const bool hit = cs <= ce;  // branch-free: an empty clip queries rank(0) twice
        part += rank1(rk, hit ? ce - lo1 + 1 : 0u) - rank1(rk, hit ? cs - lo1 : 0u);
        if (N2BM) range_set(bm2, qsk - lo2, qek - lo2);
      }
      among += part;
    }
    unsigned long long reach = 0;
    if (N2BM) {
      __syncthreads();
      for (uint32_t k = threadIdx.x; k < n2w; k += blockDim.x) reach += __popc(bm2[k]);
#pragma unroll
      for (int d = 16; d; d >>= 1) reach += __shfl_xor_sync(FULL, reach, d);
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) among += __shfl_xor_sync(FULL, among, d);
    if (lane == 0) {
      s_red[warp] = among;
      s_reach[warp] = reach;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long tri = 0, n2 = 0;
      for (int q = 0; q < NW; ++q) {
        tri += s_red[q];
        n2 += s_reach[q];
      }
      if (N2BM) {  // v itself is not in N2(v)
        if (v >= lo2 && v <= hi2 && ((bm2[(v - lo2) >> 5] >> ((v - lo2) & 31)) & 1u)) --n2;
      } else {
        n2 = a.reach2[v] - 1ull;  // |B(v, 2)| minus v itself
      }
      a.controllability[i] = n2 ? __ddiv_rn(static_cast<double>(deg), static_cast<double>(n2)) : NAN;
      a.clustering[i] = deg >= 2 ? __ddiv_rn(static_cast<double>(tri),
                                             __dmul_rn(static_cast<double>(deg), static_cast<double>(deg - 1)))
                                 : NAN;
      if (a.edges_among) a.edges_among[i] = tri;
      if (a.n2) a.n2[i] = n2;
    }
    __syncthreads();
  }
}

static int sm_count() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

cudaError_t launch_local_spans(const LocalArgs& a, cudaStream_t s) {
  span_kernel<<<sm_count() * 4, 256, 0, s>>>(a);
  if (a.v1 > a.v0) ctrl_kernel<<<sm_count() * 8, 256, 0, s>>>(a);
  return cudaGetLastError();
}

size_t local_smem_limit() { return 200 * 1024; }

template <bool SMEM, bool N2BM, int BS>
static cudaError_t launch_local_t(const LocalArgs& a, int* grid_out, cudaStream_t s) {
  const size_t bytes = SMEM ? a.stride_words * 4 : 0;
  int per = 0;
  if (SMEM) {
    cudaError_t e = cudaFuncSetAttribute(local_kernel<SMEM, N2BM, BS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(bytes));
    if (e != cudaSuccess) return e;
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, local_kernel<SMEM, N2BM, BS>, BS, bytes);
  const int g = sm_count() * (per < 1 ? 1 : per);
  if (grid_out) {  // query only (global scratch sizing)
    *grid_out = g;
    return cudaSuccess;
  }
  local_kernel<SMEM, N2BM, BS><<<g, BS, bytes, s>>>(a);
  return cudaGetLastError();
}

// 256 threads per CTA unless the shared windows exceed 56 KB (fewer than 4 CTAs/SM).
cudaError_t launch_local(const LocalArgs& a, bool smem, bool n2_bitmap, int* grid_out, cudaStream_t s) {
  const bool wide = smem && a.stride_words * 4 > 56 * 1024;
  if (smem) {
    if (wide)
      return n2_bitmap ? launch_local_t<true, true, 1024>(a, grid_out, s) : launch_local_t<true, false, 1024>(a, grid_out, s);
    return n2_bitmap ? launch_local_t<true, true, 256>(a, grid_out, s) : launch_local_t<true, false, 256>(a, grid_out, s);
  }
  return n2_bitmap ? launch_local_t<false, true, 256>(a, grid_out, s) : launch_local_t<false, false, 256>(a, grid_out, s);
}

}  // namespace sb
