// sb_local.cu -- exact local VGA metrics on the device:
//   connectivity    = deg(v)
//   control         = sum_{w in N(v)} 1/deg(w)          (exactly rounded sum)
//   controllability = deg(v) / |N2(v)|,  N2(v) = nodes within two hops, v excluded
//   clustering      = (directed edges among N(v)) / (deg(v) (deg(v) - 1))
// These are "computed exactly from the 1-hop neighbourhood and are unaffected
// by the HLL approximation" (§3.3) and must bit-equal the oracle
// (acceptance criterion 9).
//
// All three passes read the device-resident run index (runs of consecutive
// neighbour ids, built once from the LEB128 stream by run_index_kernel), so
// the per-edge work is proportional to the number of RUNS of the neighbour's
// row, not its degree (~175 runs vs ~20k ids per row on C3):
//   span_kernel   thread per node: first / last neighbour id
//   hop2_kernel   warp per node: the 2-hop id window [lo2, hi2] and control,
//                 summed in 128-bit fixed point (2^-96 units) so the result is
//                 the correctly rounded sum, independent of summation order
//   local_kernel  CTA per node: bitmap of N(v) over [lo1, hi1] + word prefix
//                 popcounts; for every w in N(v) and every run of N(w):
//                 |run & N(v)| by two rank queries (clustering) and a range-OR
//                 into the 2-hop bitmap over [lo2, hi2] (controllability).
//                 Bitmaps live in shared memory when the widest window fits,
//                 else in a per-CTA global scratch (L2-resident).
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

// Warp per node of [v0, v1): lo2 / hi2 and control.
__global__ void __launch_bounds__(256) hop2_kernel(LocalArgs a) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  for (uint64_t v = a.v0 + gw; v < a.v1; v += nw) {
    uint64_t r0, r1;
    node_runs(a, v, r0, r1);
    uint32_t lo = a.span_lo[v], hi = a.span_hi[v];
    U128 acc{0ull, 0ull};
    bool zero_deg = false;
    for (uint64_t r = r0; r < r1; ++r) {
      const uint32_t s = a.run_s[r], e = a.run_e[r];
      for (uint64_t w = s + lane; w <= e; w += 32) {
        const uint32_t dw = a.degrees[w];
        lo = min(lo, a.span_lo[w]);
        hi = max(hi, a.span_hi[w]);
        if (dw == 0) {
          zero_deg = true;  // only in an asymmetric graph: 1/0 = +inf
        } else {
          u128_add(acc, to_fixed96(__ddiv_rn(1.0, static_cast<double>(dw))));
        }
      }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      lo = min(lo, __shfl_xor_sync(FULL, lo, d));
      hi = max(hi, __shfl_xor_sync(FULL, hi, d));
    }
    acc = warp_sum128(acc);
    zero_deg = __any_sync(FULL, zero_deg);
    if (lane == 0) {
      const uint64_t i = v - a.v0;
      a.lo2[i] = lo;
      a.hi2[i] = hi;
      a.control[i] = zero_deg ? INFINITY : fixed96_to_double(acc);
      if (r1 > r0) {
        atomicMax(a.max_words + 0, (a.span_hi[v] - a.span_lo[v]) / 32 + 1);
        atomicMax(a.max_words + 1, (hi - lo) / 32 + 1);
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

// # set bits of bm at relative positions < i.
__device__ __forceinline__ uint32_t rank1(const uint32_t* bm, const uint32_t* pre, uint32_t i) {
  return pre[i >> 5] + __popc(bm[i >> 5] & ((1u << (i & 31)) - 1u));
}

template <bool SMEM>
__global__ void __launch_bounds__(256) local_kernel(LocalArgs a) {
  extern __shared__ uint32_t dyn_s[];
  __shared__ unsigned long long s_node;
  __shared__ unsigned long long s_red[2][8];
  __shared__ uint32_t s_scan[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t w1 = a.w1_words, w2 = a.w2_words;
  uint32_t* base = SMEM ? dyn_s : a.scratch + blockIdx.x * a.stride_words;
  uint32_t* bm1 = base;            // w1 + 1 words (last word stays 0)
  uint32_t* pre1 = base + w1 + 1;  // w1 + 1 words
  uint32_t* bm2 = base + 2 * (w1 + 1);
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
    const uint32_t lo2 = a.lo2[i], hi2 = a.hi2[i];
    const uint32_t n1w = (hi1 - lo1) / 32 + 1, n2w = (hi2 - lo2) / 32 + 1;
    for (uint32_t k = threadIdx.x; k <= n1w; k += blockDim.x) bm1[k] = 0u;
    for (uint32_t k = threadIdx.x; k < n2w; k += blockDim.x) bm2[k] = 0u;
    __syncthreads();
    for (uint64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
      const uint32_t s = a.run_s[r], e = a.run_e[r];
      range_set(bm1, s - lo1, e - lo1);
      range_set(bm2, s - lo2, e - lo2);
    }
    __syncthreads();
    // exclusive prefix popcount of bm1 words [0, n1w]
    {
      const uint32_t per = (n1w + 1 + blockDim.x - 1) / blockDim.x;
      const uint32_t k0 = threadIdx.x * per, k1 = min(k0 + per, n1w + 1);
      uint32_t sum = 0;
      for (uint32_t k = k0; k < k1; ++k) sum += __popc(bm1[k]);
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
        pre1[k] = run;
        run += __popc(bm1[k]);
      }
    }
    __syncthreads();
    // every w in N(v): warp j takes neighbour indices j, j + 8, ...
    unsigned long long among = 0;
    {
      uint64_t idx = 0;
      for (uint64_t r = r0; r < r1; ++r) {
        const uint32_t s = a.run_s[r], e = a.run_e[r];
        const uint64_t len = static_cast<uint64_t>(e - s) + 1;
        // first index >= idx in this run with index % 8 == warp
        uint64_t k = (static_cast<uint64_t>(warp) + 8 - idx % 8) % 8;
        for (; k < len; k += 8) {
          const uint32_t w = s + static_cast<uint32_t>(k);
          uint64_t q0, q1;
          node_runs(a, w, q0, q1);
          for (uint64_t q = q0 + lane; q < q1; q += 32) {
            const uint32_t ws = a.run_s[q], we = a.run_e[q];
            const uint32_t cs = max(ws, lo1), ce = min(we, hi1);
            if (cs <= ce) among += rank1(bm1, pre1, ce - lo1 + 1) - rank1(bm1, pre1, cs - lo1);
            range_set(bm2, ws - lo2, we - lo2);
          }
        }
        idx += len;
      }
    }
    __syncthreads();
    unsigned long long reach = 0;
    for (uint32_t k = threadIdx.x; k < n2w; k += blockDim.x) reach += __popc(bm2[k]);
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      among += __shfl_xor_sync(FULL, among, d);
      reach += __shfl_xor_sync(FULL, reach, d);
    }
    if (lane == 0) {
      s_red[0][warp] = among;
      s_red[1][warp] = reach;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long tri = 0, n2 = 0;
      for (int q = 0; q < 8; ++q) {
        tri += s_red[0][q];
        n2 += s_red[1][q];
      }
      if (v >= lo2 && v <= hi2 && ((bm2[(v - lo2) >> 5] >> ((v - lo2) & 31)) & 1u)) --n2;  // v itself
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
  if (a.v1 > a.v0) hop2_kernel<<<sm_count() * 8, 256, 0, s>>>(a);
  return cudaGetLastError();
}

size_t local_smem_limit() { return 200 * 1024; }

cudaError_t launch_local(const LocalArgs& a, bool smem, int* grid_out, cudaStream_t s) {
  const size_t bytes = smem ? a.stride_words * 4 : 0;
  int per = 0;
  if (smem) {
    cudaError_t e = cudaFuncSetAttribute(local_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(bytes));
    if (e != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, local_kernel<true>, 256, bytes);
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, local_kernel<false>, 256, 0);
  }
  const int g = sm_count() * (per < 1 ? 1 : per);
  if (grid_out) {  // query only (global scratch sizing)
    *grid_out = g;
    return cudaSuccess;
  }
  if (smem)
    local_kernel<true><<<g, 256, bytes, s>>>(a);
  else
    local_kernel<false><<<g, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sb
