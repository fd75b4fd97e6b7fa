// sb_kernels.cu -- sm_100a kernels of the HyperBall hot path.
//
//   build_items_kernel: validates the LEB128 delta-CSR once at upload and cuts
//                      every row into work items of <= `chunk` neighbours
//   init_kernel<P>   : hll_init: insert orig_id[v]
//   union_kernel<P>  : fused decode-union (PAPER.md:469-475 replaced): CTA tile
//                      of 8 consecutive nodes x one work item each, warp-
//                      cooperative LEB128 decode, 16-B coalesced row gathers,
//                      bit-serial 9-way register max on bit-sliced rows, per-node
//                      changed flag, optional P2P stores into peer replicas
//   union_interval_kernel<P> + st_build_kernel<P> : the interval variant (runs of
//                      consecutive ids folded through a per-iteration sparse table)
//   run_index_kernel : runs of consecutive ids per work item, once per graph
//   estimate_kernel<P>: hll_cardinality + hll_accumulate:
//                      integer harmonic sum -> bit-exact estimate (hll.cpp:31-37),
//                      sum_d/sum_d2 accumulation, global max increase
//   exact_init / exact_count : exact mode (bitset rows, OR union)
//   to_packed / from_packed : export/import in the reference packed layout
//   metrics_kernel   : MD / IHH / Tekl / PV / moments
#include <cstdio>
#include <cstdlib>

#include "sb_device.cuh"
#include "sb_internal.h"

namespace sb {

// ------------------------------------------------------------------ build
// Upload-time validation and work-item cutting (leb128.hpp:28-39, SPEC.md:
// 174-177, restricted to 32-bit ids).  A row is valid iff
//   * it holds exactly deg varints and ends on a terminator (no truncation,
//     no trailing bytes), none longer than 10 bytes (leb128.hpp:38),
//   * no varint after the first has value 0 (ids strictly increasing),
//   * the sum of its varints -- the last id -- is < N (so no id is >= N and no
//     32-bit wrap: every delta is >= 1).
// Canonical varints of ids < 2^32 are at most 5 bytes.  The reference decoder
// also accepts non-canonical encodings of up to 10 bytes (zero-payload
// continuation bytes, leb128.hpp:28-39); a row holding a byte with >= 5
// continuation bytes before it is re-checked by a scalar decode with exactly
// the reference's semantics (long_row_ok) -- rare, so the SWAR fast path below
// stays 5-byte only.  On an accepted row every byte at depth >= 5 has zero
// payload, so the device decoders' 4-byte look-back is exact for it.
// All four are reductions over the row's bytes, so one warp streams a row in
// 512-byte windows (16 bytes per lane, byte-parallel SWAR on 32-bit words)
// and reduces across lanes once per row; only the windows holding an item cut
// (rows with deg > chunk) run a warp scan to place the cut and its base id.
// The previous 8 bytes of the window come from the neighbour lane (or the
// previous window), since a varint's value depends on up to 4 bytes before its
// terminator.  Bytes outside the row read as 0x00: counted nowhere, and as
// look-back they look like a terminator, i.e. the row starts on a varint boundary.
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// 0x80 in every byte of x whose low 7 bits are zero.
__device__ __forceinline__ uint32_t zero_payload(uint32_t x) {
  return ~((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) & 0x80808080u;
}

// Scalar decode of one row with the reference's semantics: leb128_decode
// (leb128.hpp:28-39: truncation or > 10 bytes -> error) per varint, id =
// first or prev + delta, id < N, delta != 0 after the first, no trailing bytes.
// Deltas >= 2^32 are rejected (the u64 sum could wrap below prev: a
// non-increasing row).
__device__ bool long_row_ok(const uint8_t* stream, uint64_t pos, uint64_t end, uint32_t deg, uint64_t n,
                            uint32_t* lo) {
  uint64_t prev = 0;
  for (uint32_t k = 0; k < deg; ++k) {
    uint64_t x = 0;
    unsigned shift = 0;
    bool term = false;
    for (int i = 0; i < 10 && !term; ++i) {
      if (pos >= end) return false;
      const uint8_t b = stream[pos++];
      if (shift < 64) x |= static_cast<uint64_t>(b & 0x7fu) << shift;
      term = !(b & 0x80u);
      shift += 7;
    }
    if (!term || x >= (1ull << 32)) return false;
    const uint64_t id = k ? prev + x : x;
    if (id >= n || (k && x == 0)) return false;
    if (!k) *lo = static_cast<uint32_t>(id);
    prev = id;
  }
  return pos == end;
}

__global__ void __launch_bounds__(256, 3) build_items_kernel(BuildArgs a) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  const uint64_t node_end = a.node_end ? a.node_end : a.n_local;
  for (uint64_t node = a.node_begin + gw; node < node_end; node += nw) {
    const uint64_t pos0 = a.row_off[node];
    const uint64_t end = a.row_off[node + 1];
    const uint32_t deg = a.degrees[node];
    const uint32_t i0 = a.node_item[node];
    if (lane == 0) {
      a.item_off[i0] = pos0;
      a.item_base[i0] = 0;
      a.item_count[i0] = deg < a.chunk ? deg : a.chunk;
      a.item_node[i0] = static_cast<uint32_t>(node);
    }
    if (deg == 0 || end <= pos0) {
      if (lane == 0) {
        if (deg != 0 || end != pos0) atomicMin(a.err_node, static_cast<unsigned long long>(node));
        a.node_lo[node] = 0xffffffffu;
        a.node_hi[node] = 0u;
      }
      continue;
    }
    uint32_t cnt = 0, zeros = 0, lng = 0;  // per lane (lng: a byte at varint depth >= 5)
    unsigned long long sum = 0;            // per lane: sum of its varint contributions
    uint32_t px2 = 0, px3 = 0;             // words 2, 3 of the previous window's lane 31
    uint32_t done = 0;                     // terminators before this window (cut rows only)
    unsigned long long done_sum = 0;       // their contributions
    uint32_t next_cut = a.chunk;           // row index of the next item's first id
    // software pipeline: the next window's 16 bytes per lane are in flight
    // while this one is reduced (plus an L2 prefetch two windows ahead)
    uint4 qn = make_uint4(0u, 0u, 0u, 0u);
    if ((pos0 & ~15ull) + 16 * lane < end) qn = __ldg(reinterpret_cast<const uint4*>(a.stream + (pos0 & ~15ull) + 16 * lane));
    for (uint64_t wb = pos0 & ~15ull; wb < end; wb += 512) {
      if (lane < 4 && wb + 1024 + 128 * lane < end) prefetch_l2(a.stream + wb + 1024 + 128 * lane);
      const uint64_t lb = wb + 16 * lane;  // this lane's first byte
      uint32_t x[4] = {qn.x, qn.y, qn.z, qn.w};
      qn = make_uint4(0u, 0u, 0u, 0u);
      if (lb + 512 < end) qn = __ldg(reinterpret_cast<const uint4*>(a.stream + lb + 512));
      // valid-byte flags (0x80 per byte in [pos0, end)); invalid bytes -> 0x00
      uint32_t vm[4] = {0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u};
      if (wb < pos0 || wb + 512 > end) {  // warp-uniform: only a row's first / last window is partial
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t lo = static_cast<int64_t>(pos0) - static_cast<int64_t>(lb + 4 * i);  // bytes below pos0
          const int64_t hi = static_cast<int64_t>(end) - static_cast<int64_t>(lb + 4 * i);   // bytes below end
          uint32_t m = 0x80808080u;
          if (lo > 0) m = lo >= 4 ? 0u : m << (8 * lo);
          if (hi < 4) m &= hi <= 0 ? 0u : 0x80808080u >> (8 * (4 - hi));
          vm[i] = m;
          x[i] &= (m >> 7) * 0xffu;
        }
      }
      uint32_t p3 = __shfl_up_sync(FULL, x[3], 1), p2 = __shfl_up_sync(FULL, x[2], 1);
      if (lane == 0) {
        p3 = px3;
        p2 = px2;
      }
      px3 = __shfl_sync(FULL, x[3], 31);
      px2 = __shfl_sync(FULL, x[2], 31);
      uint32_t lcnt = 0, tw[4];
      unsigned long long lsum = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t w = x[i];
        const uint32_t wp = i >= 1 ? x[i - 1] : p3;
        const uint32_t wpp = i >= 2 ? x[i - 2] : (i == 1 ? p3 : p2);
        const uint32_t F = w & 0x80808080u, Fp = wp & 0x80808080u, Fpp = wpp & 0x80808080u;
        const uint32_t m1 = __funnelshift_l(Fp, F, 8);
        const uint32_t m2 = m1 & __funnelshift_l(Fp, F, 16);
        const uint32_t m3 = m2 & __funnelshift_l(Fp, F, 24);
        const uint32_t m4 = m3 & Fp;
        const uint32_t m5 = m4 & __funnelshift_l(Fpp, Fp, 8);
        lng |= m5 & vm[i];  // a varint longer than 5 bytes: the scalar check decides
        const uint32_t T = ~w & 0x80808080u & vm[i];
        tw[i] = T;
        lcnt += __popc(T);
        // zero-valued varint: terminator whose payload and whole look-back chain are zero
        const uint32_t z = zero_payload(w), zp = zero_payload(wp);
        const uint32_t z1 = __funnelshift_l(zp, z, 8), z2 = __funnelshift_l(zp, z, 16);
        const uint32_t z3 = __funnelshift_l(zp, z, 24), z4 = zp;
        zeros += __popc(T & z & (~m1 | z1) & (~m2 | z2) & (~m3 | z3) & (~m4 | z4));
        const uint32_t D7 = ((m1 >> 7) + (m2 >> 7) + (m3 >> 7) + (m4 >> 7)) * 7u;
        const uint32_t P = w & 0x7f7f7f7fu;
#pragma unroll
        for (int k = 0; k < 4; ++k) lsum += static_cast<unsigned long long>(byte_of(P, k)) << byte_of(D7, k);
      }
      cnt += lcnt;
      sum += lsum;
      if (next_cut < deg) {  // warp-uniform: this row is cut into several items
        uint32_t incl = lcnt;
        unsigned long long sincl = lsum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(FULL, incl, d);
          const unsigned long long ys = __shfl_up_sync(FULL, sincl, d);
          if (lane >= d) {
            incl += y;
            sincl += ys;
          }
        }
        const uint32_t excl = incl - lcnt;
        const uint32_t wtot = __shfl_sync(FULL, incl, 31);
        // every cut whose last id before it falls in this window (several when
        // chunk < 512 ids): the lane holding that id walks its bytes in order
        while (next_cut < deg && done + wtot >= next_cut) {  // warp-uniform
          const uint32_t want = next_cut - 1 - done;  // window rank of the last id before the cut
          if (want >= excl && want < incl) {
            uint32_t r = excl;
            unsigned long long part = done_sum + (sincl - lsum);
            bool found = false;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t w = x[i];
              const uint32_t wp = i >= 1 ? x[i - 1] : p3;
              const uint32_t F = w & 0x80808080u, Fp = wp & 0x80808080u;
              const uint32_t m1 = __funnelshift_l(Fp, F, 8);
              const uint32_t m2 = m1 & __funnelshift_l(Fp, F, 16);
              const uint32_t m3 = m2 & __funnelshift_l(Fp, F, 24);
              const uint32_t m4 = m3 & Fp;
              const uint32_t D = (m1 >> 7) + (m2 >> 7) + (m3 >> 7) + (m4 >> 7);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                if (!found) {
                  const uint32_t dk = (D >> (8 * k)) & 0xffu;
                  part += static_cast<unsigned long long>((w >> (8 * k)) & 0x7fu) << (7 * dk);
                  if ((tw[i] >> (8 * k + 7)) & 1u) {
                    if (r == want) {
                      found = true;
                      const uint32_t it = i0 + next_cut / a.chunk;
                      a.item_off[it] = lb + 4 * i + k + 1;
                      a.item_base[it] = static_cast<uint32_t>(part);
                      a.item_count[it] = (deg - next_cut) < a.chunk ? deg - next_cut : a.chunk;
                      a.item_node[it] = static_cast<uint32_t>(node);
                    }
                    ++r;
                  }
                }
              }
            }
          }
          next_cut += a.chunk;
        }
        done += wtot;
        done_sum += __shfl_sync(FULL, sincl, 31);
      }
    }
    // row totals
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      cnt += __shfl_xor_sync(FULL, cnt, o);
      zeros += __shfl_xor_sync(FULL, zeros, o);
      lng |= __shfl_xor_sync(FULL, lng, o);
      sum += __shfl_xor_sync(FULL, sum, o);
    }
    if (lane == 0) {
      // the first varint (the absolute first id) may be 0
      uint32_t first = 0;
      for (uint64_t b = pos0, sh = 0; b < end && b < pos0 + 5; ++b, sh += 7) {  // longer: the scalar check
        const uint8_t c = a.stream[b];
        first |= static_cast<uint32_t>(c & 0x7fu) << sh;
        if (!(c & 0x80u)) break;
      }
      const bool first_zero = first == 0;
      const bool ends_on_terminator = !(a.stream[end - 1] & 0x80u);
      const bool ok = lng ? long_row_ok(a.stream, pos0, end, deg, a.n_global, &first)
                          : cnt == deg && ends_on_terminator && zeros == (first_zero ? 1u : 0u) && sum < a.n_global;
      if (!ok) atomicMin(a.err_node, static_cast<unsigned long long>(node));
      a.node_lo[node] = first;
      a.node_hi[node] = static_cast<uint32_t>(sum);
    }
  }
}

// ------------------------------------------------------------------ init
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {  // hll.hpp:13-20
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

template <int P>
__global__ void __launch_bounds__(256) init_kernel(uint8_t* plane, uint64_t n, const uint32_t* orig) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
  constexpr int RPG = G::GB * 2;  // registers per group
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t total = n * G::GROUPS;
  for (uint64_t i = tid; i < total; i += gridDim.x * (uint64_t)blockDim.x) {
    const uint64_t v = i / G::GROUPS;
    const int g = static_cast<int>(i % G::GROUPS);
    // hll_insert (hll.cpp:21-29)
    const uint64_t h = splitmix64(orig ? static_cast<uint64_t>(orig[v]) : v);
    const uint32_t idx = static_cast<uint32_t>(h >> (64 - P));
    const uint64_t w = h << P;
    const unsigned lz = w == 0 ? (64 - P) : static_cast<unsigned>(__clzll(static_cast<long long>(w)));
    const uint32_t rho = lz + 1 < 15u ? lz + 1 : 15u;
    Grp x = grp_zero();
    if (static_cast<int>(idx / RPG) == g) {
      const uint32_t bit = 1u << (idx % RPG);
      x.b0 = (rho & 1u) ? bit : 0u;
      x.b1 = (rho & 2u) ? bit : 0u;
      x.b2 = (rho & 4u) ? bit : 0u;
      x.b3 = (rho & 8u) ? bit : 0u;
    }
    IO::st(plane + v * G::ROW + static_cast<uint64_t>(g) * G::GB, x);
  }
}

// ------------------------------------------------------------------ union
// Union kernel tuning knobs (A/B-selectable at run time for p=10):
//   U    rows per batch (loads in flight per lane per buffer)
//   DB   double-buffered batches (batch k+1 loads issued before batch k's max)
//   MINB minimum resident CTAs per SM (__launch_bounds__ register cap)
//   ACC2 two accumulators alternating between batches (shorter dependency chain)
//   KWAY bit-serial (U+1)-way max instead of the pairwise tree (kway_max)
//   OR   exact mode: rows are reachability bitsets, the union is a plain OR
//   D16  per-node feeder decodes 512-byte steps into uncompacted slots (decode_step16)
template <int U_, bool DB_, int MINB_, bool ACC2_, bool KWAY_ = false, bool OR_ = false, bool D16_ = false>
struct UCfg {
  static constexpr int U = U_;
  static constexpr bool DB = DB_;
  static constexpr int MINB = MINB_;
  static constexpr bool ACC2 = ACC2_;
  static constexpr bool KWAY = KWAY_;
  static constexpr bool OR = OR_;
  static constexpr bool D16 = D16_;
};
// U rows in flight per lane: 8 (a batch of 8 * SUB ids).  p >= 9: 128-byte
// decode windows, at most one per batch.  p < 9 (rows of <= 128 B, where the
// decode is most of the per-edge work): 512-byte decode steps (D16), 2..16
// batches per step.
template <int P>
using DefaultCfg = UCfg<8, false, 4, false, true, false, (P < 9)>;

// Per-warp id feeder: decodes one 128-byte window of the item's LEB128 stream
// at a time (decode_step4) into a shared buffer (compacted; tail padded with
// the last id, harmless because max is idempotent) and hands out batches of
// BATCH = U * SUB ids.  D16: 512-byte steps (decode_step16), one slot per byte
// in a lane-major layout of stride 17, batches up to the step's last id.
template <int P, bool SKIP, int U, bool D16 = false>
struct Feeder {
  using G = Geo<P>;
  static constexpr int BATCH = U * G::SUB;
  static constexpr int BUF = D16 ? 17 * 32 : 128 + BATCH;  // one decode step of ids + padding
  static_assert(!D16 || (!SKIP && BATCH % 16 == 0 && 512 % BATCH == 0), "D16 feeder shape");
  uint32_t* buf;
  uint64_t pos;
  uint32_t rem, base;
  int n, i;

  // Returns false when the item is exhausted.
  __device__ __forceinline__ bool next(const UnionArgs& a, int lane) {
    while (i >= n) {
      if (rem == 0) return false;
      __syncwarp();  // every lane finished reading the previous window's ids
      if constexpr (D16) {
        const Decode16 d = decode_step16(a.stream, pos, rem, base, buf, lane);
        if (d.advance == 0) {  // unreachable on a validated stream
          rem = 0;
          return false;
        }
        pos += d.advance;
        rem -= d.wanted;
        base = d.last;
        n = (d.advance + BATCH - 1) / BATCH * BATCH;  // slots past the last id repeat it
      } else {
        const Decode4 d = decode_step4<SKIP, BATCH>(a.stream, pos, rem, base, a.changed_in, buf, lane);
        if (d.advance == 0) {  // unreachable on a validated stream
          rem = 0;
          return false;
        }
        pos += d.advance;
        rem -= d.wanted;
        base = d.last;
        n = d.count;
      }
      i = 0;
      __syncwarp();
    }
    return true;
  }

  // D16: every slot holds an id of this item's node before the first decode
  // (decode_step16 only overwrites the slots of wanted terminators).
  __device__ __forceinline__ void prefill(uint32_t id, int lane) {
    if constexpr (D16) {
      __syncwarp();  // the previous item's batches are read
#pragma unroll
      for (int k = 0; k < 17; ++k) buf[32 * k + lane] = id;
    }
  }

  // Row id of slot i + q * SUB + sub (q compile-time after unrolling).
  __device__ __forceinline__ uint32_t id(int q, int sub) const {
    if constexpr (D16) {
      const uint32_t* b = buf + 17 * (i >> 4);
      if constexpr (G::SUB >= 16)
        return b[17 * (q * (G::SUB >> 4)) + 17 * (sub >> 4) + (sub & 15)];
      else
        return b[17 * ((q * G::SUB) >> 4) + ((q * G::SUB) & 15) + sub];
    } else {
      return buf[i + q * G::SUB + sub];
    }
  }
};

// Row base of this lane as an opaque 64-bit register, so each gathered row
// address is a single IMAD.WIDE.U32 (id * ROW + base) on the FMA pipe instead
// of a multiply plus a 64-bit add chain on the ALU pipe (which the LOP3 max
// already saturates).
__device__ __forceinline__ const uint8_t* opaque(const uint8_t* p) {
  asm volatile("" : "+l"(p));
  return p;
}

template <int P, int U, class F>
__device__ __forceinline__ void load_batch(Grp (&x)[U], const uint8_t* curb, const F& f, int sub) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
#pragma unroll
  for (int q = 0; q < U; ++q) x[q] = IO::ld(curb + static_cast<uint64_t>(f.id(q, sub)) * G::ROW);
}

// p = 4 (8-byte rows of four 16-bit planes): two rows per 32-bit plane word --
// row 2k in the low halves, row 2k+1 in the high ones (one PRMT per plane) --
// so one bit-serial max covers two rows; the halves are merged once per item.
template <int P, int U, class F>
__device__ __forceinline__ void load_batch_pairs(Grp (&x)[U / 2], const uint8_t* curb, const F& f, int sub) {
  using G = Geo<P>;
#pragma unroll
  for (int q = 0; q < U / 2; ++q) {
    const uint2 r0 = __ldg(reinterpret_cast<const uint2*>(curb + static_cast<uint64_t>(f.id(2 * q, sub)) * G::ROW));
    const uint2 r1 = __ldg(reinterpret_cast<const uint2*>(curb + static_cast<uint64_t>(f.id(2 * q + 1, sub)) * G::ROW));
    x[q] = Grp{__byte_perm(r0.x, r1.x, 0x5410), __byte_perm(r0.x, r1.x, 0x7632), __byte_perm(r0.y, r1.y, 0x5410),
               __byte_perm(r0.y, r1.y, 0x7632)};
  }
}

// acc <- max(acc, x[0..U)) as a balanced tree: depth log2(U)+1 maxes instead
// of a U-long serial chain through acc (the ripple LOP3s are latency-bound).
template <int U>
__device__ __forceinline__ void tree_max(Grp& acc, Grp (&x)[U]) {
#pragma unroll
  for (int s = 1; s < U; s <<= 1) {
#pragma unroll
    for (int q = 0; q + s < U; q += 2 * s) bsmax(x[q], x[q + s]);
  }
  bsmax(acc, x[0]);
}

// acc <- max(acc, x[0..U)) decided MSB-first over all K = U+1 values at once:
// M3 = OR of the b3 planes; a value stays "alive" at a register position while
// its bits so far equal the maximum's; M_k = OR of b_k over the alive values.
// With the AND folded into the OR-accumulate (one LOP3 each) this is
// ceil((K-1)/2) + 6K LOP3 (58 for K = 9) instead of 8U (64) for the tree.
// Written as explicit lop3 so ptxas keeps exactly that count: left to itself
// it turned each M_k accumulation into a tree over (b_k & alive) terms with
// the alive masks recomputed beside it (62 LOP3 per batch on the ALU pipe the
// kernel is bound by); the serial accumulate's latency is hidden by the 8
// warps per scheduler.
template <uint32_t LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(r) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return r;
}
constexpr uint32_t kOr3 = 0xfe;      // a | b | c
constexpr uint32_t kOrNot = 0xf3;    // a | ~b
constexpr uint32_t kAnd = 0xc0;      // a & b
constexpr uint32_t kOrAnd = 0xf8;    // a | (b & c)
constexpr uint32_t kAndOrNot = 0xd0; // a & (b | ~c)

template <int U>
__device__ __forceinline__ void kway_max(Grp& acc, const Grp (&x)[U]) {
  // M3: OR of the K b3 planes, three at a time
  uint32_t m3 = acc.b3;
  int q0 = 0;
  if (U % 2 == 1) {
    m3 |= x[0].b3;  // odd U: one plain OR first, then pairs
    q0 = 1;
  }
#pragma unroll
  for (int q = q0; q + 1 < U; q += 2) m3 = lop3<kOr3>(m3, x[q].b3, x[q + 1].b3);
  uint32_t al[U + 1];
  al[U] = lop3<kOrNot>(acc.b3, m3, 0u);
#pragma unroll
  for (int q = 0; q < U; ++q) al[q] = lop3<kOrNot>(x[q].b3, m3, 0u);
  uint32_t m2 = lop3<kAnd>(al[U], acc.b2, 0u);
#pragma unroll
  for (int q = 0; q < U; ++q) m2 = lop3<kOrAnd>(m2, al[q], x[q].b2);
  al[U] = lop3<kAndOrNot>(al[U], acc.b2, m2);
#pragma unroll
  for (int q = 0; q < U; ++q) al[q] = lop3<kAndOrNot>(al[q], x[q].b2, m2);
  uint32_t m1 = lop3<kAnd>(al[U], acc.b1, 0u);
#pragma unroll
  for (int q = 0; q < U; ++q) m1 = lop3<kOrAnd>(m1, al[q], x[q].b1);
  al[U] = lop3<kAndOrNot>(al[U], acc.b1, m1);
#pragma unroll
  for (int q = 0; q < U; ++q) al[q] = lop3<kAndOrNot>(al[q], x[q].b1, m1);
  uint32_t m0 = lop3<kAnd>(al[U], acc.b0, 0u);
#pragma unroll
  for (int q = 0; q < U; ++q) m0 = lop3<kOrAnd>(m0, al[q], x[q].b0);
  acc = Grp{m0, m1, m2, m3};
}

// Exact mode (bitset rows): the register max degenerates to OR.
template <bool OR>
__device__ __forceinline__ void combine(Grp& a, const Grp& b) {
  if (OR) {
    a.b0 |= b.b0;
    a.b1 |= b.b1;
    a.b2 |= b.b2;
    a.b3 |= b.b3;
  } else {
    bsmax(a, b);
  }
}

template <int U>
__device__ __forceinline__ void or_all(Grp& acc, const Grp (&x)[U]) {
#pragma unroll
  for (int q = 0; q < U; ++q) combine<true>(acc, x[q]);
}

template <class C, int U>
__device__ __forceinline__ void batch_max(Grp& acc, Grp (&x)[U]) {
  if (C::OR)
    or_all<U>(acc, x);
  else if (C::KWAY)
    kway_max<U>(acc, x);
  else
    tree_max<U>(acc, x);
}

// Writes the finished row next[v] (this lane's group) and the changed flag,
// locally and -- fused exchange -- into every peer replica over P2P, so the
// shard transfer overlaps the remaining union work instead of following it.
template <int P>
__device__ __forceinline__ void publish_row(const UnionArgs& a, const uint8_t* curb, uint8_t* nextb, uint64_t goff,
                                            uint64_t v, const Grp& acc, int lane) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
  const Grp own = IO::ld(curb + v * G::ROW);
  const bool ch = lane < G::LPR && grp_ne(acc, own);
  const bool any = __any_sync(FULL, ch);
  if (lane < G::LPR) {
    IO::st(nextb, acc);
    for (int r = 0; r < a.npeers; ++r) IO::st(a.peer_next[r] + goff + v * G::ROW, acc);
  }
  if (any && lane == 0) {
    a.changed_out[v] = 1;
    for (int r = 0; r < a.npeers; ++r) a.peer_changed[r][v] = 1;
  }
  // Peer stores are ordered before everything this thread does afterwards --
  // in particular before the iteration barrier (the 8-byte max all-reduce)
  // that releases the peers' next iteration.
  if (a.npeers) __threadfence_system();
}

// Processes one work unit: item `item` (<= chunk neighbours of one node) for
// row slice `slice`.  next[v] = max(cur[v], max_w cur[w])
// register-wise; a node split over several items is merged by the last item
// to finish (partials in `scratch`, arrival counter per node-slice).
template <int P, bool SKIP, class C>
__device__ __forceinline__ void process_item(const UnionArgs& a, uint64_t item, int slice, int lane,
                                             uint32_t* buf) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
  // 128-byte decode windows feed at most 128 ids per batch
  constexpr int U = (C::D16 && !SKIP) || C::U * G::SUB <= 128 ? C::U : 128 / G::SUB;
  using F = Feeder<P, SKIP, U, C::D16 && !SKIP>;
  const int sub = lane / G::LPR;
  const int gl = lane % G::LPR;
  const uint64_t u = item * G::SLICES + slice;
  const uint32_t node = a.item_node[item];
  const uint64_t v = a.node_begin + node;
  const uint32_t first = a.node_item[node];
  const uint32_t nit = a.node_item[node + 1] - first;
  const uint64_t goff = static_cast<uint64_t>(slice) * G::SLICE_BYTES + static_cast<uint64_t>(gl) * G::GB;
  const uint8_t* curb = opaque(a.cur + goff);
  Grp acc = (item == first) ? IO::ld(curb + v * G::ROW) : grp_zero();  // next[v] <- cur[v]
  Grp acc2 = grp_zero();
  F f;
  f.buf = buf;
  f.pos = a.item_off[item];
  f.rem = a.item_count[item];
  f.base = a.item_base[item];
  f.n = 0;
  f.i = 0;
  f.prefill(static_cast<uint32_t>(v), lane);
  if (C::DB) {
    // software pipeline: batch k+1's loads (and the next window decode when
    // needed) are in flight while batch k is reduced.
    Grp xa[U], xb[U];
    bool ha = f.next(a, lane);
    if (ha) {
      load_batch<P, U>(xa, curb, f, sub);
      f.i += F::BATCH;
    }
    while (ha) {
      const bool hb = f.next(a, lane);
      if (hb) {
        load_batch<P, U>(xb, curb, f, sub);
        f.i += F::BATCH;
      }
      batch_max<C, U>(acc, xa);
      if (!hb) break;
      ha = f.next(a, lane);
      if (ha) {
        load_batch<P, U>(xa, curb, f, sub);
        f.i += F::BATCH;
      }
      batch_max<C, U>(C::ACC2 ? acc2 : acc, xb);
    }
  } else if constexpr (G::GB == 8 && !C::OR && U % 2 == 0) {
    Grp x[U / 2];
    while (f.next(a, lane)) {
      load_batch_pairs<P, U>(x, curb, f, sub);
      f.i += F::BATCH;
      batch_max<C, U / 2>(acc, x);
    }
    Grp hi{acc.b0 >> 16, acc.b1 >> 16, acc.b2 >> 16, acc.b3 >> 16};
    acc = Grp{acc.b0 & 0xffffu, acc.b1 & 0xffffu, acc.b2 & 0xffffu, acc.b3 & 0xffffu};
    bsmax(acc, hi);
  } else {
    Grp x[U];
    while (f.next(a, lane)) {
      load_batch<P, U>(x, curb, f, sub);
      f.i += F::BATCH;
      batch_max<C, U>(acc, x);
    }
  }
  if (C::ACC2) combine<C::OR>(acc, acc2);
  if (G::SUB > 1) {
#pragma unroll
    for (int m = G::LPR; m < 32; m <<= 1) combine<C::OR>(acc, grp_shfl_xor(acc, m));
  }
  uint8_t* nextb = a.next + goff + v * G::ROW;
  bool finish = nit == 1;
  if (!finish) {
    if (lane < G::LPR) IO::st(a.scratch + u * G::SLICE_BYTES + static_cast<uint64_t>(gl) * G::GB, acc);
    __threadfence();
    uint32_t prev = 0;
    if (lane == 0) prev = atomicAdd(&a.node_counter[static_cast<uint64_t>(node) * G::SLICES + slice], 1u);
    prev = __shfl_sync(FULL, prev, 0);
    finish = prev == nit - 1;
    if (finish) {
      __threadfence();
      for (uint32_t i = first; i < first + nit; ++i) {
        if (i == item) continue;
        const uint64_t uu = static_cast<uint64_t>(i) * G::SLICES + slice;
        combine<C::OR>(acc, IO::ld_cg(a.scratch + uu * G::SLICE_BYTES + static_cast<uint64_t>(gl) * G::GB));
      }
      if (lane == 0) a.node_counter[static_cast<uint64_t>(node) * G::SLICES + slice] = 0u;
    }
  }
  if (finish) publish_row<P>(a, curb, nextb, goff, v, acc, lane);
}

// ------------------------------------------------------------------ tile-shared gathers
// A CTA takes a group of GN = 16 consecutive nodes (whole rows, one row slice)
// and sweeps the union of their neighbour lists in windows of GW_IDS ids:
//   A  warp w decodes the LEB128 rows of nodes 2w and 2w+1 straight into their
//      membership bitmaps for the window (bit per id, one shared atomicOr per
//      lane and word; a row's decode stops at the first id past the window and
//      resumes there in the next one).
//   B0 per bitmap word: the AND of every aligned block of nodes -- 8 pairs, 4
//      quads, 2 octets and the root (all 16; nodes without neighbours count as
//      holding every id).
//   B1 every id is folded into the blocks of the canonical cover of its member
//      set: block b takes the ids held by all of b but not by all of b's parent
//      (C_b = A_b & ~A_parent).  The root's ids (held by every node, ~90 % on a
//      visibility graph) are split over the 8 warps by word range; the 30 other
//      block accumulators are split over the warps by tree level.
// At the end node k's row is max(cur[k], root, k's leaf, pair, quad, octet):
// max is associative, commutative and idempotent and the covers partition each
// id's member set, so every id of N(k) is folded into exactly the blocks on
// k's path and no other id is (PAPER.md:358-360 unchanged).  Each row is
// gathered once per block of its cover -- about once per group for the root
// ids and ~2 times for the ids at the rim of the visibility disks -- instead of
// once per edge.
constexpr int GN = 16;                  // nodes per group
constexpr int GW_IDS = 8192;            // ids per window
constexpr int GW = GW_IDS / 32;         // bitmap words per node (= threads per CTA)
constexpr int GBLK = 2 * GN - 2;        // non-root blocks: 16 leaves, 8 pairs, 4 quads, 2 octets
constexpr unsigned GMIN_EDGES_PER_WINDOW = 1024;

// Instrumented build only (make stats, -DSB_GROUP_STATS): per-phase cycles and
// work counts of the group path, summed over warps (scripts/group_stats.py).
#ifdef SB_GROUP_STATS
__device__ unsigned long long g_group_stats[16];
#define SB_ST_DECL unsigned long long stc[16] = {}; long long stt = clock64();
#define SB_ST_ADD(i, v) stc[i] += (v)
#define SB_ST_LAP(i) do { const long long t_ = clock64(); stc[i] += t_ - stt; stt = t_; } while (0)
#define SB_ST_FLUSH() do { if (lane == 0) for (int i_ = 0; i_ < 16; ++i_) atomicAdd(&g_group_stats[i_], stc[i_]); } while (0)
#else
#define SB_ST_DECL
#define SB_ST_ADD(i, v) do { } while (0)
#define SB_ST_LAP(i) do { } while (0)
#define SB_ST_FLUSH() do { } while (0)
#endif

struct GroupSmem {
  uint32_t bm[GN][GW];          // membership bitmaps of the window
  uint32_t A[GN - 1][GW];       // block ANDs: pairs 0..7, quads 8..11, octets 12..13, root 14
  uint4 blk[GBLK][32];          // block accumulators (per lane; leaves 0..15, pairs 16..23, quads 24..27, octets 28..29)
  uint4 root[8][32];            // per-warp root partials (end of group)
  uint32_t rpre[GW];            // root bits: inclusive popcount prefix within each 32-word block
  uint32_t rsum[8];             // root bits per 32-word block
  uint32_t unit;                // B1 work-unit counter of the window
  uint32_t next[3][GN];         // next undecoded id per node (~0: row exhausted), by window mod 3
                                // (a double buffer is reused one window later; compute-sanitizer
                                // racecheck flags that reuse, the triple buffer is clean)
  unsigned long long pos[GN], end[GN];  // row cursors: next byte, row end, last id
  uint32_t base[GN];
  alignas(16) uint32_t q[8][64];  // per-warp id queues of the B1 folds (IdQueue)
};

// Per-warp ring of queued row ids in shared memory for the sparse B1 folds
// (p >= 10, one row slice per warp step): set bits are pushed lane-parallel --
// a lane per bitmap word, or a lane per bit of one word -- each at its rank,
// and folded 8 at a time (two broadcast LDS.128 for the ids, then one 9-way
// bit-serial max).  Replaces a warp-uniform loop over the set bits (~10
// instructions per id, 23 % of the kernel's instructions at C3).
template <int P, class C>
struct IdQueue {
  uint32_t* q;          // 64 entries
  uint32_t head, tail;  // warp-uniform; tail - head < QB between pushes
  const uint8_t* curb;
  int sub;              // p = 9: the half-warp (row group) of this lane
  // ids folded per batch: 8 per lane, lane halves taking different ids at p = 9
  static constexpr uint32_t QB = 8u * Geo<P>::SUB;

  __device__ __forceinline__ void drain(Grp& acc) {
    using G = Geo<P>;
    using IO = GrpIO<G::GB>;
    __syncwarp();
    while (tail - head >= QB) {
      const uint32_t* b = q + ((head + 8u * sub) & 63);
      const uint4 i0 = *reinterpret_cast<const uint4*>(b);
      const uint4 i1 = *reinterpret_cast<const uint4*>(b + 4);
      const uint32_t id[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
      Grp x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = IO::ld(curb + static_cast<uint64_t>(id[k]) * G::ROW);
      batch_max<C, 8>(acc, x);
      head += QB;
    }
  }
  // The last < QB queued ids (absent rows read as 0, the identity of the max).
  __device__ __forceinline__ void flush(Grp& acc) {
    using G = Geo<P>;
    using IO = GrpIO<G::GB>;
    const uint32_t n = tail - head;
    if (!n) return;
    __syncwarp();
    const int mine = static_cast<int>(n) - 8 * sub;  // this half's ids
    const uint32_t* b = q + ((head + 8u * sub) & 63);
    const uint4 i0 = *reinterpret_cast<const uint4*>(b);
    const uint4 i1 = *reinterpret_cast<const uint4*>(b + 4);
    const uint32_t id[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
    Grp x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = k < mine ? IO::ld(curb + static_cast<uint64_t>(id[k]) * G::ROW) : grp_zero();
    batch_max<C, 8>(acc, x);
    head = tail;
  }
  // One warp-uniform word w: ids id0 + bit, lane b pushes bit b.
  __device__ __forceinline__ void push_word(Grp& acc, uint32_t w, uint32_t id0, int lane) {
    __syncwarp();
    if ((w >> lane) & 1u) q[(tail + __popc(w & ((1u << lane) - 1u))) & 63] = id0 + lane;
    tail += __popc(w);
    drain(acc);
  }
  // Every lane's word cw: ids idb + bit (lane-parallel when the ids fit the ring).
  __device__ __forceinline__ void push_lanes(Grp& acc, uint32_t cw, uint32_t idb, int lane) {
    if (!__any_sync(FULL, cw != 0u)) return;
    const uint32_t n = __popc(cw);
    uint32_t incl = n;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, incl, d);
      if (lane >= d) incl += y;
    }
    const uint32_t T = __shfl_sync(FULL, incl, 31);
    if (!T) return;
    if (tail - head + T <= 64u) {
      __syncwarp();
      uint32_t pos = tail + incl - n;
      while (cw) {
        const int b = __ffs(cw) - 1;
        cw &= cw - 1u;
        q[pos & 63] = idb + b;
        ++pos;
      }
      tail += T;
      drain(acc);
      return;
    }
    uint32_t nz = __ballot_sync(FULL, cw != 0u);
    while (nz) {
      const int src = __ffs(nz) - 1;
      nz &= nz - 1u;
      push_word(acc, __shfl_sync(FULL, cw, src), __shfl_sync(FULL, idb, src), lane);
    }
  }
};

// acc <- max(acc, rows of the candidate bits) over `nw` bitmap words: id of
// bit b of word j = id0 + 32 j + b.  Batches of U * SUB candidates; a lane
// group loads its candidates' row slices (0 for a clear bit: the identity of
// the max) and folds them with the bit-serial (U+1)-way max.
template <int P, class C>
__device__ __forceinline__ void fold_bits(Grp& acc, const uint32_t* words, int nw, uint32_t id0,
                                          const uint8_t* curb, int sub) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
  constexpr int U = C::U;
  constexpr int BATCH = U * G::SUB;
  if constexpr (BATCH <= 32) {
    for (int j = 0; j < nw; ++j) {
      const uint32_t w = words[j];
      if (!w) continue;
      const uint8_t* rb = curb + static_cast<uint64_t>(id0 + 32u * j) * G::ROW;
#pragma unroll 1
      for (int c0 = 0; c0 < 32; c0 += BATCH) {
        const uint32_t bits = BATCH == 32 ? w : (w >> c0) & ((1u << (BATCH & 31)) - 1u);
        if (!bits) continue;
        Grp x[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int b = q * G::SUB + sub;
          x[q] = ((bits >> b) & 1u) ? IO::ld(rb + static_cast<uint64_t>(c0 + b) * G::ROW) : grp_zero();
        }
        batch_max<C, U>(acc, x);
      }
    }
  } else {
    constexpr int K = BATCH / 32;  // words per batch (p <= 7)
    for (int j = 0; j < nw; j += K) {
      uint32_t any = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) any |= words[j + k];
      if (!any) continue;
      Grp x[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int c = q * G::SUB + sub;
        const uint32_t w = words[j + (c >> 5)];
        x[q] = ((w >> (c & 31)) & 1u) ? IO::ld(curb + static_cast<uint64_t>(id0 + 32u * j + c) * G::ROW)
                                      : grp_zero();
      }
      batch_max<C, U>(acc, x);
    }
  }
}

// One word of candidates (the partial rows of one node).
template <int P, class C>
__device__ __forceinline__ void fold_word(Grp& acc, uint32_t w, uint32_t id0, const uint8_t* curb, int sub) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
  constexpr int QW = 32 / G::SUB;  // candidate slots per lane in one word
  constexpr int U = C::U < QW ? C::U : QW;
  constexpr int BATCH = U * G::SUB;
  const uint8_t* rb = curb + static_cast<uint64_t>(id0) * G::ROW;
#pragma unroll 1
  for (int c0 = 0; c0 < 32; c0 += BATCH) {
    const uint32_t bits = BATCH == 32 ? w : (w >> c0) & ((1u << (BATCH & 31)) - 1u);
    if (!bits) continue;
    Grp x[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int b = q * G::SUB + sub;
      x[q] = ((bits >> b) & 1u) ? IO::ld(rb + static_cast<uint64_t>(c0 + b) * G::ROW) : grp_zero();
    }
    batch_max<C, U>(acc, x);
  }
}

__device__ __forceinline__ uint4 grp_u4(const Grp& g) { return make_uint4(g.b0, g.b1, g.b2, g.b3); }
__device__ __forceinline__ Grp u4_grp(const uint4& v) { return Grp{v.x, v.y, v.z, v.w}; }

// Per-node cursor over its LEB128 row (warp-uniform): next byte, row end, last id.
struct RowPos {
  uint64_t pos, end;
  uint32_t base;
};

// Decodes node row `c` from its cursor into bitmap `bm` (ids in [B, B + GW_IDS))
// and returns the first id not consumed (~0 when the row is exhausted).  512
// bytes per step, 16 per lane, the decode_step4 arithmetic (the per-step
// costs -- the warp prefix sum, the votes, the cursor update -- paid once per
// 512 bytes); a byte belongs to the row iff it lies before the row's end
// offset, and the terminators whose id falls in the window are a prefix of the
// step's, so the cursor advances to just past the last one and the rest are
// decoded again by the next window.  Every in-window id sets
// its bit with its own shared atomicOr (lanes 16 ids apart: 2-way conflicts).
template <bool SKIP>
__device__ __forceinline__ uint32_t decode16_to_bitmap(const UnionArgs& a, RowPos& c, uint32_t B, uint32_t* bm,
                                                       int lane, unsigned& steps) {
  while (c.pos < c.end) {
    ++steps;
    // this lane's 16 bytes [pos + 16 lane, +16): 4 aligned words + the next lane's first
    const uint8_t* al = a.stream + (c.pos & ~3ull) + 16 * lane;
    uint32_t A[5];
#pragma unroll
    for (int i = 0; i < 4; ++i) A[i] = ld_stream_word(al + 4 * i);
    A[4] = __shfl_down_sync(FULL, A[0], 1);
    if (lane == 31) A[4] = ld_stream_word(al + 16);
    const uint32_t sh = static_cast<uint32_t>(c.pos & 3) * 8;
    uint32_t x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = __funnelshift_r(A[i], A[i + 1], sh);
    uint32_t prev = __shfl_up_sync(FULL, x[3], 1);
    if (lane == 0) prev = 0;  // the cursor sits on a varint boundary
    // per byte: payload << 7 * (continuation bytes just before it, <= 4)
    uint32_t pre[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t cb[4];
      varint_contrib(x[i], i ? x[i - 1] : prev, cb);
#pragma unroll
      for (int k = 0; k < 4; ++k) pre[4 * i + k] = (4 * i + k) ? pre[4 * i + k - 1] + cb[k] : cb[k];
    }
    const uint32_t lane_sum = pre[15];
    uint32_t incl = lane_sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, incl, d);
      if (lane >= d) incl += y;
    }
    // window offset of the id after this lane's preceding bytes: byte j's id is B + E + pre[j]
    const uint32_t E = c.base + incl - lane_sum - B;
    // terminators of this row (bytes before its end), 16-bit mask
    const int64_t left = static_cast<int64_t>(c.end) - static_cast<int64_t>(c.pos + 16 * lane);
    uint32_t tm = 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t T = ~x[i] & 0x80808080u;
      tm |= ((T >> 7) & 1u | (T >> 14) & 2u | (T >> 21) & 4u | (T >> 28) & 8u) << (4 * i);
    }
    tm &= left >= 16 ? 0xffffu : left <= 0 ? 0u : (1u << left) - 1u;
    // in-window terminators: all of them unless the window ends inside this step
    uint32_t inm = tm;
    if (!__all_sync(FULL, E + lane_sum < static_cast<uint32_t>(GW_IDS))) {
      inm = 0u;
#pragma unroll
      for (int j = 0; j < 16; ++j) inm |= (E + pre[j] < static_cast<uint32_t>(GW_IDS) ? 1u : 0u) << j;
      inm &= tm;
    }
    const uint32_t outm = tm & ~inm;
    // bitmap bits and the last in-window offset
    uint32_t last_off = 0u;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t off = E + pre[j];
      if ((inm >> j) & 1u) {
        bool keep = true;
        if (SKIP) keep = a.changed_in[B + off] != 0;
        if (keep) atomicOr(bm + (off >> 5), 1u << (off & 31));
        last_off = off;
      }
    }
    const uint32_t anyin = __ballot_sync(FULL, inm != 0u);
    const uint32_t anyout = __ballot_sync(FULL, outm != 0u);
    if (anyin) {  // advance past the last in-window terminator
      const int L = 31 - __clz(anyin);
      const int lk = 31 - __clz(__shfl_sync(FULL, inm, L));
      c.base = B + __shfl_sync(FULL, last_off, L);
      c.pos += 16 * L + lk + 1;
    }
    if (anyout) {  // once per row and window: the first id past the window
      uint32_t first_out = 0u;
#pragma unroll
      for (int j = 15; j >= 0; --j)
        if ((outm >> j) & 1u) first_out = E + pre[j];
      if (lane < 16) prefetch_l2(a.stream + c.pos + 128 * lane);
      return B + __shfl_sync(FULL, first_out, __ffs(anyout) - 1);
    }
    if (!anyin) {  // unreachable on a validated stream (a step always holds a terminator)
      c.pos = c.end;
      break;
    }
  }
  return 0xffffffffu;
}

// acc <- max(acc, rows of the set bits of the warp-uniform word cw): ids
// id0 + bit.  p >= 10 (one row slice per warp step): the set bits are taken 4
// at a time (one 4-row bit-serial max, 8 LOP3 per row also for sparse words);
// p < 10: batches over bit positions (fold_word).
template <int P, class C>
__device__ __forceinline__ void fold_set_bits(Grp& acc, uint32_t cw, uint32_t id0, const uint8_t* curb, int sub) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
  if constexpr (G::SUB == 1) {
    const uint8_t* rb = curb + static_cast<uint64_t>(id0) * G::ROW;
    while (cw) {
      Grp x[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (cw) {
          const int b = __ffs(cw) - 1;
          cw &= cw - 1u;
          x[q] = IO::ld(rb + static_cast<uint64_t>(b) * G::ROW);
        } else {
          x[q] = grp_zero();
        }
      }
      batch_max<C, 4>(acc, x);
    }
  } else {
    fold_word<P, C>(acc, cw, id0, curb, sub);
  }
}

// acc <- max(acc, rows of the full word at id0) for p >= 9: 8 rows per lane per
// batch (lane halves take different rows at p = 9).
template <int P, class C>
__device__ __forceinline__ void fold_word_rows(Grp& acc, uint32_t id0, const uint8_t* curb, int sub) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
  static_assert(G::SUB <= 4, "full-word folds serve p >= 8");
  const uint8_t* rb = curb + static_cast<uint64_t>(id0 + 8 * sub) * G::ROW;
#pragma unroll 1
  for (int c0 = 0; c0 < 32; c0 += 8 * G::SUB) {
    Grp x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = IO::ld(rb + static_cast<uint64_t>(c0 + q) * G::ROW);
    batch_max<C, 8>(acc, x);
  }
}

// Bits of w whose rank among its set bits is in [r0, r1).
__device__ __forceinline__ uint32_t rank_range(uint32_t w, uint32_t r0, uint32_t r1) {
  if (r1 < static_cast<uint32_t>(__popc(w))) w &= (1u << __fns(w, 0, static_cast<int>(r1) + 1)) - 1u;
  if (r0 > 0) {
    const uint32_t p = __fns(w, 0, static_cast<int>(r0));
    w &= p >= 31 ? 0u : ~((2u << p) - 1u);
  }
  return w;
}

// B1 work units, taken by the warps from a shared counter in this order: the
// 30 non-root blocks coarse levels first (octets 28..29, quads 24..27, pairs
// 16..23, leaves 0..15; one warp per block, which owns its accumulator for the
// window), then GRC slices of the root ids of equal size.  Cover sizes differ
// per block and window, so a static split leaves warps idle at the window's
// closing barrier (ncu: 22 % of the stall samples there with 8 fixed shares).
constexpr int GRC = 16;
__device__ __forceinline__ int unit_block(int u) {
  return u < 2 ? 28 + u : u < 6 ? 24 + (u - 2) : u < 14 ? 16 + (u - 6) : u - 14;
}

// Node mask of block b (leaves 0..15, pairs 16..23, quads 24..27, octets 28..29).
__device__ __forceinline__ uint32_t block_nodes(int b) {
  if (b < 16) return 1u << b;
  if (b < 24) return 0x3u << (2 * (b - 16));
  if (b < 28) return 0xfu << (4 * (b - 24));
  return 0xffu << (8 * (b - 28));
}

// C_b for word j: ids held by every node of block b but not by every node of its parent.
__device__ __forceinline__ uint32_t block_cover_word(const GroupSmem& S, int b, int j, uint32_t act) {
  if (b < 16) {  // leaf: own bitmap minus the pair's AND
    const uint32_t own = S.bm[b][j];
    return own & ~S.A[b >> 1][j];
  }
  if (b < 24) return S.A[b - 16][j] & ~S.A[8 + ((b - 16) >> 1)][j];
  if (b < 28) return S.A[b - 16][j] & ~S.A[12 + ((b - 24) >> 1)][j];
  return S.A[b - 16][j] & ~S.A[14][j];
}

template <int P, bool SKIP, class C0>
__device__ __forceinline__ void process_group16(const UnionArgs& a, uint32_t g0, int slice, int lane, int warp,
                                                uint32_t act, GroupSmem& S) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
  using C = UCfg<8, false, C0::MINB, false, C0::KWAY, C0::OR>;
  const int sub = lane / G::LPR;
  const int gl = lane % G::LPR;
  const uint64_t goff = static_cast<uint64_t>(slice) * G::SLICE_BYTES + static_cast<uint64_t>(gl) * G::GB;
  const uint8_t* curb = opaque(a.cur + goff);
  // cursors of this warp's two nodes (kept in shared memory between windows)
  if (lane < 2) {
    const int k = 2 * warp + lane;
    const uint32_t node = g0 + k;
    const bool mine = (act >> k) & 1u;
    S.pos[k] = mine ? a.row_off[node] : 0ull;
    S.end[k] = mine ? a.row_off[node + 1] : 0ull;
    S.base[k] = 0u;
    S.next[0][k] = mine ? a.node_lo[node] : 0xffffffffu;
  }
  for (int i = threadIdx.x; i < GBLK * 32; i += blockDim.x) (&S.blk[0][0])[i] = make_uint4(0u, 0u, 0u, 0u);
  Grp all = grp_zero();  // this warp's share of the root
  SB_ST_DECL
  __syncthreads();
  for (int r = 0;; ++r) {
    SB_ST_ADD(0, 1);
    uint32_t B = 0xffffffffu;
#pragma unroll
    for (int k = 0; k < GN; ++k) B = min(B, S.next[r % 3][k]);
    if (B == 0xffffffffu) break;  // every row exhausted (CTA-uniform)
    B &= ~31u;
    // A: this warp's two rows -> bitmaps
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = 2 * warp + h;
      uint32_t* bm = S.bm[k];
#pragma unroll
      for (int i = lane; i < GW; i += 32) bm[i] = 0u;
      __syncwarp();
      uint32_t nx = S.next[r % 3][k];
      if (nx - B < static_cast<uint32_t>(GW_IDS)) {
        RowPos c{S.pos[k], S.end[k], S.base[k]};
        unsigned steps = 0;
        nx = decode16_to_bitmap<SKIP>(a, c, B, bm, lane, steps);
        SB_ST_ADD(1, steps);
        __syncwarp();
        if (lane == 0) {
          S.pos[k] = c.pos;
          S.base[k] = c.base;
        }
      }
      if (lane == 0) S.next[(r + 1) % 3][k] = nx;
    }
    SB_ST_LAP(8);
    __syncthreads();
    SB_ST_LAP(9);
    // B0: block ANDs of word j = threadIdx.x (nodes without neighbours hold every id)
    {
      const int j = threadIdx.x;
      uint32_t x[GN];
#pragma unroll
      for (int k = 0; k < GN; ++k) x[k] = ((act >> k) & 1u) ? S.bm[k][j] : 0xffffffffu;
#pragma unroll
      for (int i = 0; i < 8; ++i) S.A[i][j] = x[2 * i] & x[2 * i + 1];
      uint32_t q[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) S.A[8 + i][j] = q[i] = x[4 * i] & x[4 * i + 1] & x[4 * i + 2] & x[4 * i + 3];
      const uint32_t o0 = q[0] & q[1], o1 = q[2] & q[3];
      S.A[12][j] = o0;
      S.A[13][j] = o1;
      const uint32_t rw = o0 & o1;
      S.A[14][j] = rw;
      uint32_t incl = __popc(rw);
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += y;
      }
      S.rpre[j] = incl;
      if (lane == 31) S.rsum[warp] = incl;
      if (j == 0) S.unit = 0u;
    }
    SB_ST_LAP(10);
    __syncthreads();
    SB_ST_LAP(11);
    // B1: work units from the shared counter (blocks, then root slices)
    {
      uint32_t bs = 0u, bincl = 0u, total = 0u;
      if constexpr (G::SUB <= 4) {
        bs = lane < 8 ? S.rsum[lane] : 0u;
        bincl = bs;
#pragma unroll
        for (int d = 1; d < 8; d <<= 1) {
          const uint32_t y = __shfl_up_sync(FULL, bincl, d);
          if (lane >= d) bincl += y;
        }
        total = __shfl_sync(FULL, bincl, 7);
      }
      constexpr int NRC = G::SUB <= 4 ? GRC : 8;  // root slices (p < 8: 8 ranges of 32 words)
      for (;;) {
        uint32_t u = 0u;
        if (lane == 0) u = atomicAdd(&S.unit, 1u);
        u = __shfl_sync(FULL, u, 0);
        if (u >= static_cast<uint32_t>(GBLK + NRC)) break;
        if (u >= static_cast<uint32_t>(GBLK)) {
          const int c = static_cast<int>(u) - GBLK;
          if constexpr (G::SUB <= 4) {
            // root slice c of equal id count (root ids cluster in runs, so equal
            // word ranges would not balance)
            const uint32_t lo = static_cast<uint32_t>((static_cast<uint64_t>(total) * c) / NRC);
            const uint32_t hi = static_cast<uint32_t>((static_cast<uint64_t>(total) * (c + 1)) / NRC);
            if (lo < hi) {
              // first word whose inclusive prefix exceeds x: the block by a ballot over
              // the 8 block sums, the word by a ballot inside the block
              auto locate = [&](uint32_t x, uint32_t& excl) -> int {
                const int blk = __ffs(__ballot_sync(FULL, lane < 8 && bincl > x)) - 1;
                const uint32_t bex = __shfl_sync(FULL, bincl - bs, blk);
                const int jw = __ffs(__ballot_sync(FULL, bex + S.rpre[32 * blk + lane] > x)) - 1;
                const int jj = 32 * blk + jw;
                excl = bex + S.rpre[jj] - __popc(S.A[14][jj]);
                return jj;
              };
              uint32_t ex0, ex1;
              const int j0 = locate(lo, ex0), j1 = locate(hi - 1, ex1);
              // 32 words per pass, a word per lane: full words as 4 unconditional
              // 8-row batches, the set bits of partial ones (run ends) queued
              IdQueue<P, C> Q{S.q[warp], 0u, 0u, curb, sub};
#pragma unroll 1
              for (int jb = j0; jb <= j1; jb += 32) {
                const int j = jb + lane;
                uint32_t w = j <= j1 ? S.A[14][j] : 0u;
                if (j == j0 || j == j1) w = rank_range(w, j == j0 ? lo - ex0 : 0u, j == j1 ? hi - ex1 : 32u);
                uint32_t fm = __ballot_sync(FULL, w == 0xffffffffu);
                while (fm) {
                  const int src = __ffs(fm) - 1;
                  fm &= fm - 1u;
                  fold_word_rows<P, C>(all, B + 32u * (jb + src), curb, sub);
                }
                Q.push_lanes(all, w == 0xffffffffu ? 0u : w, B + 32u * j, lane);
              }
              Q.flush(all);
              SB_ST_ADD(2, hi - lo);
            }
          } else {
            fold_bits<P, C>(all, S.A[14] + 32 * c, 32, B + 32u * 32u * c, curb, sub);
          }
          continue;
        }
        const int b = unit_block(static_cast<int>(u));
        if (!(act & block_nodes(b))) continue;  // no node of this block has neighbours
        Grp acc = u4_grp(S.blk[b][lane]);
        bool touched = false;
        // p >= 9: the cover's ids are sparse (the rims of the disks): a word per
        // lane, full words as 8-row batches, the other set bits queued
        IdQueue<P, C> Q{S.q[warp], 0u, 0u, curb, sub};
#pragma unroll 1
        for (int j0 = 0; j0 < GW; j0 += 32) {
          uint32_t cword = block_cover_word(S, b, j0 + lane, act);
          if (!__any_sync(FULL, cword != 0u)) continue;
          const uint32_t id0l = B + 32u * (j0 + lane);
          touched = true;
          if constexpr (G::SUB <= 4) {
            SB_ST_ADD(3, __reduce_add_sync(FULL, __popc(cword)));
            uint32_t fm = __ballot_sync(FULL, cword == 0xffffffffu);
            while (fm) {
              const int src = __ffs(fm) - 1;
              fm &= fm - 1u;
              fold_word_rows<P, C>(acc, B + 32u * (j0 + src), curb, sub);
            }
            Q.push_lanes(acc, cword == 0xffffffffu ? 0u : cword, id0l, lane);
          } else {
            uint32_t nz = __ballot_sync(FULL, cword != 0u);
            while (nz) {
              const int src = __ffs(nz) - 1;
              nz &= nz - 1u;
              fold_set_bits<P, C>(acc, __shfl_sync(FULL, cword, src), B + 32u * (j0 + src), curb, sub);
            }
          }
        }
        if (G::SUB <= 4) Q.flush(acc);
        if (touched) S.blk[b][lane] = grp_u4(acc);
        SB_ST_ADD(4, 1);
      }
    }
    SB_ST_LAP(12);
    __syncthreads();  // bitmaps and block ANDs are rewritten by the next window
    SB_ST_LAP(14);
  }
  // node k = max(cur[k], root partials, its leaf / pair / quad / octet)
  S.root[warp][lane] = grp_u4(all);
  __syncthreads();
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    const int k = 2 * warp + h;
    const uint32_t node = g0 + k;
    if (node >= a.n_local) break;  // warp-uniform
    const uint64_t v = a.node_begin + node;
    Grp acc = IO::ld(curb + v * G::ROW);  // next[v] <- cur[v]
    if ((act >> k) & 1u) {
      Grp x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = u4_grp(S.root[q][lane]);
      batch_max<C, 8>(acc, x);
      Grp y[4] = {u4_grp(S.blk[k][lane]), u4_grp(S.blk[16 + (k >> 1)][lane]), u4_grp(S.blk[24 + (k >> 2)][lane]),
                  u4_grp(S.blk[28 + (k >> 3)][lane])};
      batch_max<C, 4>(acc, y);
    }
    if (G::SUB > 1) {
#pragma unroll
      for (int m = G::LPR; m < 32; m <<= 1) combine<C::OR>(acc, grp_shfl_xor(acc, m));
    }
    publish_row<P>(a, curb, a.next + goff + v * G::ROW, goff, v, acc, lane);
  }
  SB_ST_LAP(15);
  SB_ST_ADD(5, 1);
  SB_ST_FLUSH();
}

// Group decision (warp 0) for the 16-node group at g0: the shared path iff >= 2
// nodes have neighbours, the group holds <= shared_max_edges edges (load
// balance) and its id span is dense in edges (>= GMIN_EDGES_PER_WINDOW per
// window: the window sweep costs per window, not per edge).  Returns the mask
// of nodes with neighbours | 0x10000 for the shared path, else 0.
__device__ __forceinline__ uint32_t group_mode16(const UnionArgs& a, uint32_t g0, int lane) {
  const uint32_t node = g0 + lane;
  const bool ex = lane < GN && node < a.n_local;
  const uint32_t deg = ex ? a.degrees[node] : 0u;
  uint32_t lo = deg ? a.node_lo[node] : 0xffffffffu;
  uint32_t hi = deg ? a.node_hi[node] : 0u;
  unsigned long long sum = deg;
#pragma unroll
  for (int o = 8; o >= 1; o >>= 1) {  // lanes 0..15
    sum += __shfl_xor_sync(FULL, sum, o);
    lo = min(lo, __shfl_xor_sync(FULL, lo, o));
    hi = max(hi, __shfl_xor_sync(FULL, hi, o));
  }
  const uint32_t act = __ballot_sync(FULL, deg != 0) & 0xffffu;
  if (__popc(act) < 2 || sum > a.shared_max_edges) return 0u;
  const unsigned long long windows = (hi - lo) / GW_IDS + 1ull;
  return sum >= GMIN_EDGES_PER_WINDOW * windows ? (act | 0x10000u) : 0u;
}

__device__ __forceinline__ bool upload_failed(const UnionArgs& a) {
  return a.err && *reinterpret_cast<const volatile unsigned long long*>(a.err) != ~0ull;
}

// Fused decode-union kernel.  Two schedules over the same work units:
//  TILE=false: each warp grabs the next (item, slice) from a global counter.
//  TILE=true : each CTA grabs a tile = (8 consecutive nodes, chunk index q,
//              slice); warp w takes node 8g+w's chunk q.  Consecutive raster
//              nodes see almost the same neighbour ids at the same stream
//              position, so the CTA's 8 warps re-read each row from L1
//              instead of L2.
template <int P, bool SKIP, class C, bool GRP>
constexpr size_t union_smem_bytes() {
  constexpr size_t ids = sizeof(uint32_t) * 8 * Feeder<P, SKIP, C::U, C::D16 && !SKIP>::BUF;
  return GRP && sizeof(GroupSmem) > ids ? sizeof(GroupSmem) : ids;
}

// GRP: the 16-node group path is compiled in (launched when the graph's
// node_lo is set); without it the per-node item path keeps its registers.
template <int P, bool SKIP, bool TILE, class C = DefaultCfg<P>, bool GRP = true>
__global__ void __launch_bounds__(256, C::MINB) union_kernel(UnionArgs a) {
  using G = Geo<P>;
  extern __shared__ __align__(16) unsigned char smem[];  // per-node feeders or the group path
  __shared__ unsigned long long s_unit[2];
  __shared__ uint32_t s_mode;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint32_t* buf = reinterpret_cast<uint32_t*>(smem) + warp * Feeder<P, SKIP, C::U, C::D16 && !SKIP>::BUF;
  if (a.stop && *reinterpret_cast<const volatile unsigned int*>(a.stop)) return;  // run finished on the device
  if (!TILE) {
    const uint64_t total = a.n_items * G::SLICES;
    for (;;) {
      unsigned long long u = 0;
      if (lane == 0) u = upload_failed(a) ? total : atomicAdd(a.work, 1ull);
      u = __shfl_sync(FULL, u, 0);
      if (u >= total) break;
      // slice-major: the warps in flight share one 512-byte slice of the plane
      // (p >= 11: a slice of every row stays in L2, the whole plane would not)
      process_item<P, SKIP, C>(a, u % a.n_items, static_cast<int>(u / a.n_items), lane, buf);
    }
  } else {
    const uint64_t total = a.n_tiles * G::SLICES;
    for (int k = 0;; ++k) {
      if (threadIdx.x == 0) s_unit[k & 1] = upload_failed(a) ? total : atomicAdd(a.work, 1ull);
      __syncthreads();
      const unsigned long long u = s_unit[k & 1];
      if (u >= total) break;
      const uint64_t t = u % a.n_tiles;  // slice-major (see the item schedule)
      const int slice = static_cast<int>(u / a.n_tiles);
      const uint32_t g0 = a.tile_node0[t];
      const uint32_t q = a.tile_q[t];
      if (GRP && a.node_lo) {  // 16-node group path when the group's rows overlap densely
        const uint32_t g16 = g0 & ~15u;
        if (warp == 0) {
          const uint32_t m = group_mode16(a, g16, lane);
          if (lane == 0) s_mode = m;
        }
        __syncthreads();
        const uint32_t m = s_mode;
        if (m) {  // the group's first tile does the whole group; its other tiles have nothing to do
          if (q == 0 && g0 == g16)
            process_group16<P, SKIP, C>(a, g16, slice, lane, warp, m & 0xffffu,
                                        *reinterpret_cast<GroupSmem*>(smem));
          continue;
        }
      }
      const uint32_t node = g0 + warp;
      if (node < a.n_local) {
        const uint32_t first = a.node_item[node];
        if (q < a.node_item[node + 1] - first)
          process_item<P, SKIP, C>(a, first + q, slice, lane, buf);
      }
    }
  }
}


// ------------------------------------------------------------------ interval mode
// Sparse table over the current plane: level k row j = max(cur[j .. j+2^k)),
// built level by level (level k = max(level k-1 [j], level k-1 [j + 2^(k-1)])).
// Rows j > n - 2^k are never addressed by a query; they copy level k-1.
template <int P, bool OR>
__global__ void st_build_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint64_t n,
                                uint64_t half) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
  const uint64_t groups = n * G::GROUPS;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < groups;
       i += gridDim.x * (uint64_t)blockDim.x) {
    const uint64_t j = i / G::GROUPS;
    Grp x = IO::ld(src + i * G::GB);
    if (j + half < n) combine<OR>(x, IO::ld(src + (i + half * G::GROUPS) * G::GB));
    IO::st(dst + i * G::GB, x);
  }
}

// The same level step over rows [r0, r1) only (the wavefront builds each
// upload chunk's table rows as soon as the rows they read are final).
template <int P, bool OR>
__global__ void st_build_rows_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint64_t n,
                                     uint64_t half, uint64_t r0, uint64_t r1) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
  const uint64_t g0 = r0 * G::GROUPS, g1 = r1 * G::GROUPS;
  for (uint64_t i = g0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < g1;
       i += gridDim.x * (uint64_t)blockDim.x) {
    const uint64_t j = i / G::GROUPS;
    Grp x = IO::ld(src + i * G::GB);
    if (j + half < n) combine<OR>(x, IO::ld(src + (i + half * G::GROUPS) * G::GB));
    IO::st(dst + i * G::GB, x);
  }
}

// Run index: one warp per work item streams the item's bytes (items tile the
// stream: item i ends where item i+1 starts) in 512-byte windows, 16 bytes per
// lane with the validation kernel's SWAR arithmetic.  The stream is validated,
// so 32-bit sums are exact: the id after byte j is a warp prefix sum of byte
// contributions, and a terminator's varint value is its segmented sum (the
// chain of continuation bytes may start in the neighbour lane).  A terminator
// starts a run unless its value is 1 (the item's first always starts one) and
// closes the previous run at (its id - its value).  Count pass: runs per item
// and the longest run; fill pass: run starts / ends at the item's offset.
template <bool FILL>
__global__ void __launch_bounds__(256, FILL ? 2 : 3) run_index_kernel(RunIndexArgs a) {
  const int lane = threadIdx.x & 31;
  const uint32_t ltm = (1u << lane) - 1u;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  for (uint64_t item = a.item_begin + gw; item < a.item_end; item += nw) {
    // a malformed upload: its items' offsets are not trustworthy addresses
    if (a.err && *reinterpret_cast<const volatile unsigned long long*>(a.err) != ~0ull) break;
    const uint64_t pos0 = a.item_off[item];
    const uint64_t end = item + 1 < a.item_end ? a.item_off[item + 1] : a.range_end_byte;
    const uint64_t out = FILL ? a.run_off[item] : 0;
    if (FILL && a.overflow && out + a.run_count[item] > a.run_cap) {  // storage sized from an estimate
      if (lane == 0) *a.overflow = 1u;
      continue;
    }
    uint32_t id_before = a.item_base[item];  // warp-uniform: id after the previous window
    uint32_t nruns = 0;                       // warp-uniform: runs started so far
    uint32_t open_start = 0;                  // first id of the open run
    uint32_t longest = 0;
    uint32_t c3 = 0, ctail = 0;               // previous window's lane 31: word 3, trailing chain value
    uint4 qn = make_uint4(0u, 0u, 0u, 0u);  // next window in flight (as in build_items_kernel)
    if ((pos0 & ~15ull) + 16 * lane < end) qn = __ldg(reinterpret_cast<const uint4*>(a.stream + (pos0 & ~15ull) + 16 * lane));
    for (uint64_t wb = pos0 & ~15ull; wb < end; wb += 512) {
      if (lane < 4 && wb + 1024 + 128 * lane < end) prefetch_l2(a.stream + wb + 1024 + 128 * lane);
      const uint64_t lb = wb + 16 * lane;
      uint32_t x[4] = {qn.x, qn.y, qn.z, qn.w};
      qn = make_uint4(0u, 0u, 0u, 0u);
      if (lb + 512 < end) qn = __ldg(reinterpret_cast<const uint4*>(a.stream + lb + 512));
      uint32_t T[4], D[4];
      uint32_t vm[4] = {0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u};
      if (wb < pos0 || wb + 512 > end) {  // warp-uniform: only an item's first / last window is partial
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t lo = static_cast<int64_t>(pos0) - static_cast<int64_t>(lb + 4 * i);
          const int64_t hi = static_cast<int64_t>(end) - static_cast<int64_t>(lb + 4 * i);
          uint32_t m = 0x80808080u;
          if (lo > 0) m = lo >= 4 ? 0u : m << (8 * lo);
          if (hi < 4) m &= hi <= 0 ? 0u : 0x80808080u >> (8 * (4 - hi));
          x[i] &= (m >> 7) * 0xffu;  // bytes outside the item read as 0x00 (terminators, not counted)
          vm[i] = m;
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) T[i] = ~x[i] & vm[i];
      uint32_t wp3 = __shfl_up_sync(FULL, x[3], 1);
      if (lane == 0) wp3 = c3;
      c3 = __shfl_sync(FULL, x[3], 31);
      // pass A: continuation depths, lane sum, trailing chain value
      uint32_t lane_sum = 0, vl = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t w = x[i], wp = i ? x[i - 1] : wp3;
        const uint32_t F = w & 0x80808080u, Fp = wp & 0x80808080u;
        const uint32_t m1 = __funnelshift_l(Fp, F, 8);
        const uint32_t m2 = m1 & __funnelshift_l(Fp, F, 16);
        const uint32_t m3 = m2 & __funnelshift_l(Fp, F, 24);
        const uint32_t m4 = m3 & Fp;
        D[i] = ((m1 >> 7) + (m2 >> 7) + (m3 >> 7) + (m4 >> 7)) * 7u;  // 7 d per byte
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t c = byte_of(w & 0x7f7f7f7fu, k) << byte_of(D[i], k);
          lane_sum += c;
          vl = ((F >> (8 * k + 7)) & 1u) ? vl + c : 0u;  // value of the chain still open after this byte
        }
      }
      // vl: value of the lane's trailing (unterminated) chain; the next lane continues it
      uint32_t tail = __shfl_up_sync(FULL, vl, 1);
      if (lane == 0) tail = ctail;
      ctail = __shfl_sync(FULL, vl, 31);
      uint32_t incl = lane_sum;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += y;
      }
      const uint32_t excl = id_before + incl - lane_sum;
      const uint32_t anyT = __ballot_sync(FULL, (T[0] | T[1] | T[2] | T[3]) != 0);
      bool first = nruns == 0 && (anyT & ltm) == 0;  // the item's first terminator is in this lane
      // pass B: ids, varint values, run starts
      uint32_t id = excl, seg = tail, ns = 0, lastS = 0, firstPrev = 0, prevS = 0;
      bool haveS = false;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t w = x[i];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t c = byte_of(w & 0x7f7f7f7fu, k) << byte_of(D[i], k);
          id += c;
          seg += c;
          if ((T[i] >> (8 * k + 7)) & 1u) {
            const uint32_t val = seg, prev = id - val;
            if (val != 1u || first) {
              if (!FILL) {
                if (haveS) longest = max(longest, prev - prevS + 1u);
                if (!haveS) firstPrev = prev;
              }
              prevS = id;
              lastS = id;
              haveS = true;
              ++ns;
            }
            first = false;
            seg = 0;
          } else if (!((w >> (8 * k + 7)) & 1u)) {
            seg = 0;  // a byte outside the item (0x00): no chain crosses it
          }
        }
      }
      uint32_t sincl = ns;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, sincl, d);
        if (lane >= d) sincl += y;
      }
      const uint32_t A = __ballot_sync(FULL, ns != 0);
      if (FILL && ns) {  // pass C: write this lane's runs
        uint32_t slot = nruns + sincl - ns;
        uint32_t id2 = excl, seg2 = tail;
        bool first2 = nruns == 0 && (anyT & ltm) == 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t w = x[i];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t c = byte_of(w & 0x7f7f7f7fu, k) << byte_of(D[i], k);
            id2 += c;
            seg2 += c;
            if ((T[i] >> (8 * k + 7)) & 1u) {
              if (seg2 != 1u || first2) {
                a.run_s[out + slot] = id2;
                if (slot) a.run_e[out + slot - 1] = id2 - seg2;
                ++slot;
              }
              first2 = false;
              seg2 = 0;
            } else if (!((w >> (8 * k + 7)) & 1u)) {
              seg2 = 0;
            }
          }
        }
      }
      if (!FILL) {
        // close the run open at this lane's first start: its first id is the last
        // start of the nearest lower lane with starts (or of an earlier window)
        const uint32_t Ab = A & ltm;
        const uint32_t pl = __shfl_sync(FULL, lastS, Ab ? 31 - __clz(Ab) : 0);
        if (ns && (Ab || nruns)) longest = max(longest, firstPrev - (Ab ? pl : open_start) + 1u);
      }
      if (A) open_start = __shfl_sync(FULL, lastS, 31 - __clz(A));
      nruns += __shfl_sync(FULL, sincl, 31);
      id_before = __shfl_sync(FULL, excl + lane_sum, 31);
    }
    if (nruns) {  // the open run ends at the item's last id
      if (FILL && lane == 0) a.run_e[out + nruns - 1] = id_before;
      if (!FILL) longest = max(longest, id_before - open_start + 1u);
    }
    if (!FILL) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) longest = max(longest, __shfl_xor_sync(FULL, longest, o));
      if (lane == 0) {
        a.run_count[item] = nruns;
        if (longest) atomicMax(a.max_run, longest);
      }
    }
  }
}

// Folds one work unit's runs: lane i stages run i of each 32-run chunk in
// registers, then runs are broadcast 4 at a time (8 sparse-table rows per
// batch, folded by the bit-serial 9-way max, or OR in exact mode).
template <int P, bool OR>
__device__ __forceinline__ void process_item_runs(const IntervalArgs& ia, uint64_t item, int slice, int lane,
                                                  const long long* lvl_off) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
  // p < 10: a row is LPR < 32 lanes wide, so the warp's SUB lane groups fold
  // different runs and are merged by xor-shuffles at the end (as the dense kernel)
  const UnionArgs& a = ia.u;
  const int sub = lane / G::LPR;
  const int gl = lane % G::LPR;
  const uint64_t u = item * G::SLICES + slice;
  const uint32_t node = a.item_node[item];
  const uint64_t v = a.node_begin + node;
  const uint32_t first = a.node_item[node];
  const uint32_t nit = a.node_item[node + 1] - first;
  const uint64_t goff = static_cast<uint64_t>(slice) * G::SLICE_BYTES + static_cast<uint64_t>(gl) * G::GB;
  const uint8_t* curb = opaque(a.cur + goff);
  Grp acc = (item == first) ? IO::ld(curb + v * G::ROW) : grp_zero();
  const uint64_t r0 = ia.run_off[item];
  uint64_t r1 = ia.run_off[item + 1];
  // an item the estimated storage could not hold was not written: its runs are
  // skipped (the index overflowed, so the caller discards this pass and reruns it)
  if (ia.run_cap && r1 > ia.run_cap) r1 = r0;
  const int K = ia.levels;
  for (uint64_t c = r0; c < r1; c += 32) {
    const int cnt = static_cast<int>(r1 - c < 32 ? r1 - c : 32);
    uint32_t ms = 0, me = 0;
    if (lane < cnt) {
      ms = ia.run_s[c + lane];
      me = ia.run_e[c + lane];
    }
    for (int q0 = 0; q0 < cnt; q0 += 4 * G::SUB) {
      Grp x[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = min(q0 + q * G::SUB + sub, cnt - 1);  // tail repeats are harmless (max is idempotent)
        uint32_t s = __shfl_sync(FULL, ms, r);
        const uint32_t e = __shfl_sync(FULL, me, r);
        uint32_t L = e - s + 1;
        while (L >= (2u << K)) {  // longer than the table covers: peel 2^K blocks
          combine<OR>(acc, IO::ld(curb + lvl_off[K] + static_cast<uint64_t>(s) * G::ROW));
          s += 1u << K;
          L -= 1u << K;
        }
        const int k = 31 - __clz(L);
        const uint8_t* lb = curb + lvl_off[k];  // level k's plane (k = 0: cur itself)
        x[2 * q] = IO::ld(lb + static_cast<uint64_t>(s) * G::ROW);
        x[2 * q + 1] = IO::ld(lb + static_cast<uint64_t>(e - (1u << k) + 1) * G::ROW);
      }
      if (OR)
        or_all<8>(acc, x);
      else
        kway_max<8>(acc, x);
    }
  }
  if (G::SUB > 1) {
#pragma unroll
    for (int m = G::LPR; m < 32; m <<= 1) combine<OR>(acc, grp_shfl_xor(acc, m));
  }
  uint8_t* nextb = a.next + goff + v * G::ROW;
  bool finish = nit == 1;
  if (!finish) {
    if (lane < G::LPR) IO::st(a.scratch + u * G::SLICE_BYTES + static_cast<uint64_t>(gl) * G::GB, acc);
    __threadfence();
    uint32_t prev = 0;
    if (lane == 0) prev = atomicAdd(&a.node_counter[static_cast<uint64_t>(node) * G::SLICES + slice], 1u);
    prev = __shfl_sync(FULL, prev, 0);
    finish = prev == nit - 1;
    if (finish) {
      __threadfence();
      for (uint32_t i = first; i < first + nit; ++i) {
        if (i == item) continue;
        const uint64_t uu = static_cast<uint64_t>(i) * G::SLICES + slice;
        combine<OR>(acc, IO::ld_cg(a.scratch + uu * G::SLICE_BYTES + static_cast<uint64_t>(gl) * G::GB));
      }
      if (lane == 0) a.node_counter[static_cast<uint64_t>(node) * G::SLICES + slice] = 0u;
    }
  }
  if (finish) publish_row<P>(a, curb, nextb, goff, v, acc, lane);
}

template <int P, bool OR>
__global__ void __launch_bounds__(256, 4) union_interval_kernel(IntervalArgs ia) {
  using G = Geo<P>;
  __shared__ unsigned long long s_unit[2];
  __shared__ long long s_lvl[12];  // byte offset of sparse-table level k from the cur plane
  if (threadIdx.x < 12)
    s_lvl[threadIdx.x] = threadIdx.x == 0 ? 0ll
                                          : static_cast<long long>(ia.st - ia.u.cur) +
                                                static_cast<long long>(threadIdx.x - 1) *
                                                    static_cast<long long>(ia.n_global * G::ROW);
  __syncthreads();
  const UnionArgs& a = ia.u;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const uint64_t total = a.n_tiles * G::SLICES;
  for (int k = 0;; ++k) {
    if (threadIdx.x == 0) s_unit[k & 1] = upload_failed(a) ? total : atomicAdd(a.work, 1ull);
    __syncthreads();
    const unsigned long long u = s_unit[k & 1];
    if (u >= total) break;
    const uint64_t t = u % a.n_tiles;  // slice-major (see union_kernel)
    const int slice = static_cast<int>(u / a.n_tiles);
    const uint32_t node = a.tile_node0[t] + warp;
    const uint32_t q = a.tile_q[t];
    if (node < a.n_local) {
      const uint32_t first = a.node_item[node];
      if (q < a.node_item[node + 1] - first)
        process_item_runs<P, OR>(ia, first + q, slice, lane, s_lvl);
    }
  }
}

// ------------------------------------------------------------------ estimate
// MODE 0: init (c -> c_cur only); 1: dense accumulate; 2: skip unchanged rows.
template <int P, int MODE>
__global__ void __launch_bounds__(256) estimate_kernel(EstArgs a) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
  __shared__ unsigned long long red[8];
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  if (a.stop && *reinterpret_cast<const volatile unsigned int*>(a.stop)) return;  // run finished on the device
  unsigned long long wmax = 0ull;  // ordered encoding; 0 < every encoded value
  unsigned long long nchanged = 0ull;
  const double m = a.m;
  const double td = static_cast<double>(a.t);
  const double tt = static_cast<double>(static_cast<uint64_t>(a.t) * a.t);
  for (uint64_t node = gw; node < a.n_local; node += nw) {
    const uint64_t v = a.node_begin + node;
    if (MODE == 2 && !a.changed[v]) {
      if (lane == 0) {
        a.c_cur[node] = a.c_prev[node];
        wmax = max(wmax, dbl_to_ord(0.0));
      }
      continue;
    }
    if (MODE != 0 && lane == 0 && a.changed[v]) ++nchanged;
    uint64_t num = 0;
    uint32_t zeros = 0;
    const uint8_t* row = a.plane + v * G::ROW;
    for (int g = lane; g < G::GROUPS; g += 32) {
      const Grp x = IO::ld(row + static_cast<uint64_t>(g) * G::GB);
      const uint32_t n0 = ~x.b0 & G::VALID, n1 = ~x.b1 & G::VALID, n2 = ~x.b2 & G::VALID, n3 = ~x.b3 & G::VALID;
      const uint32_t lo[4] = {n1 & n0, n1 & x.b0, x.b1 & n0, x.b1 & x.b0};
      const uint32_t hi[4] = {n3 & n2, n3 & x.b2, x.b3 & n2, x.b3 & x.b2};
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint32_t c = __popc(hi[r >> 2] & lo[r & 3]);
        num += static_cast<uint64_t>(c) << (15 - r);  // sum 2^(15-r) (kernels.hpp:11-16)
        if (r == 0) zeros += c;
      }
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
      num += __shfl_xor_sync(FULL, num, d);
      zeros += __shfl_xor_sync(FULL, zeros, d);
    }
    if (lane == 0) {
      // hll_estimate_from_sum (hll.cpp:31-37), same operation order, no FMA.
      const double harmonic = __ddiv_rn(static_cast<double>(num), 32768.0);
      const double raw = __ddiv_rn(__dmul_rn(__dmul_rn(a.alpha, m), m), harmonic);
      const double c = (raw <= 2.5 * m && zeros > 0) ? a.lc[zeros] : raw;
      if (MODE == 0) {
        a.c_cur[node] = c;
      } else {
        // sum_d += t * (c_t - c_{t-1}), sum_d2 += t^2 * (...)
        const double delta = __dsub_rn(c, a.c_prev[node]);
        a.c_cur[node] = c;
        a.sum_d[node] = __dadd_rn(a.sum_d[node], __dmul_rn(td, delta));
        a.sum_d2[node] = __dadd_rn(a.sum_d2[node], __dmul_rn(tt, delta));
        wmax = max(wmax, dbl_to_ord(delta));
      }
    }
  }
  if (MODE == 0) return;
  if (lane == 0) red[threadIdx.x >> 5] = wmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long b = red[0];
    for (int i = 1; i < static_cast<int>(blockDim.x >> 5); ++i) b = max(b, red[i]);
    if (b) atomicMax(a.max_ord, b);
  }
  if (lane == 0 && nchanged) atomicAdd(a.changed_count, nchanged);
}

// ------------------------------------------------------------------ layout conversion
template <int P>
__global__ void to_packed_kernel(const uint8_t* __restrict__ bits, uint8_t* __restrict__ packed,
                                 uint64_t groups) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < groups;
       i += gridDim.x * (uint64_t)blockDim.x) {
    const Grp x = IO::ld(bits + i * G::GB);
    const uint32_t pl[4] = {x.b0, x.b1, x.b2, x.b3};
    uint32_t* out = reinterpret_cast<uint32_t*>(packed + i * G::GB);
#pragma unroll
    for (int w = 0; w < G::GB / 4; ++w) {
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) word |= spread_every4(pl[b] >> (8 * w)) << b;
      out[w] = word;
    }
  }
}

template <int P>
__global__ void from_packed_kernel(const uint8_t* __restrict__ packed, uint8_t* __restrict__ bits,
                                   uint64_t groups) {
  using G = Geo<P>;
  using IO = GrpIO<G::GB>;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < groups;
       i += gridDim.x * (uint64_t)blockDim.x) {
    const uint32_t* in = reinterpret_cast<const uint32_t*>(packed + i * G::GB);
    uint32_t pl[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int w = 0; w < G::GB / 4; ++w) {
      const uint32_t word = in[w];
#pragma unroll
      for (int b = 0; b < 4; ++b) pl[b] |= gather_every4(word >> b) << (8 * w);
    }
    IO::st(bits + i * G::GB, Grp{pl[0], pl[1], pl[2], pl[3]});
  }
}

// ------------------------------------------------------------------ metrics
__global__ void metrics_kernel(MetricArgs a) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < a.n;
       i += gridDim.x * (uint64_t)blockDim.x) {
    const uint32_t nv = a.nv[i];
    const double N = static_cast<double>(nv);
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    double MD = nan, IHH = nan, TK = nan, PV = nan, M1 = nan, M2 = nan;
    if (nv >= 2) {
      MD = a.sum_d[i] / (N - 1.0);
      TK = log2((MD + 2.0) / 3.0);
      M1 = MD * static_cast<double>(a.deg[i]);
      M2 = a.sum_d2[i] / (N - 1.0);
      if (nv >= 3) {
        const double RA = 2.0 * (MD - 1.0) / (N - 2.0);
        const double pv = 1.0 - RA;
        // integration_pv in [0, 1]: an HLL estimate can put
        // MD below 1 (RA < 0), so both ends are clamped
        PV = pv > 0.0 ? (pv < 1.0 ? pv : 1.0) : 0.0;
        if (MD > 1.0) {  // integration_hh pre: MD > 1, else NaN
          const double Dk = 2.0 * (N * (log2((N + 2.0) / 3.0) - 1.0) + 1.0) / ((N - 1.0) * (N - 2.0));
          IHH = 1.0 / (RA / Dk);
        }
      }
    }
    a.md[i] = MD;
    a.ihh[i] = IHH;
    a.tekl[i] = TK;
    a.pv[i] = PV;
    a.m1[i] = M1;
    a.m2[i] = M2;
  }
}

// ------------------------------------------------------------------ launchers
// ------------------------------------------------------------------ exact mode
// Exact neighbourhood function (the "exact oracle" mode):
// the HyperBall loop with each HLL row replaced by a reachability bitset over
// a block of S = 8 * ROW sources (bit j of row v: source s0 + j reached by v
// within t hops).  union_kernel / union_interval_kernel run with the OR
// combine; exact_count_kernel turns the popcount increase into exact depth
// sums and the per-node depth histogram.
template <int P>
__global__ void __launch_bounds__(256) exact_init_kernel(ExactArgs a) {
  using G = Geo<P>;
  const uint64_t words = a.n * (G::ROW / 4);
  uint32_t* plane = reinterpret_cast<uint32_t*>(a.plane);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words;
       i += gridDim.x * (uint64_t)blockDim.x) {
    const uint64_t v = i / (G::ROW / 4), wi = i % (G::ROW / 4);
    uint32_t x = 0u;
    if (v >= a.s0 && v < a.s1) {
      const uint64_t j = v - a.s0;
      if (j / 32 == wi) x = 1u << (j % 32);
    }
    plane[i] = x;
    if (wi == 0) {
      const uint32_t in = (v >= a.s0 && v < a.s1) ? 1u : 0u;
      a.pop[v] = in;
      a.reach[v] += in;
    }
  }
}

// Depth-1 rows without a union pass (exact BFS): row v =
// ({v} U N(v)) & [s0, s1) -- what
// the first OR pass over the source rows produces -- written from v's runs
// (runs are sorted; each clipped run is a bit range: interior words plain
// stores, boundary words atomicOr, since two runs can share only a boundary word).
template <int P>
__global__ void __launch_bounds__(256) exact_init1_kernel(ExactArgs a) {
  using G = Geo<P>;
  constexpr uint32_t WORDS = G::ROW / 4;
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  const uint32_t s0 = static_cast<uint32_t>(a.s0), s1 = static_cast<uint32_t>(a.s1);
  for (uint64_t v = gw; v < a.n; v += nw) {
    uint32_t* row = reinterpret_cast<uint32_t*>(a.plane + v * G::ROW);
    for (uint32_t k = lane; k < WORDS; k += 32) row[k] = 0u;
    __syncwarp();
    if (lane == 0 && v >= s0 && v < s1) atomicOr(row + (v - s0) / 32, 1u << ((v - s0) % 32));
    const uint64_t r0 = a.run_off[a.node_item[v]], r1 = a.run_off[a.node_item[v + 1]];
    for (uint64_t r = r0; r < r1; r += 32) {
      uint32_t rs = 0xffffffffu, re = 0u;
      if (r + lane < r1) {
        rs = a.run_s[r + lane];
        re = a.run_e[r + lane];
      }
      const uint32_t cs = max(rs, s0), ce = min(re, s1 - 1u);
      if (rs != 0xffffffffu && cs <= ce) {
        const uint32_t b0 = cs - s0, b1 = ce - s0;
        const uint32_t w0 = b0 / 32, w1 = b1 / 32;
        const uint32_t m0 = 0xffffffffu << (b0 % 32), m1 = 0xffffffffu >> (31 - b1 % 32);
        if (w0 == w1) {
          atomicOr(row + w0, m0 & m1);
        } else {
          atomicOr(row + w0, m0);
          for (uint32_t w = w0 + 1; w < w1; ++w) row[w] = 0xffffffffu;
          atomicOr(row + w1, m1);
        }
      }
      if (__all_sync(FULL, rs >= s1)) break;  // sorted runs: the rest start past the block
    }
  }
}

template <int P>
__global__ void __launch_bounds__(256) exact_count_kernel(ExactArgs a) {
  using G = Geo<P>;
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  unsigned long long nchanged = 0;
  const unsigned long long t = a.t;
  for (uint64_t v = gw; v < a.n; v += nw) {
    const uint4* row = reinterpret_cast<const uint4*>(a.plane + v * G::ROW);
    uint32_t c = 0;
    for (int k = lane; k < G::ROW / 16; k += 32) {
      const uint4 x = row[k];
      c += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) c += __shfl_xor_sync(FULL, c, d);
    if (lane == 0) {
      const uint32_t delta = c - a.pop[v];  // reachability only grows
      if (delta) {
        a.pop[v] = c;
        a.sum_d[v] += t * delta;
        a.sum_d2[v] += t * t * delta;
        a.hist[v * a.hist_cap + t] += delta;
        a.reach[v] += delta;
        ++nchanged;
      }
    }
  }
  if (lane == 0 && nchanged) atomicAdd(a.changed_count, nchanged);
}

static int grid_for(const void* fn, int block, size_t smem = 0) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, block, smem);
  if (per < 1) per = 1;
  return sms * per;
}

#define SB_DISPATCH_P(p, CALL)          \
  switch (p) {                          \
    case 4: CALL(4); break;             \
    case 5: CALL(5); break;             \
    case 6: CALL(6); break;             \
    case 7: CALL(7); break;             \
    case 8: CALL(8); break;             \
    case 9: CALL(9); break;             \
    case 10: CALL(10); break;           \
    case 11: CALL(11); break;           \
    case 12: CALL(12); break;           \
    case 13: CALL(13); break;           \
    case 14: CALL(14); break;           \
    case 15: CALL(15); break;           \
    case 16: CALL(16); break;           \
    default: return cudaErrorInvalidValue; \
  }

// Neighbour-id range of nodes [n0, n1) from the validation output: out[0] =
// min first id, out[1] = max last id (rows without neighbours hold ~0 / 0, the
// neutral elements; a chunk without edges gets out[0] > out[1]).
__global__ void __launch_bounds__(256) chunk_range_kernel(const uint32_t* __restrict__ lo,
                                                          const uint32_t* __restrict__ hi, uint64_t n0, uint64_t n1,
                                                          uint32_t* out) {
  __shared__ uint32_t smn[8], smx[8];
  uint32_t mn = 0xffffffffu, mx = 0u;
  for (uint64_t v = n0 + threadIdx.x; v < n1; v += blockDim.x) {
    mn = min(mn, lo[v]);
    mx = max(mx, hi[v]);
  }
  mn = __reduce_min_sync(FULL, mn);
  mx = __reduce_max_sync(FULL, mx);
  if ((threadIdx.x & 31) == 0) {
    smn[threadIdx.x >> 5] = mn;
    smx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) {
      mn = min(mn, smn[w]);
      mx = max(mx, smx[w]);
    }
    out[0] = mn;
    out[1] = mx;
  }
}

cudaError_t launch_chunk_range(const uint32_t* lo, const uint32_t* hi, uint64_t n0, uint64_t n1, uint32_t* out,
                               cudaStream_t s) {
  chunk_range_kernel<<<1, 256, 0, s>>>(lo, hi, n0, n1, out);
  return cudaGetLastError();
}

// Alg. 1's test on the device after pass
// t of back-to-back passes: keeps the pass's max increase and changed count
// for the host, stops the run when max increase <= 0.5 (inclusive) or t is the
// depth limit, and resets the per-pass counters for the next pass.
__global__ void decide_kernel(unsigned long long* misc, unsigned int* flags, unsigned long long* rec, uint32_t t,
                              uint32_t depth) {
  if (flags[0]) return;
  const unsigned long long mo = misc[1];
  rec[0] = mo;
  rec[1] = misc[2];
  double mx = -INFINITY;  // no node contributed
  if (mo) {
    const unsigned long long u = (mo >> 63) ? (mo & 0x7fffffffffffffffull) : ~mo;
    mx = __longlong_as_double(static_cast<long long>(u));
  }
  const bool conv = mx <= 0.5;
  if (conv || (depth != 0 && t == depth)) {
    flags[1] = t;
    flags[2] = conv ? 1u : 0u;
    flags[0] = 1u;
  }
  misc[0] = misc[1] = misc[2] = misc[3] = 0ull;
}

__global__ void clear_flags_kernel(const unsigned int* flags, uint8_t* bytes, uint64_t n) {
  if (*flags) return;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    bytes[i] = 0;
}

cudaError_t launch_decide(unsigned long long* misc, unsigned int* flags, unsigned long long* rec, uint32_t t,
                          uint32_t depth, cudaStream_t s) {
  decide_kernel<<<1, 1, 0, s>>>(misc, flags, rec, t, depth);
  return cudaGetLastError();
}

cudaError_t launch_clear_flags(const unsigned int* flags, uint8_t* bytes, uint64_t n, cudaStream_t s) {
  const uint64_t blocks = (n + 255) / 256;
  clear_flags_kernel<<<static_cast<unsigned>(blocks < 1184 ? (blocks ? blocks : 1) : 1184), 256, 0, s>>>(flags, bytes, n);
  return cudaGetLastError();
}

cudaError_t launch_build_items(const BuildArgs& a, cudaStream_t s) {
  const int g = grid_for(reinterpret_cast<const void*>(build_items_kernel), 256);
  build_items_kernel<<<g, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_init(int p, uint8_t* plane, uint64_t n, const uint32_t* orig, cudaStream_t s) {
#define SB_L(P)                                                                  \
  {                                                                              \
    const int g = grid_for(reinterpret_cast<const void*>(init_kernel<P>), 256); \
    init_kernel<P><<<g, 256, 0, s>>>(plane, n, orig);                            \
  }
  SB_DISPATCH_P(p, SB_L)
#undef SB_L
  return cudaGetLastError();
}

int union_slices(int p) { return p > 10 ? 1 << (p - 10) : 1; }

// Dynamic shared memory above the 48 KB default (the group path's bitmaps and
// block accumulators), then the persistent grid for that footprint.
static int prep_union(const void* fn, size_t smem) {
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  return grid_for(fn, 256, smem);
}

cudaError_t launch_union(int p, bool skip, const UnionArgs& a, cudaStream_t s) {
  const bool tile = a.n_tiles != 0;
#define SB_UG(P, SK, TL, GR)                                                                                 \
  {                                                                                                          \
    constexpr size_t sm = union_smem_bytes<P, SK, DefaultCfg<P>, GR>();                                      \
    static int g = prep_union(reinterpret_cast<const void*>(union_kernel<P, SK, TL, DefaultCfg<P>, GR>), sm); \
    union_kernel<P, SK, TL, DefaultCfg<P>, GR><<<g, 256, sm, s>>>(a);                                        \
  }
#define SB_UL(P, SK, TL)                      \
  {                                           \
    if (TL && a.node_lo) SB_UG(P, SK, TL, true) \
    else SB_UG(P, SK, TL, false)              \
  }
#define SB_L(P)                                                     \
  {                                                                 \
    if (skip) {                                                     \
      if (tile) SB_UL(P, true, true) else SB_UL(P, true, false)     \
    } else {                                                        \
      if (tile) SB_UL(P, false, true) else SB_UL(P, false, false)   \
    }                                                               \
  }
  SB_DISPATCH_P(p, SB_L)
#undef SB_L
#undef SB_UL
  return cudaGetLastError();
}

cudaError_t launch_st_build(int p, const uint8_t* cur, uint8_t* st, uint64_t n, int levels, cudaStream_t s,
                            bool orop) {
#define SB_L(P)                                                                                  \
  {                                                                                              \
    const uint64_t groups = n * Geo<P>::GROUPS;                                                  \
    const int g = static_cast<int>(groups / 256 + 1 < 148 * 16 ? groups / 256 + 1 : 148 * 16);   \
    const uint64_t rowb = n * Geo<P>::ROW;                                                       \
    for (int k = 1; k <= levels; ++k) {                                                          \
      const uint8_t* src = k == 1 ? cur : st + static_cast<uint64_t>(k - 2) * rowb;              \
      if (orop)                                                                                  \
        st_build_kernel<P, true><<<g, 256, 0, s>>>(src, st + static_cast<uint64_t>(k - 1) * rowb, n, 1ull << (k - 1)); \
      else                                                                                       \
        st_build_kernel<P, false><<<g, 256, 0, s>>>(src, st + static_cast<uint64_t>(k - 1) * rowb, n, 1ull << (k - 1)); \
    }                                                                                            \
  }
  SB_DISPATCH_P(p, SB_L)
#undef SB_L
  return cudaGetLastError();
}

cudaError_t launch_st_build_rows(int p, const uint8_t* cur, uint8_t* st, uint64_t n, int levels, uint64_t r0,
                                 uint64_t r1, cudaStream_t s) {
  // level k of rows [r0, r1) reads level k-1 up to 2^(k-1) rows further: build
  // level k over [r0, r1 + 2^K - 2^k), so the top level covers exactly [r0, r1)
#define SB_L(P)                                                                                       \
  {                                                                                                   \
    const uint64_t rowb = n * Geo<P>::ROW;                                                            \
    for (int k = 1; k <= levels; ++k) {                                                               \
      const uint64_t e = r1 + (1ull << levels) - (1ull << k);                                         \
      const uint64_t hi = e < n ? e : n;                                                              \
      if (hi <= r0) continue;                                                                         \
      const uint64_t groups = (hi - r0) * Geo<P>::GROUPS;                                             \
      const int g = static_cast<int>(groups / 256 + 1 < 148 * 8 ? groups / 256 + 1 : 148 * 8);        \
      const uint8_t* src = k == 1 ? cur : st + static_cast<uint64_t>(k - 2) * rowb;                   \
      st_build_rows_kernel<P, false><<<g, 256, 0, s>>>(src, st + static_cast<uint64_t>(k - 1) * rowb, n, \
                                                        1ull << (k - 1), r0, hi);                     \
    }                                                                                                 \
  }
  SB_DISPATCH_P(p, SB_L)
#undef SB_L
  return cudaGetLastError();
}

cudaError_t launch_union_interval(int p, const IntervalArgs& a, cudaStream_t s, bool orop) {
#define SB_LI(P)                                                                                    \
  {                                                                                                 \
    if (orop) {                                                                                     \
      static int g = grid_for(reinterpret_cast<const void*>(union_interval_kernel<P, true>), 256);  \
      union_interval_kernel<P, true><<<g, 256, 0, s>>>(a);                                          \
    } else {                                                                                        \
      static int g = grid_for(reinterpret_cast<const void*>(union_interval_kernel<P, false>), 256); \
      union_interval_kernel<P, false><<<g, 256, 0, s>>>(a);                                         \
    }                                                                                               \
    break;                                                                                          \
  }
  switch (p) {
    case 4: SB_LI(4)
    case 5: SB_LI(5)
    case 6: SB_LI(6)
    case 7: SB_LI(7)
    case 8: SB_LI(8)
    case 9: SB_LI(9)
    case 10: SB_LI(10)
    case 11: SB_LI(11)
    case 12: SB_LI(12)
    case 13: SB_LI(13)
    case 14: SB_LI(14)
    case 15: SB_LI(15)
    case 16: SB_LI(16)
    default: return cudaErrorInvalidValue;
  }
#undef SB_LI
  return cudaGetLastError();
}

// Exact mode: OR-union over bitset rows (block of 2^(P+2) sources), P in 10..14.
template <int P>
using OrCfg = UCfg<8, false, 4, false, false, true>;

cudaError_t launch_union_or(int p, const UnionArgs& a, cudaStream_t s) {
#define SB_LO(P)                                                                                         \
  {                                                                                                      \
    constexpr size_t sm = union_smem_bytes<P, false, OrCfg<P>, true>();                                  \
    static int g = prep_union(reinterpret_cast<const void*>(union_kernel<P, false, true, OrCfg<P>>), sm); \
    union_kernel<P, false, true, OrCfg<P>><<<g, 256, sm, s>>>(a);                                       \
    break;                                                                                               \
  }
  switch (p) {
    case 10: SB_LO(10)
    case 11: SB_LO(11)
    case 12: SB_LO(12)
    case 13: SB_LO(13)
    case 14: SB_LO(14)
    default: return cudaErrorInvalidValue;
  }
#undef SB_LO
  return cudaGetLastError();
}

cudaError_t launch_exact_init(int p, const ExactArgs& a, cudaStream_t s) {
#define SB_L(P)                                                                         \
  {                                                                                     \
    const int g = grid_for(reinterpret_cast<const void*>(exact_init_kernel<P>), 256);   \
    exact_init_kernel<P><<<g, 256, 0, s>>>(a);                                          \
    break;                                                                              \
  }
  switch (p) {
    case 10: SB_L(10)
    case 11: SB_L(11)
    case 12: SB_L(12)
    case 13: SB_L(13)
    case 14: SB_L(14)
    default: return cudaErrorInvalidValue;
  }
#undef SB_L
  return cudaGetLastError();
}

cudaError_t launch_exact_init1(int p, const ExactArgs& a, cudaStream_t s) {
#define SB_L(P)                                                                         \
  {                                                                                     \
    const int g = grid_for(reinterpret_cast<const void*>(exact_init1_kernel<P>), 256);  \
    exact_init1_kernel<P><<<g, 256, 0, s>>>(a);                                         \
    break;                                                                              \
  }
  switch (p) {
    case 10: SB_L(10)
    case 11: SB_L(11)
    case 12: SB_L(12)
    case 13: SB_L(13)
    case 14: SB_L(14)
    default: return cudaErrorInvalidValue;
  }
#undef SB_L
  return cudaGetLastError();
}

cudaError_t launch_exact_count(int p, const ExactArgs& a, cudaStream_t s) {
#define SB_L(P)                                                                         \
  {                                                                                     \
    const int g = grid_for(reinterpret_cast<const void*>(exact_count_kernel<P>), 256);  \
    exact_count_kernel<P><<<g, 256, 0, s>>>(a);                                         \
    break;                                                                              \
  }
  switch (p) {
    case 10: SB_L(10)
    case 11: SB_L(11)
    case 12: SB_L(12)
    case 13: SB_L(13)
    case 14: SB_L(14)
    default: return cudaErrorInvalidValue;
  }
#undef SB_L
  return cudaGetLastError();
}

// Exclusive scan of one upload chunk's run counts into run offsets, carried
// from the chunks before it (*total), one CTA: each thread scans a contiguous
// span, the span sums are scanned across the block.
__global__ void __launch_bounds__(1024) run_offsets_kernel(const uint64_t* __restrict__ cnt, uint64_t* off,
                                                           uint64_t i0, uint64_t i1, unsigned long long* total) {
  __shared__ unsigned long long wsum[32];
  const uint64_t n = i1 - i0;
  const uint64_t per = (n + blockDim.x - 1) / blockDim.x;
  const uint64_t b = i0 + threadIdx.x * per, e = b + per < i1 ? b + per : i1;
  unsigned long long mine = 0;
  for (uint64_t i = b; i < e; ++i) mine += cnt[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long incl = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long y = __shfl_up_sync(FULL, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < static_cast<int>(blockDim.x >> 5) ? wsum[lane] : 0ull, wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long y = __shfl_up_sync(FULL, wi, d);
      if (lane >= d) wi += y;
    }
    wsum[lane] = wi - w;  // exclusive over warps
  }
  __syncthreads();
  const unsigned long long base = *total;
  unsigned long long run = base + wsum[warp] + incl - mine;
  for (uint64_t i = b; i < e; ++i) {
    off[i] = run;
    run += cnt[i];
  }
  __syncthreads();
  if (threadIdx.x == blockDim.x - 1) {  // the last thread's span ends the chunk
    *total = run;
    off[i1] = run;  // the end of the chunk's last item (the next chunk's scan writes the same)
  }
}

cudaError_t launch_run_offsets(const uint64_t* run_count, uint64_t* run_off, uint64_t i0, uint64_t i1,
                               unsigned long long* total, cudaStream_t s) {
  if (i1 <= i0) return cudaSuccess;
  run_offsets_kernel<<<1, 1024, 0, s>>>(run_count, run_off, i0, i1, total);
  return cudaGetLastError();
}

cudaError_t launch_run_index(const RunIndexArgs& a, bool fill, cudaStream_t s) {
  if (fill) {
    const int g = grid_for(reinterpret_cast<const void*>(run_index_kernel<true>), 256);
    run_index_kernel<true><<<g, 256, 0, s>>>(a);
  } else {
    const int g = grid_for(reinterpret_cast<const void*>(run_index_kernel<false>), 256);
    run_index_kernel<false><<<g, 256, 0, s>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_estimate(int p, int mode, const EstArgs& a, cudaStream_t s) {
#define SB_L(P)                                                                                 \
  {                                                                                             \
    if (mode == 0) {                                                                            \
      static int g = grid_for(reinterpret_cast<const void*>(estimate_kernel<P, 0>), 256);        \
      estimate_kernel<P, 0><<<g, 256, 0, s>>>(a);                                               \
    } else if (mode == 1) {                                                                     \
      static int g = grid_for(reinterpret_cast<const void*>(estimate_kernel<P, 1>), 256);        \
      estimate_kernel<P, 1><<<g, 256, 0, s>>>(a);                                               \
    } else {                                                                                    \
      static int g = grid_for(reinterpret_cast<const void*>(estimate_kernel<P, 2>), 256);        \
      estimate_kernel<P, 2><<<g, 256, 0, s>>>(a);                                               \
    }                                                                                           \
  }
  SB_DISPATCH_P(p, SB_L)
#undef SB_L
  return cudaGetLastError();
}

cudaError_t launch_to_packed(int p, const uint8_t* bits, uint8_t* packed, uint64_t rows, cudaStream_t s) {
#define SB_L(P)                                                                            \
  {                                                                                        \
    const uint64_t groups = rows * Geo<P>::GROUPS;                                         \
    const int g = static_cast<int>(groups / 256 + 1 < 65535 ? groups / 256 + 1 : 65535);  \
    to_packed_kernel<P><<<g, 256, 0, s>>>(bits, packed, groups);                           \
  }
  SB_DISPATCH_P(p, SB_L)
#undef SB_L
  return cudaGetLastError();
}

cudaError_t launch_from_packed(int p, const uint8_t* packed, uint8_t* bits, uint64_t rows, cudaStream_t s) {
#define SB_L(P)                                                                            \
  {                                                                                        \
    const uint64_t groups = rows * Geo<P>::GROUPS;                                         \
    const int g = static_cast<int>(groups / 256 + 1 < 65535 ? groups / 256 + 1 : 65535);  \
    from_packed_kernel<P><<<g, 256, 0, s>>>(packed, bits, groups);                         \
  }
  SB_DISPATCH_P(p, SB_L)
#undef SB_L
  return cudaGetLastError();
}

#ifdef SB_GROUP_STATS
extern "C" int sb_debug_group_stats(unsigned long long* out16, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out16, g_group_stats, sizeof(unsigned long long) * 16) != cudaSuccess) return 3;
  if (reset) {
    static const unsigned long long zero[16] = {};
    cudaMemcpyToSymbol(g_group_stats, zero, sizeof(zero));
  }
  return 0;
}
#endif

cudaError_t launch_metrics(const MetricArgs& a, cudaStream_t s) {
  const int g = static_cast<int>(a.n / 256 + 1 < 65535 ? a.n / 256 + 1 : 65535);
  metrics_kernel<<<g, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sb
