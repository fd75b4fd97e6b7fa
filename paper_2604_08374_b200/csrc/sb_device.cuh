// sb_device.cuh -- device building blocks of the B200 HyperBall path.
//
// Register layout in HBM ("bit-sliced 4-bit"): a counter row keeps the
// reference density of m/2 bytes (hll.hpp:31-32) but stores each group of 32
// registers (16 for p=4) as four bit-planes: plane b holds bit b of every
// register of the group, bit i of a plane <-> register 32*g+i.  A register-wise
// max (kernels.hpp:21-25, nibble_max_inplace) is then a 4-stage ripple
// comparator over whole 32-bit words: 8 LOP3 per 32 registers, instead of the
// masked byte-max a packed layout needs.  The reference packed layout (low
// nibble = even register, hll.hpp:50-60) is produced on export by
// bits_to_packed(); parity is always checked in the reference layout.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sb {

constexpr unsigned FULL = 0xffffffffu;

template <int P>
struct Geo {
  static constexpr int M = 1 << P;
  static constexpr int ROW = M / 2;                     // bytes per counter row (m/2)
  static constexpr int GB = P >= 5 ? 16 : 8;            // bytes per bit-sliced group
  static constexpr int GROUPS = ROW / GB;               // groups per row
  static constexpr int LPR = GROUPS >= 32 ? 32 : GROUPS;  // lanes spanning one row slice
  static constexpr int SLICES = GROUPS >= 32 ? GROUPS / 32 : 1;
  static constexpr int SUB = 32 / LPR;                  // neighbour rows per warp step
  static constexpr int SLICE_BYTES = LPR * GB;          // 512 B for p >= 10
  static constexpr uint32_t VALID = P >= 5 ? 0xffffffffu : 0x0000ffffu;
};

struct Grp {
  uint32_t b0, b1, b2, b3;
};

__device__ __forceinline__ Grp grp_zero() { return Grp{0u, 0u, 0u, 0u}; }

__device__ __forceinline__ uint32_t lop3_0c(uint32_t a, uint32_t b) {  // ~a & b
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0x0c;" : "=r"(r) : "r"(a), "r"(b), "r"(0u));
  return r;
}
__device__ __forceinline__ uint32_t lop3_8e(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;  // (~a & b) | (~(a ^ b) & c)
  asm("lop3.b32 %0, %1, %2, %3, 0x8e;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ uint32_t lop3_d8(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;  // (a & ~c) | (b & c)
  asm("lop3.b32 %0, %1, %2, %3, 0xd8;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}

// a <- register-wise max(a, b).  g = positions where b > a, computed LSB-first
// as a ripple comparator g_k = (b_k & ~a_k) | (~(a_k ^ b_k) & g_{k-1}) -- one
// LOP3 per bit-plane -- then a 4-LOP3 select: 8 LOP3 per 32 registers.
__device__ __forceinline__ void bsmax(Grp& a, const Grp& b) {
  uint32_t g = lop3_0c(a.b0, b.b0);
  g = lop3_8e(a.b1, b.b1, g);
  g = lop3_8e(a.b2, b.b2, g);
  g = lop3_8e(a.b3, b.b3, g);
  a.b0 = lop3_d8(a.b0, b.b0, g);
  a.b1 = lop3_d8(a.b1, b.b1, g);
  a.b2 = lop3_d8(a.b2, b.b2, g);
  a.b3 = lop3_d8(a.b3, b.b3, g);
}

__device__ __forceinline__ bool grp_ne(const Grp& a, const Grp& b) {
  return ((a.b0 ^ b.b0) | (a.b1 ^ b.b1) | (a.b2 ^ b.b2) | (a.b3 ^ b.b3)) != 0u;
}

__device__ __forceinline__ Grp grp_shfl_xor(const Grp& a, int m) {
  return Grp{__shfl_xor_sync(FULL, a.b0, m), __shfl_xor_sync(FULL, a.b1, m),
             __shfl_xor_sync(FULL, a.b2, m), __shfl_xor_sync(FULL, a.b3, m)};
}

// ---- group loads / stores (16 B groups; p=4 uses 8 B groups of 16-bit planes)
template <int GB>
struct GrpIO;

template <>
struct GrpIO<16> {
  __device__ __forceinline__ static Grp ld(const uint8_t* p) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    return Grp{v.x, v.y, v.z, v.w};
  }
  __device__ __forceinline__ static Grp ld_cg(const uint8_t* p) {
    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(p));
    return Grp{v.x, v.y, v.z, v.w};
  }
  __device__ __forceinline__ static void st(uint8_t* p, const Grp& g) {
    *reinterpret_cast<uint4*>(p) = make_uint4(g.b0, g.b1, g.b2, g.b3);
  }
};

template <>
struct GrpIO<8> {
  __device__ __forceinline__ static Grp unpack(uint2 v) {
    return Grp{v.x & 0xffffu, v.x >> 16, v.y & 0xffffu, v.y >> 16};
  }
  __device__ __forceinline__ static Grp ld(const uint8_t* p) {
    return unpack(__ldg(reinterpret_cast<const uint2*>(p)));
  }
  __device__ __forceinline__ static Grp ld_cg(const uint8_t* p) {
    return unpack(__ldcg(reinterpret_cast<const uint2*>(p)));
  }
  __device__ __forceinline__ static void st(uint8_t* p, const Grp& g) {
    *reinterpret_cast<uint2*>(p) = make_uint2(g.b0 | (g.b1 << 16), g.b2 | (g.b3 << 16));
  }
};

// ---- packed <-> bit-sliced conversion of one group (nwords = GB/4 packed words)
// Packed word w (little endian) holds registers 8w..8w+7, nibble k = register 8w+k.
__device__ __host__ __forceinline__ uint32_t gather_every4(uint32_t x) {
  x &= 0x11111111u;
  x = (x | (x >> 3)) & 0x03030303u;
  x = (x | (x >> 6)) & 0x000f000fu;
  x = (x | (x >> 12)) & 0x000000ffu;
  return x;
}
__device__ __host__ __forceinline__ uint32_t spread_every4(uint32_t y) {
  y &= 0xffu;
  y = (y | (y << 12)) & 0x000f000fu;
  y = (y | (y << 6)) & 0x03030303u;
  y = (y | (y << 3)) & 0x11111111u;
  return y;
}

// ---- ordered encoding of doubles for atomicMax
__device__ __host__ __forceinline__ unsigned long long dbl_to_ord(double x) {
#ifdef __CUDA_ARCH__
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
#else
  unsigned long long u;
  memcpy(&u, &x, 8);
#endif
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// Byte k of x, zero-extended (one PRMT).
__device__ __forceinline__ uint32_t byte_of(uint32_t x, int k) { return __byte_perm(x, 0u, 0x4440u + k); }

// Per byte of w: payload << 7 * (continuation bytes just before it, <= 4), the
// continuation run read from the flag bytes of w and of the previous word wp.
__device__ __forceinline__ void varint_contrib(uint32_t w, uint32_t wp, uint32_t (&c)[4]) {
  const uint32_t F = w & 0x80808080u, Fp = wp & 0x80808080u;
  const uint32_t m1 = __funnelshift_l(Fp, F, 8);
  const uint32_t m2 = m1 & __funnelshift_l(Fp, F, 16);
  const uint32_t m3 = m2 & __funnelshift_l(Fp, F, 24);
  const uint32_t m4 = m3 & Fp;
  const uint32_t D7 = ((m1 >> 7) + (m2 >> 7) + (m3 >> 7) + (m4 >> 7)) * 7u;  // 7 d per byte, <= 28
  const uint32_t P = w & 0x7f7f7f7fu;
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k] = byte_of(P, k) << byte_of(D7, k);
}

// ---- 4-bytes-per-lane LEB128 decode (hot path) ------------------------
// A 128-byte window at `pos` (a varint boundary); lane L holds bytes
// 4L..4L+3.  Because every byte's payload lands in exactly one delta, the
// absolute id at a terminator j is
//     base + sum_{k <= j} (b_k & 0x7f) << (7 * d_k),
// d_k = number of continuation bytes immediately preceding byte k -- a plain
// prefix sum over bytes, no segmented reduction.  d_k needs at most 4 bytes
// of look-back (ids < 2^32 -> at most 5 payload-carrying bytes; the bytes of a
// non-canonical varint beyond the 5th carry zero payload on a validated
// stream, so capping d_k at 4 leaves their contribution 0), i.e. the previous
// lane's word.  Only the first `remaining` terminators are taken; the window's
// trailing partial varint is re-read by the next step.
struct Decode4 {
  int wanted;     // terminators consumed from the item in this window
  int count;      // ids written to buf (== wanted unless SKIP filtered some)
  int advance;    // bytes consumed (through the last wanted terminator)
  uint32_t last;  // id of the last wanted terminator (next base)
};

__device__ __forceinline__ uint32_t ld_stream_word(const uint8_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Writes the kept ids (compacted, in order) to buf[0..count) and pads
// buf[count..count+PAD) with the last one.  Needs the stream padded by >= 136 B.
__device__ __forceinline__ uint32_t sel4(const uint32_t (&v)[4], int k) {
  return k <= 0 ? v[0] : k == 1 ? v[1] : k == 2 ? v[2] : v[3];
}

// buf must hold 128 + PAD entries.
template <bool SKIP, int PAD>
__device__ __forceinline__ Decode4 decode_step4(const uint8_t* __restrict__ stream, uint64_t pos,
                                                uint32_t remaining, uint32_t base, const uint8_t* changed,
                                                uint32_t* buf, int lane) {
  const uint8_t* al = stream + (pos & ~3ull) + 4 * lane;
  const uint32_t w0 = ld_stream_word(al);
  const uint32_t w1 = ld_stream_word(al + 4);
  const uint32_t w = __funnelshift_r(w0, w1, static_cast<uint32_t>(pos & 3) * 8);
  uint32_t wp = __shfl_up_sync(FULL, w, 1);
  if (lane == 0) wp = 0;  // the window starts on a varint boundary
  uint32_t c[4];  // per byte: payload << 7 * (run of continuation flags before it, 0..4)
  varint_contrib(w, wp, c);
  const uint32_t p1 = c[0] + c[1], p2 = p1 + c[2], lane_sum = p2 + c[3];
  uint32_t incl = lane_sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, incl, d);
    if (lane >= d) incl += y;
  }
  const uint32_t excl = base + incl - lane_sum;
  const uint32_t id[4] = {excl + c[0], excl + p1, excl + p2, excl + lane_sum};
  const uint32_t T = ~w & 0x80808080u;  // terminator flags
  const uint32_t ltm = (1u << lane) - 1u;
  // global rank of each terminator = terminators in lower lanes + earlier bytes of this lane
  uint32_t below = 0, tot = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t B = __ballot_sync(FULL, (T >> (8 * k + 7)) & 1u);
    below += __popc(B & ltm);
    tot += __popc(B);
  }
  bool want[4];
  uint32_t r = below;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool t = (T >> (8 * k + 7)) & 1u;
    want[k] = t && r < remaining;
    r += t;
  }
  // position of the last wanted terminator
  int lastk = -1;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (want[k]) lastk = k;
  const uint32_t anyw = __ballot_sync(FULL, lastk >= 0);
  Decode4 o;
  o.wanted = static_cast<int>(tot < remaining ? tot : remaining);
  o.count = 0;
  o.advance = 0;
  o.last = base;
  if (anyw == 0) return o;
  const int L = 31 - __clz(anyw);
  const int lk = __shfl_sync(FULL, lastk, L);
  o.advance = 4 * L + lk + 1;
  o.last = __shfl_sync(FULL, sel4(id, lk), L);  // lk is warp-uniform
  if (!SKIP) {
    // Every wanted id is kept, and the wanted terminators are a prefix of the
    // window's terminators: a terminator's rank is its slot, the last wanted
    // id is the padding value -- no further ballots.
    uint32_t slot = below;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (want[k]) buf[slot++] = id[k];
    o.count = o.wanted;
#pragma unroll
    for (int k = lane; k < PAD; k += 32) buf[o.wanted + k] = o.last;
    return o;
  }
  bool keep[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) keep[k] = want[k] && changed[id[k]];
  uint32_t kb = 0, kn = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t B = __ballot_sync(FULL, keep[k]);
    kb += __popc(B & ltm);
    kn += __popc(B);
  }
  uint32_t slot = kb;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (keep[k]) buf[slot++] = id[k];
  o.count = static_cast<int>(kn);
  if (kn) {
    // last kept id: highest lane with a kept id, its highest kept byte
    int hk = -1;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (keep[k]) hk = k;
    const uint32_t anyk = __ballot_sync(FULL, hk >= 0);
    const int KL = 31 - __clz(anyk);
    const int kk = __shfl_sync(FULL, hk, KL);
    const uint32_t lastkept = __shfl_sync(FULL, sel4(id, kk), KL);
#pragma unroll
    for (int k = lane; k < PAD; k += 32) buf[kn + k] = lastkept;
  }
  return o;
}

// ---- 16-bytes-per-lane LEB128 decode of the per-node feeder (p < 9) ------
// A 512-byte window at `pos` (a varint boundary); lane L holds bytes
// 16L..16L+15, decode_step4's prefix-sum arithmetic.  No compaction: slot
// buf[17 L + j] gets the id of byte j's terminator if it is one of the item's
// wanted terminators (the first `remaining`); any other slot keeps what it
// held -- an id of an earlier step of the same item, or the fill the feeder
// writes at the item's start (the node itself): folding a row twice changes
// nothing (max is idempotent).  Stride 17 keeps the stores conflict-free and
// the batch loads at 2-way.  Needs the stream padded by >= 516 B.
struct Decode16 {
  int wanted;     // terminators consumed from the item in this window
  int advance;    // bytes consumed (through the last wanted terminator)
  uint32_t last;  // id of the last wanted terminator (next base)
};

__device__ __forceinline__ Decode16 decode_step16(const uint8_t* __restrict__ stream, uint64_t pos,
                                                  uint32_t remaining, uint32_t base, uint32_t* buf, int lane) {
  const uint8_t* al = stream + (pos & ~3ull) + 16 * lane;
  uint32_t A[5];
#pragma unroll
  for (int i = 0; i < 4; ++i) A[i] = ld_stream_word(al + 4 * i);
  A[4] = __shfl_down_sync(FULL, A[0], 1);
  if (lane == 31) A[4] = ld_stream_word(al + 16);
  const uint32_t sh = static_cast<uint32_t>(pos & 3) * 8;
  uint32_t x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = __funnelshift_r(A[i], A[i + 1], sh);
  uint32_t prev = __shfl_up_sync(FULL, x[3], 1);
  if (lane == 0) prev = 0;  // the window starts on a varint boundary
  uint32_t pre[16];
  uint32_t tm = 0u;  // terminator bytes, 16-bit mask
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t w = x[i];
    uint32_t c[4];
    varint_contrib(w, i ? x[i - 1] : prev, c);
#pragma unroll
    for (int k = 0; k < 4; ++k) pre[4 * i + k] = (4 * i + k) ? pre[4 * i + k - 1] + c[k] : c[k];
    const uint32_t T = ~w & 0x80808080u;
    tm |= ((T >> 7) & 1u | (T >> 14) & 2u | (T >> 21) & 4u | (T >> 28) & 8u) << (4 * i);
  }
  const uint32_t lane_sum = pre[15];
  uint32_t incl = lane_sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, incl, d);
    if (lane >= d) incl += y;
  }
  const uint32_t excl = base + incl - lane_sum;
  const uint32_t tc = __popc(tm);
  const uint32_t ttot = __reduce_add_sync(FULL, tc);
  uint32_t wm = tm;  // wanted terminators
  if (ttot > remaining) {  // warp-uniform: the item ends inside this window
    uint32_t tinc = tc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, tinc, d);
      if (lane >= d) tinc += y;
    }
    const uint32_t below = tinc - tc;
    if (below >= remaining)
      wm = 0u;
    else if (remaining - below < tc)
      wm = tm & ((2u << __fns(tm, 0, static_cast<int>(remaining - below))) - 1u);
  }
  Decode16 o;
  o.wanted = static_cast<int>(ttot < remaining ? ttot : remaining);
  o.advance = 0;
  o.last = base;
  const uint32_t anyw = __ballot_sync(FULL, wm != 0u);
  if (anyw == 0) return o;
  const int L = 31 - __clz(anyw);
  const int lk = 31 - __clz(__shfl_sync(FULL, wm, L));
  o.advance = 16 * L + lk + 1;
  uint32_t* b = buf + 17 * lane;
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if ((wm >> j) & 1u) b[j] = excl + pre[j];
  __syncwarp();
  o.last = buf[17 * L + lk];  // the last wanted id, as just stored by lane L
  return o;
}

}  // namespace sb
