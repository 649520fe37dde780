// Device helpers shared by the sm_100a kernels (NOT shared with oracle/).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tb {

// ---------------------------------------------------------------------------
// Bicyclic monoid (§3): (a,b) = (unmatched closes, unmatched opens)
//   (a,b) ⊕ (c,d) = (a + c - min(b,c), b + d - min(b,c))
// ---------------------------------------------------------------------------
struct Bic {
  int a, b;
};
__device__ __forceinline__ Bic bic_combine(Bic x, Bic y) {
  int m = min(x.b, y.a);
  return Bic{x.a + y.a - m, x.b + y.b - m};
}

// Streaming 16-byte load that does not allocate in L1.
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Tag bytes -> element bit masks (bit i <-> byte i of 16).  Tags 0..3 carry
// two bits: lo = bit 0, hi = bit 1 (OPEN_CLIP 1 = lo, OPEN_BLEND 2 = hi,
// CLOSE 3 = both); any byte >= 4 is a leaf (R2).  Bit 0 of the four bytes of
// a and of b go to bits 24..27 and 28..31 of the product (one multiply per 8
// elements; the shifted copies never overlap, so no carries).
__host__ __device__ __forceinline__ uint32_t gather8(uint32_t a, uint32_t b) {
  return ((a & 0x01010101u) | ((b << 4) & 0x10101010u)) * 0x01020408u;
}
__host__ __device__ __forceinline__ uint32_t top_bytes(uint32_t r0, uint32_t r1) {  // byte 3 of r0, r1 -> bits 0..15
#ifdef __CUDA_ARCH__
  return __byte_perm(r0, r1, 0x0073u) & 0xffffu;
#else
  return (r0 >> 24) | ((r1 >> 16) & 0xff00u);
#endif
}
// (lo, hi) masks of 16 bytes with every byte >= 4 cleared from both
__host__ __device__ __forceinline__ void tag_bits16(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3, uint32_t& lo,
                                                    uint32_t& hi) {
  lo = top_bytes(gather8(x0, x1), gather8(x2, x3));
  hi = top_bytes(gather8(x0 >> 1, x1 >> 1), gather8(x2 >> 1, x3 >> 1));
  if ((x0 | x1 | x2 | x3) & 0xfcfcfcfcu) {
    // per byte: ((x >> 2) & 0x3f) + 0x3f has bit 6 set iff x >= 4 (no carry between bytes)
    const uint32_t j0 = (((x0 >> 2) & 0x3f3f3f3fu) + 0x3f3f3f3fu) >> 6, j1 = (((x1 >> 2) & 0x3f3f3f3fu) + 0x3f3f3f3fu) >> 6;
    const uint32_t j2 = (((x2 >> 2) & 0x3f3f3f3fu) + 0x3f3f3f3fu) >> 6, j3 = (((x3 >> 2) & 0x3f3f3f3fu) + 0x3f3f3f3fu) >> 6;
    const uint32_t junk = top_bytes(gather8(j0, j1), gather8(j2, j3));
    lo &= ~junk;
    hi &= ~junk;
  }
}
// 16 tag bytes -> (open mask, close mask)
__host__ __device__ __forceinline__ void classify16(uint4 w, uint32_t& om, uint32_t& cm) {
  uint32_t lo, hi;
  tag_bits16(w.x, w.y, w.z, w.w, lo, hi);
  om = lo ^ hi;
  cm = lo & hi;
}
// 16 tag bytes -> (open mask, close mask, blend-open mask)
__host__ __device__ __forceinline__ void classify16b(uint4 w, uint32_t& om, uint32_t& cm, uint32_t& bm) {
  uint32_t lo, hi;
  tag_bits16(w.x, w.y, w.z, w.w, lo, hi);
  om = lo ^ hi;
  cm = lo & hi;
  bm = hi & ~lo;
}

// Index of the j-th (0-based) lowest set bit of a 16-bit mask m (m has > j
// bits set): branch-free binary search on popcounts.
__device__ __forceinline__ int select_bit(uint32_t m, int j) {
  int pos = 0, c;
  c = __popc(m & 0xffu);
  if (j >= c) { j -= c; pos += 8; m >>= 8; }
  c = __popc(m & 0xfu);
  if (j >= c) { j -= c; pos += 4; m >>= 4; }
  c = __popc(m & 0x3u);
  if (j >= c) { j -= c; pos += 2; m >>= 2; }
  c = (int)(m & 1u);
  if (j >= c) pos += 1;
  return pos;
}


// ---------------------------------------------------------------------------
// Unmatched opens of a run of elements, 4 at a time.  Walking backwards with P
// = closes to the right still waiting for a partner, an open is unmatched in
// the run iff P == 0 when it is reached (§3-§4: exactly the opens of the run's
// Bic b component).  Table entry for (open nibble o, close nibble c, min(P, 4)):
// bits 0-3 = the nibble's unmatched opens, bits 4-7 = P_out - P_in + 4 (a P of 4
// or more already matches every open of the nibble).  Index = o | c << 4 | pin << 8.
// ---------------------------------------------------------------------------
constexpr int UNM4_ENTRIES = 256 * 5;
__host__ __device__ __forceinline__ uint8_t unm4_entry(int idx) {
  const int o = idx & 15, c = (idx >> 4) & 15, pin = idx >> 8;
  int P = pin, mask = 0;
  for (int j = 3; j >= 0; j--) {
    if ((c >> j) & 1) P++;
    else if ((o >> j) & 1) {
      if (P > 0) P--;
      else mask |= 1 << j;
    }
  }
  return (uint8_t)(mask | ((P - pin + 4) << 4));
}
__device__ __forceinline__ void unm4_fill(uint8_t* tab, int tid, int nthreads) {
  for (int i = tid; i < UNM4_ENTRIES; i += nthreads) tab[i] = unm4_entry(i);
}
// unmatched opens among the 32 elements of (ow, cw), walking backwards from a
// pending count P (updated)
__device__ __forceinline__ uint32_t unm32(const uint8_t* tab, uint32_t ow, uint32_t cw, int& P) {
  uint32_t um = 0;
#pragma unroll
  for (int q = 7; q >= 0; q--) {
    const uint32_t e = tab[((ow >> (4 * q)) & 15u) | (((cw >> (4 * q)) & 15u) << 4) | ((uint32_t)min(P, 4) << 8)];
    um |= (e & 15u) << (4 * q);
    P += (int)(e >> 4) - 4;
  }
  return um;
}

}  // namespace tb
