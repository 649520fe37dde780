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

// Per-byte classification of 4 tag bytes into a 4-bit mask (bit i <-> byte i).
__device__ __forceinline__ uint32_t byte_mask4(uint32_t cmp /* 0xff per hit */) {
  uint32_t m = cmp & 0x01010101u;
  return (m * 0x01020408u) >> 24;
}
// 16 tag bytes -> (open mask, close mask), bit i <-> element i.
__device__ __forceinline__ void classify16(uint4 w, uint32_t& om, uint32_t& cm) {
  uint32_t o = 0, c = 0;
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int q = 0; q < 4; q++) {
    uint32_t x = ws[q];
    uint32_t op = __vcmpeq4(x, 0x01010101u) | __vcmpeq4(x, 0x02020202u);
    uint32_t cl = __vcmpeq4(x, 0x03030303u);
    o |= byte_mask4(op) << (4 * q);
    c |= byte_mask4(cl) << (4 * q);
  }
  om = o;
  cm = c;
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
