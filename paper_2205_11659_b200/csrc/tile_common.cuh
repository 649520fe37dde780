// Per-tile building blocks shared by the paren_match and tree_bbox kernels.
//
// A tile is NT threads x K contiguous elements.  Each thread first runs a
// register walk over its K elements (the k-elements-per-thread level of the
// paper's work-efficient algorithm, §8): its stack is a bitmask of
// open positions (top = highest set bit), so push / pop / top are single
// integer operations.  The thread's result is a Bic value (a_t, b_t) (§3
// P:96-102) plus, per element, its in-thread parent or "external" mark.
#pragma once
#include "common.cuh"

namespace tb {

// Result of the register walk over 16 elements.
struct Walk16 {
  uint32_t om, cm;    // open / close masks (bit i <-> element i)
  uint32_t S;         // opens still on the thread stack at the end (unmatched in-thread)
  uint32_t plo, phi;  // nibble i: in-thread parent of element i (i < 8 / i >= 8)
  uint32_t mlo, mhi;  // nibble o: in-thread partner close of open o
  uint32_t ext;       // elements whose parent lies before the thread
  uint32_t ucm;       // closes with no in-thread open: they pop the stack at thread start
};

__device__ __forceinline__ uint4 load_tags16(const uint8_t* tags, int64_t n, int64_t tbase, bool full) {
  if (full) return ld_stream_v4(tags + tbase);
  uint32_t wv[4] = {0, 0, 0, 0};
#pragma unroll 1
  for (int i = 0; i < 16; i++) {
    const int64_t g = tbase + i;
    const uint32_t v = g < n ? tags[g] : 0u;  // padding = leaf = Bic identity
    wv[i >> 2] |= v << (8 * (i & 3));
  }
  return make_uint4(wv[0], wv[1], wv[2], wv[3]);
}

// Fig. 1 restricted to the thread's 16 elements.
__device__ __forceinline__ Walk16 walk16(uint4 raw) {
  Walk16 w;
  classify16(raw, w.om, w.cm);
  uint32_t S = 0, plo = 0, phi = 0, mlo = 0, mhi = 0, ext = 0, ucm = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) {
    const uint32_t bit = 1u << i;
    const int top = 31 - __clz(S);  // -1 when the thread stack is empty
    if (i < 8) plo |= (uint32_t)(top & 15) << (4 * i);
    else phi |= (uint32_t)(top & 15) << (4 * (i - 8));
    ext |= S ? 0u : bit;
    const bool pop = (w.cm & bit) && S;
    ucm |= ((w.cm & bit) && !S) ? bit : 0u;
    const uint32_t pv = (uint32_t)i << (4 * (top & 7));
    mlo |= (pop && top < 8) ? pv : 0u;
    mhi |= (pop && top >= 8) ? pv : 0u;
    S = (w.om & bit) ? (S | bit) : (pop ? (S ^ (1u << top)) : S);
  }
  w.S = S;
  w.plo = plo;
  w.phi = phi;
  w.mlo = mlo;
  w.mhi = mhi;
  w.ext = ext;
  w.ucm = ucm;
  return w;
}

__device__ __forceinline__ int nib(uint32_t lo, uint32_t hi, int i) {
  return (int)(((i < 8 ? lo : hi) >> (4 * (i & 7))) & 15u);
}

// Block-wide scans of the thread Bic values (warp shuffles + one barrier).
//   ex  = Bic of the tile's elements before this thread (exclusive prefix)
//   sx  = Bic of the tile's elements after this thread (exclusive suffix)
//   tot = Bic of the whole tile
template <int NW>
__device__ __forceinline__ void block_bic_scans(Bic v, Bic* wtot, Bic& ex, Bic& sx, Bic& tot, bool want_suffix) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Bic incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Bic o{__shfl_up_sync(0xffffffffu, incl.a, off), __shfl_up_sync(0xffffffffu, incl.b, off)};
    if (lane >= off) incl = bic_combine(o, incl);
  }
  Bic suf = v;
  if (want_suffix) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      Bic o{__shfl_down_sync(0xffffffffu, suf.a, off), __shfl_down_sync(0xffffffffu, suf.b, off)};
      if (lane + off < 32) suf = bic_combine(suf, o);
    }
  }
  if (lane == 31) wtot[warp] = incl;
  __syncthreads();
  Bic wpre{0, 0}, wsuf{0, 0}, t{0, 0};
#pragma unroll
  for (int w = 0; w < NW; w++) {
    const Bic x = wtot[w];
    if (w < warp) wpre = bic_combine(wpre, x);
    if (w > warp) wsuf = bic_combine(wsuf, x);
    t = bic_combine(t, x);
  }
  Bic e{__shfl_up_sync(0xffffffffu, incl.a, 1), __shfl_up_sync(0xffffffffu, incl.b, 1)};
  if (lane == 0) e = Bic{0, 0};
  ex = bic_combine(wpre, e);
  if (want_suffix) {
    Bic s{__shfl_down_sync(0xffffffffu, suf.a, 1), __shfl_down_sync(0xffffffffu, suf.b, 1)};
    if (lane == 31) s = Bic{0, 0};
    sx = bic_combine(s, wsuf);
  }
  tot = t;
}

// Thread-level owner lookup (owner rule at thread granularity): reference to
// the open at relative height x of the stack at the start of this thread.
// Returns an in-tile element offset (>= 0) or x itself (< 0) when the entry
// was pushed before the tile.  `w[k]` = min of l over lanes [lane-2^k+1, lane]
// of this warp; win/wmin/l/uo are the block's shared copies.
template <int NW, int K>
__device__ __forceinline__ int thread_ref(const int (&w)[5], int l_me, uint32_t uo_me, int x,
                                          const int (*win)[5][32], const int* wmin, const int* l,
                                          const uint32_t* uo) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int pos = lane;
#pragma unroll
  for (int k = 4; k >= 0; k--) {
    const int src = pos > 0 ? pos - 1 : 0;
    const int m = __shfl_sync(0xffffffffu, w[k], src);
    if (pos >= (1 << k) && m > x) pos -= (1 << k);
  }
  const int src = pos > 0 ? pos - 1 : 0;
  const int lV = __shfl_sync(0xffffffffu, l_me, src);
  const uint32_t uV = __shfl_sync(0xffffffffu, uo_me, src);
  if (pos > 0) return (warp * 32 + pos - 1) * K + select_bit(uV, x - lV);
  for (int W = warp - 1; W >= 0; W--) {
    if (wmin[W] <= x) {
      int p2 = 32;
#pragma unroll
      for (int k = 4; k >= 0; k--)
        if (p2 >= (1 << k) && win[W][k][p2 - 1] > x) p2 -= (1 << k);
      const int V = W * 32 + p2 - 1;
      return V * K + select_bit(uo[V], x - l[V]);
    }
  }
  return x;
}

// Windowed min of l over lanes [lane-2^k+1, lane], k = 0..4.
__device__ __forceinline__ void lane_windows(int l_t, int (&w)[5]) {
  const int lane = threadIdx.x & 31;
  w[0] = l_t;
#pragma unroll
  for (int k = 1; k < 5; k++) {
    const int h = 1 << (k - 1);
    const int o = __shfl_up_sync(0xffffffffu, w[k - 1], h);
    w[k] = lane >= h ? min(w[k - 1], o) : w[k - 1];
  }
}

}  // namespace tb
