// Cross-tile machinery of paren_match: the control block the tile scan fills
// (tile start heights, low-water marks, their 32-ary min hierarchy), and the
// owner search: for a height X of the stack at the start of tile `from`, the
// tile that pushed that entry (owner rule F1: the last tile U < from whose
// low-water mark L_U <= X).  This is the "binary search over published slice
// prefixes" of the north star, done as a 32-ary search with warp ballots.
#pragma once
#include "common.cuh"

namespace tb {

constexpr int HLEVELS = 4;  // 32^4 tiles >= 2^31 / 4096

// Global control block of one call (zeroed by the host before each launch).
struct Ctrl {
  uint32_t* lw;              // [ntiles] low-water mark L_T + 1 (0 = not yet)
  int32_t* hstart;           // [ntiles] stack height at the tile start (written with lw)
  int2* agg;                 // [ntiles] Bic value (a, b) of each tile (reduce pass)
  int2* total;               // [1] Bic value of the whole stream (after the tile scan)
  int* smin;                 // [ntiles] min low-water mark over the later tiles (INT_MAX: none)
  uint32_t* lv[HLEVELS];     // lv[k][g] = 1 + min L over tiles [g*32^k, (g+1)*32^k)
};

// Sizes (in elements) of the control arrays for `ntiles` tiles.
struct CtrlLayout {
  size_t off_lw, off_h, off_agg, off_total, off_smin, off_lv[HLEVELS], bytes;
  __host__ __device__ static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
  __host__ __device__ explicit CtrlLayout(int64_t ntiles) {
    size_t o = 0;
    off_lw = o; o = align256(o + 4 * (size_t)ntiles);
    off_h = o; o = align256(o + 4 * (size_t)ntiles);
    off_agg = o; o = align256(o + 8 * (size_t)ntiles);
    off_total = o; o = align256(o + 8);
    off_smin = o; o = align256(o + 4 * (size_t)ntiles);
    int64_t m = ntiles;
    off_lv[0] = 0;
    for (int k = 1; k < HLEVELS; k++) {
      m = (m + 31) / 32;
      off_lv[k] = o; o = align256(o + 4 * (size_t)m);
    }
    bytes = o;
  }
  __host__ __device__ Ctrl bind(void* base) const {
    char* b = (char*)base;
    Ctrl c;
    c.lw = (uint32_t*)(b + off_lw);
    c.hstart = (int32_t*)(b + off_h);
    c.agg = (int2*)(b + off_agg);
    c.total = (int2*)(b + off_total);
    c.smin = (int*)(b + off_smin);
    c.lv[0] = c.lw;
    for (int k = 1; k < HLEVELS; k++) {
      c.lv[k] = (uint32_t*)(b + off_lv[k]);
    }
    return c;
  }
};

// ---------------------------------------------------------------------------
// Owner search over a COMPLETE hierarchy (finish pass: the reduce pass has
// ended, every value is published, plain loads suffice).  Same contract as
// owner_search.  The first 32 predecessors of `from` are tested in one
// ballot; older owners are found through the 32-ary levels.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int owner_search_done(const Ctrl& c, int from, int X, int& Lout) {
  const int lane = threadIdx.x & 31;
  const uint32_t ux = (uint32_t)X;
  {
    const int t = from - 1 - lane;
    const uint32_t v = t >= 0 ? __ldg(c.lw + t) - 1u : 0xffffffffu;
    const unsigned m = __ballot_sync(0xffffffffu, t >= 0 && v <= ux);
    if (m) {
      const int k = __ffs(m) - 1;
      Lout = (int)__shfl_sync(0xffffffffu, v, k);
      return from - 1 - k;
    }
    if (from <= 32) return -1;
    from -= 32;
  }
  int idx = from;
#pragma unroll 1
  for (int k = 0; k < HLEVELS; k++) {
    const int g = idx >> 5, r = idx & 31;
    const uint32_t v = lane < r ? __ldg(c.lv[k] + ((size_t)g << 5) + lane) - 1u : 0xffffffffu;
    const unsigned m = __ballot_sync(0xffffffffu, lane < r && v <= ux);
    if (m) {
      int E = (g << 5) + (31 - __clz(m));
      uint32_t L = __shfl_sync(0xffffffffu, v, 31 - __clz(m));
#pragma unroll 1
      for (int j = k - 1; j >= 0; j--) {
        const uint32_t v2 = __ldg(c.lv[j] + ((size_t)E << 5) + lane) - 1u;
        const unsigned m2 = __ballot_sync(0xffffffffu, v2 <= ux);
        const int top = 31 - __clz(m2);
        L = __shfl_sync(0xffffffffu, v2, top);
        E = (E << 5) + top;
      }
      Lout = (int)L;
      return E;
    }
    idx = g;
    if (idx == 0) break;
  }
  return -1;
}

}  // namespace tb
