// Cross-tile machinery shared by paren_match and tree_bbox kernels:
//   * decoupled look-back over the bicyclic monoid (§3; look-back is
//     the paper's own future-work item, P:381 [Mer16]);
//   * low-water-mark hierarchy used to find, for a height X of the stack at
//     the start of tile `from`, the tile that pushed that entry (owner rule:
//     the last tile U < from whose low-water mark L_U <= X).
//     This is the "binary search over published slice prefixes" of the
//     north star, done as a 32-ary search with warp ballots.
#pragma once
#include "common.cuh"

namespace tb {

constexpr int HLEVELS = 4;  // 32^4 tiles >= 2^31 / 4096

// Global control block of one call (zeroed by the host before each launch).
struct Ctrl {
  uint32_t* counter;         // dynamic tile ids
  uint64_t* desc;            // [ntiles] Bic look-back descriptors
  uint32_t* lw;              // [ntiles] low-water mark L_T + 1 (0 = not yet)
  uint32_t* lv[HLEVELS];     // lv[k][g] = 1 + min L over tiles [g*32^k, (g+1)*32^k)
  uint32_t* cnt[HLEVELS];    // arrival counters for lv[k]
};

// Sizes (in elements) of the control arrays for `ntiles` tiles.
struct CtrlLayout {
  size_t off_counter, off_desc, off_lw, off_lv[HLEVELS], off_cnt[HLEVELS], bytes;
  __host__ __device__ static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
  __host__ __device__ explicit CtrlLayout(int64_t ntiles) {
    size_t o = 0;
    off_counter = o; o = align256(o + 16);
    off_desc = o; o = align256(o + 8 * (size_t)ntiles);
    off_lw = o; o = align256(o + 4 * (size_t)ntiles);
    int64_t m = ntiles;
    off_lv[0] = off_cnt[0] = 0;
    for (int k = 1; k < HLEVELS; k++) {
      m = (m + 31) / 32;
      off_lv[k] = o; o = align256(o + 4 * (size_t)m);
      off_cnt[k] = o; o = align256(o + 4 * (size_t)m);
    }
    bytes = o;
  }
  __host__ __device__ Ctrl bind(void* base) const {
    char* b = (char*)base;
    Ctrl c;
    c.counter = (uint32_t*)(b + off_counter);
    c.desc = (uint64_t*)(b + off_desc);
    c.lw = (uint32_t*)(b + off_lw);
    c.lv[0] = c.lw;
    c.cnt[0] = nullptr;
    for (int k = 1; k < HLEVELS; k++) {
      c.lv[k] = (uint32_t*)(b + off_lv[k]);
      c.cnt[k] = (uint32_t*)(b + off_cnt[k]);
    }
    return c;
  }
};

// ---------------------------------------------------------------------------
// Decoupled look-back (one warp).  Returns the exclusive Bic prefix of tile T
// (T >= 1).  Tile 0 publishes an inclusive descriptor straight away, so the
// walk always terminates.
// ---------------------------------------------------------------------------
__device__ __forceinline__ Bic lookback_warp(const Ctrl& c, int T) {
  const int lane = threadIdx.x & 31;
  Bic acc{0, 0};
  int j = T - 1;
  while (true) {
    const int t = j - lane;
    uint64_t d = 0;
    if (t >= 0) {
      d = ld_acquire_u64(c.desc + t);
      while (desc_flag(d) == DESC_NONE) {
        __nanosleep(20);
        d = ld_acquire_u64(c.desc + t);
      }
    }
    const unsigned inc = __ballot_sync(0xffffffffu, t >= 0 && desc_flag(d) == DESC_INC);
    const int stop = inc ? (__ffs(inc) - 1) : 31;
    Bic v = (t >= 0 && lane <= stop) ? desc_val(d) : Bic{0, 0};
    // lane k holds tile j-k; combine earlier (higher lane) first.
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      Bic o;
      o.a = __shfl_down_sync(0xffffffffu, v.a, off);
      o.b = __shfl_down_sync(0xffffffffu, v.b, off);
      if (lane + off < 32) v = bic_combine(o, v);
    }
    Bic win{__shfl_sync(0xffffffffu, v.a, 0), __shfl_sync(0xffffffffu, v.b, 0)};
    acc = bic_combine(win, acc);
    if (inc) break;
    j -= 32;
  }
  return acc;
}

// ---------------------------------------------------------------------------
// Owner search (one warp): the last tile U < from with L_U <= X (X >= 0).
// Returns U (and its L in Lout), or -1 if no tile qualifies (then the entry
// belongs to the stack that was live before tile 0, i.e. the shard's
// incoming stack).  Every visited entry is complete-before-`from`, so the
// spins only wait on tiles that are already running or done.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int owner_search(const Ctrl& c, int from, int X, int& Lout) {
  const int lane = threadIdx.x & 31;
  const uint32_t ux = (uint32_t)X;
  int idx = from;
#pragma unroll 1
  for (int k = 0; k < HLEVELS; k++) {
    const int g = idx >> 5, r = idx & 31;
    uint32_t v = 0xffffffffu;
    if (lane < r) v = wait_u32(c.lv[k] + ((size_t)g << 5) + lane) - 1u;
    const unsigned m = __ballot_sync(0xffffffffu, lane < r && v <= ux);
    if (m) {
      int E = (g << 5) + (31 - __clz(m));
      uint32_t L = __shfl_sync(0xffffffffu, v, 31 - __clz(m));
#pragma unroll 1
      for (int j = k - 1; j >= 0; j--) {
        const uint32_t v2 = wait_u32(c.lv[j] + ((size_t)E << 5) + lane) - 1u;
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

// ---------------------------------------------------------------------------
// Publish tile T's low-water mark and fold it into the hierarchy (warp 0,
// after every thread's slice writes were fenced and the block synchronised).
// The last of 32 siblings to arrive publishes the parent entry.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void publish_lowwater(const Ctrl& c, int T, int L) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    __threadfence();
    st_release_u32(c.lw + T, (uint32_t)L + 1u);
  }
  int idx = T;
#pragma unroll 1
  for (int k = 1; k < HLEVELS; k++) {
    const int g = idx >> 5;
    unsigned old = 0;
    if (lane == 0) {
      __threadfence();
      old = atomicAdd(c.cnt[k] + g, 1u);
    }
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old != 31u) return;
    __threadfence();
    uint32_t v = wait_u32(c.lv[k - 1] + ((size_t)g << 5) + lane);
    v = __reduce_min_sync(0xffffffffu, v);
    if (lane == 0) st_release_u32(c.lv[k] + g, v);
    idx = g;
  }
}

}  // namespace tb
