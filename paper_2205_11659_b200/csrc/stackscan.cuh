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
  int32_t* hstart;           // [ntiles] stack height at the tile start (written with lw)
  int2* agg;                 // [ntiles] Bic value (a, b) of each tile (reduce pass)
  int2* total;               // [1] Bic value of the whole stream (after the tile scan)
  uint32_t* lv[HLEVELS];     // lv[k][g] = 1 + min L over tiles [g*32^k, (g+1)*32^k)
  uint32_t* cnt[HLEVELS];    // arrival counters for lv[k]
};

// Sizes (in elements) of the control arrays for `ntiles` tiles.
struct CtrlLayout {
  size_t off_counter, off_desc, off_lw, off_h, off_agg, off_total, off_lv[HLEVELS], off_cnt[HLEVELS], bytes;
  __host__ __device__ static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
  __host__ __device__ explicit CtrlLayout(int64_t ntiles) {
    size_t o = 0;
    off_counter = o; o = align256(o + 16);
    off_desc = o; o = align256(o + 8 * (size_t)ntiles);
    off_lw = o; o = align256(o + 4 * (size_t)ntiles);
    off_h = o; o = align256(o + 4 * (size_t)ntiles);
    off_agg = o; o = align256(o + 8 * (size_t)ntiles);
    off_total = o; o = align256(o + 8);
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
    c.hstart = (int32_t*)(b + off_h);
    c.agg = (int2*)(b + off_agg);
    c.total = (int2*)(b + off_total);
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
// walk always terminates.  Each round trip inspects LBW = 128 predecessors
// (4 independent loads per lane): with many tiles in flight the newest
// inclusive descriptor typically lies a few hundred tiles back.
// ---------------------------------------------------------------------------
constexpr int LBG = 4;  // groups of 32 descriptors per round trip

__device__ __forceinline__ Bic warp_fold_desc(uint64_t d, bool valid, int lane, int stop) {
  // lane k holds tile (j - k); fold lanes [0, stop] with earlier tiles first
  Bic v = (valid && lane <= stop) ? desc_val(d) : Bic{0, 0};
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Bic o;
    o.a = __shfl_down_sync(0xffffffffu, v.a, off);
    o.b = __shfl_down_sync(0xffffffffu, v.b, off);
    if (lane + off < 32) v = bic_combine(o, v);
  }
  return Bic{__shfl_sync(0xffffffffu, v.a, 0), __shfl_sync(0xffffffffu, v.b, 0)};
}

__device__ __forceinline__ Bic lookback_warp(const Ctrl& c, int T) {
  const int lane = threadIdx.x & 31;
  Bic acc{0, 0};
  int j = T - 1;
  while (true) {
    uint64_t d[LBG];
#pragma unroll
    for (int g = 0; g < LBG; g++) {
      const int t = j - 32 * g - lane;
      d[g] = t >= 0 ? ld_relaxed_u64(c.desc + t) : desc_pack(DESC_INC, Bic{0, 0});
    }
#pragma unroll
    for (int g = 0; g < LBG; g++) {
      const int t = j - 32 * g - lane;
      // descriptors carry their own payload: relaxed (strong) loads suffice
      while (desc_flag(d[g]) == DESC_NONE) d[g] = ld_relaxed_u64(c.desc + t);
      const unsigned inc = __ballot_sync(0xffffffffu, desc_flag(d[g]) == DESC_INC);
      const int stop = inc ? (__ffs(inc) - 1) : 31;
      acc = bic_combine(warp_fold_desc(d[g], t >= 0, lane, stop), acc);
      if (inc) return acc;
    }
    j -= 32 * LBG;
  }
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

// Low-water marks of the 32 tiles before `base` (lane j <-> tile base-1-j),
// read once and kept in a register; 0 = not yet published.  Searches from
// any `from` in (base-32, base] are answered from it while it covers them,
// waiting only for the tiles that are actually needed (closest first).
struct LwWindow {
  int base;
  uint32_t v;  // lw + 1 as published, 0 = unknown
};

__device__ __forceinline__ LwWindow lw_window_load(const Ctrl& c, int base) {
  const int lane = threadIdx.x & 31;
  const int t = base - 1 - lane;
  LwWindow w;
  w.base = base;
  w.v = t >= 0 ? ld_acquire_u32(c.lw + t) : 0xffffffffu;  // 0xffffffff: no tile
  return w;
}

// Search via the window first; falls back to the hierarchy if the answer is
// older than the window.
__device__ __forceinline__ int owner_search_win(const Ctrl& c, LwWindow& w, int from, int X, int& Lout) {
  const int lane = threadIdx.x & 31;
  const uint32_t ux = (uint32_t)X;
  const int t = w.base - 1 - lane;
  const bool cand = t < from && t >= 0;
  while (true) {
    // closest candidate lane whose value is known and qualifies, with all
    // closer candidates known (and not qualifying)
    const bool known = w.v != 0u;
    const bool q = cand && known && (w.v - 1u) <= ux;
    const unsigned mq = __ballot_sync(0xffffffffu, q);
    const unsigned mu = __ballot_sync(0xffffffffu, cand && !known);
    const unsigned first_q = mq & (~mq + 1u);          // lowest qualifying lane
    const unsigned before = first_q ? (first_q - 1u) : 0xffffffffu;
    if (mq && (mu & before) == 0u) {
      const int k = __ffs(mq) - 1;
      Lout = (int)(__shfl_sync(0xffffffffu, w.v, k) - 1u);
      return w.base - 1 - k;
    }
    if (!mq && !mu) break;  // nothing in the window qualifies
    // wait for the unknown candidates that matter (closer than any hit)
    if (cand && !known && (mq == 0u || ((1u << lane) & before))) w.v = wait_u32(c.lw + t);
  }
  if (w.base - 32 <= 0) return -1;
  return owner_search(c, min(from, w.base - 32), X, Lout);
}

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

// ---------------------------------------------------------------------------
// Publish tile T's inclusive descriptor and low-water mark (one thread, after
// the block synchronised on its slice writes).  The release store orders all
// of the CTA's earlier writes (bar.sync + gpu-scope release, as in CUTLASS's
// semaphores) before both stores; the relaxed low-water store after the
// release fence forms a release pattern for readers that acquire it.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void publish_inclusive(const Ctrl& c, int T, Bic incl, int L, bool desc_too) {
  if (desc_too) st_release_u64(c.desc + T, desc_pack(DESC_INC, incl));
  else __threadfence();
  st_relaxed_u32(c.lw + T, (uint32_t)L + 1u);
}

// Fold tile T's published low-water mark into the 32-ary hierarchy (warp;
// off the critical path).  The last of 32 siblings to arrive publishes the
// parent entry.
__device__ __forceinline__ void hierarchy_arrive(const Ctrl& c, int T) {
  const int lane = threadIdx.x & 31;
  int idx = T;
#pragma unroll 1
  for (int k = 1; k < HLEVELS; k++) {
    const int g = idx >> 5;
    unsigned old = 0;
    if (lane == 0) old = atom_add_acqrel_u32(c.cnt[k] + g, 1u);
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old != 31u) return;
    uint32_t v = wait_u32(c.lv[k - 1] + ((size_t)g << 5) + lane);
    v = __reduce_min_sync(0xffffffffu, v);
    if (lane == 0) st_release_u32(c.lv[k] + g, v);
    idx = g;
  }
}

}  // namespace tb
