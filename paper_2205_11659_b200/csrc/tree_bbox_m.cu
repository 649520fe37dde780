// tree_bbox from matching (sm_100a): clip intersections and blend unions
// (§6, §9) computed from the parent / match arrays that
// paren_match produces (§2: parent = Fig. 1's out, match = the
// classical partner).
//
// With the parent of every element known, the clip of an element is
//     ctx(e) = box(e) ∩ ctx(parent(e))        (clip opens and leaves)
//     ctx(b) = ctx(parent(b))                  (blend opens carry no box, R7)
// and the union of a node (o, c = match(o)) is the union of the clipped leaves
// strictly between o and c (R8).  Both are evaluated tile by tile:
//
// bbm_reduce   one CTA per tile.  The tile's opens whose close lies beyond the
//              tile ("tile-unmatched": the slice of P:229-233) get their
//              tile-local cumulative clip lc = ∩ of the clip boxes of the
//              slice entries below and at them, written in place into
//              node_bbox[o] (a placeholder the later passes read), and the tile
//              records its link = the parent of its bottom slice entry.
// bbm_tc       TC(T) = ctx(link_T) = lc(link_T) ∩ TC(tile of link_T): a forest
//              over tiles resolved by pointer jumping (cooperative grid).  This
//              replaces the paper's exclusive scan of per-partition top boxes
//              (P:292).
// bbm_main     one CTA per tile, no waiting on other tiles:
//   B  per-thread walk over its 8 elements: the clip relative to the
//      thread's external ancestor X (the parent of the current outermost
//      in-thread group), in place in shared memory;
//   C  the context of each thread's link (X of its last outermost group) by
//      pointer jumping over the tile's threads;
//   D  pending elements: ctx(X) = rel(X) ∩ TL[thread of X] inside the tile,
//      lc(X) ∩ TC(tile of X) outside it (componentwise idempotent, so reading
//      a slot while its owner finalises it is harmless);
//   E  per-thread union walk (sequential stack algorithm) over the
//      thread's elements: in-thread nodes are finished, closes of outer nodes
//      record the thread's prefix union, opens left open record the union of
//      the thread's leaves after them;
//   F  window unions over threads (warp shuffles); for every slice entry the
//      union of the tile's leaves after it (su); the tile's union (a 32-ary
//      hierarchy over tile unions is built by bbm_hier afterwards);
//   G  closes of nodes opened in an earlier thread: suffix union of the open's
//      thread ∪ whole threads in between ∪ this thread's prefix (F4); closes
//      of nodes opened in an earlier tile: the tile prefix before the close,
//      listed for bbm_close;
//   H  coalesced copy-out.
// bbm_close    one CTA per tile (warps take 32 listed closes at a time): prefix ∪ su(open) ∪ the
//              whole tiles in between (hierarchy); blend opens receive it.
// bbm_final    blend opens never closed (R4): union of everything after them
//              (the open's tile suffix ∪ the hierarchy over all later tiles).
#include <algorithm>
#include <climits>
#include <cooperative_groups.h>
#include "boxes.cuh"
#include "common.cuh"
#include "kernels.h"

namespace tb {
namespace bbm {

constexpr int NT = 128;
constexpr int K = 8;
constexpr int TILE = NT * K;
constexpr int NW = NT / 32;
constexpr int LV = 5;    // 32-ary levels of the tile-union hierarchy (32^5 tiles > 2^31 / TILE)

struct Params {
  const uint8_t* tags;
  const float4* boxes;
  const int32_t* match;
  const int32_t* parent;
  float4* out;
  int64_t n;
  int ntiles;
  float4* u[LV];         // u[0][T] = union of tile T's clipped leaves; u[k] over 32^k tiles
  int32_t* link;         // [ntiles] parent of the tile's bottom slice entry (-1: root / none)
  float4* tc;            // [ntiles] ctx(link)
  float4* su;            // [n] union of the tile's clipped leaves after each slice entry
  int32_t* xc;           // [ntiles][TILE] closes of nodes opened in an earlier tile
  int32_t* xcnt;         // [ntiles] their count
  int32_t* never;        // [n] blend opens never closed (R4)
  uint32_t* nnever;      // their count
  uint64_t* trace;       // optional per-tile phase timestamps (debug)
};

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define BBM_TRACE(T, s)                                                          \
  do {                                                                           \
    if (p.trace && threadIdx.x == 0) p.trace[(size_t)(T) * 16 + (s)] = gtime();  \
  } while (0)

// tag byte classes of 8 elements: om = opens (clip or blend), bm = blend
// opens, cm = closes; everything else is a leaf (R2)
__device__ __forceinline__ void classify8(uint2 raw, uint32_t& om, uint32_t& cm, uint32_t& bm) {
  uint32_t o = 0, c = 0, b = 0;
  const uint32_t ws[2] = {raw.x, raw.y};
#pragma unroll
  for (int q = 0; q < 2; q++) {
    const uint32_t x = ws[q];
    const uint32_t bl = __vcmpeq4(x, 0x02020202u);
    o |= byte_mask4(__vcmpeq4(x, 0x01010101u) | bl) << (4 * q);
    c |= byte_mask4(__vcmpeq4(x, 0x03030303u)) << (4 * q);
    b |= byte_mask4(bl) << (4 * q);
  }
  om = o;
  cm = c;
  bm = b;
}

__device__ __forceinline__ uint2 load_tags8(const uint8_t* tags, int64_t n, int64_t tbase) {
  if (tbase + 8 <= n) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(tags + tbase));
    return r;
  }
  uint32_t wv[2] = {0, 0};
  for (int i = 0; i < 8; i++) {
    const int64_t g = tbase + i;
    const uint32_t v = g < n ? tags[g] : 0u;
    wv[i >> 2] |= v << (8 * (i & 3));
  }
  return make_uint2(wv[0], wv[1]);
}

// 8 consecutive int32 (16-byte aligned when full); -1 past the end
__device__ __forceinline__ void load_i8(const int32_t* a, int64_t n, int64_t tbase, int (&v)[K]) {
  if (tbase + 8 <= n) {
    const int4 x = __ldg(reinterpret_cast<const int4*>(a + tbase));
    const int4 y = __ldg(reinterpret_cast<const int4*>(a + tbase) + 1);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
  } else {
#pragma unroll
    for (int i = 0; i < K; i++) v[i] = (tbase + i < n) ? __ldg(a + tbase + i) : -1;
  }
}

// Union over tiles [a, b] by one warp (a, b warp-uniform; the hierarchy is
// complete): per level the lanes load the partial groups at both ends.
__device__ float4 range_union_tiles_warp(const Params& p, int a, int b) {
  const int lane = threadIdx.x & 31;
  float4 acc = bEMPTY();
  int k = 0;
  while (a <= b) {
    const float4* val = p.u[k];
    if ((a >> 5) == (b >> 5) || k == LV - 1) {
      for (int i = a + lane; i <= b; i += 32) acc = unite(acc, __ldcg(val + i));
      break;
    }
    if (a & 31) {
      const int e = a | 31;
      const int i = a + lane;
      if (i <= e) acc = unite(acc, __ldcg(val + i));
      a = e + 1;
    }
    if ((b & 31) != 31) {
      const int s0 = b & ~31;
      const int i = s0 + lane;
      if (i <= b) acc = unite(acc, __ldcg(val + i));
      b = s0 - 1;
    }
    if (a > b) break;
    a >>= 5;
    b = ((b + 1) >> 5) - 1;
    k++;
  }
  return warp_unite_all(acc);
}

// ----------------------------------------------------------------------------
// bbm_reduce: slice clips (lc) in place, tile links
// ----------------------------------------------------------------------------
// One warp per tile, 32 consecutive elements per lane, tags only: the lane's
// Bic from a 4-element table, warp scans give how many of the lane's unmatched
// opens survive to the tile end (the bottom ones of its stack, §3-§4
// P:96-138); only lanes owning survivors walk their elements.
constexpr int RK = TILE / 32;  // elements per lane in bbm_reduce
__global__ void __launch_bounds__(128) bbm_reduce(Params p) {
  __shared__ uint8_t bic4[256];  // Bic of 4 elements: index = open nibble | close nibble << 4; a | b << 4
  const int lane = threadIdx.x & 31;
  {
    const int t = threadIdx.x;
#pragma unroll
    for (int r = 0; r < 2; r++) {
      const int idx = t + 128 * r;
      Bic v{0, 0};
#pragma unroll
      for (int j = 0; j < 4; j++) v = bic_combine(v, Bic{(idx >> (4 + j)) & 1, (idx >> j) & 1});
      bic4[idx] = (uint8_t)(v.a | (v.b << 4));
    }
  }
  __syncthreads();
  const int T = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (T >= p.ntiles) return;
  const int64_t base = (int64_t)T * TILE, lbase = base + (int64_t)lane * RK;
  uint32_t om = 0, cm = 0, bmask = 0;  // opens, closes, blend opens of the lane's 32 elements
  if (lbase + RK <= p.n) {
    const uint4 t0 = __ldg(reinterpret_cast<const uint4*>(p.tags + lbase));
    const uint4 t1 = __ldg(reinterpret_cast<const uint4*>(p.tags + lbase) + 1);
    const uint32_t tw[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const uint32_t x = tw[q];
      const uint32_t bl = __vcmpeq4(x, 0x02020202u);
      om |= byte_mask4(__vcmpeq4(x, 0x01010101u) | bl) << (4 * q);
      cm |= byte_mask4(__vcmpeq4(x, 0x03030303u)) << (4 * q);
      bmask |= byte_mask4(bl) << (4 * q);
    }
  } else {
    for (int i = 0; i < RK; i++) {
      const int64_t g = lbase + i;
      if (g >= p.n) break;
      const uint8_t t = p.tags[g];
      if (t == 1 || t == 2) om |= 1u << i;
      if (t == 2) bmask |= 1u << i;
      if (t == 3) cm |= 1u << i;
    }
  }
  Bic lb{0, 0};
#pragma unroll
  for (int q = 0; q < 8; q++) {
    const uint32_t e = bic4[((om >> (4 * q)) & 15u) | (((cm >> (4 * q)) & 15u) << 4)];
    lb = bic_combine(lb, Bic{(int)(e & 15u), (int)(e >> 4)});
  }
  // exclusive suffix over lanes: Bic of the tile's elements after this lane
  Bic suf = lb;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const Bic o{__shfl_down_sync(0xffffffffu, suf.a, off), __shfl_down_sync(0xffffffffu, suf.b, off)};
    if (lane + off < 32) suf = bic_combine(suf, o);
  }
  Bic sx{__shfl_down_sync(0xffffffffu, suf.a, 1), __shfl_down_sync(0xffffffffu, suf.b, 1)};
  if (lane == 31) sx = Bic{0, 0};
  const int s_l = max(lb.b - sx.a, 0);  // survivors: the bottom s_l opens of the lane's stack
  uint32_t sm = 0;
  if (s_l > 0) {
    uint32_t S = 0;
#pragma unroll
    for (int i = 0; i < RK; i++) {
      const uint32_t bit = 1u << i;
      if (om & bit) S |= bit;
      else if ((cm & bit) && S) S ^= 1u << (31 - __clz(S));
    }
    for (int k = 0; k < s_l; k++) {
      const uint32_t low = S & (~S + 1u);
      sm |= low;
      S ^= low;
    }
  }
  // lane aggregate of the slice clips, exclusive ∩-scan over lanes
  float4 agg = bINF();
  for (uint32_t q = sm & ~bmask; q; q &= q - 1) agg = isect(agg, __ldg(p.boxes + lbase + __ffs(q) - 1));
  float4 x = agg;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float4 o = shfl_up_box(x, off);
    if (lane >= off) x = isect(x, o);
  }
  float4 acc = shfl_up_box(x, 1);
  if (lane == 0) acc = bINF();
  for (uint32_t q = sm; q; q &= q - 1) {
    const int i = __ffs(q) - 1;
    if (!((bmask >> i) & 1u)) acc = isect(acc, __ldg(p.boxes + lbase + i));
    p.out[lbase + i] = acc;
  }
  const int first = __reduce_min_sync(0xffffffffu, sm ? (lane * RK + __ffs(sm) - 1) : INT_MAX);
  if (lane == 0) p.link[T] = (first == INT_MAX) ? -1 : __ldg(p.parent + base + first);
}

// ----------------------------------------------------------------------------
// bbm_tc: TC(T) = ctx(link_T) by pointer jumping over tiles (cooperative)
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) bbm_tc(Params p, float4* acc2, int* ptr2, int* flag) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int nt = p.ntiles;
  const int gt = (int)(blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
  const int nthr = (int)(gridDim.x * (int64_t)blockDim.x);
  float4* acc[2] = {acc2, acc2 + nt};
  int* ptr[2] = {ptr2, ptr2 + nt};
  for (int V = gt; V < nt; V += nthr) {
    const int X = __ldg(p.link + V);
    acc[0][V] = X >= 0 ? __ldg(p.out + X) : bINF();  // lc(X), written by bbm_reduce
    ptr[0][V] = X >= 0 ? X / TILE : -1;
  }
  int cb = 0;
  for (int round = 0; round < 40; round++) {
    if (gt == 0) flag[round & 1] = 0;
    grid.sync();
    int any = 0;
    for (int V = gt; V < nt; V += nthr) {
      float4 a = __ldcg(acc[cb] + V);
      int q = __ldcg(ptr[cb] + V);
      if (q >= 0) {
        a = isect(a, __ldcg(acc[cb] + q));
        q = __ldcg(ptr[cb] + q);
        any |= q >= 0;
      }
      acc[cb ^ 1][V] = a;
      ptr[cb ^ 1][V] = q;
    }
    any = __syncthreads_or(any);
    if (any && threadIdx.x == 0) atomicOr(flag + (round & 1), 1);
    cb ^= 1;
    grid.sync();
    if (__ldcg(flag + (round & 1)) == 0) break;
  }
  for (int V = gt; V < nt; V += nthr) p.tc[V] = __ldcg(acc[cb] + V);
}

// ----------------------------------------------------------------------------
// bbm_main
// ----------------------------------------------------------------------------
struct Smem {
  float4 val[TILE];  // boxes -> clips -> outputs (swizzled slots)
  union {
    struct {         // C: pointer jumping over threads
      float4 acc[2][NT];
      int ptr[2][NT];
    } pj;
    float4 tl[NT];   // D: ctx of each thread's link
    struct {         // F-G
      float4 win[5][NT];  // union of thread unions over lanes [lane - 2^k + 1, lane] (clipped to the warp)
      float4 suf[NT];     // inclusive suffix within the warp
    } un;
  } u;
  float4 wtu[NW];
  float4 wmid[NW][NW];  // union of the warps strictly between two warps
  uint32_t bmk[NT];  // blend opens of each thread
  uint32_t lmk[NT];  // leaves of each thread
  int nx;            // closes of earlier tiles' nodes listed for bbm_close
};

// element i of thread t lives at slot 8t + (i ^ (t & 7)): conflict-free both for
// the coalesced copies and for the per-thread accesses
__device__ __forceinline__ int slot(int t, int i) { return (t << 3) | (i ^ (t & 7)); }
__device__ __forceinline__ int slot_of(int e) { return slot(e >> 3, e & 7); }

// union of the clipped leaves of whole threads [a, b]: the suffix of a's warp,
// the warps strictly between (table), the window part of b's warp ending at
// b — selects rather than branches, since every lane asks a different range
__device__ __forceinline__ float4 range_union_threads(const Smem& s, int a, int b) {
  if (a > b) return bEMPTY();
  const int wa = a >> 5, wb = b >> 5;
  const int a2 = (wa == wb) ? a : (wb << 5);  // start of the part inside b's warp
  const int len = b - a2 + 1;
  const int k = min(31 - __clz(len), 4);
  const float4 right = (len == 32) ? s.wtu[wb] : unite(s.u.un.win[k][b], s.u.un.win[k][a2 + (1 << k) - 1]);
  if (wa == wb) return right;
  return unite(unite(s.u.un.suf[a], right), s.wmid[wa][wb]);
}

__global__ void __launch_bounds__(NT, 6) bbm_main(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockIdx.x;
  const int64_t base = (int64_t)T * TILE;
  const int64_t tstart = base + (int64_t)tid * K;
  const int64_t tend = base + TILE;
  const int nvalid = (int)(p.n - base < TILE ? p.n - base : TILE);
  BBM_TRACE(T, 0);

  // ---- A. load -------------------------------------------------------------
  uint32_t om, cm, bm;
  classify8(load_tags8(p.tags, p.n, tstart), om, cm, bm);
  uint32_t lm = ~om & ~cm & 0xffu;
  {
    const int64_t rem = p.n - tstart;
    if (rem < K) lm &= rem <= 0 ? 0u : ((1u << rem) - 1u);
  }
  int mt[K], pr[K];
  load_i8(p.match, p.n, tstart, mt);
  load_i8(p.parent, p.n, tstart, pr);
  // contexts of out-of-tile parents (lc in node_bbox ∩ TC of their tile):
  // the last two distinct ones are fetched now, used in C/D
  int xa = -1, xb = -1;
#pragma unroll
  for (int i = 0; i < K; i++) {
    if ((((om | lm) >> i) & 1u) && pr[i] >= 0 && pr[i] < base && pr[i] != xa) {
      xb = xa;
      xa = pr[i];
    }
  }
  float4 ga = bINF(), gb = bINF();
  if (xa >= 0) ga = isect(__ldcg(p.out + xa), __ldg(p.tc + xa / TILE));
  if (xb >= 0) gb = isect(__ldcg(p.out + xb), __ldg(p.tc + xb / TILE));
  // boxes into the slots, coalesced (512 contiguous bytes per warp instruction)
#pragma unroll
  for (int j = 0; j < K; j++) {
    const int e = j * NT + tid;
    s.val[slot_of(e)] = e < nvalid ? __ldg(p.boxes + base + e) : bINF();
  }
  s.bmk[tid] = bm;
  s.lmk[tid] = lm;
  if (tid == 0) s.nx = 0;
  uint32_t thr_un = 0;  // opens closed beyond this thread (or never)
#pragma unroll
  for (int i = 0; i < K; i++)
    if (((om >> i) & 1u) && (mt[i] < 0 || mt[i] >= tstart + K)) thr_un |= 1u << i;
  __syncthreads();

  // ---- B. clips relative to the thread's external ancestor -------------------
  int curX = -1;
  uint32_t pend = 0;
#pragma unroll
  for (int i = 0; i < K; i++) {
    if (((om | lm) >> i) & 1u) {
      const int par = pr[i];
      float4 b = bINF();
      if (par < tstart) {
        curX = par;
      } else {
        b = s.val[slot(tid, par - (int)tstart)];
      }
      float4& me = s.val[slot(tid, i)];
      me = ((bm >> i) & 1u) ? b : isect(me, b);
      if (curX >= 0) pend |= 1u << i;
    }
  }
  __syncthreads();
  BBM_TRACE(T, 1);

  // ---- C. ctx of each thread's link (pointer jumping over threads) ------------
  {
    float4 acc = bINF();
    int ptr = -1;
    if (thr_un && curX >= 0) {
      if (curX < base) {
        acc = curX == xa ? ga : (curX == xb ? gb : isect(__ldcg(p.out + curX), __ldg(p.tc + curX / TILE)));
      } else {
        const int x = curX - (int)base;
        acc = s.val[slot_of(x)];
        ptr = x / K;
      }
    }
    int cb = 0;
    s.u.pj.acc[0][tid] = acc;
    s.u.pj.ptr[0][tid] = ptr;
    int any = __syncthreads_or(ptr >= 0);
    while (any) {
      if (ptr >= 0) {
        acc = isect(acc, s.u.pj.acc[cb][ptr]);
        ptr = s.u.pj.ptr[cb][ptr];
      }
      s.u.pj.acc[cb ^ 1][tid] = acc;
      s.u.pj.ptr[cb ^ 1][tid] = ptr;
      cb ^= 1;
      any = __syncthreads_or(ptr >= 0);
    }
    s.u.tl[tid] = acc;  // every read of pj happened before the last barrier
  }
  __syncthreads();
  BBM_TRACE(T, 2);

  // ---- D. finish pending clips: rel ∩ ctx(X) ------------------------------------
  if (pend) {
    int X = -1, cx = INT_MIN;
    float4 g = bINF();
#pragma unroll
    for (int i = 0; i < K; i++) {
      if (((om | lm) >> i) & 1u) {
        if (pr[i] < tstart) X = pr[i];
        if ((pend >> i) & 1u) {
          if (X != cx) {
            cx = X;
            if (X < base) {
              g = X == xa ? ga : (X == xb ? gb : isect(__ldcg(p.out + X), __ldg(p.tc + X / TILE)));
            } else {
              const int x = X - (int)base;
              g = isect(s.val[slot_of(x)], s.u.tl[x / K]);
            }
          }
          float4& me = s.val[slot(tid, i)];
          me = isect(me, g);
        }
      }
    }
  }
  __syncthreads();
  BBM_TRACE(T, 3);

  // ---- E. unions inside the thread ---------------------------------------------------
  // A node opened and closed in this thread gets the union of the leaves between
  // (the slots hold final clips now); a close of an outer node records the
  // thread's prefix union (completed in G).
  float4 PT = bEMPTY();  // union of this thread's clipped leaves so far
  uint32_t ecm = 0;
#pragma unroll
  for (int i = 0; i < K; i++) {
    const uint32_t bit = 1u << i;
    if (lm & bit) {
      PT = unite(PT, s.val[slot(tid, i)]);
    } else if (cm & bit) {
      const int m = mt[i];
      if (m >= tstart) {
        const int o = m - (int)tstart;
        float4 U = bEMPTY();
        uint32_t lb = lm & (bit - 1u) & ~((2u << o) - 1u);  // leaves strictly between
        while (lb) {
          const int j = __ffs(lb) - 1;
          lb &= lb - 1;
          U = unite(U, s.val[slot(tid, j)]);
        }
        s.val[slot(tid, i)] = U;
        if ((bm >> o) & 1u) s.val[slot(tid, o)] = U;
      } else if (m >= 0) {
        s.val[slot(tid, i)] = PT;  // completed by the open's thread (F) or in G
        if (m < base) ecm |= bit;
      } else {
        s.val[slot(tid, i)] = bEMPTY();  // R3
      }
    }
  }
  BBM_TRACE(T, 4);

  // ---- F. unions over threads; slice suffix unions; tile union ----------------------
  {
    float4 w = PT, suf = PT;
    s.u.un.win[0][tid] = w;
#pragma unroll
    for (int k = 1; k <= 5; k++) {
      const int off = 1 << (k - 1);
      const float4 a = shfl_up_box(w, off);
      if (lane >= off) w = unite(w, a);
      if (k < 5) s.u.un.win[k][tid] = w;
      const float4 b = make_float4(__shfl_down_sync(0xffffffffu, suf.x, off),
                                   __shfl_down_sync(0xffffffffu, suf.y, off),
                                   __shfl_down_sync(0xffffffffu, suf.z, off),
                                   __shfl_down_sync(0xffffffffu, suf.w, off));
      if (lane + off < 32) suf = unite(suf, b);
    }
    s.u.un.suf[tid] = suf;
    if (lane == 31) s.wtu[warp] = w;
  }
  __syncthreads();
  BBM_TRACE(T, 8);
  if (tid < NW * NW) {
    const int x = tid / NW, y = tid % NW;
    float4 m = bEMPTY();
    for (int w = x + 1; w < y; w++) m = unite(m, s.wtu[w]);
    s.wmid[x][y] = m;
  }
  __syncthreads();
  BBM_TRACE(T, 9);
  {
    // Opens left open at this thread's end, from the top down with R = union of
    // this thread's leaves after them: a slice entry publishes su = R ∪ the
    // threads after this one; an open closed by a later thread of the tile
    // finishes that close: R ∪ the threads in between ∪ the closer's prefix.
    uint32_t qt = 0, qi = 0, nvm = 0;
#pragma unroll
    for (int i = 0; i < K; i++) {
      if ((thr_un >> i) & 1u) {
        if (mt[i] < 0 || mt[i] >= tend) qt |= 1u << i;
        else qi |= 1u << i;
      }
      if (((bm >> i) & 1u) && mt[i] < 0) nvm |= 1u << i;
    }
    if (qt | qi) {
      const float4 after = qt ? range_union_threads(s, tid + 1, NT - 1) : bEMPTY();
      float4 R = bEMPTY();
#pragma unroll
      for (int i = K - 1; i >= 0; i--) {
        const uint32_t bit = 1u << i;
        if (qt & bit) {
          p.su[tstart + i] = unite(R, after);
          if (nvm & bit) p.never[atomicAdd(p.nnever, 1u)] = (int)(tstart + i);
        } else if (qi & bit) {
          const int c = mt[i] - (int)base;
          float4& cv = s.val[slot_of(c)];
          const float4 U = unite(unite(R, range_union_threads(s, tid + 1, c / K - 1)), cv);
          cv = U;
          if ((bm >> i) & 1u) s.val[slot(tid, i)] = U;
        }
        if ((lm & bit) && ((qt | qi) & (bit - 1u))) R = unite(R, s.val[slot(tid, i)]);
      }
    }
  }
  BBM_TRACE(T, 10);
  if (tid == 0) {
    float4 tu = s.wtu[0];
#pragma unroll
    for (int w = 1; w < NW; w++) tu = unite(tu, s.wtu[w]);
    p.u[0][T] = tu;
  }
  BBM_TRACE(T, 5);

  // ---- G. closes of nodes opened in an earlier thread (finished here) or an
  //      earlier tile (the tile's prefix before the close stored, the close
  //      listed for bbm_close) --------------------------------------------------------
  if (ecm) {
    const float4 pre = range_union_threads(s, 0, tid - 1);
    uint32_t q = ecm;
#pragma unroll 1
    while (q) {
      const int i = __ffs(q) - 1;
      q &= q - 1;
      float4& me = s.val[slot(tid, i)];
      me = unite(me, pre);
      p.xc[(int64_t)T * TILE + atomicAdd(&s.nx, 1)] = (int)(tstart + i);
    }
  }
  __syncthreads();
  if (tid == 0) p.xcnt[T] = s.nx;
  BBM_TRACE(T, 6);

  // ---- H. copy-out.  A slice blend open is stored with its true context: later
  //      tiles read ctx = node_bbox[o] ∩ TC(tile of o), the same whether they see
  //      lc (bbm_reduce) or the context (∩ is idempotent per component); its
  //      union replaces it in bbm_close / bbm_final. ------------------------------------
#pragma unroll
  for (int j = 0; j < K; j++) {
    const int e = j * NT + tid;
    if (e < nvalid) __stcs(p.out + base + e, s.val[slot_of(e)]);
  }
  BBM_TRACE(T, 7);
}

// ----------------------------------------------------------------------------
// bbm_hier: level k of the 32-ary hierarchy of tile unions from level k - 1
// (one warp per group; launched once per level)
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) bbm_hier(Params p, int k, int m /* nodes at level k - 1 */) {
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x * 8 + (threadIdx.x >> 5);
  if ((g << 5) >= m) return;
  const int c = (g << 5) + lane;
  float4 v = c < m ? __ldcg(p.u[k - 1] + c) : bEMPTY();
  v = warp_unite_all(v);
  if (lane == 0) p.u[k][g] = v;
}

// ----------------------------------------------------------------------------
// bbm_close: closes of nodes opened in an earlier tile (one CTA per tile):
// union = prefix of the close's tile (stored by bbm_main) ∪ the open's tile
// suffix after it ∪ the whole tiles in between (F4); blend opens get it too.
// Lanes sharing the open's tile share one warp-cooperative range union.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(128) bbm_close(Params p) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int T = blockIdx.x;
  const int cnt = __ldg(p.xcnt + T);
  int cto = -1;  // warp cache: the last range resolved (deep chains repeat one open tile)
  float4 cR = bEMPTY();
  for (int j0 = warp * 32; j0 < cnt; j0 += 128) {
    const int j = j0 + lane;
    const bool valid = j < cnt;
    int c = 0, o = 0, To = 0;
    float4 P = bEMPTY(), su = bEMPTY();
    uint8_t kind = 0;
    if (valid) {
      c = __ldg(p.xc + (int64_t)T * TILE + j);
      o = __ldg(p.match + c);
      To = o / TILE;
      P = __ldcg(p.out + c);
      su = __ldcg(p.su + o);
      kind = __ldg(p.tags + o);
    }
    float4 R = bEMPTY();
    bool pending = valid && To < T - 1;
    if (pending && To == cto) {
      R = cR;
      pending = false;
    }
    uint32_t mask;
    while ((mask = __ballot_sync(0xffffffffu, pending)) != 0u) {
      const int tl = __shfl_sync(0xffffffffu, To, __ffs(mask) - 1);
      const float4 Rl = range_union_tiles_warp(p, tl + 1, T - 1);
      if (pending && To == tl) {
        R = Rl;
        pending = false;
      }
      cto = tl;
      cR = Rl;
    }
    if (valid) {
      const float4 U = unite(unite(P, su), R);
      p.out[c] = U;
      if (kind == 2) p.out[o] = U;  // blend open
    }
  }
}

// ----------------------------------------------------------------------------
// blend opens never closed (R4)
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) bbm_final(Params p) {
  // one warp per open: its tile's suffix after it ∪ every later tile
  const uint32_t cnt = __ldcg(p.nnever);
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * 8;
  for (uint32_t q = blockIdx.x * 8 + (threadIdx.x >> 5); q < cnt; q += nwarps) {
    const int o = __ldcg(p.never + q);
    const int To = o / TILE;
    const float4 after = To + 1 < p.ntiles ? range_union_tiles_warp(p, To + 1, p.ntiles - 1) : bEMPTY();
    if (lane == 0) p.out[o] = unite(__ldcg(p.su + o), after);
  }
}

// ----------------------------------------------------------------------------
// workspace
// ----------------------------------------------------------------------------
struct Layout {
  int64_t ntiles;
  size_t zero_off, zero_bytes;
  size_t off_nnever;
  size_t off_u[LV], off_link, off_tc, off_su, off_xc, off_xcnt, off_never, off_tcacc, off_tcptr, off_tcflag, bytes;
  explicit Layout(int64_t n) {
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    ntiles = (n + TILE - 1) / TILE;
    size_t o = 0;
    zero_off = o;
    off_nnever = o; o = al(o + 4);
    zero_bytes = o - zero_off;
    int64_t m = ntiles;
    for (int k = 0; k < LV; k++) {
      off_u[k] = o; o = al(o + 16 * (size_t)m);
      m = (m + 31) / 32;
    }
    off_link = o; o = al(o + 4 * (size_t)ntiles);
    off_tc = o; o = al(o + 16 * (size_t)ntiles);
    off_xcnt = o; o = al(o + 4 * (size_t)ntiles);
    off_tcacc = o; o = al(o + 32 * (size_t)ntiles);
    off_tcptr = o; o = al(o + 8 * (size_t)ntiles);
    off_tcflag = o; o = al(o + 16);
    off_su = o; o = al(o + 16 * (size_t)n);
    off_xc = o; o = al(o + 4 * (size_t)ntiles * TILE);
    off_never = o; o = al(o + 4 * (size_t)n);
    bytes = o;
  }
};

void main_setup() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(bbm_main, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    done = true;
  }
}

int tc_blocks() {
  static int nb = 0;
  if (nb == 0) {
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bbm_tc, 256, 0);
    nb = sms * std::max(occ, 1);
  }
  return nb;
}

}  // namespace bbm

size_t bbm_workspace_bytes(int64_t n) {
  if (n <= 0) return 0;
  return bbm::Layout(n).bytes;
}

int bbm_tile_elems() { return bbm::TILE; }

cudaError_t bbm_launch(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                       int64_t n, float* node_bbox, void* ws, cudaStream_t stream, uint64_t* trace) {
  if (n <= 0) return cudaSuccess;
  bbm::Layout L(n);
  char* b = (char*)ws;
  bbm::Params p;
  p.tags = tags;
  p.boxes = reinterpret_cast<const float4*>(leaf_bbox);
  p.match = match;
  p.parent = parent;
  p.out = reinterpret_cast<float4*>(node_bbox);
  p.n = n;
  p.ntiles = (int)L.ntiles;
  p.nnever = (uint32_t*)(b + L.off_nnever);
  for (int k = 0; k < bbm::LV; k++) {
    p.u[k] = (float4*)(b + L.off_u[k]);
  }
  p.link = (int32_t*)(b + L.off_link);
  p.tc = (float4*)(b + L.off_tc);
  p.su = (float4*)(b + L.off_su);
  p.never = (int32_t*)(b + L.off_never);
  p.xc = (int32_t*)(b + L.off_xc);
  p.xcnt = (int32_t*)(b + L.off_xcnt);
  p.trace = trace;
  cudaError_t err = cudaMemsetAsync(b + L.zero_off, 0, L.zero_bytes, stream);
  if (err != cudaSuccess) return err;
  TB_LAUNCH(stream, "bbm_reduce", (bbm::bbm_reduce<<<(unsigned)((L.ntiles + 3) / 4), 128, 0, stream>>>(p)));
  {
    float4* acc2 = (float4*)(b + L.off_tcacc);
    int* ptr2 = (int*)(b + L.off_tcptr);
    int* flag = (int*)(b + L.off_tcflag);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((L.ntiles + 255) / 256, bbm::tc_blocks()));
    void* args[] = {(void*)&p, (void*)&acc2, (void*)&ptr2, (void*)&flag};
    void* tok;
    prof_begin(stream, "bbm_tc", &tok);
    err = cudaLaunchCooperativeKernel((const void*)bbm::bbm_tc, dim3(blocks), dim3(256), args, 0, stream);
    prof_end(stream, tok);
    if (err != cudaSuccess) return err;
  }
  bbm::main_setup();
  TB_LAUNCH(stream, "bbm_main",
            (bbm::bbm_main<<<(unsigned)L.ntiles, bbm::NT, sizeof(bbm::Smem), stream>>>(p)));
  {
    int64_t m = L.ntiles;
    for (int k = 1; k < bbm::LV && m > 1; k++) {
      const int64_t groups = (m + 31) / 32;
      TB_LAUNCH(stream, "bbm_hier",
                (bbm::bbm_hier<<<(unsigned)((groups + 7) / 8), 256, 0, stream>>>(p, k, (int)m)));
      m = groups;
    }
  }
  TB_LAUNCH(stream, "bbm_close", (bbm::bbm_close<<<(unsigned)L.ntiles, 128, 0, stream>>>(p)));
  TB_LAUNCH(stream, "bbm_final", (bbm::bbm_final<<<148, 256, 0, stream>>>(p)));
  return cudaGetLastError();
}

}  // namespace tb
