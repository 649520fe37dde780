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
static const int kMinus1 = -1;
namespace bbm {

#ifndef BBM_K
#define BBM_K 8
#endif
constexpr int K = BBM_K;           // elements per thread of bbm_main
constexpr int NT = 1024 / K;       // its threads per tile
#ifndef BBM_MINB
#define BBM_MINB (BBM_K == 16 ? 9 : 6)
#endif
constexpr int MINB = BBM_MINB;     // resident CTAs per SM (shared memory / registers)
constexpr int TILE = NT * K;
static_assert(TILE == 1024 && (K == 8 || K == 16), "bbm tiles are 1024 elements");
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
  int t0, t1;            // tiles of this launch: [t0, t1) (chunked pipeline; else [0, ntiles))
  float4* u[LV];         // u[0][T] = union of tile T's clipped leaves; u[k] over 32^k tiles
  int32_t* link;         // [ntiles] the tile's bottom slice entry (tile-local, -1: none); its parent is the link
  float4* tc;            // [ntiles] ctx(link)
  float4* su;            // [n] union of the tile's clipped leaves after each slice entry
  int32_t* xc;           // [ntiles][TILE] closes of nodes opened in an earlier tile
  int32_t* xcnt;         // [ntiles] their count
  int32_t* never;        // [n] blend opens never closed (R4)
  uint32_t* nnever;      // their count
  uint64_t* trace;       // optional per-tile phase timestamps (debug)
  // shard mode; zero / null for one device.  match / parent hold
  // GLOBAL indices; arrays are indexed locally (global - off).
  int64_t off;             // global index of element 0
  const int32_t* ext_idx;  // [n_ext] open entries of earlier chunks, ascending
  const float4* ext_ctx;   // their true contexts
  int n_ext;
  ShardPop* pops;          // closes of nodes opened in an earlier chunk (for the exchange)
  uint32_t* npops;
  int fs_list;             // shard phase 1: bbm_reduce lists the chunk's final-stack opens per tile in xc / xcnt
};

// True context of an open X of an earlier chunk (binary search in the
// imported table; INF when there is none, i.e. the chunk-local frame).  Not
// inlined: only shard mode takes it, for elements whose parent lies in an
// earlier chunk.
__device__ __noinline__ float4 ext_lookup(const int32_t* idx, const float4* ctx, int cnt, int X) {
  int lo = 0, hi = cnt;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(idx + mid) < X) lo = mid + 1;
    else hi = mid;
  }
  return (lo < cnt && __ldg(idx + lo) == X) ? __ldg(ctx + lo) : bINF();
}
__device__ __forceinline__ float4 ext_ctx(const Params& p, int X) {
  return ext_lookup(p.ext_idx, p.ext_ctx, p.n_ext, X);
}

// node_bbox[X] of a slice entry X is read by later tiles while X's own tile may
// be storing X's true context over lc(X) (F6): both values give the same
// result, and the accesses are relaxed (morally strong) so they do not race.
__device__ __forceinline__ float4 ld_relaxed_box(const float4* p) {
  float4 v;
  asm volatile("ld.relaxed.gpu.global.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_box(float4* p, float4 v) {
  asm volatile("st.relaxed.gpu.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// Context of an open X outside the current tile: node_bbox[X] holds lc(X) or
// its true context (F6), completed by TC of X's tile; earlier chunks: imported.
template <bool SHARD>
__device__ __forceinline__ float4 outer_ctx(const Params& p, int X) {
  if (SHARD && X < p.off) return ext_ctx(p, X);
  const int64_t x = SHARD ? X - p.off : X;
  return isect(ld_relaxed_box(p.out + x), __ldg(p.tc + x / TILE));
}

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define BBM_TRACE(T, s)                                                          \
  do {                                                                           \
    if (p.trace && threadIdx.x == 0) p.trace[(size_t)(T) * 16 + (s)] = gtime();  \
  } while (0)

// tag byte classes of K elements (K / 4 words): om = opens (clip or blend),
// bm = blend opens, cm = closes; everything else is a leaf (R2)
__device__ __forceinline__ void classifyK(const uint32_t (&ws)[K / 4], uint32_t& om, uint32_t& cm, uint32_t& bm) {
  static_assert(K == 8 || K == 16, "classifyK");
  const uint4 w = K == 16 ? make_uint4(ws[0], ws[1], ws[2 % (K / 4)], ws[3 % (K / 4)]) : make_uint4(ws[0], ws[1], 0u, 0u);
  classify16b(w, om, cm, bm);
}

__device__ __forceinline__ void load_tagsK(const uint8_t* tags, int64_t n, int64_t tbase, uint32_t (&wv)[K / 4]) {
  if (tbase + K <= n) {
    if constexpr (K == 16) {
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(wv[0]), "=r"(wv[1]), "=r"(wv[2]), "=r"(wv[3])
                   : "l"(tags + tbase));
    } else {
      asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(wv[0]), "=r"(wv[1]) : "l"(tags + tbase));
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < K / 4; q++) wv[q] = 0;
  for (int i = 0; i < K; i++) {
    const int64_t g = tbase + i;
    const uint32_t v = g < n ? tags[g] : 0u;
    wv[i >> 2] |= v << (8 * (i & 3));
  }
}

// K consecutive int32 (16-byte aligned when full); -1 past the end
__device__ __forceinline__ void load_iK(const int32_t* a, int64_t n, int64_t tbase, int (&v)[K]) {
  if (tbase + K <= n) {
#pragma unroll
    for (int q = 0; q < K / 4; q++) {
      const int4 x = __ldg(reinterpret_cast<const int4*>(a + tbase) + q);
      v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
    }
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
  const int T = p.t0 + blockIdx.x * 4 + (threadIdx.x >> 5);
  if (T >= p.t1) return;
  const int64_t base = (int64_t)T * TILE, lbase = base + (int64_t)lane * RK;
  uint32_t om = 0, cm = 0, bmask = 0;  // opens, closes, blend opens of the lane's 32 elements
  if (lbase + RK <= p.n) {
    const uint4 t0 = __ldg(reinterpret_cast<const uint4*>(p.tags + lbase));
    const uint4 t1 = __ldg(reinterpret_cast<const uint4*>(p.tags + lbase) + 1);
    uint32_t o1, c1, b1;
    classify16b(t0, om, cm, bmask);
    classify16b(t1, o1, c1, b1);
    om |= o1 << 16;
    cm |= c1 << 16;
    bmask |= b1 << 16;
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
  if (p.fs_list) {
    // shard phase 1: the survivors closed after the chunk or never are the
    // tile's part of the chunk's final stack (ascending; xc / xcnt are free
    // until phase 2)
    uint32_t fm = 0;
    for (uint32_t q = sm; q; q &= q - 1) {
      const int i = __ffs(q) - 1;
      const int mm = __ldg(p.match + lbase + i);
      if (mm < 0 || mm >= p.off + p.n) fm |= 1u << i;
    }
    const int c = __popc(fm);
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    int pos = x - c;
    for (uint32_t q = fm; q; q &= q - 1) p.xc[base + pos++] = lane * RK + __ffs(q) - 1;
    if (lane == 31) p.xcnt[T] = x;
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
  if (lane == 0) p.link[T] = (first == INT_MAX) ? -1 : first;  // bbm_tc takes its parent (tags + boxes only here)
}

// ----------------------------------------------------------------------------
// bbm_tc: TC(T) = ctx(link_T) by pointer jumping over tiles (cooperative)
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) bbm_tc(Params p, float4* acc2, int* ptr2, int* flag) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  // tiles [t0, t1); TC of every tile before t0 is final (earlier launches of
  // the chunked pipeline), so chains stop there
  const int nt = p.ntiles, t0 = p.t0, t1 = p.t1;
  const int gt = (int)(blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
  const int nthr = (int)(gridDim.x * (int64_t)blockDim.x);
  // the two buffers by selects (a runtime index into a pointer array would place it in local memory)
  auto acc = [&](int b) { return b ? acc2 + nt : acc2; };
  auto ptr = [&](int b) { return b ? ptr2 + nt : ptr2; };
  for (int V = t0 + gt; V < t1; V += nthr) {
    const int f = __ldg(p.link + V);  // the tile's first slice entry (local), -1: none
    const int X = f >= 0 ? __ldg(p.parent + (int64_t)V * TILE + f) : -1;  // its parent: global index
    // lc(X), written by bbm_reduce (or X's context: F6); an open of an earlier
    // chunk: imported context
    float4 a = bINF();
    int q = -1;
    if (X >= p.off) {
      a = ld_relaxed_box(p.out + (X - p.off));
      q = (int)((X - p.off) / TILE);
      if (q < t0) {
        a = isect(a, __ldcg(p.tc + q));
        q = -1;
      }
    } else if (X >= 0) {
      a = ext_ctx(p, X);
    }
    acc(0)[V] = a;
    ptr(0)[V] = q;
  }
  int cb = 0;
  for (int round = 0; round < 40; round++) {
    if (gt == 0) flag[round & 1] = 0;
    grid.sync();
    int any = 0;
    for (int V = t0 + gt; V < t1; V += nthr) {
      float4 a = __ldcg(acc(cb) + V);
      int q = __ldcg(ptr(cb) + V);
      if (q >= 0) {
        a = isect(a, __ldcg(acc(cb) + q));
        q = __ldcg(ptr(cb) + q);
        any |= q >= 0;
      }
      acc(cb ^ 1)[V] = a;
      ptr(cb ^ 1)[V] = q;
    }
    any = __syncthreads_or(any);
    if (any && threadIdx.x == 0) atomicOr(flag + (round & 1), 1);
    cb ^= 1;
    grid.sync();
    if (__ldcg(flag + (round & 1)) == 0) break;
  }
  for (int V = t0 + gt; V < t1; V += nthr) p.tc[V] = __ldcg(acc(cb) + V);
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
  int nx;            // closes of earlier tiles' nodes listed for bbm_close
};

// element i of thread t lives at slot Kt + (i ^ (t & 7)): conflict-free both for
// the coalesced copies (8 consecutive elements of one thread per 128-byte
// wavefront) and for the per-thread accesses (8 threads, distinct slot & 7)
// (bit form: K is a power of two >= 8 and indices are non-negative, so
// slot(t, i) = (t*K | t & 7) ^ i and slot_of(e) = e ^ ((e / K) & 7) — no
// signed-division fixups, one LOP3 per access once t's part is hoisted)
constexpr int LOGK = K == 8 ? 3 : 4;
__device__ __forceinline__ int slot(int t, int i) { return ((t << LOGK) | (t & 7)) ^ i; }
__device__ __forceinline__ int slot_of(int e) { return e ^ (int)(((unsigned)e >> LOGK) & 7u); }
__device__ __forceinline__ int thr_of(int e) { return (int)((unsigned)e >> LOGK); }

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

template <bool SHARD>
__global__ void __launch_bounds__(NT, MINB) bbm_main(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = p.t0 + blockIdx.x;
  const int64_t base = (int64_t)T * TILE;  // local indices (arrays)
  const int64_t tstart = base + (int64_t)tid * K;
  const int nvalid = (int)(p.n - base < TILE ? p.n - base : TILE);
  // global indices (compared with match / parent values)
  // (the last tile of a shard chunk ends at the chunk end: a partner beyond it
  // is in the next chunk, not in this tile or thread)
  // (32-bit: global indices fit in int32, n <= 2^31 - 1; the ends are clamped
  // to the chunk end, a no-op on one device)
  const int64_t gend = p.off + p.n;
  const int gbase = (int)(p.off + base), gtstart = (int)(p.off + tstart);
  const int gtend = (int)min((int64_t)gbase + TILE, gend);
  const int gthr_end = (int)min((int64_t)gtstart + K, gend);
  BBM_TRACE(T, 0);

  // ---- A. load -------------------------------------------------------------
  uint32_t om, cm, bm;
  {
    uint32_t tw[K / 4];
    load_tagsK(p.tags, p.n, tstart, tw);
    classifyK(tw, om, cm, bm);
  }
  uint32_t lm = ~om & ~cm & ((1u << K) - 1u);
  {
    const int64_t rem = p.n - tstart;
    if (rem < K) lm &= rem <= 0 ? 0u : ((1u << rem) - 1u);
  }
  int mt[K], pr[K];
  load_iK(p.match, p.n, tstart, mt);
  load_iK(p.parent, p.n, tstart, pr);
  // contexts of out-of-tile parents (lc in node_bbox ∩ TC of their tile):
  // the last two distinct ones are fetched now, used in C/D
  int xa = -1, xb = -1;
#pragma unroll
  for (int i = 0; i < K; i++) {
    if ((((om | lm) >> i) & 1u) && pr[i] >= 0 && pr[i] < gbase && pr[i] != xa) {
      xb = xa;
      xa = pr[i];
    }
  }
  float4 ga = bINF(), gb = bINF();
  if (xa >= 0) ga = outer_ctx<SHARD>(p, xa);
  if (xb >= 0) gb = outer_ctx<SHARD>(p, xb);
  // boxes into the slots, coalesced (512 contiguous bytes per warp instruction)
#pragma unroll
  for (int j = 0; j < K; j++) {
    const int e = j * NT + tid;
    s.val[slot_of(e)] = e < nvalid ? __ldg(p.boxes + base + e) : bINF();
  }
  if (tid == 0) s.nx = 0;
  uint32_t thr_un = 0;  // opens closed beyond this thread (or never)
#pragma unroll
  for (int i = 0; i < K; i++)
    if (((om >> i) & 1u) && (mt[i] < 0 || mt[i] >= gthr_end)) thr_un |= 1u << i;
  __syncthreads();

  // ---- B. clips relative to the thread's external ancestor -------------------
  int curX = -1;
  uint32_t pend = 0;
#pragma unroll
  for (int i = 0; i < K; i++) {
    if (((om | lm) >> i) & 1u) {
      const int par = pr[i];
      float4 b = bINF();
      if (par < gtstart) {
        curX = par;
      } else {
        b = s.val[slot(tid, (int)(par - gtstart))];
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
      if (curX < gbase) {
        acc = curX == xa ? ga : (curX == xb ? gb : outer_ctx<SHARD>(p, curX));
      } else {
        const int x = (int)(curX - gbase);
        acc = s.val[slot_of(x)];
        ptr = thr_of(x);
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

  // ---- D. finish pending clips: rel ∩ ctx(X).  Other threads read only this
  //      thread's thread-unmatched opens (as their contexts); those all belong
  //      to the thread's last external group (context tl[tid]) and are
  //      finished after the barrier, so no slot is read while it is written.
  const uint32_t pend_now = pend & ~thr_un;
  if (pend_now) {
    int X = -1, cx = INT_MIN;
    float4 g = bINF();
#pragma unroll
    for (int i = 0; i < K; i++) {
      if (((om | lm) >> i) & 1u) {
        if (pr[i] < gtstart) X = pr[i];
        if ((pend_now >> i) & 1u) {
          if (X != cx) {
            cx = X;
            if (X < gbase) {
              g = X == xa ? ga : (X == xb ? gb : outer_ctx<SHARD>(p, X));
            } else {
              const int x = (int)(X - gbase);
              g = isect(s.val[slot_of(x)], s.u.tl[thr_of(x)]);
            }
          }
          float4& me = s.val[slot(tid, i)];
          me = isect(me, g);
        }
      }
    }
  }
  __syncthreads();
  if (pend & thr_un) {
    const float4 g = s.u.tl[tid];
    uint32_t q = pend & thr_un;
#pragma unroll 1
    while (q) {
      const int i = __ffs(q) - 1;
      q &= q - 1;
      float4& me = s.val[slot(tid, i)];
      me = isect(me, g);
    }
  }
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
    {  // leaves: a select, not a branch (every lane reads its slot)
      const float4 u = unite(PT, s.val[slot(tid, i)]);
      PT = (lm & bit) ? u : PT;
    }
    if (cm & bit) {
      const int m = mt[i];
      float4 st = m >= 0 ? PT : bEMPTY();  // outer node: completed in F or G; R3: EMPTY
      if (m >= gtstart) {
        const int o = (int)(m - gtstart);
        float4 U = bEMPTY();
        uint32_t lb = lm & (bit - 1u) & ~((2u << o) - 1u);  // leaves strictly between
        while (lb) {
          const int j = __ffs(lb) - 1;
          lb &= lb - 1;
          U = unite(U, s.val[slot(tid, j)]);
        }
        st = U;
        if ((bm >> o) & 1u) s.val[slot(tid, o)] = U;
      }
      ecm |= ((unsigned)m < (unsigned)gbase) ? bit : 0u;
      s.val[slot(tid, i)] = st;
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
        if (mt[i] < 0 || mt[i] >= gtend) qt |= 1u << i;
        else qi |= 1u << i;
      }
      if (((bm >> i) & 1u) && mt[i] < 0) nvm |= 1u << i;
    }
    if (qt | qi) {
      const float4 after = qt ? range_union_threads(s, tid + 1, NT - 1) : bEMPTY();
      float4 R = bEMPTY();
      uint64_t pk = 0;  // up to 4 pending (close, open position) entries, 16 bits each
      int npk = 0;
#pragma unroll
      for (int i = K - 1; i >= 0; i--) {
        const uint32_t bit = 1u << i;
        if (qt & bit) {
          p.su[tstart + i] = unite(R, after);
        } else if (qi & bit) {
          const int c = (int)(mt[i] - gbase);
          float4& cv = s.val[slot_of(c)];
          if (npk < 4) {  // the thread range is added below, with the lanes in step
            cv = unite(R, cv);
            pk |= (uint64_t)(c | (i << 10)) << (16 * npk);
            npk++;
          } else {
            const float4 U = unite(unite(R, range_union_threads(s, tid + 1, thr_of(c) - 1)), cv);
            cv = U;
            if ((bm >> i) & 1u) s.val[slot(tid, i)] = U;
          }
        }
        if ((lm & bit) && ((qt | qi) & (bit - 1u))) R = unite(R, s.val[slot(tid, i)]);
      }
      if (nvm) {  // blend opens never closed (R4), listed for bbm_final (any order)
        unsigned k = atomicAdd(p.nnever, (unsigned)__popc(nvm));
#pragma unroll 1
        for (uint32_t q = nvm; q; q &= q - 1) p.never[k++] = (int)(tstart + __ffs(q) - 1);
      }
#pragma unroll 1
      for (int k = 0; k < npk; k++) {
        const int e = (int)(pk >> (16 * k)) & 0xffff;
        const int c = e & 1023, i = e >> 10;
        float4& cv = s.val[slot_of(c)];
        const float4 U = unite(cv, range_union_threads(s, tid + 1, thr_of(c) - 1));
        cv = U;
        if ((bm >> i) & 1u) s.val[slot(tid, i)] = U;
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
    if (e < nvalid) st_relaxed_box(p.out + base + e, s.val[slot_of(e)]);
  }
  BBM_TRACE(T, 7);
}

// ----------------------------------------------------------------------------
// bbm_hier: level k of the 32-ary hierarchy of tile unions from level k - 1
// (one warp per group; launched once per level).  Groups [g0, g1) are the ones
// touching the launch's tiles; a group still missing later tiles is rebuilt by
// a later launch and never read before (range unions take whole groups inside
// finished tiles only).
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) bbm_hier(Params p, int k, int m /* nodes at level k - 1 */, int g0, int g1) {
  const int lane = threadIdx.x & 31;
  const int g = g0 + blockIdx.x * 8 + (threadIdx.x >> 5);
  if (g >= g1 || (g << 5) >= m) return;
  const int c = (g << 5) + lane;
  float4 v = c < m ? __ldcg(p.u[k - 1] + c) : bEMPTY();
  v = warp_unite_all(v);
  if (lane == 0) p.u[k][g] = v;
}

// ----------------------------------------------------------------------------
// bbm_close: closes of nodes opened in an earlier tile (one CTA per tile):
// union = prefix of the close's tile (stored by bbm_main) ∪ the open's tile
// suffix after it ∪ the whole tiles in between (F4); blend opens get it too.
// Lanes sharing the open's tile share one warp-cooperative range union.  One
// warp per tile (a tile lists ~17 closes on C5), 32 closes at a time.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(128) bbm_close(Params p) {
  const int lane = threadIdx.x & 31;
  const int T = p.t0 + blockIdx.x * 4 + (threadIdx.x >> 5);
  if (T >= p.t1) return;
  const int cnt = __ldg(p.xcnt + T);
  int cto = INT_MIN;  // warp cache: the last range resolved (deep chains repeat one open tile); To = -1 is a key
  float4 cR = bEMPTY();
  for (int j0 = 0; j0 < cnt; j0 += 32) {
    const int j = j0 + lane;
    const bool valid = j < cnt;
    int c = 0, o = 0, To = 0;
    float4 P = bEMPTY(), su = bEMPTY();
    uint8_t kind = 0;
    if (valid) {
      c = __ldg(p.xc + (int64_t)T * TILE + j);  // local
      o = __ldg(p.match + c);                   // global
      P = __ldcg(p.out + c);
      if (o >= p.off) {
        const int64_t ol = o - p.off;
        To = (int)(ol / TILE);
        su = __ldcg(p.su + ol);
        kind = __ldg(p.tags + ol);
      } else {
        To = -1;  // opened in an earlier chunk: this chunk's part is every tile before
      }
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
      if (o >= p.off) {
        p.out[c] = U;
        if (kind == 2) p.out[o - p.off] = U;  // blend open
      } else {  // shard mode: finished after the exchange
        const uint32_t q = atomicAdd(p.npops, 1u);
        ShardPop r;
        r.pre = U;
        r.c = (int)(p.off + c);
        r.o = o;
        r.pad0 = r.pad1 = 0;
        p.pops[q] = r;
      }
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
// bbm_patch_host (chunked host pipeline): node_bbox entries written after
// their chunk was copied out -- blend opens that receive their union from a
// close in a later chunk (bbm_close) or that are never closed (bbm_final) --
// stored again straight into the (mapped, pinned) host result.  One warp per
// tile over its listed closes; then the never-closed list.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) bbm_patch_host(Params p, float4* hout, int ctiles) {
  const int lane = threadIdx.x & 31;
  const int nwarps = gridDim.x * 8;
  for (int T = blockIdx.x * 8 + (threadIdx.x >> 5); T < p.ntiles; T += nwarps) {
    const int cnt = __ldg(p.xcnt + T);
    for (int j = lane; j < cnt; j += 32) {
      const int c = __ldg(p.xc + (int64_t)T * TILE + j);
      const int o = __ldg(p.match + c);
      if (o >= 0 && (o / TILE) / ctiles < T / ctiles && __ldg(p.tags + o) == 2) hout[o] = __ldcg(p.out + o);
    }
  }
  const uint32_t nv = __ldcg(p.nnever);
  for (uint32_t q = blockIdx.x * 256 + threadIdx.x; q < nv; q += gridDim.x * 256) {
    const int o = __ldcg(p.never + q);
    hout[o] = __ldcg(p.out + o);
  }
}

// ----------------------------------------------------------------------------
// shard mode: a chunk's final stack, the chunk context chain,
// exported unions, fix-up of nodes that span chunks
// ----------------------------------------------------------------------------
// The chunk's final stack = its opens closed after the chunk or never (§3-§4,
// P:96-138), ascending: listed per tile by bbm_reduce (xc / xcnt), positioned
// by an exclusive scan of the counts, written with the chunk-local cumulative
// clip lc ∩ TC_local (one warp per tile).
__global__ void __launch_bounds__(128) bbm_fs_write(Params p, const int* offs, ShardOpen* fs, int* link_out) {
  const int lane = threadIdx.x & 31;
  const int T = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (T >= p.ntiles) return;
  const int cnt = __ldg(p.xcnt + T);
  if (cnt == 0) return;
  const int64_t base = (int64_t)T * TILE;
  const int o0 = __ldg(offs + T);
  const float4 tcT = __ldg(p.tc + T);
  for (int j = lane; j < cnt; j += 32) {
    const int64_t x = base + __ldg(p.xc + base + j);
    ShardOpen r;
    r.v = isect(__ldcg(p.out + x), tcT);  // lc ∩ TC_local
    r.idx = (int)(p.off + x);
    r.pad0 = r.pad1 = r.pad2 = 0;
    fs[o0 + j] = r;
    if (o0 + j == 0) *link_out = __ldg(p.parent + x);  // the chunk's link (earlier chunk or root)
  }
}

// position of global index X in a chunk's ascending list (-1 if absent)
__device__ __forceinline__ int find_open(const ShardOpen* l, int cnt, int X) {
  int lo = 0, hi = cnt;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (l[mid].idx < X) lo = mid + 1;
    else hi = mid;
  }
  return (lo < cnt && l[lo].idx == X) ? lo : -1;
}

__device__ __forceinline__ int chunk_of(const int4* hdr, int G, int X) {
  int h = 0;
  while (h + 1 < G && hdr[h + 1].x <= X) h++;
  return h;
}

// TCc(h) = ctx(link_h) = lcc(link_h) ∩ TCc(chunk of link_h): the clip chain over
// chunks (in order); then the import table of chunk g: every final-stack open
// of chunks h < g with its true context lcc ∩ TCc(h).  hdr[h] = {off, n, b, link}.
__global__ void __launch_bounds__(256) bbm_compose(const int4* hdr, int G, int g, const ShardOpen* allfs, int maxb,
                                                   int32_t* ext_idx, float4* ext_ctx) {
  __shared__ float4 tcc[64];
  __shared__ int start[65];
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int h = 0; h < G; h++) {
      const int4 hd = hdr[h];
      float4 t = bINF();
      if (hd.w >= 0) {
        const int h2 = chunk_of(hdr, G, hd.w);
        const int q = find_open(allfs + (size_t)h2 * maxb, hdr[h2].z, hd.w);
        if (q >= 0) t = isect(allfs[(size_t)h2 * maxb + q].v, tcc[h2]);
      }
      tcc[h] = t;
      start[h] = acc;
      acc += hd.z;
    }
    start[G] = acc;
  }
  __syncthreads();
  const int total = start[g];
  for (int i = blockIdx.x * 256 + threadIdx.x; i < total; i += gridDim.x * 256) {
    int h = 0;
    while (start[h + 1] <= i) h++;
    const ShardOpen r = allfs[(size_t)h * maxb + (i - start[h])];
    ext_idx[i] = r.idx;
    ext_ctx[i] = isect(r.v, tcc[h]);
  }
}

// Export after the local passes: for each final-stack open the union of the
// chunk's clipped leaves after it (one warp per open), and the chunk's union.
__global__ void __launch_bounds__(256) bbm_export(Params p, const ShardOpen* fs, int b, ShardOpen* suc, float4* tu) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (w == b) {
    const float4 t = p.ntiles > 0 ? range_union_tiles_warp(p, 0, p.ntiles - 1) : bEMPTY();
    if (lane == 0) *tu = t;
    return;
  }
  if (w > b) return;
  const int o = fs[w].idx;
  const int64_t ol = o - p.off;
  const int To = (int)(ol / TILE);
  const float4 after = To + 1 < p.ntiles ? range_union_tiles_warp(p, To + 1, p.ntiles - 1) : bEMPTY();
  if (lane == 0) {
    ShardOpen r;
    r.v = unite(__ldcg(p.su + ol), after);
    r.idx = o;
    r.pad0 = r.pad1 = r.pad2 = 0;
    suc[w] = r;
  }
}

__device__ __forceinline__ float4 chunk_range(const float4* alltu, int a, int b) {
  float4 v = bEMPTY();
  for (int h = a; h <= b; h++) v = unite(v, alltu[h]);
  return v;
}

// Fix-up of nodes spanning chunks (chunk g), after exchange 2:
//   own closes of earlier chunks' nodes: suffix of the open's chunk ∪ chunks
//     between ∪ this chunk's prefix (F4 over chunks);
//   own blend opens closed in a later chunk: the same union, from that chunk's
//     record;
//   own blend opens never closed (R4): ∪ every later chunk.
__global__ void __launch_bounds__(256) bbm_fixup(Params p, const int4* hdr, int G, int g, const ShardOpen* allsuc,
                                                 int maxb, const float4* alltu, const ShardPop* allpops,
                                                 const int* npops, int maxp) {
  const int64_t tid = blockIdx.x * (int64_t)256 + threadIdx.x, nthr = (int64_t)gridDim.x * 256;
  // own pops
  for (int64_t i = tid; i < npops[g]; i += nthr) {
    const ShardPop r = allpops[(size_t)g * maxp + i];
    const int h = chunk_of(hdr, G, r.o);
    const int q = find_open(allsuc + (size_t)h * maxb, hdr[h].z, r.o);
    float4 U = unite(r.pre, chunk_range(alltu, h + 1, g - 1));
    if (q >= 0) U = unite(U, allsuc[(size_t)h * maxb + q].v);
    p.out[r.c - p.off] = U;
  }
  // later chunks' pops of this chunk's blend opens
  for (int k = g + 1; k < G; k++) {
    for (int64_t i = tid; i < npops[k]; i += nthr) {
      const ShardPop r = allpops[(size_t)k * maxp + i];
      if (r.o < p.off || r.o >= p.off + p.n) continue;
      const int64_t ol = r.o - p.off;
      if (p.tags[ol] != 2) continue;
      const int q = find_open(allsuc + (size_t)g * maxb, hdr[g].z, r.o);
      float4 U = unite(r.pre, chunk_range(alltu, g + 1, k - 1));
      if (q >= 0) U = unite(U, allsuc[(size_t)g * maxb + q].v);
      p.out[ol] = U;
    }
  }
  // blend opens never closed: the chunk-local part is in node_bbox (bbm_final)
  if (g + 1 < G) {
    const float4 later = chunk_range(alltu, g + 1, G - 1);
    const uint32_t cnt = __ldcg(p.nnever);
    for (int64_t i = tid; i < cnt; i += nthr) {
      const int o = __ldcg(p.never + i);
      p.out[o] = unite(__ldcg(p.out + o), later);
    }
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
  size_t off_fsoff;
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
    off_fsoff = o; o = al(o + 4 * (size_t)(ntiles + 1));
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
  if (once_per_device(1)) {
    cudaFuncSetAttribute(bbm_main<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    cudaFuncSetAttribute(bbm_main<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
  }
}

int tc_blocks() {  // co-resident CTAs of the cooperative kernel on the current device
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bbm_tc, 256, 0);
  return sms * std::max(occ, 1);
}

}  // namespace bbm

size_t bbm_workspace_bytes(int64_t n) {
  if (n <= 0) return 0;
  return bbm::Layout(n).bytes;
}

int bbm_tile_elems() { return bbm::TILE; }

namespace {

bbm::Params make_params(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                        int64_t n, float* node_bbox, void* ws, const BbmShard* sh, uint64_t* trace) {
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
  p.t0 = 0;
  p.t1 = (int)L.ntiles;
  p.nnever = (uint32_t*)(b + L.off_nnever);
  for (int k = 0; k < bbm::LV; k++) p.u[k] = (float4*)(b + L.off_u[k]);
  p.link = (int32_t*)(b + L.off_link);
  p.tc = (float4*)(b + L.off_tc);
  p.su = (float4*)(b + L.off_su);
  p.never = (int32_t*)(b + L.off_never);
  p.xc = (int32_t*)(b + L.off_xc);
  p.xcnt = (int32_t*)(b + L.off_xcnt);
  p.trace = trace;
  p.off = sh ? sh->off : 0;
  p.ext_idx = sh ? sh->ext_idx : nullptr;
  p.ext_ctx = sh ? sh->ext_ctx : nullptr;
  p.n_ext = sh ? sh->n_ext : 0;
  p.pops = sh ? sh->pops : nullptr;
  p.npops = sh ? sh->npops : nullptr;
  p.fs_list = 0;
  return p;
}

cudaError_t launch_tc(const bbm::Params& p, void* ws, cudaStream_t stream) {
  bbm::Layout L(p.n);
  char* b = (char*)ws;
  float4* acc2 = (float4*)(b + L.off_tcacc);
  int* ptr2 = (int*)(b + L.off_tcptr);
  int* flag = (int*)(b + L.off_tcflag);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((p.t1 - p.t0 + 255) / 256, bbm::tc_blocks()));
  bbm::Params pc = p;
  void* args[] = {(void*)&pc, (void*)&acc2, (void*)&ptr2, (void*)&flag};
  void* tok;
  prof_begin(stream, "bbm_tc", &tok);
  cudaError_t err = cudaLaunchCooperativeKernel((const void*)bbm::bbm_tc, dim3(blocks), dim3(256), args, 0, stream);
  prof_end(stream, tok);
  return err;
}

// bbm_main, the union hierarchy and bbm_close over tiles [p.t0, p.t1)
cudaError_t launch_range(const bbm::Params& p, cudaStream_t stream) {
  const unsigned nt = (unsigned)(p.t1 - p.t0);
  bbm::main_setup();
  if (p.off == 0 && p.n_ext == 0 && p.pops == nullptr)
    TB_LAUNCH(stream, "bbm_main", (bbm::bbm_main<false><<<nt, bbm::NT, sizeof(bbm::Smem), stream>>>(p)));
  else
    TB_LAUNCH(stream, "bbm_main", (bbm::bbm_main<true><<<nt, bbm::NT, sizeof(bbm::Smem), stream>>>(p)));
  {
    int64_t m = p.ntiles;
    for (int k = 1; k < bbm::LV && m > 1; k++) {
      const int sh = 5 * k;
      const int g0 = p.t0 >> sh, g1 = ((p.t1 - 1) >> sh) + 1;  // groups touching the range
      TB_LAUNCH(stream, "bbm_hier",
                (bbm::bbm_hier<<<(unsigned)((g1 - g0 + 7) / 8), 256, 0, stream>>>(p, k, (int)m, g0, g1)));
      m = (m + 31) / 32;
    }
  }
  TB_LAUNCH(stream, "bbm_close", (bbm::bbm_close<<<(nt + 3) / 4, 128, 0, stream>>>(p)));
  return cudaGetLastError();
}

// bbm_main, the union hierarchy, bbm_close, bbm_final
cudaError_t launch_rest(const bbm::Params& p, cudaStream_t stream) {
  cudaError_t err = launch_range(p, stream);
  if (err != cudaSuccess) return err;
  TB_LAUNCH(stream, "bbm_final", (bbm::bbm_final<<<sm_count(), 256, 0, stream>>>(p)));
  return cudaGetLastError();
}

}  // namespace

cudaError_t bbm_launch_reduce(const uint8_t* tags, const float* leaf_bbox, int64_t n, float* node_bbox, void* ws,
                              cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  bbm::Layout L(n);
  bbm::Params p = make_params(tags, leaf_bbox, nullptr, nullptr, n, node_bbox, ws, nullptr, nullptr);
  cudaError_t err = cudaMemsetAsync((char*)ws + L.zero_off, 0, L.zero_bytes, stream);
  if (err != cudaSuccess) return err;
  TB_LAUNCH(stream, "bbm_reduce", (bbm::bbm_reduce<<<(unsigned)((L.ntiles + 3) / 4), 128, 0, stream>>>(p)));
  return cudaGetLastError();
}

cudaError_t bbm_launch_rest(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                            int64_t n, float* node_bbox, void* ws, cudaStream_t stream, uint64_t* trace) {
  if (n <= 0) return cudaSuccess;
  bbm::Params p = make_params(tags, leaf_bbox, match, parent, n, node_bbox, ws, nullptr, trace);
  cudaError_t err = launch_tc(p, ws, stream);
  if (err != cudaSuccess) return err;
  return launch_rest(p, stream);
}

cudaError_t bbm_launch(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                       int64_t n, float* node_bbox, void* ws, cudaStream_t stream, uint64_t* trace) {
  cudaError_t err = bbm_launch_reduce(tags, leaf_bbox, n, node_bbox, ws, stream);
  if (err != cudaSuccess) return err;
  return bbm_launch_rest(tags, leaf_bbox, match, parent, n, node_bbox, ws, stream, trace);
}

int bbm_tiles(int64_t n) { return (int)((n + bbm::TILE - 1) / bbm::TILE); }

cudaError_t bbm_begin(void* ws, int64_t n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  bbm::Layout L(n);
  return cudaMemsetAsync((char*)ws + L.zero_off, 0, L.zero_bytes, stream);
}

cudaError_t bbm_tiles_launch(const uint8_t* tags, const float* leaf_bbox, const int32_t* match,
                             const int32_t* parent, int64_t n, float* node_bbox, void* ws, int t0, int t1,
                             cudaStream_t stream) {
  if (n <= 0 || t0 >= t1) return cudaSuccess;
  bbm::Params p = make_params(tags, leaf_bbox, match, parent, n, node_bbox, ws, nullptr, nullptr);
  p.t0 = t0;
  p.t1 = t1;
  TB_LAUNCH(stream, "bbm_reduce", (bbm::bbm_reduce<<<(unsigned)((t1 - t0 + 3) / 4), 128, 0, stream>>>(p)));
  cudaError_t err = launch_tc(p, ws, stream);
  if (err != cudaSuccess) return err;
  return launch_range(p, stream);
}

cudaError_t bbm_end(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                    int64_t n, float* node_bbox, void* ws, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  bbm::Params p = make_params(tags, leaf_bbox, match, parent, n, node_bbox, ws, nullptr, nullptr);
  TB_LAUNCH(stream, "bbm_final", (bbm::bbm_final<<<sm_count(), 256, 0, stream>>>(p)));
  return cudaGetLastError();
}

cudaError_t bbm_patch_host_launch(const uint8_t* tags, const int32_t* match, int64_t n, const float* node_bbox,
                                  void* ws, float* host_mapped, int chunk_tiles, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  bbm::Params p = make_params(tags, nullptr, match, nullptr, n, const_cast<float*>(node_bbox), ws, nullptr, nullptr);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((p.ntiles + 7) / 8, sm_count() * 8));
  TB_LAUNCH(stream, "bbm_patch_host", (bbm::bbm_patch_host<<<blocks, 256, 0, stream>>>(
                                          p, reinterpret_cast<float4*>(host_mapped), chunk_tiles)));
  return cudaGetLastError();
}

cudaError_t bbm_shard_phase1(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                             int64_t n, int64_t off, float* node_bbox, void* ws, ShardOpen* fs, int** b_dev,
                             int* link_dev, cudaStream_t stream) {
  bbm::Layout L(std::max<int64_t>(n, 1));
  char* b = (char*)ws;
  int* offs = (int*)(b + L.off_fsoff);
  *b_dev = offs + L.ntiles;
  if (n <= 0) {
    cudaError_t e = cudaMemsetAsync(offs + L.ntiles, 0, 4, stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(link_dev, &kMinus1, 4, cudaMemcpyHostToDevice, stream);
    return e;
  }
  BbmShard sh{off, nullptr, nullptr, 0, nullptr, nullptr};
  bbm::Params p = make_params(tags, leaf_bbox, match, parent, n, node_bbox, ws, &sh, nullptr);
  p.fs_list = 1;
  cudaError_t err = cudaMemsetAsync((char*)ws + L.zero_off, 0, L.zero_bytes, stream);
  if (err == cudaSuccess) err = cudaMemcpyAsync(link_dev, &kMinus1, 4, cudaMemcpyHostToDevice, stream);
  if (err != cudaSuccess) return err;
  const unsigned g4 = (unsigned)((L.ntiles + 3) / 4);
  TB_LAUNCH(stream, "bbm_reduce", (bbm::bbm_reduce<<<g4, 128, 0, stream>>>(p)));
  err = launch_tc(p, ws, stream);  // no imported contexts yet: chunk-local TC
  if (err != cudaSuccess) return err;
  err = excl_scan_launch(p.xcnt, (int)L.ntiles, offs, "bbm_scan_counts", stream);
  if (err != cudaSuccess) return err;
  TB_LAUNCH(stream, "bbm_fs_write", (bbm::bbm_fs_write<<<g4, 128, 0, stream>>>(p, offs, fs, link_dev)));
  return cudaGetLastError();
}

cudaError_t bbm_compose_launch(const int4* hdr, int G, int g, const ShardOpen* allfs, int maxb, int n_ext,
                               int32_t* ext_idx, float4* ext_ctx, cudaStream_t stream) {
  const int blocks = std::max(1, std::min((n_ext + 255) / 256, 1024));
  TB_LAUNCH(stream, "bbm_compose",
            (bbm::bbm_compose<<<blocks, 256, 0, stream>>>(hdr, G, g, allfs, maxb, ext_idx, ext_ctx)));
  return cudaGetLastError();
}

cudaError_t bbm_shard_phase2(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                             int64_t n, float* node_bbox, void* ws, const BbmShard* sh, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  bbm::Layout L(n);
  bbm::Params p = make_params(tags, leaf_bbox, match, parent, n, node_bbox, ws, sh, nullptr);
  cudaError_t err = cudaMemsetAsync((char*)ws + L.zero_off, 0, L.zero_bytes, stream);  // R4 list count
  if (err == cudaSuccess) err = launch_tc(p, ws, stream);
  if (err != cudaSuccess) return err;
  return launch_rest(p, stream);
}

cudaError_t bbm_export_launch(const uint8_t* tags, const float* leaf_bbox, const int32_t* match,
                              const int32_t* parent, int64_t n, float* node_bbox, void* ws, const BbmShard* sh,
                              const ShardOpen* fs, int b, ShardOpen* suc, float4* tu, cudaStream_t stream) {
  if (n <= 0) {
    const float inf = __builtin_inff();
    const float4 e = make_float4(inf, inf, -inf, -inf);
    return cudaMemcpyAsync(tu, &e, sizeof(e), cudaMemcpyHostToDevice, stream);
  }
  bbm::Params p = make_params(tags, leaf_bbox, match, parent, n, node_bbox, ws, sh, nullptr);
  TB_LAUNCH(stream, "bbm_export", (bbm::bbm_export<<<(unsigned)(b / 8 + 1), 256, 0, stream>>>(p, fs, b, suc, tu)));
  return cudaGetLastError();
}

cudaError_t bbm_fixup_launch(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                             int64_t n, float* node_bbox, void* ws, const BbmShard* sh, const int4* hdr, int G, int g,
                             const ShardOpen* allsuc, int maxb, const float4* alltu, const ShardPop* allpops,
                             const int* npops, int maxp, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  bbm::Params p = make_params(tags, leaf_bbox, match, parent, n, node_bbox, ws, sh, nullptr);
  TB_LAUNCH(stream, "bbm_fixup", (bbm::bbm_fixup<<<sm_count(), 256, 0, stream>>>(p, hdr, G, g, allsuc, maxb, alltu,
                                                                         allpops, npops, maxp)));
  return cudaGetLastError();
}

}  // namespace tb
