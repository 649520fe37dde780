// tree_bbox for sm_100a: clip intersections and blend unions (§6 P:192-221,
// §9) on top of the same tile machinery as paren_match.
//
// Tile = 256 threads x 8 contiguous elements = 2048 elements.  Boxes are
// carried as totalOrder integer keys (boxes.cuh).
//
// bb_reduce (pass 1; reads the tags and, gathered, the boxes of each tile's
//   unmatched opens): per-thread register walk -> Bic; block scans; the
//   tile's stack slice with, per entry, its original index, kind and the
//   tile-local cumulative clip lc = ∩ of the clip boxes of slice entries 0..p
//   (the "inclusive intersection scan" the paper's first bbox dispatch puts
//   in its slices); decoupled look-back -> stack height at the tile
//   start; low-water mark + 32-ary hierarchy (as paren_match).
// bb_finish (pass 2; persistent CTAs, reads tags + boxes, writes node_bbox):
//   1. incoming stack top (a_T + 1 entries) copied from predecessors' slices
//      (owner rule); its TRUE clips = lc ∩ TC(owner), where TC(U) is the true
//      clip just below tile U's low-water mark.  TC of the deepest owner is
//      found by a warp-parallel look-back along the owner chain that stops at
//      the first tile that already published its TC; this tile then publishes
//      its own TC.  (The paper rebuilds the snapshot by an exclusive scan of
//      per-partition top boxes; this is the single-pass equivalent.)
//   2. thread-level chains (a thread's outermost external entry lives in an
//      earlier thread) are resolved by pointer jumping over the 256 threads.
//   3. each thread runs the sequential two-box stack algorithm of the
//      introduction over its 8 elements, starting from its resolved
//      external stack: leaf = box ∩ clip(top), clip open pushes
//      box ∩ clip(top), blend open pushes clip(top), a close yields the
//      union of its node's clipped leaves at the close and, for
//      blend nodes, at the open.
//   4. nodes opened in an earlier thread or tile get their unions from
//      suffix unions (published per slice entry) ∪ range unions over whole
//      threads (sparse table) / whole tiles (32-ary hierarchy of per-tile
//      unions, published as tiles finish step 3) ∪ this thread's prefix union.
// bb_final: blend nodes still open at the end of the stream (R4) get the
//   union of everything after them.
#include <algorithm>
#include <climits>
#include <cooperative_groups.h>
#include "boxes.cuh"
#include "kernels.h"
#include "stackscan.cuh"
#include "tile_common.cuh"

namespace tb {
namespace bb {

constexpr int NT = 128;
constexpr int K = 8;
constexpr int TILE = NT * K;
constexpr int NW = NT / 32;
constexpr int SREC = TILE + 1;  // slice records per tile

struct SliceRec {
  float4 lc; // tile-local cumulative clip
  int idx;   // original element index
  int kind;  // 1 = blend open, 0 = clip open
  int pad0, pad1;
};

// Finish-pass state published by tiles (flags zeroed per call).
struct FState {
  uint32_t* counter;        // dynamic tile ids of the finish pass
  uint32_t* tcf;            // [ntiles] TC published
  uint32_t* suf;            // [ntiles] suffix unions published
  uint32_t* uf[HLEVELS];    // [k][g] union hierarchy published (k = 0: per tile)
  uint32_t* ucnt[HLEVELS];  // arrival counters (k >= 1)
  float4* tc;               // [ntiles] true clip just below the tile's low-water mark
  float4* u[HLEVELS];       // [k][g] union of true-clipped leaves (k = 0: per tile)
  float4* su;               // [ntiles * TILE] true union of leaves after each slice entry
  int32_t* bcount;          // [ntiles] slice length (written by pass 1)
};

// Per-CTA scratch of the persistent finish pass (global, L2-resident).
struct Scratch {
  float4* cin;    // [TILE+1] clip of the incoming entry at depth d (lc, then true)
  int4* meta;     // [TILE+1] {index, kind, run, slice position}
  float4* accin;  // [TILE+1] union of leaves from the entry's open to the tile start
  float4* uoc;    // [TILE]   thread-local cumulative clip of each thread-unmatched open
  float4* uosu;   // [TILE]   union of the thread's leaves after each thread-unmatched open
  int4* run;      // [TILE+1] {tile, L, lo, hi}
  float4* runtc;  // [TILE+1] TC of the run's tile
  float4* runr;   // [TILE+1] union over the tiles between the run's tile and this tile
};
constexpr size_t SCRATCH_BYTES = 16 * (size_t)(7 * (TILE + 1) + TILE) + 1024;

// A close that pops an entry of an earlier chunk (shard mode).
struct BbPop {
  int4 a;     // {close global index, open global index, open kind, source chunk}
  int4 b;     // {position in the source chunk's slice, 0, 0, 0}
  float4 pu;  // union of this chunk's clipped leaves before the close
};

struct Params {
  const uint8_t* tags;
  const float4* boxes;
  float4* out;
  int64_t n;
  int ntiles;
  Ctrl ctrl;
  SliceRec* slice;  // [ntiles * SREC]
  FState f;
  char* scratch;
  uint64_t* trace;  // optional per-tile phase timestamps (debug)
  // shard mode (zero / null when unsharded): the stack live before the chunk
  int64_t offset;           // global index of element 0
  int H0;                   // stack height at the chunk start
  int init_lo;              // entries provided for heights [init_lo, H0)
  const float4* init_clip;  // their true clips
  const int4* init_meta;    // {global index, kind, source chunk, position in its slice}
  BbPop* pops;              // closes popping a provided entry (finished by the shard fix-up)
};

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define BB_TRACE(T, slot)                                                           \
  do {                                                                              \
    if (p.trace && threadIdx.x == 0) p.trace[(size_t)(T) * 16 + (slot)] = gtime();  \
  } while (0)

// ----------------------------------------------------------------------------
// small helpers
// ----------------------------------------------------------------------------
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

__device__ __forceinline__ uint2 load_tags8(const uint8_t* tags, int64_t n, int64_t tbase, bool full) {
  if (full) {
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

// Bic walk over 8 elements: S = opens left on the thread stack, ucm = closes
// that pop the stack at thread start.
__device__ __forceinline__ void walk8(uint32_t om, uint32_t cm, uint32_t& S_out, uint32_t& ucm_out) {
  uint32_t S = 0, ucm = 0;
#pragma unroll
  for (int i = 0; i < K; i++) {
    const uint32_t bit = 1u << i;
    const int top = 31 - __clz(S);
    const bool pop = (cm & bit) && S;
    ucm |= ((cm & bit) && !S) ? bit : 0u;
    S = (om & bit) ? (S | bit) : (pop ? (S ^ (1u << top)) : S);
  }
  S_out = S;
  ucm_out = ucm;
}

__device__ __forceinline__ float4 ld_box_cg(const float4* p) { return __ldcg(p); }

// Exclusive block scan of an int (sum).
template <int NW_>
__device__ __forceinline__ int block_excl_sum(int v, int* wsum, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += o;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  int pre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < NW_; w++) {
    const int s = wsum[w];
    if (w < warp) pre += s;
    tot += s;
  }
  total = tot;
  return pre + x - v;
}

// Exclusive block ∩-scan of a box (thread order).
template <int NW_>
__device__ __forceinline__ float4 block_excl_isect(float4 v, float4* wbox) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4 x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float4 o = shfl_up_box(x, off);
    if (lane >= off) x = isect(x, o);
  }
  if (lane == 31) wbox[warp] = x;
  __syncthreads();
  float4 pre = bINF();
#pragma unroll
  for (int w = 0; w < NW_; w++)
    if (w < warp) pre = isect(pre, wbox[w]);
  float4 e = shfl_up_box(x, 1);
  if (lane == 0) e = bINF();
  return isect(pre, e);
}

// ----------------------------------------------------------------------------
// pass 1
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) bb_reduce(Params p) {
  __shared__ Bic wtot[NW];
  __shared__ float4 wbox[NW];
  const int tid = threadIdx.x;
  const int T = blockIdx.x;
  const int64_t base = (int64_t)T * TILE;
  const int64_t tbase = base + (int64_t)tid * K;
  const bool full = base + TILE <= p.n;

  uint32_t om, cm, bm, S, ucm;
  classify8(load_tags8(p.tags, p.n, tbase, full), om, cm, bm);
  walk8(om, cm, S, ucm);
  const int a_t = __popc(ucm), b_t = __popc(S);
  Bic ex, sx, tot;
  block_bic_scans<NW>(Bic{a_t, b_t}, wtot, ex, sx, tot, true);
  if (tid == 0) {
    p.ctrl.agg[T] = make_int2(tot.a, tot.b);  // the tile scan turns these into heights
    p.f.bcount[T] = tot.b;
  }
  // surviving unmatched opens of this thread: the s_t lowest bits of S
  const int s_t = max(b_t - sx.a, 0);
  uint32_t surv = 0;
  {
    uint32_t m = S;
    for (int k = 0; k < s_t; k++) {
      surv |= m & (~m + 1u);
      m &= m - 1;
    }
  }
  float4 bx[K];
  float4 own = bINF();
#pragma unroll
  for (int i = 0; i < K; i++) {
    bx[i] = bINF();
    if (((surv & ~bm) >> i) & 1u) bx[i] = (__ldg(p.boxes + tbase + i));
    own = isect(own, bx[i]);
  }
  float4 acc = block_excl_isect<NW>(own, wbox);
  {
    const int l_t = ex.b - ex.a - a_t;
    int k = 0;
#pragma unroll
    for (int i = 0; i < K; i++) {
      if ((surv >> i) & 1u) {
        acc = isect(acc, bx[i]);
        SliceRec r;
        r.lc = (acc);
        r.idx = (int)(p.offset + tbase + i);
        r.kind = (int)((bm >> i) & 1u);
        r.pad0 = r.pad1 = 0;
        p.slice[(int64_t)T * SREC + (l_t + k + tot.a)] = r;
        k++;
      }
    }
  }
}

// ----------------------------------------------------------------------------
// hierarchy of per-tile unions (finish pass)
// ----------------------------------------------------------------------------
__device__ __forceinline__ float4 wait_box(const uint32_t* flag, const float4* val) {
  while (ld_acquire_u32(flag) == 0u) {
  }
  return ld_box_cg(val);
}

// Union over tiles [a, b] (warp-cooperative; waits for unpublished entries).
__device__ __forceinline__ float4 range_union_tiles(const FState& f, int a, int b) {
  const int lane = threadIdx.x & 31;
  float4 acc = bEMPTY();
  int k = 0;
  while (a <= b) {
    const uint32_t* fl = f.uf[k];
    const float4* val = f.u[k];
    if ((a >> 5) == (b >> 5) || k == HLEVELS - 1) {
      for (int i = a + lane; i <= b; i += 32) acc = unite(acc, wait_box(fl + i, val + i));
      break;
    }
    if (a & 31) {
      const int e = a | 31;
      const int i = a + lane;
      if (i <= e) acc = unite(acc, wait_box(fl + i, val + i));
      a = e + 1;
    }
    if ((b & 31) != 31) {
      const int s = b & ~31;
      const int i = s + lane;
      if (i <= b) acc = unite(acc, wait_box(fl + i, val + i));
      b = s - 1;
    }
    if (a > b) break;
    a >>= 5;
    b = ((b + 1) >> 5) - 1;
    k++;
  }
  return warp_unite_all(acc);
}

// Publish the tile's union and fold it into the hierarchy (warp; the last of
// 32 siblings publishes the parent).
__device__ __forceinline__ void publish_union(const FState& f, int T, float4 tu) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    f.u[0][T] = (tu);
    __threadfence();
    st_release_u32(f.uf[0] + T, 1u);
  }
  int idx = T;
#pragma unroll 1
  for (int k = 1; k < HLEVELS; k++) {
    const int g = idx >> 5;
    unsigned old = 0;
    if (lane == 0) old = atom_add_acqrel_u32(f.ucnt[k] + g, 1u);
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old != 31u) return;
    const int c = (g << 5) + lane;
    float4 v = wait_box(f.uf[k - 1] + c, f.u[k - 1] + c);
    v = warp_unite_all(v);
    if (lane == 0) {
      f.u[k][g] = (v);
      __threadfence();
      st_release_u32(f.uf[k] + g, 1u);
    }
    idx = g;
  }
}

// ----------------------------------------------------------------------------
// tile clip chain: TC(V) = true clip of the entry just below tile V's
// low-water mark (height L_V - 1 of the stack at V's start; INF at the root).
// TC(V) = lc_W(X - L_W) ∩ TC(W) with W the owner of height X = L_V - 1 (F1),
// a forest over tiles; resolved by pointer jumping (cooperative grid, one
// grid-wide barrier per doubling round).  Replaces the per-partition
// "exclusive scan of top boxes" of the paper's second bbox dispatch.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) bb_tc(Params p, float4* acc2, int* ptr2, int* flag) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)((gridDim.x * (int64_t)blockDim.x) >> 5);
  const int nt = p.ntiles;
  float4* acc[2] = {acc2, acc2 + nt};
  int* ptr[2] = {ptr2, ptr2 + nt};
  // links (one warp per tile: the owner search is warp-cooperative)
  for (int V = gw; V < nt; V += nwarps) {
    const int X = (int)(__ldg(p.ctrl.lw + V) - 1u) - 1;
    float4 a = bINF();
    int q = -1;
    if (X >= 0) {
      int LW = 0;
      const int W = owner_search_done(p.ctrl, V, X, LW);
      if (W >= 0) {
        a = __ldg(&p.slice[(int64_t)W * SREC + (X - LW)].lc);
        q = W;
      } else if (X < p.H0 && X >= p.init_lo) {
        a = __ldg(p.init_clip + (X - p.init_lo));
      }
    }
    if (lane == 0) {
      acc[0][V] = a;
      ptr[0][V] = q;
    }
  }
  const int gt = (int)(blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
  const int nthr = (int)(gridDim.x * (int64_t)blockDim.x);
  int cb = 0;
  for (int round = 0; round < 32; round++) {
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
  for (int V = gt; V < nt; V += nthr) p.f.tc[V] = __ldcg(acc[cb] + V);
}

// ----------------------------------------------------------------------------
// pass 2 (persistent)
// ----------------------------------------------------------------------------
struct Smem {
  float4 box[TILE];  // the tile's boxes (swizzled), replaced in place by its outputs
  float4 tl[NT];     // true clip of each thread's link entry
  int win[NW][5][32];
  int wmin[NW];
  int l[NT];
  uint32_t uo[NT];
  uint32_t bmk[NT];
  int uoff[NT];
  int link[NT];
  uint32_t skip[NT];  // tile-unmatched blend opens: written by a later tile or bb_final
  union {
    struct {  // phase D: pointer jumping over threads
      float4 acc[2][NT];
      int ptr[2][NT];
      int esc[2][NT];
    } pj;
    struct {  // phases F-H: unions over whole threads
      float4 win[6][NT];  // union of thread unions over lanes [lane-2^k+1, lane] (clipped to the warp)
      float4 suf[NT];     // inclusive suffix within the warp
    } un;
  } u;
  float4 wtu[NW];    // per-warp unions
  Bic wtot[NW];
  int wsum[NW];
  int tile, nruns;
};

// element i of thread t lives at slot 8t + (i ^ (t & 7)): conflict-free both
// for the coalesced copies (8 consecutive elements = one row) and for the
// per-thread accesses (8 consecutive threads hit 8 distinct 16-byte columns)
__device__ __forceinline__ int slot(int t, int i) { return (t << 3) | (i ^ (t & 7)); }
__device__ __forceinline__ int slot_of(int e) { return slot(e >> 3, e & 7); }

__device__ __forceinline__ int rank_in(uint32_t m, int bit) { return __popc(m & ((1u << bit) - 1u)); }

// Union of the clipped leaves of whole threads [a, b] (a <= b + 1).
__device__ __forceinline__ float4 range_union_threads(const Smem& s, int a, int b) {
  if (a > b) return bEMPTY();
  const int wa = a >> 5, wb = b >> 5;
  if (wa == wb) {
    const int k = 31 - __clz(b - a + 1);
    return unite(s.u.un.win[k][b], s.u.un.win[k][a + (1 << k) - 1]);
  }
  float4 v = unite(s.u.un.suf[a], s.u.un.win[5][b]);
  for (int w = wa + 1; w < wb; w++) v = unite(v, s.wtu[w]);
  return v;
}

__global__ void __launch_bounds__(NT, 6) bb_finish(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Scratch sc;
  {
    float4* b = reinterpret_cast<float4*>(p.scratch + (size_t)blockIdx.x * SCRATCH_BYTES);
    sc.cin = b;
    sc.meta = reinterpret_cast<int4*>(sc.cin + (TILE + 1));
    sc.accin = reinterpret_cast<float4*>(sc.meta + (TILE + 1));
    sc.run = reinterpret_cast<int4*>(sc.accin + (TILE + 1));
    sc.runtc = reinterpret_cast<float4*>(sc.run + (TILE + 1));
    sc.runr = sc.runtc + (TILE + 1);
    sc.uoc = sc.runr + (TILE + 1);
    sc.uosu = sc.uoc + TILE;
  }

  while (true) {
    if (tid == 0) s.tile = (int)atomicAdd(p.f.counter, 1u);
    __syncthreads();
    const int T = s.tile;
    if (T >= p.ntiles) break;
    const int64_t base = (int64_t)T * TILE;
    const int64_t tbase = base + (int64_t)tid * K;
    const bool full = base + TILE <= p.n;
    const int nvalid = full ? TILE : (int)(p.n - base);

    BB_TRACE(T, 0);
    // ---- A. load: tags to registers, boxes to shared memory (coalesced) --
    uint32_t om, cm, bm, S, ucm;
    classify8(load_tags8(p.tags, p.n, tbase, full), om, cm, bm);
#pragma unroll
    for (int j = 0; j < K; j++) {
      const int e = j * NT + tid;
      s.box[slot_of(e)] = e < nvalid ? __ldg(p.boxes + base + e) : bINF();
    }
    walk8(om, cm, S, ucm);
    const int a_t = __popc(ucm), b_t = __popc(S);

    // ---- B. scans, thread references ----------------------------------------
    Bic ex, sx, tot;
    block_bic_scans<NW>(Bic{a_t, b_t}, s.wtot, ex, sx, tot, true);  // (barrier: boxes staged)
    const int aT = tot.a;
    const int r_t = ex.b - ex.a;
    const int l_t = r_t - a_t;
    int tot_uo;
    const int uoff = block_excl_sum<NW>(b_t, s.wsum, tot_uo);
    int wl[5];
    lane_windows(l_t, wl);
#pragma unroll
    for (int k = 0; k < 5; k++) s.win[warp][k][lane] = wl[k];
    {
      const int o = __shfl_sync(0xffffffffu, wl[4], 15);
      if (lane == 31) s.wmin[warp] = min(wl[4], o);
    }
    s.l[tid] = l_t;
    s.uo[tid] = S;
    s.bmk[tid] = bm;
    s.uoff[tid] = uoff;
    const int s_t = max(b_t - sx.a, 0);  // this thread's opens that survive the tile
    {
      uint32_t surv = 0, m = S;
      for (int k = 0; k < s_t; k++) {
        surv |= m & (~m + 1u);
        m &= m - 1;
      }
      s.skip[tid] = surv & bm;
    }
    // thread-local cumulative clip of each thread-unmatched open
    {
      float4 acc = bINF();
      int k = 0;
#pragma unroll
      for (int i = 0; i < K; i++) {
        if ((S >> i) & 1u) {
          if (!((bm >> i) & 1u)) acc = isect(acc, s.box[slot(tid, i)]);
          sc.uoc[uoff + k] = acc;
          k++;
        }
      }
    }
    const int H = __ldg(p.ctrl.hstart + T);
    const int lo = max(H - 1 - aT, 0);
    for (int d = H + tid; d <= aT; d += NT) {
      sc.cin[d] = bINF();
      sc.meta[d] = make_int4(-1, 0, -1, 0);
    }
    __syncthreads();
    const int top_ref = thread_ref<NW, K>(wl, l_t, S, r_t - 1, s.win, s.wmin, s.l, s.uo);
    const int link_ref = thread_ref<NW, K>(wl, l_t, S, l_t - 1, s.win, s.wmin, s.l, s.uo);
    s.link[tid] = link_ref;

    BB_TRACE(T, 1);
    // ---- C. incoming stack: runs of predecessors' slices ------------------
    if (warp == 0) {
      int cur = H - 1, from = T, nr = 0;
      while (cur >= lo) {
        int LU = 0;
        const int U = owner_search_done(p.ctrl, from, cur, LU);
        const int rlo = max(LU, lo);
        if (lane == 0) sc.run[nr] = make_int4(U, U >= 0 ? LU : p.init_lo, U >= 0 ? rlo : lo, cur);
        nr++;
        if (U < 0) break;  // the rest lies in the stack provided by the shard exchange
        cur = LU - 1;
        from = U;
      }
      if (lane == 0) s.nruns = nr;
    }
    __syncthreads();
    const int nr = s.nruns;
    for (int r = warp; r < nr; r += NW) {
      const int4 rr = __ldcg(sc.run + r);
      const int cnt = rr.w - rr.z + 1;
      for (int i = lane; i < cnt; i += 32) {
        const int h = rr.w - i;
        const int d = H - 1 - h;
        if (rr.x >= 0) {
          const SliceRec rec = p.slice[(int64_t)rr.x * SREC + (h - rr.y)];
          sc.cin[d] = rec.lc;
          sc.meta[d] = make_int4(rec.idx, rec.kind, r, h - rr.y);
        } else {  // live before the chunk: true clip provided by the shard exchange
          const int q = h - p.init_lo;
          sc.cin[d] = __ldg(p.init_clip + q);
          sc.meta[d] = make_int4(__ldg(p.init_meta + q).x, __ldg(p.init_meta + q).y, r, q);
        }
      }
    }
    __syncthreads();
    BB_TRACE(T, 2);
    // TC of each run's tile: deepest precomputed (bb_tc), the others from the run below
    if (warp == 0 && nr > 0) {
      const int4 rb = __ldcg(sc.run + nr - 1);
      float4 tc = rb.x >= 0 ? __ldg(p.f.tc + rb.x) : bINF();
      if (lane == 0) sc.runtc[nr - 1] = tc;
      for (int r = nr - 2; r >= 0; r--) {
        const int4 rbelow = __ldcg(sc.run + r + 1);
        tc = isect(__ldcg(sc.cin + (H - 1 - rbelow.w)), tc);
        if (lane == 0) sc.runtc[r] = tc;
      }
    }
    __syncthreads();
    for (int d = tid; d < min(aT + 1, H); d += NT) {
      const int run = __ldcg(sc.meta + d).z;
      sc.cin[d] = isect(__ldcg(sc.cin + d), __ldcg(sc.runtc + run));
    }
    __syncthreads();

    BB_TRACE(T, 3);
    // ---- D. thread chains: clip of each thread's link entry ---------------
    {
      int ptr = -1, esc = 0;
      float4 acc = bINF();
      if (link_ref >= 0) {
        const int W = link_ref / K;
        ptr = W;
        acc = __ldcg(sc.uoc + s.uoff[W] + rank_in(s.uo[W], link_ref % K));
      } else {
        esc = link_ref;
      }
      int cb = 0;
      s.u.pj.acc[0][tid] = acc;
      s.u.pj.ptr[0][tid] = ptr;
      s.u.pj.esc[0][tid] = esc;
      int any = __syncthreads_or(ptr >= 0);
      while (any) {
        if (ptr >= 0) {
          acc = isect(acc, s.u.pj.acc[cb][ptr]);
          esc = s.u.pj.esc[cb][ptr];
          ptr = s.u.pj.ptr[cb][ptr];
        }
        s.u.pj.acc[cb ^ 1][tid] = acc;
        s.u.pj.ptr[cb ^ 1][tid] = ptr;
        s.u.pj.esc[cb ^ 1][tid] = esc;
        cb ^= 1;
        any = __syncthreads_or(ptr >= 0);
      }
      s.tl[tid] = isect(acc, __ldcg(sc.cin + (-esc - 1)));
    }
    __syncthreads();

    // true clip of an entry of this thread's start stack
    auto entry_clip = [&](int ref) -> float4 {
      if (ref >= 0) {
        const int V = ref / K;
        return isect(__ldcg(sc.uoc + s.uoff[V] + rank_in(s.uo[V], ref % K)), s.tl[V]);
      }
      return __ldcg(sc.cin + (-ref - 1));
    };
    auto next_down = [&](int ref) -> int {
      if (ref >= 0) {
        const int V = ref / K;
        const uint32_t below = s.uo[V] & ((1u << (ref % K)) - 1u);
        return below ? V * K + (31 - __clz(below)) : s.link[V];
      }
      return ref - 1;
    };

    BB_TRACE(T, 4);
    // ---- E. per-thread two-box stack walk ----------------------------
    // The thread's stack is the bitmask St of its open positions; the clip of
    // the top is the effective clip of the deepest clip open on it (a blend
    // passes its parent's clip through), else the clip of the external top.
    // A node closed inside the thread gets the union of the clipped leaves
    // strictly inside it.  Results replace the boxes in shared memory; a
    // close that pops an external entry records the thread's prefix union.
    uint32_t lm = ~om & ~cm & 0xffu;  // leaves
    if (!full) {
      const int64_t rem = p.n - tbase;
      lm &= rem >= K ? 0xffu : (rem <= 0 ? 0u : ((1u << rem) - 1u));
    }
    const uint32_t clipm = om & ~bm;
    float4 tu_thr = bEMPTY();  // union of this thread's clipped leaves
    {
      int ref = top_ref;
      float4 cext = entry_clip(ref);
      float4 ctop = cext;
      uint32_t St = 0;
#pragma unroll
      for (int i = 0; i < K; i++) {
        const uint32_t bit = 1u << i;
        float4& me = s.box[slot(tid, i)];
        if (om & bit) {
          if (!(bm & bit)) {
            ctop = isect(me, ctop);
            me = ctop;
          }
          St |= bit;
        } else if (cm & bit) {
          if (St) {
            const int o = 31 - __clz(St);
            float4 U = bEMPTY();
#pragma unroll
            for (int j = 0; j < i; j++)
              if (((lm >> j) & 1u) && j > o) U = unite(U, s.box[slot(tid, j)]);
            me = U;
            if ((bm >> o) & 1u) s.box[slot(tid, o)] = U;
            St ^= 1u << o;
            const uint32_t cs = St & clipm;
            ctop = cs ? s.box[slot(tid, 31 - __clz(cs))] : cext;
          } else {
            me = tu_thr;  // prefix union; completed in H
            ref = next_down(ref);
            cext = entry_clip(ref);
            ctop = cext;
          }
        } else if ((lm >> i) & 1u) {
          const float4 v = isect(me, ctop);
          me = v;
          tu_thr = unite(tu_thr, v);
        }
      }
      // unions after each thread-unmatched open (St = those opens)
      float4 suf = bEMPTY();
#pragma unroll
      for (int j = K - 1; j >= 0; j--) {
        if ((St >> j) & 1u) sc.uosu[uoff + __popc(St & ((1u << j) - 1u))] = suf;
        if ((lm >> j) & 1u) suf = unite(suf, s.box[slot(tid, j)]);
      }
    }

    // ---- F. unions over whole threads; publish tile union and suffix unions --
    {
      // windows of 2^k lanes ending at each lane (k = 0..5, clipped at lane 0;
      // level 5 is the inclusive in-warp prefix)
      float4 w = tu_thr, suf = tu_thr;
      s.u.un.win[0][tid] = w;
#pragma unroll
      for (int k = 1; k <= 5; k++) {
        const int off = 1 << (k - 1);
        const float4 a = shfl_up_box(w, off);
        if (lane >= off) w = unite(w, a);
        s.u.un.win[k][tid] = w;
        const float4 b = make_float4(__shfl_down_sync(0xffffffffu, suf.x, off),
                                     __shfl_down_sync(0xffffffffu, suf.y, off),
                                     __shfl_down_sync(0xffffffffu, suf.z, off),
                                     __shfl_down_sync(0xffffffffu, suf.w, off));
        if (lane + off < 32) suf = unite(suf, b);
      }
      s.u.un.suf[tid] = suf;
      if (lane == 31) s.wtu[warp] = w;  // w = inclusive prefix over the whole warp
    }
    __syncthreads();
    BB_TRACE(T, 5);
    if (s_t > 0) {
      const float4 after = range_union_threads(s, tid + 1, NT - 1);
      for (int k = 0; k < s_t; k++)
        p.f.su[(int64_t)T * TILE + (l_t + k + aT)] = unite(__ldcg(sc.uosu + uoff + k), after);
    }
    __syncthreads();
    if (warp == 0) {
      if (lane == 0) {
        __threadfence();
        st_release_u32(p.f.suf + T, 1u);
      }
      float4 tu = lane < NW ? s.wtu[lane] : bEMPTY();
      publish_union(p.f, T, warp_unite_all(tu));
    }

    // ---- G. unions reaching back into earlier tiles -------------------------
    BB_TRACE(T, 6);
    for (int r = warp; r < nr; r += NW) {
      const int4 rr = __ldcg(sc.run + r);
      const float4 mid = range_union_tiles(p.f, rr.x + 1, T - 1);
      if (lane == 0) sc.runr[r] = mid;
    }
    __syncthreads();
    for (int d = tid; d < min(aT, H); d += NT) {
      const int4 m = __ldcg(sc.meta + d);
      const int U = __ldcg(sc.run + m.z).x;
      float4 v = __ldcg(sc.runr + m.z);
      if (U >= 0) {
        while (ld_acquire_u32(p.f.suf + U) == 0u) {
        }
        v = unite(ld_box_cg(p.f.su + (int64_t)U * TILE + m.w), v);
      }
      sc.accin[d] = v;
    }
    __syncthreads();

    BB_TRACE(T, 7);
    // ---- H. closes that pop entries of earlier threads / tiles -------------
    if (ucm) {
      int ref = top_ref;
#pragma unroll
      for (int i = 0; i < K; i++) {
        if ((ucm >> i) & 1u) {
          const int64_t g = tbase + i;
          float4& me = s.box[slot(tid, i)];
          float4 U;
          if (ref >= 0) {
            const int V = ref / K;
            const float4 su = __ldcg(sc.uosu + s.uoff[V] + rank_in(s.uo[V], ref % K));
            U = unite(unite(su, range_union_threads(s, V + 1, tid - 1)), me);
            if ((s.bmk[V] >> (ref % K)) & 1u) s.box[slot(V, ref % K)] = U;
          } else {
            const int dd = -ref - 1;
            if (dd >= H) {
              U = bEMPTY();  // nothing to close (R3)
            } else {
              const int4 m = __ldcg(sc.meta + dd);
              U = unite(unite(__ldcg(sc.accin + dd), range_union_threads(s, 0, tid - 1)), me);
              if (__ldcg(sc.run + m.z).x >= 0) {
                if (m.y) p.out[m.x - p.offset] = U;  // blend open of an earlier tile
              } else {
                // the open lives in an earlier chunk: U so far is this chunk's part
                const int k = p.H0 - H + dd;
                const int4 im = __ldg(p.init_meta + m.w);
                BbPop rec;
                rec.a = make_int4((int)(p.offset + g), im.x, im.y, im.z);
                rec.b = make_int4(im.w, 0, 0, 0);
                rec.pu = U;
                p.pops[k] = rec;
              }
            }
          }
          me = U;
          ref = next_down(ref);
        }
      }
    }
    __syncthreads();

    // ---- copy-out (coalesced), skipping tile-unmatched blend opens --------
#pragma unroll
    for (int j = 0; j < K; j++) {
      const int e = j * NT + tid;
      if (e < nvalid && !((s.skip[e >> 3] >> (e & 7)) & 1u)) __stcs(p.out + base + e, s.box[slot_of(e)]);
    }
    BB_TRACE(T, 8);
    __syncthreads();
  }
}

// ----------------------------------------------------------------------------
// pass 3: blend nodes still open at the end of the stream (R4)
// ----------------------------------------------------------------------------
__device__ __forceinline__ int range_min_L(const Ctrl& c, int a, int b) {
  const int lane = threadIdx.x & 31;
  int acc = INT_MAX;
  int k = 0;
  while (a <= b) {
    const uint32_t* v = c.lv[k];
    if ((a >> 5) == (b >> 5) || k == HLEVELS - 1) {
      for (int i = a + lane; i <= b; i += 32) acc = min(acc, (int)(__ldg(v + i) - 1u));
      break;
    }
    if (a & 31) {
      const int e = a | 31, i = a + lane;
      if (i <= e) acc = min(acc, (int)(__ldg(v + i) - 1u));
      a = e + 1;
    }
    if ((b & 31) != 31) {
      const int s0 = b & ~31, i = s0 + lane;
      if (i <= b) acc = min(acc, (int)(__ldg(v + i) - 1u));
      b = s0 - 1;
    }
    if (a > b) break;
    a >>= 5;
    b = ((b + 1) >> 5) - 1;
    k++;
  }
  return __reduce_min_sync(0xffffffffu, acc);
}

__global__ void __launch_bounds__(128) bb_final(Params p) {
  const int lane = threadIdx.x & 31;
  const int W = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (W >= p.ntiles) return;
  const int bW = __ldg(p.f.bcount + W);
  if (bW == 0) return;
  const int LW = (int)(__ldg(p.ctrl.lw + W) - 1u);
  const int minL = (W + 1 < p.ntiles) ? range_min_L(p.ctrl, W + 1, p.ntiles - 1) : INT_MAX;
  const int nsurv = min(bW, max(minL - LW, 0));  // entries at heights < minL survive
  if (nsurv == 0) return;
  const float4 after = (W + 1 < p.ntiles) ? range_union_tiles(p.f, W + 1, p.ntiles - 1) : bEMPTY();
  for (int q = lane; q < nsurv; q += 32) {
    const SliceRec rec = p.slice[(int64_t)W * SREC + q];
    if (rec.kind) {
      const float4 v = unite(ld_box_cg(p.f.su + (int64_t)W * TILE + q), after);
      p.out[rec.idx] = (v);
    }
  }
}

// ----------------------------------------------------------------------------
// shard support: chunk summary, chunk export, composition of
// the incoming stack, fix-up of nodes that span chunks
// ----------------------------------------------------------------------------
// One entry of a chunk's final stack (its unmatched opens, bottom to top).
struct SumRec {
  float4 clip;  // chunk-local cumulative clip (true clip if the chunk began at the root)
  int idx;      // global index
  int kind;     // 1 = blend
  int tile;     // owning tile in the chunk
  int pos;      // position in that tile's slice
};

// After bb_reduce (chunk-local frame): header (a, b) and the chunk's final
// stack; the clip of an entry = its tile-local cumulative clip ∩ the clip of
// the entry just below its run (runs are processed bottom-up).
__global__ void __launch_bounds__(NT) bb_summary(Params p, int32_t* hdr, SumRec* recs, int4* runs) {
  __shared__ int s_nr;
  __shared__ float4 s_tc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int2 t2 = __ldcg(p.ctrl.total);  // Bic value of the chunk (tile scan)
  const Bic tot{t2.x, t2.y};
  if (tid == 0) {
    hdr[0] = tot.a;
    hdr[1] = tot.b;
  }
  if (warp == 0) {
    int cur = tot.b - 1, from = p.ntiles, nr = 0;
    while (cur >= 0) {
      int LU = 0;
      const int U = owner_search_done(p.ctrl, from, cur, LU);
      if (lane == 0) runs[nr] = make_int4(U, LU, LU, cur);
      nr++;
      cur = LU - 1;
      from = U;
    }
    if (lane == 0) s_nr = nr;
  }
  __syncthreads();
  const int nr = s_nr;
  float4 tc = bINF();
  for (int r = nr - 1; r >= 0; r--) {
    const int4 rr = __ldcg(runs + r);
    for (int h = rr.z + tid; h <= rr.w; h += NT) {
      const SliceRec rec = p.slice[(int64_t)rr.x * SREC + (h - rr.y)];
      SumRec o;
      o.clip = isect(rec.lc, tc);
      o.idx = rec.idx;
      o.kind = rec.kind;
      o.tile = rr.x;
      o.pos = h - rr.y;
      recs[h] = o;
    }
    __syncthreads();
    if (tid == 0) s_tc = __ldcg(&recs[rr.w].clip);
    __syncthreads();
    tc = s_tc;
  }
}

// After bb_finish (chunk-local frame): the chunk's union of clipped leaves and,
// per final-stack entry, the union of the chunk's leaves after it:
//   su(entry) = su_tile(entry) ∪ (union of the tiles after its tile).
__global__ void __launch_bounds__(1024) bb_export(Params p, const SumRec* recs, int b, float4* suf_tiles,
                                                  float4* out_tu, float4* out_su) {
  __shared__ float4 wtot[32];
  __shared__ float4 carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry = bEMPTY();
  __syncthreads();
  // suffix unions over tiles: suf_tiles[t] = union of tiles (t, ntiles)
  for (int hi = p.ntiles - 1; hi >= 0; hi -= 1024) {
    const int t = hi - tid;
    float4 v = t >= 0 ? ld_box_cg(p.f.u[0] + t) : bEMPTY();
    // inclusive scan from high t to low t (tid order)
    float4 x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const float4 o = shfl_up_box(x, off);
      if (lane >= off) x = unite(x, o);
    }
    if (lane == 31) wtot[warp] = x;
    __syncthreads();
    float4 pre = carry;
    for (int w = 0; w < warp; w++) pre = unite(pre, wtot[w]);
    float4 ex = shfl_up_box(x, 1);
    if (lane == 0) ex = bEMPTY();
    if (t >= 0) suf_tiles[t] = unite(pre, ex);
    __syncthreads();
    if (tid == 0) {
      float4 c = carry;
      for (int w = 0; w < 32; w++) c = unite(c, wtot[w]);
      carry = c;
    }
    __syncthreads();
  }
  if (tid == 0) *out_tu = carry;
  __syncthreads();
  for (int q = tid; q < b; q += 1024) {
    const SumRec r = recs[q];
    out_su[q] = unite(ld_box_cg(p.f.su + (int64_t)r.tile * TILE + r.pos), __ldcg(suf_tiles + r.tile));
  }
}

// Rank g: true clips TC of every earlier chunk (just below its low-water
// mark, owner rule over chunks), then the provided stack entries for
// heights [lo, H): clip = chunk-local clip ∩ TC(owner chunk).
__global__ void __launch_bounds__(256) bb_compose(const SumRec* allrecs, int maxb, const int* L, int g, int lo,
                                                  int H, float4* init_clip, int4* init_meta) {
  __shared__ float4 tc[64];
  if (threadIdx.x == 0) {
    for (int h = 0; h < g; h++) {
      const int X = L[h] - 1;
      float4 v = bINF();
      if (X >= 0) {
        int o = h - 1;
        while (o > 0 && L[o] > X) o--;
        v = isect(allrecs[(int64_t)o * maxb + (X - L[o])].clip, tc[o]);
      }
      tc[h] = v;
    }
  }
  __syncthreads();
  for (int X = lo + threadIdx.x; X < H; X += blockDim.x) {
    int o = g - 1;
    while (o > 0 && L[o] > X) o--;
    const int q = X - L[o];
    const SumRec r = allrecs[(int64_t)o * maxb + q];
    init_clip[X - lo] = isect(r.clip, tc[o]);
    init_meta[X - lo] = make_int4(r.idx, r.kind, o, q);
  }
}

// Rank g: finish the nodes that span chunks.
//   own pops:           out[close] = su_h(open) ∪ TU(h+1..g-1) ∪ pu
//   later chunks' pops of own blend opens: out[open] = the same union
//   own blend opens open at the end of the stream: su_g ∪ TU(g+1..G-1)
__global__ void bb_fixup(int G, int g, int64_t off, int b_g, int min_L_after, int L_g, const float4* tu,
                         const float4* allsu, int maxb, const BbPop* allpops, int maxp, const int* npops,
                         const SumRec* myrecs, float4* out) {
  auto turange = [&](int a, int bb) {
    float4 v = bEMPTY();
    for (int k = a; k <= bb; k++) v = unite(v, tu[k]);
    return v;
  };
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int k = g; k < G; k++) {
    for (int64_t i = i0; i < npops[k]; i += stride) {
      const BbPop r = allpops[(int64_t)k * maxp + i];
      const int h = r.a.w, q = r.b.x;
      if (k == g) {
        const float4 U = unite(unite(allsu[(int64_t)h * maxb + q], turange(h + 1, g - 1)), r.pu);
        out[r.a.x - off] = U;
      } else if (h == g && r.a.z) {
        const float4 U = unite(unite(allsu[(int64_t)g * maxb + q], turange(g + 1, k - 1)), r.pu);
        out[r.a.y - off] = U;
      }
    }
  }
  for (int64_t q = i0; q < b_g; q += stride) {
    if ((int64_t)L_g + q < (int64_t)min_L_after && myrecs[q].kind) {
      out[myrecs[q].idx - off] = unite(allsu[(int64_t)g * maxb + q], turange(g + 1, G - 1));
    }
  }
}

// ----------------------------------------------------------------------------
// workspace
// ----------------------------------------------------------------------------
struct Layout {
  size_t ctrl_bytes, fzero_off, fzero_bytes, data_off, bytes;
  size_t off_counter, off_tcf, off_suf, off_uf[HLEVELS], off_ucnt[HLEVELS];
  size_t off_tc, off_u[HLEVELS], off_su, off_bcount, off_slice, off_scratch, off_tcacc, off_tcptr, off_tcflag;
  int64_t ntiles;
  int nblocks;
  static size_t al(size_t x) { return (x + 255) & ~size_t(255); }
  Layout(int64_t n, int nblocks_) : nblocks(nblocks_) {
    ntiles = (n + TILE - 1) / TILE;
    ctrl_bytes = CtrlLayout(ntiles).bytes;
    size_t o = al(ctrl_bytes);
    fzero_off = o;
    off_counter = o; o = al(o + 16);
    off_tcf = o; o = al(o + 4 * (size_t)ntiles);
    off_suf = o; o = al(o + 4 * (size_t)ntiles);
    int64_t m = ntiles;
    for (int k = 0; k < HLEVELS; k++) {
      off_uf[k] = o; o = al(o + 4 * (size_t)m);
      off_ucnt[k] = o; o = al(o + 4 * (size_t)m);
      m = (m + 31) / 32;
    }
    fzero_bytes = o - fzero_off;
    data_off = o;
    off_tc = o; o = al(o + 16 * (size_t)ntiles);
    m = ntiles;
    for (int k = 0; k < HLEVELS; k++) {
      off_u[k] = o; o = al(o + 16 * (size_t)m);
      m = (m + 31) / 32;
    }
    off_bcount = o; o = al(o + 4 * (size_t)ntiles);
    off_tcacc = o; o = al(o + 32 * (size_t)ntiles);
    off_tcptr = o; o = al(o + 8 * (size_t)ntiles);
    off_tcflag = o; o = al(o + 16);
    off_su = o; o = al(o + 16 * (size_t)ntiles * TILE);
    off_slice = o; o = al(o + sizeof(SliceRec) * (size_t)ntiles * SREC);
    off_scratch = o; o = al(o + SCRATCH_BYTES * (size_t)nblocks);
    bytes = o;
  }
};

int finish_blocks() {
  static int nb = 0;
  if (nb == 0) {
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(bb_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bb_finish, NT, sizeof(Smem));
    nb = sms * (occ > 0 ? occ : 1);
  }
  return nb;
}

}  // namespace bb

size_t bb_workspace_bytes(int64_t n) {
  if (n <= 0) return 0;
  return bb::Layout(n, bb::finish_blocks()).bytes;
}

static bb::Params bb_params(const uint8_t* tags, const float* leaf_bbox, int64_t n, float* node_bbox, void* ws,
                           const BbShard* sh, uint64_t* trace) {
  bb::Layout L(n, bb::finish_blocks());
  char* b = (char*)ws;
  bb::Params p;
  p.tags = tags;
  p.boxes = reinterpret_cast<const float4*>(leaf_bbox);
  p.out = reinterpret_cast<float4*>(node_bbox);
  p.n = n;
  p.ntiles = (int)L.ntiles;
  p.ctrl = CtrlLayout(L.ntiles).bind(ws);
  p.slice = (bb::SliceRec*)(b + L.off_slice);
  p.f.counter = (uint32_t*)(b + L.off_counter);
  p.f.tcf = (uint32_t*)(b + L.off_tcf);
  p.f.suf = (uint32_t*)(b + L.off_suf);
  for (int k = 0; k < HLEVELS; k++) {
    p.f.uf[k] = (uint32_t*)(b + L.off_uf[k]);
    p.f.ucnt[k] = (uint32_t*)(b + L.off_ucnt[k]);
    p.f.u[k] = (float4*)(b + L.off_u[k]);
  }
  p.f.tc = (float4*)(b + L.off_tc);
  p.f.su = (float4*)(b + L.off_su);
  p.f.bcount = (int32_t*)(b + L.off_bcount);
  p.scratch = b + L.off_scratch;
  p.trace = trace;
  p.offset = sh ? sh->offset : 0;
  p.H0 = sh ? sh->H0 : 0;
  p.init_lo = sh ? sh->init_lo : 0;
  p.init_clip = sh ? (const float4*)sh->init_clip : nullptr;
  p.init_meta = sh ? (const int4*)sh->init_meta : nullptr;
  p.pops = sh ? (bb::BbPop*)sh->pops : nullptr;
  return p;
}

cudaError_t bb_reduce_launch(const uint8_t* tags, const float* leaf_bbox, int64_t n, void* ws, const BbShard* sh,
                             cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  bb::Layout L(n, bb::finish_blocks());
  cudaError_t err = cudaMemsetAsync((char*)ws + L.fzero_off, 0, L.fzero_bytes, stream);
  if (err != cudaSuccess) return err;
  bb::Params p = bb_params(tags, leaf_bbox, n, nullptr, ws, sh, nullptr);
  TB_LAUNCH(stream, "bb_reduce", (bb::bb_reduce<<<(unsigned)L.ntiles, bb::NT, 0, stream>>>(p)));
  err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  return tile_scan_launch(p.ctrl, L.ntiles, 0, p.H0, stream);
}

cudaError_t bb_finish_launch(const uint8_t* tags, const float* leaf_bbox, int64_t n, float* node_bbox, void* ws,
                             const BbShard* sh, cudaStream_t stream, uint64_t* trace) {
  if (n <= 0) return cudaSuccess;
  const int nb_max = bb::finish_blocks();
  bb::Layout L(n, nb_max);
  bb::Params p = bb_params(tags, leaf_bbox, n, node_bbox, ws, sh, trace);
  {
    // tile clip chains (cooperative: one grid-wide barrier per doubling round)
    static int tc_blocks = 0;
    if (tc_blocks == 0) {
      int dev = 0, sms = 0, occ = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bb::bb_tc, 256, 0);
      tc_blocks = sms * std::max(occ, 1);
    }
    char* b = (char*)ws;
    float4* acc2 = (float4*)(b + L.off_tcacc);
    int* ptr2 = (int*)(b + L.off_tcptr);
    int* flag = (int*)(b + L.off_tcflag);
    const int64_t need = (L.ntiles * 32 + 255) / 256;  // one warp per tile in the link phase
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(need, tc_blocks));
    void* args[] = {(void*)&p, (void*)&acc2, (void*)&ptr2, (void*)&flag};
    void* tok;
    prof_begin(stream, "bb_tc", &tok);
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)bb::bb_tc, dim3(blocks), dim3(256), args, 0, stream);
    prof_end(stream, tok);
    if (e != cudaSuccess) return e;
  }
  const int nfin = (int)std::min<int64_t>(L.ntiles, (int64_t)nb_max);
  TB_LAUNCH(stream, "bb_finish", (bb::bb_finish<<<(unsigned)nfin, bb::NT, sizeof(bb::Smem), stream>>>(p)));
  if (!sh)
    TB_LAUNCH(stream, "bb_final", (bb::bb_final<<<(unsigned)((L.ntiles + 3) / 4), 128, 0, stream>>>(p)));
  return cudaGetLastError();
}

cudaError_t bb_launch(const uint8_t* tags, const float* leaf_bbox, int64_t n, float* node_bbox, void* ws,
                      cudaStream_t stream, uint64_t* trace) {
  cudaError_t err = bb_reduce_launch(tags, leaf_bbox, n, ws, nullptr, stream);
  if (err == cudaSuccess) err = bb_finish_launch(tags, leaf_bbox, n, node_bbox, ws, nullptr, stream, trace);
  return err;
}

int bb_tile_elems() { return bb::TILE; }
size_t bb_sumrec_bytes() { return sizeof(bb::SumRec); }
size_t bb_pop_bytes() { return sizeof(bb::BbPop); }

cudaError_t bb_summary_launch(const uint8_t* tags, const float* leaf_bbox, int64_t n, void* ws, int32_t* hdr,
                              void* recs, int4* runs, cudaStream_t stream) {
  if (n <= 0) return cudaMemsetAsync(hdr, 0, 8, stream);
  bb::Params p = bb_params(tags, leaf_bbox, n, nullptr, ws, nullptr, nullptr);
  TB_LAUNCH(stream, "bb_summary", (bb::bb_summary<<<1, bb::NT, 0, stream>>>(p, hdr, (bb::SumRec*)recs, runs)));
  return cudaGetLastError();
}

cudaError_t bb_export_launch(const uint8_t* tags, const float* leaf_bbox, int64_t n, void* ws, const void* recs,
                             int b, float4* suf_tiles, float4* out_tu, float4* out_su, cudaStream_t stream) {
  if (n <= 0) {
    const float inf = __builtin_inff();
    float4 e = make_float4(inf, inf, -inf, -inf);
    return cudaMemcpyAsync(out_tu, &e, sizeof(e), cudaMemcpyHostToDevice, stream);
  }
  bb::Params p = bb_params(tags, leaf_bbox, n, nullptr, ws, nullptr, nullptr);
  TB_LAUNCH(stream, "bb_export",
            (bb::bb_export<<<1, 1024, 0, stream>>>(p, (const bb::SumRec*)recs, b, suf_tiles, out_tu, out_su)));
  return cudaGetLastError();
}

cudaError_t bb_compose_launch(const void* allrecs, int maxb, const int* L, int g, int lo, int H, float4* init_clip,
                              int4* init_meta, cudaStream_t stream) {
  TB_LAUNCH(stream, "bb_compose",
            (bb::bb_compose<<<1, 256, 0, stream>>>((const bb::SumRec*)allrecs, maxb, L, g, lo, H, init_clip,
                                                   init_meta)));
  return cudaGetLastError();
}

cudaError_t bb_fixup_launch(int G, int g, int64_t off, int b_g, int min_L_after, int L_g, const float4* tu,
                            const float4* allsu, int maxb, const void* allpops, int maxp, const int* npops,
                            const void* myrecs, float4* out, cudaStream_t stream) {
  TB_LAUNCH(stream, "bb_fixup",
            (bb::bb_fixup<<<256, 256, 0, stream>>>(G, g, off, b_g, min_L_after, L_g, tu, allsu, maxb,
                                                   (const bb::BbPop*)allpops, maxp, npops,
                                                   (const bb::SumRec*)myrecs, out)));
  return cudaGetLastError();
}

}  // namespace tb
