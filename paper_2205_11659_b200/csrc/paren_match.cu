// paren_match for sm_100a: reduce pass + finish pass over the tags.
//
// Tile = 256 threads x 16 contiguous elements = 4096 elements.
//
// pm_reduce (pass 1, reads 1 B/element):
//   register walk per thread -> Bic (a_t, b_t) (§3); forward and
//   reverse warp scans; the tile's stack slice Stk(enum(s)[p..p+w]) (§7.1
//   its unmatched opens, ascending) is written to the workspace and
//   the tile's Bic value published.  tile_scan (one CTA, tilescan.cu) turns the
//   tile values into the stack height H at each tile start and the low-water
//   marks L = max(H - a_T, 0) with their 32-ary min hierarchy.  (A single-pass
//   decoupled look-back, the paper's future-work item P:381, was built in
//   round 1 and measured slower than reduce + scan at these sizes.)
// pm_finish (pass 2, reads 1 B/element, writes 8 B/element):
//   the same register walk; thread-level owner lookups resolve references to
//   earlier threads of the tile; the needed top of the incoming stack (a_T+1
//   entries, the k-suffix of P:127) is copied from predecessors' slices found
//   by owner search (suffix relation P:131-138: the entry at height h at the
//   start of tile T lives in the last tile U < T with L_U <= h, at slice
//   position h - L_U); a second register pass writes parent (Fig. 1 out,
//   P:78-90) and match with 16-byte stores.  Cross-tile partners are
//   written into the earlier tile's match[] slot (overwriting pass 1's -1).
// No inter-CTA waiting in pass 2: pass 1's results are complete at launch.
#include <climits>
#include "kernels.h"
#include "stackscan.cuh"
#include "tile_common.cuh"

namespace tb {
namespace pm {

constexpr int NT = 256;
constexpr int K = 16;
constexpr int TILE = NT * K;
constexpr int NW = NT / 32;
constexpr int RUNCAP = 32;
constexpr int SKIP = INT_MIN;

struct Params {
  const uint8_t* tags;
  int64_t n;
  int32_t* match;
  int32_t* parent;
  int32_t* slice;  // [ntiles * TILE]
  Ctrl ctrl;
  Bic init;                   // prefix before the first element (shard mode)
  const int32_t* init_stack;  // entries at heights [init_lo, init.b) (global indices)
  int init_lo;
  int64_t offset;             // global index of element 0 (shard mode)
  int2* pairs;                // shard mode: (open, close) for closes that pop init_stack entries
};

// ----------------------------------------------------------------------------
// pass 1
// ----------------------------------------------------------------------------
// One warp per tile, 128 consecutive elements per lane: the lane's Bic from a
// 4-element table, warp shuffles for the scans (no block barrier).  A lane
// whose bottom s_l unmatched opens survive the tile finds them with a second
// table, walking backwards 4 elements at a time (common.cuh unm32).
constexpr int RL = TILE / 32;  // elements per lane in pm_reduce
__global__ void __launch_bounds__(256) pm_reduce(Params p) {
  __shared__ uint8_t bic4[256];  // Bic of 4 elements: index = open nibble | close nibble << 4; a | b << 4
  __shared__ uint8_t unm4[UNM4_ENTRIES];
  const int lane = threadIdx.x & 31;
  {
    const int t = threadIdx.x;
    Bic v{0, 0};
#pragma unroll
    for (int j = 0; j < 4; j++) v = bic_combine(v, Bic{(t >> (4 + j)) & 1, (t >> j) & 1});
    bic4[t] = (uint8_t)(v.a | (v.b << 4));
    unm4_fill(unm4, t, 256);
  }
  __syncthreads();
  const int ntiles = (int)((p.n + TILE - 1) / TILE);
  const int T = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (T >= ntiles) return;
  const int64_t base = (int64_t)T * TILE, lbase = base + (int64_t)lane * RL;
  uint32_t om[RL / 32], cm[RL / 32];
  {
    uint4 raw[RL / 16];
    // L1-allocating loads: the lane stride is 128 B, so the first load brings
    // the warp's 4 KB into L1 and the other seven hit it
#pragma unroll
    for (int q = 0; q < RL / 16; q++) {
      const int64_t g = lbase + 16 * q;
      raw[q] = g + 16 <= p.n ? __ldg(reinterpret_cast<const uint4*>(p.tags + g)) : load_tags16(p.tags, p.n, g, false);
    }
#pragma unroll
    for (int q = 0; q < RL / 16; q++) {
      uint32_t o, c;
      classify16(raw[q], o, c);
      if (q & 1) {
        om[q >> 1] |= o << 16;
        cm[q >> 1] |= c << 16;
      } else {
        om[q >> 1] = o;
        cm[q >> 1] = c;
      }
    }
  }
  Bic lb{0, 0};
#pragma unroll
  for (int w = 0; w < RL / 32; w++) {
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const uint32_t e = bic4[((om[w] >> (4 * q)) & 15u) | (((cm[w] >> (4 * q)) & 15u) << 4)];
      lb = bic_combine(lb, Bic{(int)(e & 15u), (int)(e >> 4)});
    }
  }
  Bic incl = lb, suf = lb;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const Bic a{__shfl_up_sync(0xffffffffu, incl.a, off), __shfl_up_sync(0xffffffffu, incl.b, off)};
    if (lane >= off) incl = bic_combine(a, incl);
    const Bic b{__shfl_down_sync(0xffffffffu, suf.a, off), __shfl_down_sync(0xffffffffu, suf.b, off)};
    if (lane + off < 32) suf = bic_combine(suf, b);
  }
  const Bic tot{__shfl_sync(0xffffffffu, incl.a, 31), __shfl_sync(0xffffffffu, incl.b, 31)};
  Bic ex{__shfl_up_sync(0xffffffffu, incl.a, 1), __shfl_up_sync(0xffffffffu, incl.b, 1)};
  Bic sx{__shfl_down_sync(0xffffffffu, suf.a, 1), __shfl_down_sync(0xffffffffu, suf.b, 1)};
  if (lane == 0) ex = Bic{0, 0};
  if (lane == 31) sx = Bic{0, 0};
  if (lane == 0) p.ctrl.agg[T] = make_int2(tot.a, tot.b);  // the tile scan turns these into heights
  // slice: this lane's unmatched opens that survive to the tile end sit at
  // relative heights l + k, slice position l + k + a_T (k = rank from the bottom)
  const int l = ex.b - ex.a - lb.a;
  const int s_l = max(lb.b - sx.a, 0);
  if (s_l > 0) {
    // the lane's unmatched opens (backward, 4 at a time); the bottom s_l survive
    uint32_t um[RL / 32];
    int P = 0;
#pragma unroll
    for (int w = RL / 32 - 1; w >= 0; w--) um[w] = unm32(unm4, om[w], cm[w], P);
    int k = 0;
#pragma unroll
    for (int w = 0; w < RL / 32; w++) {
      uint32_t m = um[w];
      while (m && k < s_l) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const int64_t x = lbase + 32 * w + j;
        p.slice[base + (l + k + tot.a)] = (int)(p.offset + x);
        k++;
      }
    }
  }
}

// ----------------------------------------------------------------------------
// pass 2
// ----------------------------------------------------------------------------
struct Smem {
  int inc[TILE + 1];     // incoming stack: inc[d] = entry at depth d from the top
  int extv[K + 1][NT];   // extv[d][t] = entry at depth d of the stack at thread t's start
  int win[NW][5][32];    // per-warp low-water windows
  int wmin[NW];
  int l[NT];
  uint32_t uo[NT];
  int link[NT];
  Bic wtot[NW];
  int runU[RUNCAP], runL[RUNCAP], runLo[RUNCAP], runHi[RUNCAP];
  int nruns, more;
};

// Warp 0: up to RUNCAP runs of the incoming stack from height `cur` down to
// `lo`; a run is a contiguous piece of one predecessor's slice.
__device__ __forceinline__ int find_runs(Smem& s, const Ctrl& c, int cur, int& from, int lo, int init_lo) {
  const int lane = threadIdx.x & 31;
  int nr = 0;
  while (cur >= lo && nr < RUNCAP) {
    int LU = 0;
    const int U = owner_search_done(c, from, cur, LU);
    if (lane == 0) {
      s.runU[nr] = U;
      s.runHi[nr] = cur;
      s.runL[nr] = U >= 0 ? LU : init_lo;
      s.runLo[nr] = U >= 0 ? max(LU, lo) : lo;
    }
    if (U < 0) {
      cur = lo - 1;
    } else {
      cur = LU - 1;
      from = U;
    }
    nr++;
  }
  if (lane == 0) {
    s.nruns = nr;
    s.more = cur;
  }
  return cur;
}

#ifndef PM_FINISH_MINB
#define PM_FINISH_MINB 4  // CTAs per SM (64 registers)
#endif
template <bool SHARD>
__global__ void __launch_bounds__(NT, PM_FINISH_MINB) pm_finish(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockIdx.x;
  const int64_t base = (int64_t)T * TILE;
  const int64_t tbase = base + (int64_t)tid * K;
  const bool full = base + TILE <= p.n;

  const uint4 raw = load_tags16(p.tags, p.n, tbase, full);
  // The incoming-stack range needs only H and the tile's a_T, both published by
  // pass 1 (agg[T] is this tile's Bic), so warp 0 starts the owner search
  // while the tag loads are in flight; its L2 round trips overlap the walk and
  // the block scan instead of following them.
  const int H = __ldg(p.ctrl.hstart + T);
  const int aT = __ldg(p.ctrl.agg + T).x;
  const int lo = max(H - 1 - aT, 0);  // lowest referenced height that exists
  int cur = H - 1, from = T;
  if (warp == 0) cur = find_runs(s, p.ctrl, cur, from, lo, p.init_lo);
  const Walk16 w = walk16(raw);
  const int a_t = __popc(w.ucm), b_t = __popc(w.S);
  Bic ex, sx, tot;
  block_bic_scans<NW>(Bic{a_t, b_t}, s.wtot, ex, sx, tot, false);
  const int r_t = ex.b - ex.a;
  const int l_t = r_t - a_t;
  (void)b_t;

  int wl[5];
  lane_windows(l_t, wl);
#pragma unroll
  for (int k = 0; k < 5; k++) s.win[warp][k][lane] = wl[k];
  {
    const int o = __shfl_sync(0xffffffffu, wl[4], 15);
    if (lane == 31) s.wmin[warp] = min(wl[4], o);
  }
  s.l[tid] = l_t;
  s.uo[tid] = w.S;
  __syncthreads();

  const int top_ref = thread_ref<NW, K>(wl, l_t, w.S, r_t - 1, s.win, s.wmin, s.l, s.uo);
  s.link[tid] = thread_ref<NW, K>(wl, l_t, w.S, l_t - 1, s.win, s.wmin, s.l, s.uo);
  for (int d = H + tid; d <= aT; d += NT) s.inc[d] = -1;  // below the root
  __syncthreads();

  // materialise the needed top of the incoming stack
  while (true) {
    const int nr = s.nruns;
    for (int r = 0; r < nr; r++) {
      const int U = s.runU[r], LU = s.runL[r], hlo = s.runLo[r], hhi = s.runHi[r];
      const int cnt = hhi - hlo + 1;
      const int32_t* src = U >= 0 ? p.slice + (int64_t)U * TILE : p.init_stack;
      for (int i = tid; i < cnt; i += NT) {
        const int h = hhi - i;
        const int v = __ldg(src + (h - LU));
        s.inc[H - 1 - h] = U >= 0 ? v : -(v + 2);  // init-stack entries are tagged (<= -2)
      }
    }
    const int more = s.more;
    __syncthreads();
    if (more < lo) break;
    if (warp == 0) cur = find_runs(s, p.ctrl, cur, from, lo, p.init_lo);
    __syncthreads();
  }

  // entries of the stack at this thread's start that it pops (depths 0..a_t):
  // one device, their global indices (-1: root); shard mode, references
  // (>= 0 in-tile element, < 0 incoming depth -ref-1) resolved where used
  const int gbase0 = (int)(p.offset + base);
  {
    // in-tile entries first (owner chain), then consecutive incoming depths
    int ref = top_ref, d = 0;
    for (; d <= a_t && ref >= 0; d++) {
      s.extv[d][tid] = SHARD ? ref : gbase0 + ref;
      const int V = ref >> 4;
      const uint32_t below = s.uo[V] & ((1u << (ref & 15)) - 1u);
      ref = below ? (V << 4) + (31 - __clz(below)) : s.link[V];
    }
    for (; d <= a_t; d++, ref--) s.extv[d][tid] = SHARD ? ref : s.inc[-ref - 1];
  }

  // parent / match
  const uint32_t mo = w.om & ~w.S;
  const int tb32 = (int)(p.offset + tbase);  // global indices fit in int32 (N <= 2^31 - 1)
  const int gbase = (int)(p.offset + base);
  // value of a reference: global index, -1 for the root, or (shard mode) an
  // entry of the stack provided by the exchange
  auto resolve = [&](int ref, bool& from_init) -> int {
    from_init = false;
    if (ref >= 0) return gbase + ref;
    const int e = s.inc[-ref - 1];
    if (SHARD && e <= -2) {
      from_init = true;
      return -e - 2;
    }
    return e;
  };
  int dcur = 0;
  int ref = s.extv[0][tid];
  bool vinit;
  int val = SHARD ? resolve(ref, vinit) : ref;
#pragma unroll
  for (int q = 0; q < K / 4; q++) {
    int pv[4], mv[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int i = 4 * q + j;
      const uint32_t bit = 1u << i;
      const int local_par = tb32 + nib(w.plo, w.phi, i);
      pv[j] = (w.ext & bit) ? val : local_par;
      int m = (w.om & bit) ? ((mo & bit) ? tb32 + nib(w.mlo, w.mhi, i) : SKIP) : -1;
      const bool uc = (w.ucm & bit) != 0u;
      m = (w.cm & bit) ? (uc ? val : local_par) : m;
      dcur += uc;
      if (uc) {
        ref = s.extv[dcur][tid];
        val = SHARD ? resolve(ref, vinit) : ref;
      }
      mv[j] = m;
    }
    if (full) {
      __stcs(reinterpret_cast<int4*>(p.parent + tbase) + q, make_int4(pv[0], pv[1], pv[2], pv[3]));
      if (((w.S >> (4 * q)) & 15u) == 0) {
        __stcs(reinterpret_cast<int4*>(p.match + tbase) + q, make_int4(mv[0], mv[1], mv[2], mv[3]));
      } else {
#pragma unroll
        for (int j = 0; j < 4; j++)
          if (mv[j] != SKIP) p.match[tbase + 4 * q + j] = mv[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int64_t g = tbase + 4 * q + j;
        if (g < p.n) {
          p.parent[g] = pv[j];
          if (mv[j] != SKIP) p.match[g] = mv[j];
        }
      }
    }
  }
  // closes whose partner opened in an earlier thread / tile write match[open]
  // (the d-th such close pops the entry at depth d of the thread's start stack)
  {
    uint32_t q = w.ucm;
    int d = 0;
#pragma unroll 1
    while (q) {
      const int i = __ffs(q) - 1;
      q &= q - 1;
      const int r = s.extv[d][tid];
      bool from_init = false;
      const int v = SHARD ? resolve(r, from_init) : r;
      if (v >= 0) {
        if (!SHARD || !from_init) {
          p.match[v - p.offset] = tb32 + i;
        } else {  // partner lives in an earlier shard: record (open, close) for the exchange
          const int k = p.init.b - H + (-r - 1);
          p.pairs[k] = make_int2(v, tb32 + i);
        }
      }
      d++;
    }
  }
  // opens never closed (R4) get match = -1: this tile's slice entries that
  // survive to the end of the stream (F1), its bottom min(b_T, smin_T - L_T);
  // nothing else writes those slots
  if (warp == NW - 1) {
    const int L = (int)__ldg(p.ctrl.lw + T) - 1;
    const int bT = __ldg(p.ctrl.agg + T).y;
    const int sm = __ldg(p.ctrl.smin + T);
    const int surv = min(bT, max(sm == INT_MAX ? bT : sm - L, 0));
    for (int k = lane; k < surv; k += 32) p.match[__ldcg(p.slice + (int64_t)T * TILE + k) - p.offset] = -1;
  }
}

// Chunk summary for sharding: the chunk's final stack (its unmatched opens,
// bottom to top, global indices) = heights [0, b) of the stack after the last
// tile.  By the owner rule (F1) tile U's slice entries that survive to the end
// are its bottom min(b_U, smin_U - L_U) ones, at heights L_U + k; the ranges of
// different tiles are disjoint, so each tile copies its survivors into place
// (one warp per tile; pm_finish marks never-closed opens by the same rule).
__global__ void __launch_bounds__(256) pm_summary(Params p, int ntiles, int32_t* hdr, int32_t* opens) {
  const int lane = threadIdx.x & 31;
  const int U = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (U == 0 && lane == 0) {
    const int2 t2 = __ldcg(p.ctrl.total);  // Bic value of the chunk (tile scan)
    hdr[0] = t2.x;
    hdr[1] = t2.y;
  }
  if (U >= ntiles) return;
  const int L = (int)__ldg(p.ctrl.lw + U) - 1;
  const int bU = __ldg(p.ctrl.agg + U).y;
  const int sm = __ldg(p.ctrl.smin + U);
  const int surv = min(bU, max(sm == INT_MAX ? bU : sm - L, 0));
  for (int k = lane; k < surv; k += 32) opens[L + k] = __ldcg(p.slice + (int64_t)U * TILE + k);
}

}  // namespace pm

size_t pm_workspace_bytes(int64_t n) {
  const int64_t ntiles = (n + pm::TILE - 1) / pm::TILE;
  CtrlLayout L(ntiles);
  return L.bytes + CtrlLayout::align256(sizeof(int32_t) * (size_t)ntiles * pm::TILE);
}

size_t pm_ctrl_bytes(int64_t n) {
  const int64_t ntiles = (n + pm::TILE - 1) / pm::TILE;
  return CtrlLayout(ntiles).bytes;
}

static pm::Params pm_params(const uint8_t* tags, int64_t n, int32_t* match, int32_t* parent, void* ws,
                            const ShardInit* init) {
  const int64_t ntiles = (n + pm::TILE - 1) / pm::TILE;
  CtrlLayout L(ntiles);
  pm::Params p;
  p.tags = tags;
  p.n = n;
  p.match = match;
  p.parent = parent;
  p.slice = (int32_t*)((char*)ws + L.bytes);
  p.ctrl = L.bind(ws);
  p.init = init ? Bic{init->a, init->h} : Bic{0, 0};
  p.init_stack = init ? init->stack : nullptr;
  p.init_lo = init ? init->lo : 0;
  p.offset = init ? init->offset : 0;
  p.pairs = init ? init->pairs : nullptr;
  return p;
}

static cudaError_t pm_configure() {
  if (once_per_device(0)) {
    cudaError_t err = cudaFuncSetAttribute(pm::pm_finish<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)sizeof(pm::Smem));
    if (err == cudaSuccess)
      err = cudaFuncSetAttribute(pm::pm_finish<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(pm::Smem));

    if (err != cudaSuccess) return err;
  }
  return cudaSuccess;
}

// tile scan (heights from the prefix `init`); the per-tile aggregates and
// slices of pm_reduce do not depend on `init`, so the shard protocol's phase 2
// reuses phase 1's
cudaError_t pm_rescan_launch(int64_t n, int32_t* match, void* ws, const ShardInit* init, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int64_t ntiles = (n + pm::TILE - 1) / pm::TILE;
  pm::Params p = pm_params(nullptr, n, match, nullptr, ws, init);
  return tile_scan_launch(p.ctrl, ntiles, p.init.a, p.init.b, stream);
}

cudaError_t pm_reduce_only_launch(const uint8_t* tags, int64_t n, int32_t* match, void* ws, const ShardInit* init,
                                  cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int64_t ntiles = (n + pm::TILE - 1) / pm::TILE;
  pm::Params p = pm_params(tags, n, match, nullptr, ws, init);
  cudaError_t err = pm_configure();
  if (err != cudaSuccess) return err;
  TB_LAUNCH(stream, "pm_reduce", (pm::pm_reduce<<<(unsigned)((ntiles + 7) / 8), 256, 0, stream>>>(p)));
  return cudaGetLastError();
}

cudaError_t pm_reduce_launch(const uint8_t* tags, int64_t n, int32_t* match, void* ws, const ShardInit* init,
                             cudaStream_t stream) {
  cudaError_t err = pm_reduce_only_launch(tags, n, match, ws, init, stream);
  if (err != cudaSuccess) return err;
  return pm_rescan_launch(n, match, ws, init, stream);
}

cudaError_t pm_finish_launch(const uint8_t* tags, int64_t n, int32_t* match, int32_t* parent, void* ws,
                             const ShardInit* init, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  cudaError_t err = pm_configure();
  if (err != cudaSuccess) return err;
  const int64_t ntiles = (n + pm::TILE - 1) / pm::TILE;
  pm::Params p = pm_params(tags, n, match, parent, ws, init);
  if (p.init_stack == nullptr && p.pairs == nullptr)  // no stack provided by a shard exchange
    TB_LAUNCH(stream, "pm_finish", (pm::pm_finish<false><<<(unsigned)ntiles, pm::NT, sizeof(pm::Smem), stream>>>(p)));
  else
    TB_LAUNCH(stream, "pm_finish", (pm::pm_finish<true><<<(unsigned)ntiles, pm::NT, sizeof(pm::Smem), stream>>>(p)));
  return cudaGetLastError();
}

cudaError_t pm_summary_launch(const uint8_t* tags, int64_t n, void* ws, int32_t* hdr, int32_t* opens,
                              cudaStream_t stream) {
  cudaError_t err = pm_configure();
  if (err != cudaSuccess) return err;
  const int64_t ntiles = (n + pm::TILE - 1) / pm::TILE;
  if (ntiles == 0) return cudaMemsetAsync(hdr, 0, 8, stream);
  pm::Params p = pm_params(tags, n, nullptr, nullptr, ws, nullptr);
  TB_LAUNCH(stream, "pm_summary",
            (pm::pm_summary<<<(unsigned)((ntiles + 7) / 8), 256, 0, stream>>>(p, (int)ntiles, hdr, opens)));
  return cudaGetLastError();
}

cudaError_t pm_launch(const uint8_t* tags, int64_t n, int32_t* match, int32_t* parent, void* ws,
                      const ShardInit* init, cudaStream_t stream) {
  cudaError_t err = pm_reduce_launch(tags, n, match, ws, init, stream);
  if (err == cudaSuccess) err = pm_finish_launch(tags, n, match, parent, ws, init, stream);
  return err;
}

}  // namespace tb
