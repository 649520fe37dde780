// paren_match kernel for sm_100a — one pass over the tags.
//
// Per tile of TILE = 4096 elements (256 threads x 16 contiguous elements):
//  1. 16-byte streaming load of the tags; one register walk per thread over
//     its 16 elements with a 4-bit-per-entry stack in a 64-bit register (the
//     k-elements-per-thread idea of §8).  It records, per element,
//     the in-thread parent (nibble) or "external", the in-thread partner of
//     every matched open, and the thread's Bic value (a_t, b_t) (§3).
//  2. Warp-shuffle + shared-memory scans of the thread Bic values, forward
//     (heights at each thread start) and reverse (which unmatched opens
//     survive the tile: the §7.1 slice rule P:231-233).
//  3. The tile aggregate is published at once (decoupled look-back);
//     the tile's stack slice Stk(enum(s)[p..p+w]) is written to the
//     workspace; thread-level owner lookups (binary lifting over warp-shuffled
//     low-water windows) resolve references to earlier threads of the tile.
//  4. Look-back gives the stack height H at the tile start; the low-water mark
//     max(H - a_T, 0) is published into a 32-ary hierarchy.
//  5. The needed top of the incoming stack (a_T + 1 entries; the k-suffix of
//     P:127) is materialised in shared memory from predecessors' slices found
//     by owner search (suffix relation P:131-138).
//  6. A second register pass resolves external references and writes parent
//     (Fig. 1 out) and match with 16-byte stores.
// See DESIGN.md §2 for the derivations (owner rule, relative heights).
#include <climits>
#include "stackscan.cuh"
#include "kernels.h"

namespace tb {
namespace pm {

constexpr int NT = 256;
constexpr int K = 16;
constexpr int TILE = NT * K;
constexpr int NW = NT / 32;
constexpr int RUNCAP = 32;
constexpr int SKIP = INT_MIN;

struct Smem {
  int inc[TILE + 1];        // incoming stack, inc[d] = entry at depth d from the top
  int win[NW][5][32];       // per-warp low-water windows: min l over lanes [j-2^k+1, j]
  int wmin[NW];             // per-warp min l
  int l[NT];                // thread relative low-water marks
  uint32_t uo[NT];          // per-thread unmatched-open masks
  int link[NT];             // reference to the entry just below a thread's first unmatched open
  int extv[K + 1][NT];      // extv[d][t]: index of the entry at depth d of thread t's start stack
  Bic wtot[NW];
  int runU[RUNCAP], runL[RUNCAP], runLo[RUNCAP], runHi[RUNCAP];
  int nruns, more;
  int tile;
  Bic excl;
};

// Warp 0: collect up to RUNCAP runs of the incoming stack, from height `cur`
// down to `lo`, each run being a contiguous piece of one predecessor's slice
// (owner rule); returns the height still to do (< lo when finished).
__device__ __forceinline__ int find_runs(Smem& s, const Ctrl& c, LwWindow& win, int cur, int& from,
                                         int lo, int init_lo) {
  const int lane = threadIdx.x & 31;
  int nr = 0;
  while (cur >= lo && nr < RUNCAP) {
    int LU = 0;
    const int U = owner_search_win(c, win, from, cur, LU);
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

struct Params {
  const uint8_t* tags;
  int64_t n;
  int32_t* match;
  int32_t* parent;
  int32_t* slice;  // [ntiles * TILE]
  Ctrl ctrl;
  Bic init;                   // prefix before the first element (shard mode)
  const int32_t* init_stack;  // entries at heights [init_lo, init.b)
  int init_lo;
  uint64_t* trace;            // optional per-tile phase timestamps (debug)
};

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PM_TRACE(slot)                                                     \
  do {                                                                     \
    if (p.trace && (threadIdx.x & 31) == 0) p.trace[(size_t)T * 16 + (slot)] = gtime(); \
  } while (0)

// Reference to the open at relative height x of the stack at the start of
// thread `tid`: an in-tile element offset (>= 0), or x itself (< 0) when the
// entry was pushed before the tile ("escaped"; resolved after look-back).
// Owner rule at thread granularity: the last thread V < tid with l_V <= x.
__device__ __forceinline__ int thread_ref(const Smem& s, const int (&w)[5], int l_me, uint32_t uo_me,
                                          int x, int lane, int warp) {
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
    if (s.wmin[W] <= x) {
      int p2 = 32;
#pragma unroll
      for (int k = 4; k >= 0; k--)
        if (p2 >= (1 << k) && s.win[W][k][p2 - 1] > x) p2 -= (1 << k);
      const int V = W * 32 + p2 - 1;
      return V * K + select_bit(s.uo[V], x - s.l[V]);
    }
  }
  return x;
}

__global__ void __launch_bounds__(NT, 4) paren_match_kernel(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) s.tile = (int)atomicAdd(p.ctrl.counter, 1u);
  __syncthreads();
  const int T = s.tile;
  const int64_t base = (int64_t)T * TILE;
  const int64_t tbase = base + (int64_t)tid * K;
  const bool full = base + TILE <= p.n;
  if (tid == 0) PM_TRACE(0);

  // ---- 1. load, classify, register walk -----------------------------------
  uint4 raw;
  if (full) {
    raw = ld_stream_v4(p.tags + tbase);
  } else {
    uint32_t wv[4] = {0, 0, 0, 0};
    for (int i = 0; i < K; i++) {
      const int64_t g = tbase + i;
      const uint32_t v = g < p.n ? p.tags[g] : 0u;
      wv[i >> 2] |= v << (8 * (i & 3));
    }
    raw = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
  uint32_t om, cm;
  classify16(raw, om, cm);

  // Thread stack as a bitmask of open positions (top = highest set bit).
  uint32_t S = 0;
  uint32_t plo = 0, phi = 0;  // nibble i: in-thread parent of element i (i < 8 / i >= 8)
  uint32_t mlo = 0, mhi = 0;  // nibble o: in-thread partner (close) of open o
  uint32_t ext = 0;           // element's parent lies before the thread
  uint32_t ucm = 0;           // closes with no in-thread open (pop the external stack)
#pragma unroll
  for (int i = 0; i < K; i++) {
    const uint32_t bit = 1u << i;
    const int top = 31 - __clz(S);  // -1 when the thread stack is empty
    if (i < 8) plo |= (uint32_t)(top & 15) << (4 * i);
    else phi |= (uint32_t)(top & 15) << (4 * (i - 8));
    ext |= S ? 0u : bit;
    const bool pop = (cm & bit) && S;
    ucm |= ((cm & bit) && !S) ? bit : 0u;
    const uint32_t pv = (uint32_t)i << (4 * (top & 7));
    mlo |= (pop && top < 8) ? pv : 0u;
    mhi |= (pop && top >= 8) ? pv : 0u;
    S = (om & bit) ? (S | bit) : (pop ? (S ^ (1u << top)) : S);
  }
  const uint32_t uo = S;         // opens unmatched inside the thread (left on its stack)
  const uint32_t mo = om & ~S;   // opens matched inside the thread
  const int a_t = __popc(ucm), b_t = __popc(uo);

  // ---- 2. forward / reverse Bic scans --------------------------------------
  const Bic v{a_t, b_t};
  Bic incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Bic o{__shfl_up_sync(0xffffffffu, incl.a, off), __shfl_up_sync(0xffffffffu, incl.b, off)};
    if (lane >= off) incl = bic_combine(o, incl);
  }
  Bic suf = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Bic o{__shfl_down_sync(0xffffffffu, suf.a, off), __shfl_down_sync(0xffffffffu, suf.b, off)};
    if (lane + off < 32) suf = bic_combine(suf, o);
  }
  if (lane == 31) s.wtot[warp] = incl;
  __syncthreads();
  Bic wpre{0, 0}, wsuf{0, 0}, tot{0, 0};
#pragma unroll
  for (int w = 0; w < NW; w++) {
    const Bic x = s.wtot[w];
    if (w < warp) wpre = bic_combine(wpre, x);
    if (w > warp) wsuf = bic_combine(wsuf, x);
    tot = bic_combine(tot, x);
  }
  Bic ex{__shfl_up_sync(0xffffffffu, incl.a, 1), __shfl_up_sync(0xffffffffu, incl.b, 1)};
  if (lane == 0) ex = Bic{0, 0};
  ex = bic_combine(wpre, ex);  // exclusive in-tile prefix of this thread
  Bic sx{__shfl_down_sync(0xffffffffu, suf.a, 1), __shfl_down_sync(0xffffffffu, suf.b, 1)};
  if (lane == 31) sx = Bic{0, 0};
  sx = bic_combine(sx, wsuf);  // exclusive in-tile suffix of this thread
  const int aT = tot.a;

  // ---- 3a. publish the aggregate (tile 0: inclusive) ----------------------
  if (tid == 0) PM_TRACE(1);
  if (tid == 0) {
    if (T == 0) st_release_u64(p.ctrl.desc, desc_pack(DESC_INC, bic_combine(p.init, tot)));
    else st_release_u64(p.ctrl.desc + T, desc_pack(DESC_AGG, tot));
  }

  // ---- 3b. slice (tile's unmatched opens, ascending) + match placeholders --
  const int r_t = ex.b - ex.a;  // relative height at thread start
  const int l_t = r_t - a_t;    // relative low-water mark of the thread
  {
    const int s_t = max(b_t - sx.a, 0);  // opens surviving to the tile end
    uint32_t m = uo;
    for (int k = 0; k < s_t; k++) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      const int64_t gi = tbase + bit;
      p.slice[base + (l_t + k + aT)] = (int32_t)gi;
      p.match[gi] = -1;  // placeholder; the tile holding the close overwrites it
    }
  }

  // ---- 3c. per-warp low-water windows for thread-level owner lookups ------
  int w[5];
  w[0] = l_t;
#pragma unroll
  for (int k = 1; k < 5; k++) {
    const int h = 1 << (k - 1);
    const int o = __shfl_up_sync(0xffffffffu, w[k - 1], h);
    w[k] = lane >= h ? min(w[k - 1], o) : w[k - 1];
  }
#pragma unroll
  for (int k = 0; k < 5; k++) s.win[warp][k][lane] = w[k];
  {
    const int o = __shfl_sync(0xffffffffu, w[4], 15);
    if (lane == 31) s.wmin[warp] = min(w[4], o);
  }
  s.l[tid] = l_t;
  s.uo[tid] = uo;
  __syncthreads();

  // ---- 4. warp 0: look-back, low-water publication, first owner runs ------
  //      (overlaps with the other warps' in-tile lookups below)
  int cur = 0, from = T, lo = 0;
  LwWindow lwin;
  if (warp == 0) {
    PM_TRACE(2);
    const Bic excl = (T == 0) ? p.init : lookback_warp(p.ctrl, T);
    PM_TRACE(3);
    if (lane == 0) publish_inclusive(p.ctrl, T, bic_combine(excl, tot), max(excl.b - aT, 0), T > 0);
    __syncwarp();
    named_bar_arrive(1, 64);  // warp 1 folds L_T into the hierarchy meanwhile
    PM_TRACE(4);
    if (lane == 0) s.excl = excl;
    lo = max(excl.b - 1 - aT, 0);
    lwin = lw_window_load(p.ctrl, T);
    cur = find_runs(s, p.ctrl, lwin, excl.b - 1, from, lo, p.init_lo);
    PM_TRACE(5);
  }
  if (warp == 1) PM_TRACE(6);
  const int top_ref = thread_ref(s, w, l_t, uo, r_t - 1, lane, warp);
  const int link_ref = thread_ref(s, w, l_t, uo, l_t - 1, lane, warp);
  s.link[tid] = link_ref;
  if (warp == 1) {
    named_bar_sync(1, 64);
    hierarchy_arrive(p.ctrl, T);
  }
  if (warp == 1) PM_TRACE(7);
  __syncthreads();
  if (tid == 0) PM_TRACE(8);
  const int H = s.excl.b;

  // ---- 5. materialise the needed top of the incoming stack ----------------
  for (int d = H + tid; d <= aT; d += NT) s.inc[d] = -1;  // below the root
  while (true) {
    const int nr = s.nruns;
    for (int r = 0; r < nr; r++) {
      const int U = s.runU[r], LU = s.runL[r], hlo = s.runLo[r], hhi = s.runHi[r];
      const int cnt = hhi - hlo + 1;
      const int32_t* src = U >= 0 ? p.slice + (int64_t)U * TILE : p.init_stack;
      for (int i = tid; i < cnt; i += NT) {
        const int h = hhi - i;
        s.inc[H - 1 - h] = ld_cg_s32(src + (h - LU));
      }
    }
    const int more = s.more;
    __syncthreads();
    if (more < max(H - 1 - aT, 0)) break;
    if (warp == 0) cur = find_runs(s, p.ctrl, lwin, cur, from, lo, p.init_lo);
    __syncthreads();
  }

  if (tid == 0) PM_TRACE(9);
  // ---- 6. entries of the stack at thread start that this thread pops -----
  {
    int ref = top_ref;
    for (int d = 0; d <= a_t; d++) {
      s.extv[d][tid] = ref >= 0 ? (int)(base + ref) : s.inc[-ref - 1];
      if (ref >= 0) {
        const int V = ref >> 4;
        const uint32_t below = s.uo[V] & ((1u << (ref & 15)) - 1u);
        ref = below ? (V << 4) + (31 - __clz(below)) : s.link[V];
      } else {
        ref -= 1;
      }
    }
  }

  // ---- 7. parent / match, 16-byte stores ------------------------------------
  {
    const int tb32 = (int)tbase;  // element indices fit in int32 (n <= 2^31 - 1)
    int dcur = 0;
    int val = s.extv[0][tid];
#pragma unroll
    for (int q = 0; q < K / 4; q++) {
      int pv[4], mv[4];
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int i = 4 * q + j;
        const uint32_t bit = 1u << i;
        const int pnib = (int)(((i < 8 ? plo : phi) >> (4 * (i & 7))) & 15u);
        const int mnib = (int)(((i < 8 ? mlo : mhi) >> (4 * (i & 7))) & 15u);
        const int local_par = tb32 + pnib;
        pv[j] = (ext & bit) ? val : local_par;
        int m = (om & bit) ? ((mo & bit) ? tb32 + mnib : SKIP) : -1;
        const bool uc = (ucm & bit) != 0u;
        m = (cm & bit) ? (uc ? val : local_par) : m;
        if (uc && val >= 0) p.match[val] = tb32 + i;  // open of an earlier thread / tile
        dcur += uc;
        if (uc) val = s.extv[dcur][tid];
        mv[j] = m;
      }
      if (full) {
        __stcs(reinterpret_cast<int4*>(p.parent + tbase) + q, make_int4(pv[0], pv[1], pv[2], pv[3]));
        if (((uo >> (4 * q)) & 15u) == 0) {
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
  }
  if (tid == 0) PM_TRACE(10);
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

cudaError_t pm_launch(const uint8_t* tags, int64_t n, int32_t* match, int32_t* parent, void* ws,
                      const ShardInit* init, cudaStream_t stream, uint64_t* trace) {
  if (n <= 0) return cudaSuccess;
  const int64_t ntiles = (n + pm::TILE - 1) / pm::TILE;
  CtrlLayout L(ntiles);
  cudaError_t err = cudaMemsetAsync(ws, 0, L.bytes, stream);
  if (err != cudaSuccess) return err;
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
  p.trace = trace;
  static bool configured = false;
  const int smem = (int)sizeof(pm::Smem);
  if (!configured) {
    err = cudaFuncSetAttribute(pm::paren_match_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    configured = true;
  }
  pm::paren_match_kernel<<<(unsigned)ntiles, pm::NT, smem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace tb
