// paren_match for sm_100a: reduce pass + finish pass over the tags.
//
// Tile = 256 threads x 16 contiguous elements = 4096 elements.
//
// pm_reduce (pass 1, reads 1 B/element):
//   register walk per thread -> Bic (a_t, b_t) (§3); forward and
//   reverse block scans; the tile's stack slice Stk(enum(s)[p..p+w]) (§7.1
//   its unmatched opens, ascending) is written to the workspace and
//   each of those opens gets a -1 placeholder in match[]; decoupled look-back
//   (single pass over the tiles, the paper's future-work item P:381) gives the
//   stack height H at the tile start; the low-water mark L = max(H - a_T, 0)
//   is published into a 32-ary min hierarchy.
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
#include <cstdlib>
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
  const int32_t* init_stack;  // entries at heights [init_lo, init.b)
  int init_lo;
  int dbg;                    // debug: bit0 skip look-back, bit1 skip hierarchy, bit2 skip slice
};

// ----------------------------------------------------------------------------
// pass 1
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) pm_reduce(Params p) {
  __shared__ Bic wtot[NW];
  __shared__ int s_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = (int)atomicAdd(p.ctrl.counter, 1u);  // issue order = tile order
  __syncthreads();
  const int T = s_tile;
  const int64_t base = (int64_t)T * TILE;
  const int64_t tbase = base + (int64_t)tid * K;
  const bool full = base + TILE <= p.n;

  const Walk16 w = walk16(load_tags16(p.tags, p.n, tbase, full));
  const int a_t = __popc(w.ucm), b_t = __popc(w.S);
  Bic ex, sx, tot;
  block_bic_scans<NW>(Bic{a_t, b_t}, wtot, ex, sx, tot, true);
  if (tid == 0) {
    if (T == 0) st_release_u64(p.ctrl.desc, desc_pack(DESC_INC, bic_combine(p.init, tot)));
    else st_release_u64(p.ctrl.desc + T, desc_pack(DESC_AGG, tot));
  }
  // slice: this thread's unmatched opens that survive to the tile end sit at
  // relative heights l_t + k, slice position l_t + k + a_T.
  {
    const int l_t = ex.b - ex.a - a_t;
    const int s_t = max(b_t - sx.a, 0);
    uint32_t m = w.S;
    for (int k = 0; k < ((p.dbg & 4) ? 0 : s_t); k++) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      const int gi = (int)(tbase + bit);
      p.slice[base + (l_t + k + tot.a)] = gi;
      p.match[gi] = -1;  // placeholder: a later tile's close may overwrite it in pass 2
    }
  }
  if (warp == 0) {
    const Bic excl = (T == 0 || (p.dbg & 1)) ? p.init : lookback_warp(p.ctrl, T);
    if (lane == 0) {
      p.ctrl.hstart[T] = excl.b;
      publish_inclusive(p.ctrl, T, bic_combine(excl, tot), max(excl.b - tot.a, 0), T > 0);
    }
    if (!(p.dbg & 2)) hierarchy_arrive(p.ctrl, T);
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

__global__ void __launch_bounds__(NT, 4) pm_finish(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockIdx.x;
  const int64_t base = (int64_t)T * TILE;
  const int64_t tbase = base + (int64_t)tid * K;
  const bool full = base + TILE <= p.n;

  const Walk16 w = walk16(load_tags16(p.tags, p.n, tbase, full));
  const int a_t = __popc(w.ucm), b_t = __popc(w.S);
  Bic ex, sx, tot;
  block_bic_scans<NW>(Bic{a_t, b_t}, s.wtot, ex, sx, tot, false);
  const int aT = tot.a;
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
  const int H = __ldg(p.ctrl.hstart + T);
  const int lo = max(H - 1 - aT, 0);  // lowest referenced height that exists
  int cur = H - 1, from = T;
  __syncthreads();

  if (warp == 0) cur = find_runs(s, p.ctrl, cur, from, lo, p.init_lo);
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
        s.inc[H - 1 - h] = __ldg(src + (h - LU));
      }
    }
    const int more = s.more;
    __syncthreads();
    if (more < lo) break;
    if (warp == 0) cur = find_runs(s, p.ctrl, cur, from, lo, p.init_lo);
    __syncthreads();
  }

  // entries of the stack at this thread's start that it pops (depths 0..a_t)
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

  // parent / match
  const uint32_t mo = w.om & ~w.S;
  const int tb32 = (int)tbase;
  int dcur = 0;
  int val = s.extv[0][tid];
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
      if (uc && val >= 0) p.match[val] = tb32 + i;  // partner opened in an earlier thread / tile
      dcur += uc;
      if (uc) val = s.extv[dcur][tid];
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
                      const ShardInit* init, cudaStream_t stream) {
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
  {
    const char* e = getenv("TB_DEBUG_PM");
    p.dbg = e ? atoi(e) : 0;
  }
  static bool configured = false;
  const int smem = (int)sizeof(pm::Smem);
  if (!configured) {
    err = cudaFuncSetAttribute(pm::pm_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    configured = true;
  }
  TB_LAUNCH(stream, "pm_reduce", (pm::pm_reduce<<<(unsigned)ntiles, pm::NT, 0, stream>>>(p)));
  TB_LAUNCH(stream, "pm_finish", (pm::pm_finish<<<(unsigned)ntiles, pm::NT, smem, stream>>>(p)));
  return cudaGetLastError();
}

}  // namespace tb
