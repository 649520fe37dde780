// paren_match kernel for sm_100a — one pass over the tags.
//
// Per tile of TILE = 4096 elements (256 threads x 16 contiguous elements):
//  1. 16-byte streaming load of the tags; per-thread Bic fold (§3)
//     with a 4-bit-per-entry register stack (the k-elements-per-thread idea of
//     §8, with the thread's stack in one 64-bit register).
//  2. Warp-shuffle + shared-memory scans of the thread Bic values, forward
//     (prefix heights) and reverse (which unmatched opens survive the tile,
//     the §7.1 slice rule P:231-233).
//  3. The tile aggregate is published at once; the tile's unmatched opens
//     (its stack slice, Stk(enum(s)[p..p+w]) P:229) are written to the
//     workspace; thread-level owner lookups resolve in-tile references.
//  4. Decoupled look-back gives the stack height H at the tile start; the
//     low-water mark max(H - a_T, 0) is published into a 32-ary hierarchy.
//  5. The needed top of the incoming stack (a_T + 1 entries, P:127 k-suffix)
//     is materialised in shared memory from predecessors' slices, found by
//     owner search (suffix relation P:131-138).
//  6. Sequential walk per thread produces parent (Fig. 1 out) and match; the
//     results are staged in shared memory and written with 16-byte stores.
// See DESIGN.md §2 for the derivations (F1 owner rule, relative heights).
#include <climits>
#include "stackscan.cuh"
#include "kernels.h"

namespace tb {
namespace pm {

constexpr int NT = 256;
constexpr int K = 16;
constexpr int TILE = NT * K;
constexpr int NW = NT / 32;
constexpr int LOGNT = 8;
constexpr int RUNCAP = 32;
constexpr int SKIP = INT_MIN;  // match slot filled by a later tile

struct Smem {
  int par[TILE];
  int mat[TILE];
  int inc[TILE + 1];           // incoming stack, inc[d] = entry at depth d
  int mn[LOGNT][NT];           // sparse table of thread low-water marks
  int link[NT];
  uint32_t uo[NT];             // per-thread unmatched-open masks
  Bic wtot[NW];
  int runU[RUNCAP], runL[RUNCAP], runLo[RUNCAP], runHi[RUNCAP];
  int nruns, more;
  int tile;
  Bic excl;
};

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
};

// Find the last thread V < t with l_V <= x (binary lifting on the sparse
// table).  Returns V or -1.
__device__ __forceinline__ int thread_owner(const Smem& s, int t, int x) {
  int pos = t;
#pragma unroll
  for (int k = LOGNT - 1; k >= 0; k--) {
    if (pos >= (1 << k) && s.mn[k][pos - 1] > x) pos -= (1 << k);
  }
  return pos - 1;
}

__global__ void __launch_bounds__(NT, 3) paren_match_kernel(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) s.tile = (int)atomicAdd(p.ctrl.counter, 1u);
  __syncthreads();
  const int T = s.tile;
  const int64_t base = (int64_t)T * TILE;
  const int64_t tbase = base + (int64_t)tid * K;
  const bool full = base + TILE <= p.n;

  // ---- 1. load + classify ------------------------------------------------
  uint4 raw;
  if (full) {
    raw = ld_stream_v4(p.tags + tbase);
  } else {
    uint32_t wv[4] = {0, 0, 0, 0};
    for (int i = 0; i < K; i++) {
      int64_t g = tbase + i;
      uint32_t v = g < p.n ? p.tags[g] : 0u;
      wv[i >> 2] |= v << (8 * (i & 3));
    }
    raw = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
  uint32_t om, cm;
  classify16(raw, om, cm);

  // per-thread Bic + unmatched-open mask (register nibble stack)
  int a_t = 0, sp = 0;
  uint64_t stk = 0;
#pragma unroll
  for (int i = 0; i < K; i++) {
    if ((om >> i) & 1u) {
      stk = (stk << 4) | (uint64_t)i;
      sp++;
    } else if ((cm >> i) & 1u) {
      if (sp) {
        stk >>= 4;
        sp--;
      } else {
        a_t++;
      }
    }
  }
  const int b_t = sp;
  uint32_t uo = 0;
  for (int j = 0; j < sp; j++) uo |= 1u << ((stk >> (4 * j)) & 15u);

  // ---- 2. forward / reverse Bic scans --------------------------------------
  Bic v{a_t, b_t};
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
    Bic x = s.wtot[w];
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
  const int aT = tot.a, bT = tot.b;

  // ---- 3a. publish the aggregate (tile 0: inclusive) ----------------------
  if (tid == 0) {
    if (T == 0) st_release_u64(p.ctrl.desc, desc_pack(DESC_INC, bic_combine(p.init, tot)));
    else st_release_u64(p.ctrl.desc + T, desc_pack(DESC_AGG, tot));
  }

  // ---- 3b. slice (tile's unmatched opens, ascending) + match placeholders --
  const int r_t = ex.b - ex.a;  // relative height at thread start
  const int l_t = r_t - a_t;    // relative low-water mark
  const int s_t = max(b_t - sx.a, 0);
  uint32_t tu = 0;  // tile-unmatched opens of this thread
  {
    uint32_t m = uo;
    for (int k = 0; k < s_t; k++) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      tu |= 1u << bit;
      const int64_t gi = tbase + bit;
      p.slice[base + (l_t + k + aT)] = (int32_t)gi;
      p.match[gi] = -1;  // placeholder; a later tile may overwrite
    }
  }
  s.uo[tid] = uo;
  s.mn[0][tid] = l_t;
  if (tu) __threadfence();
  __syncthreads();

  // ---- 3c. thread-level owner table -----------------------------------
#pragma unroll
  for (int k = 1; k < LOGNT; k++) {
    const int h = 1 << (k - 1);
    int m = s.mn[k - 1][tid];
    if (tid >= h) m = min(m, s.mn[k - 1][tid - h]);
    s.mn[k][tid] = m;
    __syncthreads();
  }
  // top of stack at thread start (height r_t - 1) and link (height l_t - 1)
  int top_ref, link_ref = 0;
  {
    int x = r_t - 1;
    int V = thread_owner(s, tid, x);
    top_ref = V >= 0 ? V * K + select_bit(s.uo[V], x - s.mn[0][V]) : x;
    if (b_t > 0) {
      x = l_t - 1;
      V = thread_owner(s, tid, x);
      link_ref = V >= 0 ? V * K + select_bit(s.uo[V], x - s.mn[0][V]) : x;
    }
  }
  s.link[tid] = link_ref;

  // ---- 4. look-back, low-water publication -------------------------------
  if (warp == 0) {
    Bic excl = (T == 0) ? p.init : lookback_warp(p.ctrl, T);
    if (T > 0 && lane == 0) st_release_u64(p.ctrl.desc + T, desc_pack(DESC_INC, bic_combine(excl, tot)));
    const int H = excl.b;
    publish_lowwater(p.ctrl, T, max(H - aT, 0));
    if (lane == 0) s.excl = excl;
  }
  __syncthreads();
  const int H = s.excl.b;

  // ---- 5. materialise the needed top of the incoming stack ----------------
  {
    const int need_lo = H - 1 - aT;  // lowest height referenced (may be < 0)
    const int lo = max(need_lo, 0);
    for (int d = H + tid; d <= aT; d += NT) s.inc[d] = -1;  // below the root
    int cur = H - 1, from = T;
    while (true) {
      if (warp == 0) {
        int nr = 0;
        while (cur >= lo && nr < RUNCAP) {
          int LU = 0;
          const int U = owner_search(p.ctrl, from, cur, LU);
          if (lane == 0) {
            s.runU[nr] = U;
            s.runHi[nr] = cur;
            if (U >= 0) {
              s.runL[nr] = LU;
              s.runLo[nr] = max(LU, lo);
            } else {
              s.runL[nr] = p.init_lo;
              s.runLo[nr] = lo;
            }
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
          s.more = cur >= lo;
        }
      }
      __syncthreads();
      const int nr = s.nruns;
      for (int r = 0; r < nr; r++) {
        const int U = s.runU[r], LU = s.runL[r], hlo = s.runLo[r], hhi = s.runHi[r];
        const int cnt = hhi - hlo + 1;
        if (U >= 0) {
          const int32_t* src = p.slice + (int64_t)U * TILE;
          for (int i = tid; i < cnt; i += NT) {
            const int h = hhi - i;
            s.inc[H - 1 - h] = ld_cg_s32(src + (h - LU));
          }
        } else {
          for (int i = tid; i < cnt; i += NT) {
            const int h = hhi - i;
            s.inc[H - 1 - h] = p.init_stack[h - LU];
          }
        }
      }
      const int more = s.more;
      __syncthreads();
      if (!more) break;
    }
  }

  // ---- 6. sequential walk: parent / match --------------------------------
  {
    int ref = top_ref;
    uint64_t st = 0;
    int depth = 0;
    const int e0 = tid * K;
#pragma unroll
    for (int i = 0; i < K; i++) {
      const int e = e0 + i;
      const int64_t gi = tbase + i;
      int par;
      if (depth) par = (int)(tbase + (int)(st & 15u));
      else par = ref >= 0 ? (int)(base + ref) : s.inc[-ref - 1];
      s.par[e] = par;
      if ((om >> i) & 1u) {
        st = (st << 4) | (uint64_t)i;
        depth++;
        // A tile-unmatched open is matched (if ever) by a later tile, which
        // writes global match[] itself; every other open's slot is written
        // by its close (same thread, or a later thread of this tile).
        if ((tu >> i) & 1u) s.mat[e] = SKIP;
      } else if ((cm >> i) & 1u) {
        if (depth) {
          const int o = (int)(st & 15u);
          st >>= 4;
          depth--;
          s.mat[e] = (int)(tbase + o);
          s.mat[e0 + o] = (int)gi;
        } else {
          s.mat[e] = par;
          if (par >= 0) {
            if (ref >= 0) {
              s.mat[ref] = (int)gi;
            } else {
              p.match[par] = (int)gi;  // open lives in an earlier tile
            }
          }
          // step one entry down the stack at thread start
          if (ref >= 0) {
            const int V = ref / K;
            const uint32_t below = s.uo[V] & ((1u << (ref % K)) - 1u);
            ref = below ? V * K + (31 - __clz(below)) : s.link[V];
          } else {
            ref -= 1;
          }
        }
      } else {
        s.mat[e] = -1;
      }
    }
  }
  __syncthreads();

  // ---- 7. stores -----------------------------------------------------------
  if (full) {
    int4* gpar = reinterpret_cast<int4*>(p.parent + base);
    int4* gmat = reinterpret_cast<int4*>(p.match + base);
    const int4* spar = reinterpret_cast<const int4*>(s.par);
    const int4* smat = reinterpret_cast<const int4*>(s.mat);
#pragma unroll
    for (int j = 0; j < TILE / 4 / NT; j++) {
      const int q = j * NT + tid;
      __stcs(gpar + q, spar[q]);
      const int4 m = smat[q];
      if (m.x != SKIP && m.y != SKIP && m.z != SKIP && m.w != SKIP) {
        __stcs(gmat + q, m);
      } else {
        int32_t* gm = p.match + base + 4 * q;
        if (m.x != SKIP) gm[0] = m.x;
        if (m.y != SKIP) gm[1] = m.y;
        if (m.z != SKIP) gm[2] = m.z;
        if (m.w != SKIP) gm[3] = m.w;
      }
    }
  } else {
    for (int e = tid; e < TILE; e += NT) {
      const int64_t gi = base + e;
      if (gi >= p.n) break;
      p.parent[gi] = s.par[e];
      if (s.mat[e] != SKIP) p.match[gi] = s.mat[e];
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
