// Tile-level scan of the bicyclic monoid (§3) between the reduce and
// finish passes.  Each tile's reduce pass only publishes its Bic value (no
// inter-tile waiting); this single-CTA kernel turns them into, per tile, the
// stack height at its start H_T (exclusive prefix .b), its low-water mark
// L_T = max(H_T - a_T, 0), and the 32-ary min hierarchy over L used by the
// owner search (F1).  Two warp-shuffle passes over each warp's contiguous
// range of tiles with a block-level exclusive scan of the warp totals in
// between — a reduce-then-scan at tile granularity.
#include <climits>
#include "kernels.h"
#include "stackscan.cuh"

namespace tb {
namespace ts {

constexpr int NT = 1024, NW = NT / 32;

__device__ __forceinline__ Bic warp_incl_scan(Bic v, int lane) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Bic o{__shfl_up_sync(0xffffffffu, v.a, off), __shfl_up_sync(0xffffffffu, v.b, off)};
    if (lane >= off) v = bic_combine(o, v);
  }
  return v;
}

__global__ void __launch_bounds__(NT) tile_scan(Ctrl c, int ntiles, Bic init, int64_t* apre) {
  __shared__ Bic wt[NW];
  __shared__ int wmin[NW];
  __shared__ long long wsum[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int span = ((ntiles + NW - 1) / NW + 31) & ~31;
  const int t0 = warp * span, t1 = min(t0 + span, ntiles);
  // pass A: total of this warp's range
  Bic carry{0, 0};
  long long asum = 0;  // sum of (a_T + 1) over the warp's range (apre)
  for (int t = t0; t < t1; t += 32) {
    const int i = t + lane;
    const int2 g = i < t1 ? __ldcg(c.agg + i) : make_int2(0, 0);
    const Bic x = warp_incl_scan(Bic{g.x, g.y}, lane);
    const Bic last{__shfl_sync(0xffffffffu, x.a, 31), __shfl_sync(0xffffffffu, x.b, 31)};
    carry = bic_combine(carry, last);
    if (apre) asum += __reduce_add_sync(0xffffffffu, i < t1 ? (unsigned)(g.x + 1) : 0u);
  }
  if (lane == 0) {
    wt[warp] = carry;
    wsum[warp] = asum;
  }
  __syncthreads();
  long long abase = 0;
  if (apre) {
    for (int w = 0; w < warp; w++) abase += wsum[w];
    if (warp == NW - 1 && lane == 0) apre[ntiles] = abase + asum;
  }
  Bic pre = init;
  for (int w = 0; w < warp; w++) pre = bic_combine(pre, wt[w]);
  if (warp == NW - 1 && lane == 0) {
    Bic tot = init;
    for (int w = 0; w < NW; w++) tot = bic_combine(tot, wt[w]);
    *c.total = make_int2(tot.a, tot.b);
  }
  // pass B: exclusive prefix of every tile -> start height, low-water mark
  int lmin = INT_MAX;
  for (int t = t0; t < t1; t += 32) {
    const int i = t + lane;
    const int2 g = i < t1 ? __ldcg(c.agg + i) : make_int2(0, 0);
    const Bic x = warp_incl_scan(Bic{g.x, g.y}, lane);
    Bic ex{__shfl_up_sync(0xffffffffu, x.a, 1), __shfl_up_sync(0xffffffffu, x.b, 1)};
    if (lane == 0) ex = Bic{0, 0};
    const Bic e = bic_combine(pre, ex);
    if (apre) {
      // exclusive prefix of (a_T + 1): offset of tile i's incoming list
      int v = i < t1 ? g.x + 1 : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= off) v += y;
      }
      const int own = i < t1 ? g.x + 1 : 0;
      if (i < t1) apre[i] = abase + (v - own);
      abase += __shfl_sync(0xffffffffu, v, 31);
    }
    if (i < t1) {
      c.hstart[i] = e.b;
      c.lw[i] = (uint32_t)max(e.b - g.x, 0) + 1u;
      lmin = min(lmin, max(e.b - g.x, 0));
    }
    const Bic last{__shfl_sync(0xffffffffu, x.a, 31), __shfl_sync(0xffffffffu, x.b, 31)};
    pre = bic_combine(pre, last);
  }
  // pass C: smin[i] = min L over tiles > i (which of a tile's slice entries
  // survive to the end of the stream, F1), backwards over each warp's range
  lmin = __reduce_min_sync(0xffffffffu, lmin);
  if (lane == 0) wmin[warp] = lmin;
  __syncthreads();
  int after = INT_MAX;
  for (int w = warp + 1; w < NW; w++) after = min(after, wmin[w]);
  for (int t = t0 + ((t1 - t0 - 1) & ~31); t1 > t0 && t >= t0; t -= 32) {
    const int i = t + lane;
    const int v = i < t1 ? (int)__ldcg(c.lw + i) - 1 : INT_MAX;
    int x = v;  // min over lanes >= lane
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_down_sync(0xffffffffu, x, off);
      if (lane + off < 32) x = min(x, y);
    }
    int ex = __shfl_down_sync(0xffffffffu, x, 1);
    if (lane == 31) ex = INT_MAX;
    if (i < t1) c.smin[i] = min(ex, after);
    after = min(after, __shfl_sync(0xffffffffu, x, 0));
  }
  // 32-ary min hierarchy over the low-water marks (full groups are complete)
  int m = ntiles;
  for (int k = 1; k < HLEVELS; k++) {
    __syncthreads();
    const int groups = (m + 31) / 32;
    for (int g = warp; g < groups; g += NW) {
      const int i = g * 32 + lane;
      uint32_t v = i < m ? __ldcg(c.lv[k - 1] + i) : 0xffffffffu;
      v = __reduce_min_sync(0xffffffffu, v);
      if (lane == 0) c.lv[k][g] = v;
    }
    m = groups;
  }
}

}  // namespace ts

cudaError_t tile_scan_launch(const Ctrl& c, int64_t ntiles, int init_a, int init_h, cudaStream_t stream,
                             int64_t* apre) {
  if (ntiles <= 0) return cudaSuccess;
  TB_LAUNCH(stream, "tile_scan",
            (ts::tile_scan<<<1, ts::NT, 0, stream>>>(c, (int)ntiles, Bic{init_a, init_h}, apre)));
  return cudaGetLastError();
}

}  // namespace tb
