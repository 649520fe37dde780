// Culling + binning of the clipped leaf boxes (the
// motivating use of the boxes, "input to visibility culling and binning",
// P:15; reading R16): a leaf whose node_bbox is non-empty and overlaps
// the viewport is listed in every bin its box overlaps (open overlap).  Three
// passes: per-bin counts (which also list the binned leaves), exclusive scan,
// fill over the listed leaves (the order inside a bin is not specified).  Bin ranges are computed
// in fp64 from the definition, so bin edges agree exactly with the oracle.
#include <algorithm>
#include <climits>
#include <cstdint>
#include "kernels.h"

namespace tb {
namespace bins {

struct P {
  const uint8_t* tags;
  const float4* box;
  int64_t n;
  int gw, gh;
  float bs;
  int32_t* counts;
  int32_t* offsets;
  int32_t* cursor;
  int32_t* items;
};

// bin range of a leaf's clipped box b (false: culled).  Bin edges in fp64 from
// the definition (R16).
__device__ __forceinline__ bool rect_of(const P& p, float4 b, int& x0, int& x1, int& y0, int& y1) {
  if (!(b.x < b.z && b.y < b.w)) return false;  // empty clipped box: culled
  if (!(b.z > 0.f && b.w > 0.f && b.x < p.gw * p.bs && b.y < p.gh * p.bs)) return false;  // off-screen
  const double bs = p.bs;
  double fa = floor((double)b.x / bs), fb = ceil((double)b.z / bs) - 1.0;
  x0 = (int)fmax(fa, 0.0);
  x1 = (int)fmin(fb, (double)(p.gw - 1));
  fa = floor((double)b.y / bs);
  fb = ceil((double)b.w / bs) - 1.0;
  y0 = (int)fmax(fa, 0.0);
  y1 = (int)fmin(fb, (double)(p.gh - 1));
  return true;
}

// Every thread takes 8 consecutive elements per step (grid-stride): the tags
// and all eight boxes are loaded together -- not only the leaves' boxes, which
// would wait for the tags; leaves and non-leaves interleave, so the same DRAM
// sectors are read either way.  f(e, x0, x1, y0, y1) for every binned leaf;
// count and fill walk the same elements per CTA.
constexpr int BE = 8;
template <class F>
__device__ __forceinline__ void for_binned_leaves(const P& p, F&& f) {
  const int64_t stride = (int64_t)gridDim.x * 256 * BE;
  const bool al = (reinterpret_cast<uintptr_t>(p.tags) & 7u) == 0 && (reinterpret_cast<uintptr_t>(p.box) & 15u) == 0;
  for (int64_t e0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) * BE; e0 < p.n; e0 += stride) {
    uint32_t tw[2] = {0x03030303u, 0x03030303u};  // past the end: closes (never binned)
    float4 b[BE];
    if (e0 + BE <= p.n && al) {
      const uint2 t2 = __ldg(reinterpret_cast<const uint2*>(p.tags + e0));
      tw[0] = t2.x;
      tw[1] = t2.y;
#pragma unroll
      for (int i = 0; i < BE; i++) b[i] = __ldg(p.box + e0 + i);
    } else {
#pragma unroll
      for (int i = 0; i < BE; i++) {
        b[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e0 + i < p.n) {
          tw[i >> 2] = (tw[i >> 2] & ~(0xffu << (8 * (i & 3)))) | ((uint32_t)p.tags[e0 + i] << (8 * (i & 3)));
          b[i] = __ldg(p.box + e0 + i);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < BE; i++) {
      const uint32_t t = (tw[i >> 2] >> (8 * (i & 3))) & 0xffu;
      int x0, x1, y0, y1;
      if (t != 1u && t != 2u && t != 3u && rect_of(p, b[i], x0, x1, y0, y1)) f(e0 + i, x0, x1, y0, y1);
    }
  }
}

// streaming fill (fallback when the listed leaves overflowed the list)
__global__ void __launch_bounds__(256) bin_fill_k(P p) {
  for_binned_leaves(p, [&](int64_t e, int x0, int x1, int y0, int y1) {
    for (int y = y0; y <= y1; y++)
      for (int x = x0; x <= x1; x++) {
        const int k = y * p.gw + x;
        p.items[p.offsets[k] + atomicAdd(p.cursor + k, 1)] = (int32_t)e;
      }
  });
}

// Grids of up to SMB bins count in a per-CTA shared-memory histogram (one
// global atomic per bin and CTA).  The count pass also lists every binned leaf
// (warp-aggregated append, up to `cap`): the fill pass then walks that list
// only -- after culling few leaves remain -- instead of streaming all boxes
// again; a list that overflowed falls back to the streaming fill.
constexpr int SMB = 4096;

__device__ __forceinline__ void list_leaf(int32_t* cand, uint32_t* ncand, int64_t cap, int64_t e) {
  const unsigned act = __activemask();
  const int lane = threadIdx.x & 31, leader = __ffs(act) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(ncand, (uint32_t)__popc(act));
  base = __shfl_sync(act, base, leader);
  const int64_t at = (int64_t)base + __popc(act & ((1u << lane) - 1u));
  if (at < cap) cand[at] = (int32_t)e;
}

template <bool PRIV>
__global__ void __launch_bounds__(256) bin_count_list_k(P p, int32_t* cand, uint32_t* ncand, int64_t cap) {
  __shared__ int h[PRIV ? SMB : 1];
  const int nb = p.gw * p.gh;
  if (PRIV) {
    for (int k = threadIdx.x; k < nb; k += 256) h[k] = 0;
    __syncthreads();
  }
  for_binned_leaves(p, [&](int64_t e, int x0, int x1, int y0, int y1) {
    list_leaf(cand, ncand, cap, e);
    for (int y = y0; y <= y1; y++)
      for (int x = x0; x <= x1; x++) atomicAdd(PRIV ? h + y * p.gw + x : p.counts + y * p.gw + x, 1);
  });
  if (PRIV) {
    __syncthreads();
    for (int k = threadIdx.x; k < nb; k += 256)
      if (h[k]) atomicAdd(p.counts + k, h[k]);
  }
}

__global__ void __launch_bounds__(256) bin_fill_list_k(P p, const int32_t* cand, const uint32_t* ncand) {
  const int64_t cnt = *ncand;
  for (int64_t q = blockIdx.x * (int64_t)256 + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * 256) {
    const int32_t e = __ldg(cand + q);
    int x0, x1, y0, y1;
    if (!rect_of(p, __ldg(p.box + e), x0, x1, y0, y1)) continue;  // always binned (listed by the count pass)
    for (int y = y0; y <= y1; y++)
      for (int x = x0; x <= x1; x++) {
        const int k = y * p.gw + x;
        p.items[p.offsets[k] + atomicAdd(p.cursor + k, 1)] = e;
      }
  }
}

}  // namespace bins

constexpr int64_t kCandCap = 1 << 22;  // listed leaves (16 MB)
static int64_t g_cand_cap = kCandCap;  // tests lower it to reach the streaming fill

int64_t bins_debug_cap(int64_t cap) {
  const int64_t old = g_cand_cap;
  if (cap >= 1 && cap <= kCandCap) g_cand_cap = cap;
  return old;
}

size_t bins_workspace_bytes(int nb) {  // fill cursors, candidate count, candidate list
  return sizeof(int32_t) * ((size_t)nb + 4 + (size_t)kCandCap);
}

cudaError_t bins_launch(const uint8_t* tags, const float* node_bbox, int64_t n, int gw, int gh, float bs,
                        int32_t* counts, int32_t* offsets, int32_t* cursor, int32_t* items, int64_t capacity,
                        int64_t* total, cudaStream_t stream) {
  // cursor: workspace of bins_workspace_bytes(gw * gh)
  bins::P p{tags, reinterpret_cast<const float4*>(node_bbox), n, gw, gh, bs, counts, offsets, cursor, items};
  const int nb = gw * gh;
  uint32_t* ncand = reinterpret_cast<uint32_t*>(cursor + nb);
  int32_t* cand = cursor + nb + 4;
  const int64_t cap = std::min<int64_t>(g_cand_cap, std::max<int64_t>(n, 1));
  const unsigned grid = (unsigned)(sm_count() * 8);
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int32_t) * (size_t)nb, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(ncand, 0, sizeof(uint32_t), stream);
  if (e == cudaSuccess && n > 0) {
    if (nb <= bins::SMB)
      TB_LAUNCH(stream, "bin_count", (bins::bin_count_list_k<true><<<grid, 256, 0, stream>>>(p, cand, ncand, cap)));
    else
      TB_LAUNCH(stream, "bin_count", (bins::bin_count_list_k<false><<<grid, 256, 0, stream>>>(p, cand, ncand, cap)));
  }
  if (e == cudaSuccess) e = excl_scan_launch(counts, nb, offsets, "bin_scan", stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(cursor, 0, sizeof(int32_t) * (size_t)nb, stream);
  int32_t hv[2] = {0, 0};
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hv[0], offsets + nb, 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hv[1], ncand, 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return e;
  *total = hv[0];
  if (hv[0] <= capacity && n > 0 && hv[0] > 0) {
    if ((uint32_t)hv[1] <= (uint64_t)cap) {
      const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(((uint32_t)hv[1] + 255) / 256, grid));
      TB_LAUNCH(stream, "bin_fill", (bins::bin_fill_list_k<<<g, 256, 0, stream>>>(p, cand, ncand)));
    } else {
      TB_LAUNCH(stream, "bin_fill", (bins::bin_fill_k<<<grid, 256, 0, stream>>>(p)));
    }
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace tb
