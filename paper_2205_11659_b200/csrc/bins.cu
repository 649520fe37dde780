// Culling + binning of the clipped leaf boxes (the
// motivating use of the boxes, "input to visibility culling and binning",
// P:15; reading R16): a leaf whose node_bbox is non-empty and overlaps
// the viewport is listed in every bin its box overlaps (open overlap).  Three
// passes: per-bin counts (atomics), exclusive scan (one CTA), fill (atomic
// cursors: the order inside a bin is not specified).  Bin ranges are computed
// in fp64 from the definition, so bin edges agree exactly with the oracle.
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

__device__ __forceinline__ bool rect(const P& p, int64_t e, int& x0, int& x1, int& y0, int& y1) {
  const uint8_t t = p.tags[e];
  if (t == 1 || t == 2 || t == 3) return false;
  const float4 b = __ldg(p.box + e);
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

__global__ void __launch_bounds__(256) bin_count_k(P p) {
  for (int64_t e = blockIdx.x * (int64_t)256 + threadIdx.x; e < p.n; e += (int64_t)gridDim.x * 256) {
    int x0, x1, y0, y1;
    if (!rect(p, e, x0, x1, y0, y1)) continue;
    for (int y = y0; y <= y1; y++)
      for (int x = x0; x <= x1; x++) atomicAdd(p.counts + y * p.gw + x, 1);
  }
}


__global__ void __launch_bounds__(256) bin_fill_k(P p) {
  for (int64_t e = blockIdx.x * (int64_t)256 + threadIdx.x; e < p.n; e += (int64_t)gridDim.x * 256) {
    int x0, x1, y0, y1;
    if (!rect(p, e, x0, x1, y0, y1)) continue;
    for (int y = y0; y <= y1; y++)
      for (int x = x0; x <= x1; x++) {
        const int k = y * p.gw + x;
        p.items[p.offsets[k] + atomicAdd(p.cursor + k, 1)] = (int32_t)e;
      }
  }
}

}  // namespace bins

cudaError_t bins_launch(const uint8_t* tags, const float* node_bbox, int64_t n, int gw, int gh, float bs,
                        int32_t* counts, int32_t* offsets, int32_t* cursor, int32_t* items, int64_t capacity,
                        int64_t* total, cudaStream_t stream) {
  bins::P p{tags, reinterpret_cast<const float4*>(node_bbox), n, gw, gh, bs, counts, offsets, cursor, items};
  const int nb = gw * gh;
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int32_t) * (size_t)nb, stream);
  const unsigned grid = 148 * 8;
  if (e == cudaSuccess && n > 0) TB_LAUNCH(stream, "bin_count", (bins::bin_count_k<<<grid, 256, 0, stream>>>(p)));
  if (e == cudaSuccess) e = excl_scan_launch(counts, nb, offsets, "bin_scan", stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(cursor, 0, sizeof(int32_t) * (size_t)nb, stream);
  int32_t t = 0;
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(&t, offsets + nb, 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return e;
  *total = t;
  if (t <= capacity && n > 0 && t > 0) {
    TB_LAUNCH(stream, "bin_fill", (bins::bin_fill_k<<<grid, 256, 0, stream>>>(p)));
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace tb
