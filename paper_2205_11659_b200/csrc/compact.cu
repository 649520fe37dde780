// Stream compaction front end (the step upstream of
// the hot path): a full scene stream of command bytes -> the elements
// the bounding-box path needs (a caller-supplied keep map over byte values),
// compacted, with their boxes and an index map back into the full stream.
// Three passes: per-block kept counts, an exclusive scan over blocks (one
// CTA), a block-local scan + scatter that preserves order.  (Fusing the flag
// scan into the path's tile loaders, so compaction costs no extra HBM pass, is
// the next step.)
#include <climits>
#include <cstdint>
#include "kernels.h"

namespace tb {
namespace cpt {

constexpr int NT = 256, K = 16, BLK = NT * K;  // 4096 elements per block

struct KeepMap {
  uint8_t m[256];
};

__device__ __forceinline__ uint32_t kept16(const uint8_t* tags, int64_t n, int64_t g, const uint8_t* km) {
  uint32_t f = 0;
  if (g + 16 <= n) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(tags + g));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; q++)
#pragma unroll
      for (int b = 0; b < 4; b++) f |= (uint32_t)(km[(w[q] >> (8 * b)) & 255u] != 0) << (4 * q + b);
  } else {
    for (int i = 0; i < 16; i++)
      if (g + i < n && km[tags[g + i]]) f |= 1u << i;
  }
  return f;
}

__global__ void __launch_bounds__(NT) count_k(const uint8_t* tags, int64_t n, KeepMap kmv, int* cnt) {
  __shared__ uint8_t km[256];
  __shared__ int ws[NT / 32];
  km[threadIdx.x] = kmv.m[threadIdx.x];
  __syncthreads();
  const int64_t g = (int64_t)blockIdx.x * BLK + (int64_t)threadIdx.x * K;
  int c = __popc(kept16(tags, n, g, km));
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < NT / 32; w++) t += ws[w];
    cnt[blockIdx.x] = t;
  }
}


// Warp-cooperative scatter: each warp owns 512 contiguous elements, counted
// first (16 per lane), then walked in 16 rounds of 32 consecutive elements --
// one per lane, a ballot gives each kept element its output slot -- so reads
// and the compacted writes are both contiguous across the warp.
__global__ void __launch_bounds__(NT) scatter_k(const uint8_t* tags, const float4* boxes, int64_t n, KeepMap kmv,
                                                const int* offs, uint8_t* tags_out, float4* boxes_out,
                                                int32_t* index_out) {
  __shared__ uint8_t km[256];
  __shared__ int ws[NT / 32];
  km[threadIdx.x] = kmv.m[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t w0 = (int64_t)blockIdx.x * BLK + (int64_t)warp * (32 * K);
  const uint32_t f = kept16(tags, n, w0 + lane * K, km);
  const int c = __reduce_add_sync(0xffffffffu, __popc(f));
  if (lane == 0) ws[warp] = c;
  __syncthreads();
  int pos = offs[blockIdx.x];
  for (int w = 0; w < warp; w++) pos += ws[w];
#pragma unroll 4
  for (int r = 0; r < K; r++) {
    const int64_t e = w0 + r * 32 + lane;
    // element e is bit (lane & 15) of lane 2r + lane / 16's kept mask
    const uint32_t fl = __shfl_sync(0xffffffffu, f, 2 * r + (lane >> 4));
    const bool k = (fl >> (lane & 15)) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, k);
    if (k) {
      const int at = pos + __popc(bal & ((1u << lane) - 1u));
      tags_out[at] = tags[e];
      if (boxes) boxes_out[at] = __ldg(boxes + e);
      index_out[at] = (int32_t)e;
    }
    pos += __popc(bal);
  }
}

}  // namespace cpt

size_t compact_workspace_bytes(int64_t n) { return 4 * (size_t)(2 * ((n + cpt::BLK - 1) / cpt::BLK) + 2); }

cudaError_t compact_launch(const uint8_t* tags, const float* boxes, int64_t n, const uint8_t* keep_map,
                           uint8_t* tags_out, float* boxes_out, int32_t* index_out, int64_t* n_out, void* ws,
                           cudaStream_t stream) {
  cpt::KeepMap km;
  for (int i = 0; i < 256; i++) km.m[i] = keep_map[i];
  const int nb = (int)((n + cpt::BLK - 1) / cpt::BLK);
  int* cnt = (int*)ws;
  int* offs = cnt + nb + 1;
  if (n > 0) TB_LAUNCH(stream, "compact_count", (cpt::count_k<<<nb, cpt::NT, 0, stream>>>(tags, n, km, cnt)));
  cudaError_t e0 = excl_scan_launch(cnt, nb, offs, "compact_scan", stream);
  if (e0 != cudaSuccess) return e0;
  if (n > 0)
    TB_LAUNCH(stream, "compact_scatter",
              (cpt::scatter_k<<<nb, cpt::NT, 0, stream>>>(tags, reinterpret_cast<const float4*>(boxes), n, km,
                                                          offs, tags_out, reinterpret_cast<float4*>(boxes_out),
                                                          index_out)));
  int32_t t = 0;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(&t, offs + nb, 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  *n_out = t;
  return e;
}

}  // namespace tb
