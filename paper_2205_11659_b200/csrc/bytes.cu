// Byte classification for parsing workloads (the
// paper's "parsing" use of parenthesis matching): raw text bytes
// -> tag bytes through a caller-supplied 256-entry class map (e.g. '{' '[' ->
// open, '}' ']' -> close, everything else -> leaf), after which paren_match
// runs unchanged.  One streaming pass, 16 bytes per thread per step.
#include <algorithm>
#include <cstdint>
#include "kernels.h"

namespace tb {

struct ClassMap {
  uint8_t m[256];
};

__global__ void __launch_bounds__(256) classify_bytes_k(const uint8_t* in, int64_t n, ClassMap cm, uint8_t* out) {
  __shared__ uint8_t t[256];
  t[threadIdx.x] = cm.m[threadIdx.x];
  __syncthreads();
  const int64_t nvec = n >> 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += stride) {
    uint4 x = __ldcs(reinterpret_cast<const uint4*>(in) + v);
    uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const uint32_t b = w[k];
      w[k] = (uint32_t)t[b & 255u] | ((uint32_t)t[(b >> 8) & 255u] << 8) | ((uint32_t)t[(b >> 16) & 255u] << 16) |
             ((uint32_t)t[b >> 24] << 24);
    }
    __stcs(reinterpret_cast<uint4*>(out) + v, make_uint4(w[0], w[1], w[2], w[3]));
  }
  for (int64_t i = (nvec << 4) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = t[in[i]];
}

cudaError_t classify_bytes_launch(const uint8_t* in, int64_t n, const uint8_t* class_map, uint8_t* out,
                                  cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  ClassMap cm;
  for (int i = 0; i < 256; i++) cm.m[i] = class_map[i];
  const int64_t nvec = (n >> 4) + 1;
  const unsigned blocks = (unsigned)std::min<int64_t>((nvec + 255) / 256, sm_count() * 8);
  TB_LAUNCH(stream, "classify_bytes", (classify_bytes_k<<<blocks, 256, 0, stream>>>(in, n, cm, out)));
  return cudaGetLastError();
}

}  // namespace tb
