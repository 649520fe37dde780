// Exclusive prefix sum of a small int32 array in one CTA (per-tile / per-bin /
// per-block counts of the auxiliary passes): out[i] = sum(in[0..i)),
// out[n] = total.  Warp shuffles + one block-level combine per 1024 entries.
#include "kernels.h"

namespace tb {

__global__ void __launch_bounds__(1024) excl_scan_k(const int* in, int n, int* out) {
  __shared__ int ws[32];
  __shared__ int carry_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int carry = 0;
  for (int b0 = 0; b0 < n; b0 += 1024) {
    const int i = b0 + tid;
    const int v = i < n ? in[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    int pre = carry;
    for (int w = 0; w < warp; w++) pre += ws[w];
    if (i < n) out[i] = pre + x - v;
    if (tid == 1023) carry_s = pre + x;
    __syncthreads();
    carry = carry_s;
    __syncthreads();
  }
  if (tid == 0) out[n] = carry;
}

cudaError_t excl_scan_launch(const int* in, int n, int* out, const char* name, cudaStream_t stream) {
  TB_LAUNCH(stream, name, (excl_scan_k<<<1, 1024, 0, stream>>>(in, n, out)));
  return cudaGetLastError();
}

}  // namespace tb
