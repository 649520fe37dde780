// Exclusive prefix sum of an int32 array (per-tile / per-bin / per-block counts
// of the auxiliary passes): out[i] = sum(in[0..i)), out[n] = total.
// Reduce-then-scan over blocks of SB entries, no workspace: pass 1 stores each
// block's sum in the block's first output slot; pass 2 (one CTA) turns those
// slots into exclusive block offsets and writes out[n]; pass 3 reads its
// block's offset before any thread of the block overwrites that slot, then
// scans the block (4 entries per thread, warp shuffles, one combine).
#include "kernels.h"

namespace tb {

namespace {
constexpr int SB = 4096;  // entries per block
constexpr int ST = 1024;  // threads per block

__device__ __forceinline__ int warp_incl(int x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}
}  // namespace

__global__ void __launch_bounds__(ST) scan_sums_k(const int* in, int n, int* out) {
  __shared__ int ws[ST / 32];
  const int64_t base = (int64_t)blockIdx.x * SB;
  int s = 0;
#pragma unroll
  for (int r = 0; r < SB / ST; r++) {
    const int64_t g = base + r * ST + threadIdx.x;
    if (g < n) s += in[g];
  }
  s = __reduce_add_sync(0xffffffffu, s);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int t = __reduce_add_sync(0xffffffffu, ws[threadIdx.x]);
    if (threadIdx.x == 0) out[base] = t;
  }
}

__global__ void __launch_bounds__(ST) scan_offsets_k(int n, int* out) {
  __shared__ int ws[ST / 32];
  __shared__ int carry_s;
  const int nb = (n + SB - 1) / SB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int carry = 0;
  for (int b0 = 0; b0 < nb; b0 += ST) {
    const int b = b0 + tid;
    const int v = b < nb ? out[(int64_t)b * SB] : 0;
    const int x = warp_incl(v);
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    int pre = carry;
    for (int w = 0; w < warp; w++) pre += ws[w];
    if (b < nb) out[(int64_t)b * SB] = pre + x - v;
    if (tid == ST - 1) carry_s = pre + x;
    __syncthreads();
    carry = carry_s;
    __syncthreads();
  }
  if (tid == 0) out[n] = carry;
}

__global__ void __launch_bounds__(ST) scan_apply_k(const int* in, int n, int* out) {
  __shared__ int ws[ST / 32];
  __shared__ int off_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * SB, g0 = base + 4 * tid;
  if (tid == 0) off_s = out[base];
  int v[4];
#pragma unroll
  for (int j = 0; j < 4; j++) v[j] = g0 + j < n ? in[g0 + j] : 0;
  const int t = v[0] + v[1] + v[2] + v[3];
  const int x = warp_incl(t);
  if (lane == 31) ws[warp] = x;
  __syncthreads();  // also orders the read of out[base] before the writes below
  int pre = off_s;
  for (int w = 0; w < warp; w++) pre += ws[w];
  pre += x - t;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    if (g0 + j < n) out[g0 + j] = pre;
    pre += v[j];
  }
}

cudaError_t excl_scan_launch(const int* in, int n, int* out, const char* name, cudaStream_t stream) {
  if (n <= 0) return cudaMemsetAsync(out, 0, sizeof(int), stream);
  const unsigned nb = (unsigned)((n + SB - 1) / SB);
  TB_LAUNCH(stream, name, (scan_sums_k<<<nb, ST, 0, stream>>>(in, n, out)));
  TB_LAUNCH(stream, name, (scan_offsets_k<<<1, ST, 0, stream>>>(n, out)));
  TB_LAUNCH(stream, name, (scan_apply_k<<<nb, ST, 0, stream>>>(in, n, out)));
  return cudaGetLastError();
}

}  // namespace tb
