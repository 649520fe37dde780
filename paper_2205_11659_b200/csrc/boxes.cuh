// Bounding-box algebra on the device (§6): intersection for clips,
// raw union for blends, on float4 (x0, y0, x1, y1).  fminf/fmaxf compile to
// FMNMX, whose semantics on sm_100 (measured, tools/probe/minmax_probe.cu) are
// exactly DESIGN R12: -0 below +0, a NaN operand ignored, two NaNs -> the
// canonical NaN.  So every result is bit-identical to the oracle.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tb {

__device__ __forceinline__ float4 bINF() {
  return make_float4(-__int_as_float(0x7f800000), -__int_as_float(0x7f800000), __int_as_float(0x7f800000),
                     __int_as_float(0x7f800000));
}
__device__ __forceinline__ float4 bEMPTY() {
  return make_float4(__int_as_float(0x7f800000), __int_as_float(0x7f800000), -__int_as_float(0x7f800000),
                     -__int_as_float(0x7f800000));
}
__device__ __forceinline__ float4 isect(float4 a, float4 b) {
  return make_float4(fmaxf(a.x, b.x), fmaxf(a.y, b.y), fminf(a.z, b.z), fminf(a.w, b.w));
}
__device__ __forceinline__ float4 unite(float4 a, float4 b) {
  return make_float4(fminf(a.x, b.x), fminf(a.y, b.y), fmaxf(a.z, b.z), fmaxf(a.w, b.w));
}

__device__ __forceinline__ float4 shfl_up_box(float4 v, int d) {
  return make_float4(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d),
                     __shfl_up_sync(0xffffffffu, v.z, d), __shfl_up_sync(0xffffffffu, v.w, d));
}
__device__ __forceinline__ float4 shfl_xor_box(float4 v, int m) {
  return make_float4(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m),
                     __shfl_xor_sync(0xffffffffu, v.z, m), __shfl_xor_sync(0xffffffffu, v.w, m));
}
__device__ __forceinline__ float4 warp_unite_all(float4 v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v = unite(v, shfl_xor_box(v, m));
  return v;
}

}  // namespace tb
