// Bounding-box algebra on the device (§6): intersection for clips,
// raw union for blends.  Coordinates are carried as 32-bit integer keys whose
// signed order is the IEEE 754 totalOrder of the fp32 values
// (key = bits ^ ((bits >> 31) & 0x7fffffff), an involution), so every min/max
// is a single integer instruction and -0 < +0 holds exactly (DESIGN R12).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tb {

struct KBox {
  int x0, y0, x1, y1;
};

__device__ __forceinline__ int fkey(int bits) { return bits ^ ((bits >> 31) & 0x7fffffff); }
__device__ __forceinline__ KBox to_kbox(float4 f) {
  return KBox{fkey(__float_as_int(f.x)), fkey(__float_as_int(f.y)), fkey(__float_as_int(f.z)),
              fkey(__float_as_int(f.w))};
}
__device__ __forceinline__ float4 to_float4(KBox k) {
  return make_float4(__int_as_float(fkey(k.x0)), __int_as_float(fkey(k.y0)), __int_as_float(fkey(k.x1)),
                     __int_as_float(fkey(k.y1)));
}
__device__ __forceinline__ int4 to_int4(KBox k) { return make_int4(k.x0, k.y0, k.x1, k.y1); }
__device__ __forceinline__ KBox from_int4(int4 v) { return KBox{v.x, v.y, v.z, v.w}; }

// keys of -inf / +inf
constexpr int KNEG_INF = (int)0x807fffff;
constexpr int KPOS_INF = 0x7f800000;
__device__ __forceinline__ KBox kINF() { return KBox{KNEG_INF, KNEG_INF, KPOS_INF, KPOS_INF}; }
__device__ __forceinline__ KBox kEMPTY() { return KBox{KPOS_INF, KPOS_INF, KNEG_INF, KNEG_INF}; }

__device__ __forceinline__ KBox isect(KBox a, KBox b) {
  return KBox{max(a.x0, b.x0), max(a.y0, b.y0), min(a.x1, b.x1), min(a.y1, b.y1)};
}
__device__ __forceinline__ KBox unite(KBox a, KBox b) {
  return KBox{min(a.x0, b.x0), min(a.y0, b.y0), max(a.x1, b.x1), max(a.y1, b.y1)};
}

__device__ __forceinline__ KBox shfl_box(KBox v, int src) {
  return KBox{__shfl_sync(0xffffffffu, v.x0, src), __shfl_sync(0xffffffffu, v.y0, src),
              __shfl_sync(0xffffffffu, v.x1, src), __shfl_sync(0xffffffffu, v.y1, src)};
}
__device__ __forceinline__ KBox shfl_up_box(KBox v, int d) {
  return KBox{__shfl_up_sync(0xffffffffu, v.x0, d), __shfl_up_sync(0xffffffffu, v.y0, d),
              __shfl_up_sync(0xffffffffu, v.x1, d), __shfl_up_sync(0xffffffffu, v.y1, d)};
}
__device__ __forceinline__ KBox shfl_down_box(KBox v, int d) {
  return KBox{__shfl_down_sync(0xffffffffu, v.x0, d), __shfl_down_sync(0xffffffffu, v.y0, d),
              __shfl_down_sync(0xffffffffu, v.x1, d), __shfl_down_sync(0xffffffffu, v.y1, d)};
}
__device__ __forceinline__ KBox warp_isect_all(KBox v) {
  return KBox{__reduce_max_sync(0xffffffffu, v.x0), __reduce_max_sync(0xffffffffu, v.y0),
              __reduce_min_sync(0xffffffffu, v.x1), __reduce_min_sync(0xffffffffu, v.y1)};
}
__device__ __forceinline__ KBox warp_unite_all(KBox v) {
  return KBox{__reduce_min_sync(0xffffffffu, v.x0), __reduce_min_sync(0xffffffffu, v.y0),
              __reduce_max_sync(0xffffffffu, v.x1), __reduce_max_sync(0xffffffffu, v.y1)};
}

}  // namespace tb
