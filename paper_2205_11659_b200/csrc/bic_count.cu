// Global Bic of a tag stream (validation helper behind tb_count_unmatched):
// (a, b) = fold of open -> (0,1), close -> (1,0) under ⊕ (§3).
// Pass 1: one Bic per 4096-element block; pass 2: one warp folds the block
// values in order (⊕ is associative but not commutative).
#include "common.cuh"
#include "kernels.h"

namespace tb {
namespace bc {

constexpr int NT = 256, K = 16, TILE = NT * K;

__global__ void __launch_bounds__(NT) block_bic(const uint8_t* tags, int64_t n, int2* part) {
  __shared__ Bic wt[NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * TILE + (int64_t)tid * K;
  uint32_t wv[4] = {0, 0, 0, 0};
  for (int i = 0; i < K; i++) {
    const int64_t g = base + i;
    const uint32_t v = g < n ? tags[g] : 0u;
    wv[i >> 2] |= v << (8 * (i & 3));
  }
  uint32_t om, cm;
  classify16(make_uint4(wv[0], wv[1], wv[2], wv[3]), om, cm);
  Bic acc{0, 0};
  for (int i = 0; i < K; i++) {
    Bic e{(int)((cm >> i) & 1u), (int)((om >> i) & 1u)};
    acc = bic_combine(acc, e);
  }
  for (int off = 1; off < 32; off <<= 1) {
    Bic o{__shfl_down_sync(0xffffffffu, acc.a, off), __shfl_down_sync(0xffffffffu, acc.b, off)};
    if (lane + off < 32) acc = bic_combine(acc, o);
  }
  if (lane == 0) wt[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    Bic t{0, 0};
    for (int w = 0; w < NT / 32; w++) t = bic_combine(t, wt[w]);
    part[blockIdx.x] = make_int2(t.a, t.b);
  }
}

__global__ void fold_parts(const int2* part, int64_t m, int64_t* out) {
  const int lane = threadIdx.x;
  Bic acc{0, 0};
  for (int64_t j = 0; j < m; j += 32) {
    Bic v{0, 0};
    if (j + lane < m) v = Bic{part[j + lane].x, part[j + lane].y};
    for (int off = 1; off < 32; off <<= 1) {
      Bic o{__shfl_down_sync(0xffffffffu, v.a, off), __shfl_down_sync(0xffffffffu, v.b, off)};
      if (lane + off < 32) v = bic_combine(v, o);
    }
    Bic w{__shfl_sync(0xffffffffu, v.a, 0), __shfl_sync(0xffffffffu, v.b, 0)};
    acc = bic_combine(acc, w);
  }
  if (lane == 0) {
    out[0] = acc.a;
    out[1] = acc.b;
  }
}

}  // namespace bc

size_t bic_count_workspace_bytes(int64_t n) {
  const int64_t m = (n + bc::TILE - 1) / bc::TILE;
  return (size_t)m * sizeof(int2) + 256;
}

cudaError_t bic_count_launch(const uint8_t* tags, int64_t n, void* ws, int64_t* d_out2,
                             cudaStream_t stream) {
  const int64_t m = (n + bc::TILE - 1) / bc::TILE;
  if (m > 0) TB_LAUNCH(stream, "bic_block", (bc::block_bic<<<(unsigned)m, bc::NT, 0, stream>>>(tags, n, (int2*)ws)));
  TB_LAUNCH(stream, "bic_fold", (bc::fold_parts<<<1, 32, 0, stream>>>((const int2*)ws, m, d_out2)));
  return cudaGetLastError();
}

}  // namespace tb
