// tree_transform: a generic monoid payload composed down the tree (SURVEY
// §8(f) NEXT row 2; "it can compute any monoid"), here 2D affine
// transforms — non-commutative and non-idempotent, so none of the box path's
// idempotence tricks (DESIGN F6) are available.  Reading R15:
//     world(e) = world(parent(e)) ∘ local(e)   (leaves and opens; root = I)
//     world(close) = world(its open)           (unmatched close: I, R3)
// computed from paren_match's parent / match (like tree_bbox_matched):
// tt_reduce   one warp per tile: the tile's slice entries (opens closed beyond
//             the tile or never) get their tile-local cumulative
//             product lc (an ordered warp scan), kept in a separate array;
//             the tile's link = the parent of its bottom slice entry.
// tt_tc       TC(T) = world(link_T) = TC(tile of link_T) ∘ lc(link_T): pointer
//             jumping over tiles, composing earlier contexts on the left.
// tt_main     one CTA per tile, transforms staged through shared memory (SoA,
//             coalesced in and out): each thread composes its elements relative
//             to its external ancestor X; thread links by pointer jumping; every
//             element's world = ctx(X) ∘ rel in place — the only slots other
//             threads read (thread-unmatched opens) are finished after a barrier;
//             then each close takes its open's world (in the tile: its slot;
//             in an earlier tile: TC ∘ lc of that slice entry).
#include <algorithm>
#include <climits>
#include <cooperative_groups.h>
#include "common.cuh"
#include "kernels.h"

namespace tb {
namespace tt {

constexpr int NT = 128;
constexpr int K = 8;
constexpr int TILE = NT * K;
constexpr int RK = TILE / 32;  // elements per lane in tt_reduce

struct Xf {
  float a, b, c, d, tx, ty;  // p -> [[a, b], [c, d]] p + (tx, ty)
};
__device__ __forceinline__ Xf xf_id() { return Xf{1.f, 0.f, 0.f, 1.f, 0.f, 0.f}; }
// (A ∘ B)(p) = A(B(p))
__device__ __forceinline__ Xf compose(const Xf& A, const Xf& B) {
  Xf r;
  r.a = fmaf(A.a, B.a, A.b * B.c);
  r.b = fmaf(A.a, B.b, A.b * B.d);
  r.c = fmaf(A.c, B.a, A.d * B.c);
  r.d = fmaf(A.c, B.b, A.d * B.d);
  r.tx = fmaf(A.a, B.tx, fmaf(A.b, B.ty, A.tx));
  r.ty = fmaf(A.c, B.tx, fmaf(A.d, B.ty, A.ty));
  return r;
}
__device__ __forceinline__ Xf shfl_up_xf(const Xf& v, int d) {
  return Xf{__shfl_up_sync(0xffffffffu, v.a, d),  __shfl_up_sync(0xffffffffu, v.b, d),
            __shfl_up_sync(0xffffffffu, v.c, d),  __shfl_up_sync(0xffffffffu, v.d, d),
            __shfl_up_sync(0xffffffffu, v.tx, d), __shfl_up_sync(0xffffffffu, v.ty, d)};
}
__device__ __forceinline__ Xf load_xf(const float* p, int64_t i) {
  const float2* q = reinterpret_cast<const float2*>(p + 6 * i);
  const float2 u = __ldg(q), v = __ldg(q + 1), w = __ldg(q + 2);
  return Xf{u.x, u.y, v.x, v.y, w.x, w.y};
}
__device__ __forceinline__ void store_xf(float* p, int64_t i, const Xf& x) {
  float2* q = reinterpret_cast<float2*>(p + 6 * i);
  q[0] = make_float2(x.a, x.b);
  q[1] = make_float2(x.c, x.d);
  q[2] = make_float2(x.tx, x.ty);
}

struct Params {
  const uint8_t* tags;
  const float* local;  // [n][6]
  const int32_t* match;
  const int32_t* parent;
  float* out;  // [n][6]
  int64_t n;
  int ntiles;
  int32_t* link;  // [ntiles]
  Xf* tc;         // [ntiles]
  Xf* lcg;        // [n] (sparse: slice entries)
};

__device__ __forceinline__ bool is_open(uint8_t t) { return t == 1 || t == 2; }

__global__ void __launch_bounds__(128) tt_reduce(Params p) {
  const int lane = threadIdx.x & 31;
  const int T = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (T >= p.ntiles) return;
  const int64_t base = (int64_t)T * TILE, lbase = base + (int64_t)lane * RK, tend = base + TILE;
  uint32_t om = 0;  // the lane's opens (tags as two 16-byte loads)
  if (lbase + RK <= p.n) {
    const uint4 t0 = __ldg(reinterpret_cast<const uint4*>(p.tags + lbase));
    const uint4 t1 = __ldg(reinterpret_cast<const uint4*>(p.tags + lbase) + 1);
    uint32_t o1, c0, c1;
    classify16(t0, om, c0);
    classify16(t1, o1, c1);
    om |= o1 << 16;
  } else {
    for (int i = 0; i < RK && lbase + i < p.n; i++)
      if (is_open(p.tags[lbase + i])) om |= 1u << i;
  }
  uint32_t sm = 0;  // opens closed beyond the tile or never
  for (uint32_t q = om; q; q &= q - 1) {
    const int i = __ffs(q) - 1;
    const int m = __ldg(p.match + lbase + i);
    if (m < 0 || m >= tend) sm |= 1u << i;
  }
  Xf agg = xf_id();
  for (uint32_t q = sm; q; q &= q - 1) agg = compose(agg, load_xf(p.local, lbase + __ffs(q) - 1));
  Xf x = agg;  // inclusive product over lanes 0..lane, earlier lanes on the left
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const Xf o = shfl_up_xf(x, off);
    if (lane >= off) x = compose(o, x);
  }
  Xf acc = shfl_up_xf(x, 1);
  if (lane == 0) acc = xf_id();
  for (uint32_t q = sm; q; q &= q - 1) {
    const int i = __ffs(q) - 1;
    acc = compose(acc, load_xf(p.local, lbase + i));
    p.lcg[lbase + i] = acc;
  }
  const int first = __reduce_min_sync(0xffffffffu, sm ? (lane * RK + __ffs(sm) - 1) : INT_MAX);
  if (lane == 0) p.link[T] = (first == INT_MAX) ? -1 : __ldg(p.parent + base + first);
}

__global__ void __launch_bounds__(256) tt_tc(Params p, Xf* acc2, int* ptr2, int* flag) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int nt = p.ntiles;
  const int gt = (int)(blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
  const int nthr = (int)(gridDim.x * (int64_t)blockDim.x);
  // the two buffers by selects (a runtime index into a pointer array would place it in local memory)
  auto acc = [&](int b) { return b ? acc2 + nt : acc2; };
  auto ptr = [&](int b) { return b ? ptr2 + nt : ptr2; };
  for (int V = gt; V < nt; V += nthr) {
    const int X = __ldg(p.link + V);
    acc(0)[V] = X >= 0 ? p.lcg[X] : xf_id();
    ptr(0)[V] = X >= 0 ? X / TILE : -1;
  }
  int cb = 0;
  for (int round = 0; round < 40; round++) {
    if (gt == 0) flag[round & 1] = 0;
    grid.sync();
    int any = 0;
    for (int V = gt; V < nt; V += nthr) {
      Xf a = acc(cb)[V];
      int q = __ldcg(ptr(cb) + V);
      if (q >= 0) {
        a = compose(acc(cb)[q], a);  // the earlier context on the left
        q = __ldcg(ptr(cb) + q);
        any |= q >= 0;
      }
      acc(cb ^ 1)[V] = a;
      ptr(cb ^ 1)[V] = q;
    }
    any = __syncthreads_or(any);
    if (any && threadIdx.x == 0) atomicOr(flag + (round & 1), 1);
    cb ^= 1;
    grid.sync();
    if (__ldcg(flag + (round & 1)) == 0) break;
  }
  for (int V = gt; V < nt; V += nthr) p.tc[V] = acc(cb)[V];
}

// Shared memory holds the tile's transforms as six float arrays (SoA); thread t's
// element i sits at index 8t + (i ^ ((t >> 2) & 7)), so the 32 lanes of a warp
// reading their i-th element hit 32 distinct banks.
struct Smem {
  float v[6][TILE];  // local, then relative to the thread's external ancestor, then world
  Xf tl[NT];         // world of each thread's link
  Xf acc[2][NT];
  int ptr[2][NT];
};
__device__ __forceinline__ int sidx(int t, int i) { return (t << 3) | (i ^ ((t >> 2) & 7)); }
__device__ __forceinline__ Xf sget(const Smem& s, int j) {
  return Xf{s.v[0][j], s.v[1][j], s.v[2][j], s.v[3][j], s.v[4][j], s.v[5][j]};
}
__device__ __forceinline__ void sput(Smem& s, int j, const Xf& x) {
  s.v[0][j] = x.a;
  s.v[1][j] = x.b;
  s.v[2][j] = x.c;
  s.v[3][j] = x.d;
  s.v[4][j] = x.tx;
  s.v[5][j] = x.ty;
}

__device__ __forceinline__ Xf outer_ctx(const Params& p, int X) {  // an open of an earlier tile
  return compose(p.tc[X / TILE], p.lcg[X]);
}

__global__ void __launch_bounds__(NT) tt_main(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x;
  const int T = blockIdx.x;
  const int64_t base = (int64_t)T * TILE, tstart = base + (int64_t)tid * K;
  const int nvalid = (int)(p.n - base < TILE ? p.n - base : TILE);
  // the tile's transforms, coalesced: 6 * TILE floats as float4s (AoS in HBM)
  {
    const float* src = p.local + 6 * base;
    const int nf = 6 * nvalid;
    const bool vec = nvalid == TILE;  // 6*TILE*4 bytes from a 16-byte aligned base
    for (int f4 = tid; f4 < (6 * TILE) / 4; f4 += NT) {
      float w[4];
      if (vec) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(src) + f4);
        w[0] = q.x; w[1] = q.y; w[2] = q.z; w[3] = q.w;
      } else {
#pragma unroll
        for (int k = 0; k < 4; k++) w[k] = (4 * f4 + k < nf) ? __ldg(src + 4 * f4 + k) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int f = 4 * f4 + k, e = f / 6, c = f - 6 * e;
        s.v[c][sidx(e >> 3, e & 7)] = w[k];
      }
    }
  }
  uint8_t tg[K];
  int pr[K], mt[K];
  if (tstart + K <= p.n) {  // 8 tags, 8 parents, 8 matches as vectors (16-byte aligned)
    const uint2 t8 = __ldg(reinterpret_cast<const uint2*>(p.tags + tstart));
    const int4 p0 = __ldg(reinterpret_cast<const int4*>(p.parent + tstart));
    const int4 p1 = __ldg(reinterpret_cast<const int4*>(p.parent + tstart) + 1);
    const int4 m0 = __ldg(reinterpret_cast<const int4*>(p.match + tstart));
    const int4 m1 = __ldg(reinterpret_cast<const int4*>(p.match + tstart) + 1);
#pragma unroll
    for (int i = 0; i < K; i++) tg[i] = (uint8_t)(((i < 4 ? t8.x : t8.y) >> (8 * (i & 3))) & 0xffu);
    pr[0] = p0.x; pr[1] = p0.y; pr[2] = p0.z; pr[3] = p0.w; pr[4] = p1.x; pr[5] = p1.y; pr[6] = p1.z; pr[7] = p1.w;
    mt[0] = m0.x; mt[1] = m0.y; mt[2] = m0.z; mt[3] = m0.w; mt[4] = m1.x; mt[5] = m1.y; mt[6] = m1.z; mt[7] = m1.w;
  } else {
#pragma unroll
    for (int i = 0; i < K; i++) {
      const int64_t g = tstart + i;
      const bool ok = g < p.n;
      tg[i] = ok ? p.tags[g] : 0;
      pr[i] = ok ? __ldg(p.parent + g) : -1;
      mt[i] = ok ? __ldg(p.match + g) : -1;
    }
  }
  uint32_t valid = 0, thr_un = 0, pend = 0;
#pragma unroll
  for (int i = 0; i < K; i++) {
    if (tstart + i < p.n) valid |= 1u << i;
    if (is_open(tg[i]) && (mt[i] < 0 || mt[i] >= tstart + K)) thr_un |= 1u << i;
  }
  __syncthreads();
  // relative products, in place
  int curX = -1;
#pragma unroll
  for (int i = 0; i < K; i++) {
    if (((valid >> i) & 1u) && tg[i] != 3) {
      const int par = pr[i];
      if (par < tstart) {
        curX = par;
      } else {
        sput(s, sidx(tid, i), compose(sget(s, sidx(tid, par - (int)tstart)), sget(s, sidx(tid, i))));
      }
      if (curX >= 0) pend |= 1u << i;
    }
  }
  __syncthreads();
  // world of each thread's link (pointer jumping; earlier context on the left)
  {
    Xf acc = xf_id();
    int ptr = -1;
    if (thr_un && curX >= 0) {
      if (curX < base) {
        acc = outer_ctx(p, curX);
      } else {
        const int x = curX - (int)base;
        acc = sget(s, sidx(x >> 3, x & 7));
        ptr = x / K;
      }
    }
    int cb = 0;
    s.acc[0][tid] = acc;
    s.ptr[0][tid] = ptr;
    int any = __syncthreads_or(ptr >= 0);
    while (any) {
      if (ptr >= 0) {
        acc = compose(s.acc[cb][ptr], acc);
        ptr = s.ptr[cb][ptr];
      }
      s.acc[cb ^ 1][tid] = acc;
      s.ptr[cb ^ 1][tid] = ptr;
      cb ^= 1;
      any = __syncthreads_or(ptr >= 0);
    }
    s.tl[tid] = acc;
  }
  __syncthreads();
  // worlds in place.  Other threads read only this thread's thread-unmatched
  // opens (their contexts); those belong to its last external group (context
  // tl[tid]) and are finished after the barrier.
  {
    const uint32_t now = pend & ~thr_un;
    int X = -1, cx = INT_MIN;
    Xf g = xf_id();
#pragma unroll
    for (int i = 0; i < K; i++) {
      if (!((valid >> i) & 1u) || tg[i] == 3) continue;
      if (pr[i] < tstart) X = pr[i];
      if ((now >> i) & 1u) {
        if (X != cx) {
          cx = X;
          if (X < base) {
            g = outer_ctx(p, X);
          } else {
            const int x = X - (int)base;
            g = compose(s.tl[x / K], sget(s, sidx(x >> 3, x & 7)));
          }
        }
        sput(s, sidx(tid, i), compose(g, sget(s, sidx(tid, i))));
      }
    }
  }
  __syncthreads();
  if (pend & thr_un) {
    const Xf g = s.tl[tid];
    uint32_t q = pend & thr_un;
#pragma unroll 1
    while (q) {
      const int i = __ffs(q) - 1;
      q &= q - 1;
      sput(s, sidx(tid, i), compose(g, sget(s, sidx(tid, i))));
    }
  }
  __syncthreads();
  // closes take their open's world (R15; unmatched: I): an open of this tile
  // from its (final) slot, an open of an earlier tile -- a slice entry there --
  // as TC ∘ lc
  {
#pragma unroll
    for (int i = 0; i < K; i++) {
      if (((valid >> i) & 1u) && tg[i] == 3) {
        const int o = mt[i];
        Xf w = xf_id();
        if (o >= base) {
          const int x = o - (int)base;
          w = sget(s, sidx(x >> 3, x & 7));
        } else if (o >= 0) {
          w = outer_ctx(p, o);
        }
        sput(s, sidx(tid, i), w);
      }
    }
  }
  __syncthreads();
  // coalesced copy-out
  {
    float* dst = p.out + 6 * base;
    const int nf = 6 * nvalid;
    for (int f4 = tid; f4 < (6 * TILE) / 4; f4 += NT) {
      float w[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int f = 4 * f4 + k, e = f / 6, c = f - 6 * e;
        w[k] = s.v[c][sidx(e >> 3, e & 7)];
      }
      if (nvalid == TILE) {
        reinterpret_cast<float4*>(dst)[f4] = make_float4(w[0], w[1], w[2], w[3]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; k++)
          if (4 * f4 + k < nf) dst[4 * f4 + k] = w[k];
      }
    }
  }
}

struct Layout {
  int64_t ntiles;
  size_t off_link, off_tc, off_lcg, off_acc, off_ptr, off_flag, bytes;
  explicit Layout(int64_t n) {
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    ntiles = (n + TILE - 1) / TILE;
    size_t o = 0;
    off_link = o; o = al(o + 4 * (size_t)ntiles);
    off_tc = o; o = al(o + sizeof(Xf) * (size_t)ntiles);
    off_acc = o; o = al(o + 2 * sizeof(Xf) * (size_t)ntiles);
    off_ptr = o; o = al(o + 8 * (size_t)ntiles);
    off_flag = o; o = al(o + 16);
    off_lcg = o; o = al(o + sizeof(Xf) * (size_t)n);
    bytes = o;
  }
};

int tc_blocks() {  // co-resident CTAs of the cooperative kernel on the current device
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tt_tc, 256, 0);
  return sms * std::max(occ, 1);
}

}  // namespace tt

size_t tt_workspace_bytes(int64_t n) { return n > 0 ? tt::Layout(n).bytes : 0; }

cudaError_t tt_launch(const uint8_t* tags, const float* local, const int32_t* match, const int32_t* parent,
                      int64_t n, float* world, void* ws, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  tt::Layout L(n);
  char* b = (char*)ws;
  tt::Params p;
  p.tags = tags;
  p.local = local;
  p.match = match;
  p.parent = parent;
  p.out = world;
  p.n = n;
  p.ntiles = (int)L.ntiles;
  p.link = (int32_t*)(b + L.off_link);
  p.tc = (tt::Xf*)(b + L.off_tc);
  p.lcg = (tt::Xf*)(b + L.off_lcg);
  TB_LAUNCH(stream, "tt_reduce", (tt::tt_reduce<<<(unsigned)((L.ntiles + 3) / 4), 128, 0, stream>>>(p)));
  {
    tt::Xf* acc2 = (tt::Xf*)(b + L.off_acc);
    int* ptr2 = (int*)(b + L.off_ptr);
    int* flag = (int*)(b + L.off_flag);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((L.ntiles + 255) / 256, tt::tc_blocks()));
    void* args[] = {(void*)&p, (void*)&acc2, (void*)&ptr2, (void*)&flag};
    void* tok;
    prof_begin(stream, "tt_tc", &tok);
    cudaError_t err = cudaLaunchCooperativeKernel((const void*)tt::tt_tc, dim3(blocks), dim3(256), args, 0, stream);
    prof_end(stream, tok);
    if (err != cudaSuccess) return err;
  }
  if (once_per_device(2))
    cudaFuncSetAttribute(tt::tt_main, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(tt::Smem));
  TB_LAUNCH(stream, "tt_main", (tt::tt_main<<<(unsigned)L.ntiles, tt::NT, sizeof(tt::Smem), stream>>>(p)));
  return cudaGetLastError();
}

}  // namespace tb
