// tree_fold: a generic monoid payload multiplied UP the tree (SURVEY §8(f)
// NEXT row 2, the "up" half: blends are upward flow; the union
// structure run in reverse; "it can compute any monoid").
// Reading R17: 2x2 matrices over the integers mod 2^32, ordered products --
// exactly associative, neither commutative nor idempotent, so none of the box
// path's overlapping-window tricks (min/max are idempotent, F4) apply: every
// range below is split into DISJOINT pieces combined left to right.
//   node value(o, c) = product of the leaf payloads strictly inside (o, c)
// from paren_match's match:
// tf_tile   one CTA per 2048-element tile, 16 consecutive elements per thread:
//           thread products; ordered prefix / suffix products over the threads
//           and a disjoint sparse table over them (any thread range in two
//           lookups); nodes inside one thread by a direct product; nodes inside
//           the tile: (suffix of the open's thread) · (threads between) ·
//           (prefix of the close's thread); nodes leaving the tile: the tile
//           suffix after the open / the tile prefix before the close, parked in
//           the output slots, the close (or never-closed open) listed
// tf_hier   32-ary hierarchy of ordered tile products
// tf_cross  one warp per tile's list: value = S(o) · (tiles between) · P(c)
//           with the tiles between split over the hierarchy (ordered warp
//           products); never-closed opens take the tiles to the stream end (R4)
#include <algorithm>
#include "common.cuh"
#include "kernels.h"

namespace tb {
namespace tf {

constexpr int NT = 128;
constexpr int K = 16;
constexpr int W = NT * K;  // 2048
constexpr int LOGW = 11;
constexpr int LV = 5;      // levels of tile products: 32^5 tiles > 2^31 / W
constexpr int DL = 8;      // disjoint sparse table levels over the 128 threads (0: the threads)

using M = uint4;  // (a, b, c, d) = [[a, b], [c, d]] mod 2^32
__device__ __forceinline__ M mid() { return make_uint4(1u, 0u, 0u, 1u); }
__device__ __forceinline__ M mul(const M& X, const M& Y) {
  return make_uint4(X.x * Y.x + X.y * Y.z, X.x * Y.y + X.y * Y.w, X.z * Y.x + X.w * Y.z, X.z * Y.y + X.w * Y.w);
}
__device__ __forceinline__ M shfl_m(const M& v, int src) {
  return make_uint4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                    __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
}
__device__ __forceinline__ M shfl_up_m(const M& v, int d) {
  return make_uint4(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d),
                    __shfl_up_sync(0xffffffffu, v.z, d), __shfl_up_sync(0xffffffffu, v.w, d));
}
__device__ __forceinline__ M shfl_down_m(const M& v, int d) {
  return make_uint4(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d),
                    __shfl_down_sync(0xffffffffu, v.z, d), __shfl_down_sync(0xffffffffu, v.w, d));
}
// ordered product of the lanes' values (lane 0 leftmost), result in every lane
__device__ __forceinline__ M warp_prod(M v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const M o = shfl_down_m(v, off);
    if ((lane & (2 * off - 1)) == 0) v = mul(v, o);
  }
  return shfl_m(v, 0);
}

struct Params {
  const uint8_t* tags;
  const M* x;
  const int32_t* match;
  int64_t n;
  int ntiles;
  M* out;
  M* tp[LV];         // ordered tile products, 32-ary levels
  int32_t* list;     // [ntiles * W] per tile: closes whose open lies in an earlier tile, opens never closed
  int32_t* nlist;    // [ntiles]
};

struct Smem {
  M xs[W];           // the tile's payloads (swizzled slots: conflict-free per-thread rows)
  M pre[NT];         // product of threads [0, t)
  M suf[NT];         // product of threads (t, NT)
  M dl[DL][NT];      // disjoint sparse table: level h, thread t: t's half-block product toward the middle
  int cnt;
};

// element i of thread t: slot ((i & 8) << 7) | 8 t + ((i & 7) ^ (t & 7)) -- 8
// consecutive lanes read 8 distinct 16-byte bank groups
__device__ __forceinline__ int slot(int t, int i) { return ((i & 8) << 7) | (t << 3) | ((i & 7) ^ (t & 7)); }

// product of threads [l, r] (l <= r): two lookups in the disjoint sparse table
__device__ __forceinline__ M thread_range(const Smem& s, int l, int r) {
  if (l > r) return mid();
  if (l == r) return s.dl[0][l];
  const int h = 32 - __clz(l ^ r);  // the level whose block splits l | r
  return mul(s.dl[h][l], s.dl[h][r]);
}

__global__ void __launch_bounds__(NT) tf_tile(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31;
  const int T = blockIdx.x;
  const int64_t base = (int64_t)T * W;
  const int nvalid = (int)(p.n - base < W ? p.n - base : W);
  const int tl0 = tid * K;
  if (tid == 0) s.cnt = 0;
  // payloads in (coalesced), tags and match of the thread's 16 elements
#pragma unroll 4
  for (int j = 0; j < K; j++) {
    const int e = j * NT + tid;
    s.xs[slot(e >> 4, e & 15)] = e < nvalid ? __ldg(p.x + base + e) : mid();
  }
  uint32_t om = 0, cm = 0, lm = 0;
  {
    uint4 raw = make_uint4(0, 0, 0, 0);
    if (tl0 + K <= nvalid) {
      raw = __ldg(reinterpret_cast<const uint4*>(p.tags + base + tl0));
    } else {
      uint32_t wv[4] = {0, 0, 0, 0};
      for (int i = 0; i < K && tl0 + i < nvalid; i++) wv[i >> 2] |= (uint32_t)p.tags[base + tl0 + i] << (8 * (i & 3));
      raw = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
    classify16(raw, om, cm);
    const int nv = max(0, min(K, nvalid - tl0));
    const uint32_t valid = nv >= K ? 0xffffu : ((1u << nv) - 1u);
    om &= valid;
    cm &= valid;
    lm = valid & ~(om | cm);
  }
  int32_t mt[K];
#pragma unroll
  for (int q = 0; q < K / 4; q++) {
    int4 v = make_int4(-1, -1, -1, -1);
    if (tl0 + 4 * q + 4 <= nvalid) {
      v = __ldg(reinterpret_cast<const int4*>(p.match + base + tl0) + q);
    } else {
      int* w = &v.x;
      for (int j = 0; j < 4; j++)
        if (tl0 + 4 * q + j < nvalid) w[j] = p.match[base + tl0 + 4 * q + j];
    }
    mt[4 * q] = v.x;
    mt[4 * q + 1] = v.y;
    mt[4 * q + 2] = v.z;
    mt[4 * q + 3] = v.w;
  }
  const int64_t gb = base + tl0;  // global index of element 0 of the thread
  __syncthreads();

  // Outputs go to the slots of xs (a leaf's output is its payload, opens and
  // closes carry no payload) and leave in one coalesced copy at the end.
  // Forward walk of the thread: its product; nodes inside the thread (a stack
  // of their running products); the prefix before each close of an open
  // outside the thread (parked in the close's slot until pass 2)
  M P = mid();
  {
    // the innermost open in-thread node's product in a register (tp), the
    // enclosing ones below it (entry j of thread t in dl[j][t]: the sparse
    // table is built after the walk; the bank depends on t only); every element
    // runs the same predicated sequence: a leaf multiplies P and tp, an open
    // of an in-thread node pushes, its close pops
    static_assert(DL >= K / 2, "the walk's stack lives in dl");
    M tp = mid();
    int d = 0;
#pragma unroll
    for (int i = 0; i < K; i++) {
      const bool isl = (lm >> i) & 1u, iso = (om >> i) & 1u, isc = (cm >> i) & 1u;
      const int64_t o = mt[i];
      const bool push = iso && o >= 0 && o < gb + K;  // an open closed in this thread
      const bool pop = isc && o >= gb;                // the close of one
      const M v = isl ? s.xs[slot(tid, i)] : mid();
      P = mul(P, v);
      const M tv = mul(tp, v);
      if (push) {
        if (d > 0) s.dl[d - 1][tid] = tp;
        d++;
        tp = mid();
      } else if (pop) {
        s.xs[slot(tid, i)] = tv;
        s.xs[slot(tid, (int)(o - gb))] = tv;
        d--;
        tp = d > 0 ? mul(s.dl[d - 1][tid], tv) : mid();
      } else {
        tp = tv;
        if (isc) s.xs[slot(tid, i)] = o < 0 ? mid() : P;  // R3; or the thread prefix before the close (pass 2)
      }
    }
  }
  // disjoint sparse table over the threads: level 0 = the thread products;
  // level h (blocks of 2^h, halves of 2^(h-1)): a left-half thread holds the
  // product from it to the half's end, a right-half thread from the half's
  // start to it (segmented ordered scans: shuffles inside a warp, one carry
  // across the two warps of a 64-thread half)
  s.dl[0][tid] = P;
#pragma unroll
  for (int h = 1; h < DL; h++) {
    const int half = 1 << (h - 1);
    const bool right = (tid >> (h - 1)) & 1;
    const int seg = min(half, 32);
    const int ls = lane & (seg - 1);  // position inside the warp-level segment
    // inclusive prefix and suffix within the segment, in every lane (the
    // shuffles need the whole warp); right-half lanes keep the prefix
    M pv = P, sv = P;
#pragma unroll
    for (int off = 1; off < seg; off <<= 1) {  // seg is a constant of the unrolled level
      const M a = shfl_up_m(pv, off), b = shfl_down_m(sv, off);
      if (ls >= off) pv = mul(a, pv);
      if (ls + off < seg) sv = mul(sv, b);
    }
    M v = right ? pv : sv;
    // halves of 64 add the other warp of the half
    s.dl[h][tid] = v;
    if (half == 64) {
      __syncthreads();
      if (right && (tid & 32)) v = mul(s.dl[h][tid - lane - 1], v);        // · prefix of the half's first warp
      if (!right && !(tid & 32)) v = mul(v, s.dl[h][(tid | 31) + 1]);     // · suffix of the half's second warp
      __syncthreads();
      s.dl[h][tid] = v;
    }
  }
  __syncthreads();
  s.pre[tid] = thread_range(s, 0, tid - 1);
  s.suf[tid] = thread_range(s, tid + 1, NT - 1);
  if (tid == 0) p.tp[0][T] = thread_range(s, 0, NT - 1);
  __syncthreads();

  // pass 1 (backward walk): the open side of nodes leaving the thread -- the
  // rest of the thread after the open, then the threads up to the close's
  // thread (or the tile end: closed in a later tile or never)
  {
    M S = mid();
#pragma unroll
    for (int i = K - 1; i >= 0; i--) {
      if ((om >> i) & 1u) {
        const int64_t c = mt[i];
        if (c < 0 || c >= gb + K) {
          const M r = c >= 0 && c < base + W ? thread_range(s, tid + 1, (int)((c - base) >> 4) - 1) : s.suf[tid];
          s.xs[slot(tid, i)] = mul(S, r);
        }
      }
      if ((lm >> i) & 1u) S = mul(s.xs[slot(tid, i)], S);
    }
  }
  __syncthreads();  // the open sides are in their slots
  // pass 2: closes of opens in an earlier thread of the tile (open side parked
  // in out[o], this thread's prefix in out[c]); closes of earlier tiles' opens
  // get the tile prefix and are listed, as are opens never closed
#pragma unroll
  for (int i = 0; i < K; i++) {
    const int64_t g = gb + i;
    if ((cm >> i) & 1u) {
      const int64_t o = mt[i];
      if (o >= 0 && o < gb) {
        const M v = s.xs[slot(tid, i)];
        if (o >= base) {
          const int lo = (int)(o - base);
          M& so = s.xs[slot(lo >> 4, lo & 15)];
          const M u = mul(so, v);
          s.xs[slot(tid, i)] = u;
          so = u;
        } else {
          s.xs[slot(tid, i)] = mul(s.pre[tid], v);
          p.list[base + atomicAdd(&s.cnt, 1)] = (int32_t)g;
        }
      }
    } else if (((om >> i) & 1u) && mt[i] < 0) {
      p.list[base + atomicAdd(&s.cnt, 1)] = (int32_t)g;
    }
  }
  __syncthreads();
  if (tid == 0) p.nlist[T] = s.cnt;
#pragma unroll 4
  for (int j = 0; j < K; j++) {  // coalesced copy-out
    const int e = j * NT + tid;
    if (e < nvalid) p.out[base + e] = s.xs[slot(e >> 4, e & 15)];
  }
}

__global__ void __launch_bounds__(256) tf_hier(const M* src, M* dst, int m /* nodes at level k - 1 */) {
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x * 8 + (threadIdx.x >> 5);
  if ((g << 5) >= m) return;
  const int c = (g << 5) + lane;
  const M v = warp_prod(c < m ? __ldcg(src + c) : mid());
  if (lane == 0) dst[g] = v;
}

// ordered product of tiles a .. b by one thread (a > b: identity): disjoint
// pieces, a's partial group and b's partial group at each level
__device__ __forceinline__ M range_tiles(const Params& p, int a, int b) {
  M left = mid(), right = mid();
#pragma unroll
  for (int k = 0; k < LV; k++) {  // unrolled: p.tp[k] stays a parameter-space load
    if (a <= b) {
      const M* t = p.tp[k];
      if ((a >> 5) == (b >> 5)) {
        for (int i = a; i <= b; i++) left = mul(left, __ldcg(t + i));
        a = b + 1;
      } else {
        if (a & 31) {
          for (int i = a; i <= (a | 31); i++) left = mul(left, __ldcg(t + i));
          a = (a >> 5) + 1;
        } else {
          a >>= 5;
        }
        if ((b & 31) != 31) {
          M r = mid();
          for (int i = b & ~31; i <= b; i++) r = mul(r, __ldcg(t + i));
          right = mul(r, right);
          b = (b >> 5) - 1;
        } else {
          b >>= 5;
        }
      }
    }
  }
  return mul(left, right);
}

// one warp per tile, one listed element per lane
__global__ void __launch_bounds__(128) tf_cross(Params p) {
  const int lane = threadIdx.x & 31;
  const int T = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (T >= p.ntiles) return;
  const int cnt = __ldg(p.nlist + T);
  const int64_t base = (int64_t)T * W;
  for (int j = lane; j < cnt; j += 32) {
    const int64_t e = __ldg(p.list + base + j);
    const int32_t o = __ldg(p.match + e);
    if (p.tags[e] == 3) {  // a close of an earlier tile's open: S(o) · tiles between · P(e)
      const M u = mul(mul(__ldcg(p.out + o), range_tiles(p, (int)(o >> LOGW) + 1, T - 1)), __ldcg(p.out + e));
      p.out[e] = u;
      p.out[o] = u;
    } else {  // an open never closed (R4): every later tile
      p.out[e] = mul(__ldcg(p.out + e), range_tiles(p, T + 1, p.ntiles - 1));
    }
  }
}

struct Layout {
  size_t tp[LV], list, nlist, bytes;
  explicit Layout(int64_t n) {
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const int64_t nt = (n + W - 1) / W;
    size_t o = 0;
    int64_t m = nt;
    for (int k = 0; k < LV; k++) {
      tp[k] = o;
      o = al(o + 16 * (size_t)std::max<int64_t>(m, 1));
      m = (m + 31) / 32;
    }
    list = o; o = al(o + 4 * (size_t)nt * W);
    nlist = o; o = al(o + 4 * (size_t)nt);
    bytes = o;
  }
};

}  // namespace tf

size_t tf_workspace_bytes(int64_t n) { return n > 0 ? tf::Layout(n).bytes : 0; }

cudaError_t tf_launch(const uint8_t* tags, const uint32_t* x, const int32_t* match, int64_t n, uint32_t* out,
                      void* ws, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const tf::Layout L(n);
  tf::Params p;
  p.tags = tags;
  p.x = reinterpret_cast<const tf::M*>(x);
  p.match = match;
  p.n = n;
  p.ntiles = (int)((n + tf::W - 1) / tf::W);
  p.out = reinterpret_cast<tf::M*>(out);
  for (int k = 0; k < tf::LV; k++) p.tp[k] = reinterpret_cast<tf::M*>((char*)ws + L.tp[k]);
  p.list = reinterpret_cast<int32_t*>((char*)ws + L.list);
  p.nlist = reinterpret_cast<int32_t*>((char*)ws + L.nlist);
  const int nt = p.ntiles;
  if (once_per_device(4)) {
    cudaError_t e0 = cudaFuncSetAttribute(tf::tf_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(tf::Smem));
    if (e0 != cudaSuccess) return e0;
  }
  TB_LAUNCH(stream, "tf_tile", (tf::tf_tile<<<(unsigned)nt, tf::NT, sizeof(tf::Smem), stream>>>(p)));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int m = nt;
  for (int k = 1; k < tf::LV && m > 1; k++) {
    const int groups = (m + 31) / 32;
    TB_LAUNCH(stream, "tf_hier", (tf::tf_hier<<<(unsigned)((groups + 7) / 8), 256, 0, stream>>>(p.tp[k - 1], p.tp[k], m)));
    m = groups;
  }
  TB_LAUNCH(stream, "tf_cross", (tf::tf_cross<<<(unsigned)((nt + 3) / 4), 128, 0, stream>>>(p)));
  return cudaGetLastError();
}

}  // namespace tb
