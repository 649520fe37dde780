// paren_match + tree_bbox in one tile pass (sm_100a).
//
// The matching (§2-§8 of the paper: Fig. 1's parent, and the
// classical partner) and the two box passes (§6, §9: the clip
// intersection of P:24/P:201/P:292 and the blend union of P:24/P:196/P:216-221,
// stored at the close and scattered to a blend open) are computed by
// the same kernel from the tags and boxes of one tile, so each element's tag
// and box are read once and match, parent and node_bbox written once.
//
//   fz_reduce  one warp per 2048-element tile, tags only (+ the boxes of the
//              tile's unmatched opens): the tile's Bic value (§3) and
//              its stack slice (§7.1: unmatched opens, ascending)
//              with each entry's tile-local cumulative clip lc.
//   fz_ctrl    (cooperative, one CTA per SM) the tile scan: start heights H_T,
//              low-water marks L_T and their 32-ary hierarchy (owner rule F1),
//              pop offsets; each tile's link owner and incoming stack as runs
//              of one owner tile (the suffix relation of P:131-138); TC(T) =
//              the context of the stack entry just below its slice, by
//              pointer jumping over tiles (F11; replaces the paper's scan of
//              partition top boxes).
//   fz_main    one CTA per tile: register walk (Fig. 1 per thread), block Bic
//              scan, thread-level owner lookups (F2), thread link contexts by
//              pointer jumping over threads, the start stacks' pops, one
//              forward walk that clips, unions and emits parent/match, the
//              suffix unions of opens closed in a later thread or tile, the
//              cross-thread closes; TMA in and out.
//   fz_hier    32-ary hierarchy of tile unions (one launch: the last block
//              builds the upper levels).
//   fz_close   closes of nodes opened in an earlier tile: tile prefix ∪ the
//              open's tile suffix ∪ the whole tiles between (F4/F7); blend
//              opens and match[open] receive the result; blend opens never
//              closed (R4) get the union of everything after them.
// Variants of the same kernels: the matching alone (fz_match, no boxes);
// scene mode (sc_count / sc_scan / sc_compact in front: the passes run on the
// compacted stream); shard mode (fused_shard.cuh: the imported stack above h0).
#include <algorithm>
#include <climits>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "boxes.cuh"
#include "common.cuh"
#include "kernels.h"
#include "stackscan.cuh"
#include "tile_common.cuh"

namespace tb {
namespace fz {

constexpr int K = 16;          // elements per thread
constexpr int LOGK = 4;
constexpr int NT = 128;        // threads per tile
constexpr int NW = NT / 32;
constexpr int W = NT * K;      // tile = 2048 elements
constexpr int LOGW = 11;
constexpr int LV = 5;          // 32-ary levels of tile unions: 32^5 tiles > 2^31 / W
static_assert(W == (1 << LOGW) && K == (1 << LOGK), "tile shape");

struct Params {
  const uint8_t* tags;
  const float4* boxes;
  int64_t n;
  int ntiles;
  int32_t* match;      // may be null (tree_bbox alone)
  int32_t* parent;     // may be null
  float4* out;
  Ctrl ctrl;
  int64_t* aoff;       // [ntiles + 1] exclusive prefix of a_T (pop records); incoming list of T at aoff[T] + T
  int32_t* slice_idx;  // [ntiles * W] global index | blend << 31
  float4* slice_box;   // [ntiles * W] lc: ∩ of the clip boxes of the slice entries at and below (fz_reduce)
  float4* slice_su;    // [ntiles * W] union of the tile's clipped leaves after the entry (fz_main)
  int2* pop;           // [aoff[ntiles]] close popping incoming depth D: (close, slice ref of its open); root: (-1, -1)
  float4* tu[LV];      // tile unions, 32-ary hierarchy
  float4* pj_acc;      // [2 * ntiles] pointer jumping over tiles
  int32_t* pj_ptr;     // [2 * ntiles]
  int32_t* pj_own;     // [ntiles] link owner: the tile that pushed the entry just below the tile's slice (-1: root)
  int2* runs;          // [ntiles * RMAX] the tile's incoming stack by owner: (owner U, L_U), heights [L_U, previous L)
  int32_t* nruns;      // [ntiles] number of runs covering the a_T + 1 top entries (may exceed RMAX)
  float4* tc;          // [ntiles] TC(T) = context of that entry
  int32_t* flag;       // [3]
  int4* blk;           // [gridDim of fz_ctrl] block aggregates (a, b, sum lo, sum hi)
  int32_t* blkmin;     // [gridDim of fz_ctrl] min low-water mark of the block's tiles
  int chunk;           // fz_ctrl: tiles per block (multiple of 32)
  uint64_t* trace;     // optional (debug): fz_ctrl phase timestamps, block 0
  int use_tma;         // fz_main: full tiles move their boxes with TMA (tensor maps below)
  // shard mode (fused_shard.cuh; all zero / null on one device): the chunk's
  // first element has global index goff; heights are offset by h0 and the
  // h0 entries below are the imported stack, a virtual slice at vbase
  int goff;
  int h0;
  int vbase;           // ntiles * W: slice reference of imported height 0
  int32_t* shd;        // [SHD] shd[1]: overflow of the shard capacity (compose step)
  int32_t* tcend;      // [ntiles] end of TC's pointer chain: -1 root, -2 - h imported height h
  int32_t* exc;        // [h0] shard: the close popping imported height h (-1: none)
  float4* exu;         // [h0] shard: its union over this chunk (the prefix before the close)
  // scene mode (stream compaction fused into the loaders):
  // the passes run on the COMPACTED stream -- tile T holds kept elements
  // [T W, T W + W) -- whose tags and full-stream indices sc_compact writes (two
  // of the outputs); fz_reduce / fz_main gather the boxes through those
  // indices, so no box is compacted over HBM.  n / ntiles are the full
  // stream's (capacity); the kept count is on the device.
  int nobox;              // matching only (fused_match_launch): no boxes, no contexts, no unions
  int pf_tiles;           // fz_main: resident CTAs on the device (the L2 prefetch distance in tiles)
  int scene;
  int keep03;              // the keep table is bytes 0-3 exactly (a compare)
  const uint32_t* keepw;   // [8] 256-bit keep table
  int64_t* nkp;            // the kept count
  const uint8_t* tags_in;  // the full stream
  const float4* boxes_in;  // its boxes
  int32_t* kcin;           // [ntiles] kept elements per full-stream tile
  int64_t* kpin;           // [ntiles + 1] their exclusive prefix
  uint8_t* tags_out;       // [n] the compacted tags
  int32_t* index_out;      // [n] full-stream index of each kept element
};
constexpr int SHD = 64;
// TMA descriptors of fz_main: per array (leaf boxes in, node boxes out) one 2D
// map per half of the thread rows: {32 floats, n/16 rows}, row stride 256 B,
// box {32, NT}, 128-byte swizzle (the slot layout of Smem::val)
struct Maps {
  CUtensorMap in[2];
  CUtensorMap out[2];
};
constexpr int MAXCTRL = 4096;  // fz_ctrl blocks (co-resident CTAs) provided for
constexpr int RMAX = 8;        // runs of the incoming stack kept per tile (more: followed in fz_main)

// ----------------------------------------------------------------------------
// workspace
// ----------------------------------------------------------------------------
struct Layout {
  size_t ctrl, aoff, sidx, sbox, ssu, pop, tu[LV], pja, pjp, pjo, tcs, rns, nrs, flag, blk, blkmin, shd, tce, kpw, nk,
      kci, kpi, bytes;
  int64_t ntiles;
  explicit Layout(int64_t n, int h0 = 0, bool nobox = false) {
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    ntiles = (n + W - 1) / W;
    const size_t cap = (size_t)ntiles * W + (size_t)h0;  // + the imported stack (shard mode)
    const size_t ntc = (size_t)ntiles + ((size_t)h0 + W - 1) / W;
    const size_t npop = (size_t)n;                    // Σ a_T <= closes
    size_t o = 0;
    shd = o; o = al(o + 4 * SHD);  // first: at the same offset for every n (fused_shard_status)
    ctrl = o; o = al(o + CtrlLayout(ntiles).bytes);
    aoff = o; o = al(o + 8 * ((size_t)ntiles + 1));
    sidx = o; o = al(o + 4 * cap);
    sbox = o; o = al(o + (nobox ? 0 : 16 * cap));  // matching only: no slice boxes / unions
    ssu = o; o = al(o + (nobox ? 0 : 16 * cap));
    pop = o; o = al(o + 8 * npop);
    int64_t m = ntiles;
    for (int k = 0; k < LV; k++) {
      tu[k] = o; o = al(o + 16 * (size_t)m);
      m = (m + 31) / 32;
    }
    pja = o; o = al(o + 32 * (size_t)ntiles);
    pjp = o; o = al(o + 8 * (size_t)ntiles);
    pjo = o; o = al(o + 4 * (size_t)ntiles);
    tcs = o; o = al(o + 16 * ntc);
    rns = o; o = al(o + 8 * RMAX * (size_t)ntiles);
    nrs = o; o = al(o + 4 * (size_t)ntiles);
    flag = o; o = al(o + 16);
    blk = o; o = al(o + 16 * MAXCTRL);
    blkmin = o; o = al(o + 4 * MAXCTRL);
    tce = o; o = al(o + 4 * (size_t)ntiles);
    kpw = o; o = al(o + 32);
    nk = o; o = al(o + 8);
    kci = o; o = al(o + 4 * (size_t)ntiles);
    kpi = o; o = al(o + 8 * ((size_t)ntiles + 1));
    bytes = o;
  }
};

static Params make_params(const uint8_t* tags, const float* boxes, int64_t n, int32_t* match, int32_t* parent,
                          float* out, void* ws, int h0 = 0, int goff = 0, bool nobox = false) {
  const Layout L(n, h0, nobox);
  char* b = (char*)ws;
  Params p;
  p.tags = tags;
  p.boxes = (const float4*)boxes;
  p.n = n;
  p.ntiles = (int)L.ntiles;
  p.match = match;
  p.parent = parent;
  p.out = (float4*)out;
  p.ctrl = CtrlLayout(L.ntiles).bind(b + L.ctrl);
  p.aoff = (int64_t*)(b + L.aoff);
  p.slice_idx = (int32_t*)(b + L.sidx);
  p.slice_box = (float4*)(b + L.sbox);
  p.slice_su = (float4*)(b + L.ssu);
  p.pop = (int2*)(b + L.pop);
  for (int k = 0; k < LV; k++) p.tu[k] = (float4*)(b + L.tu[k]);
  p.pj_acc = (float4*)(b + L.pja);
  p.pj_ptr = (int32_t*)(b + L.pjp);
  p.pj_own = (int32_t*)(b + L.pjo);
  p.tc = (float4*)(b + L.tcs);
  p.runs = (int2*)(b + L.rns);
  p.nruns = (int32_t*)(b + L.nrs);
  p.flag = (int32_t*)(b + L.flag);
  p.blk = (int4*)(b + L.blk);
  p.blkmin = (int32_t*)(b + L.blkmin);
  p.chunk = 32;
  p.trace = nullptr;
  p.use_tma = 0;
  p.goff = goff;
  p.h0 = h0;
  p.vbase = (int)(L.ntiles * W);
  p.shd = (int32_t*)(b + L.shd);
  p.tcend = (int32_t*)(b + L.tce);
  p.exc = nullptr;
  p.exu = nullptr;
  p.nobox = 0;
  p.pf_tiles = 0;
  p.scene = 0;
  p.keep03 = 0;
  p.keepw = (const uint32_t*)(b + L.kpw);
  p.nkp = (int64_t*)(b + L.nk);
  p.tags_in = nullptr;
  p.boxes_in = nullptr;
  p.kcin = (int32_t*)(b + L.kci);
  p.kpin = (int64_t*)(b + L.kpi);
  p.tags_out = nullptr;
  p.index_out = nullptr;
  return p;
}


// ----------------------------------------------------------------------------
// fz_reduce: tile Bic values, slices and their local cumulative clips
// ----------------------------------------------------------------------------
__device__ uint8_t g_unm4[UNM4_ENTRIES];  // common.cuh unm4_entry, filled once per device

// position of the j-th (0-based) set bit of m (m has more than j set bits)
__device__ __forceinline__ int select_bit32(uint32_t m, int j) {
  int pos = 0, c = __popc(m & 0xffffu);
  if (j >= c) { j -= c; pos = 16; m >>= 16; }
  c = __popc(m & 0xffu);
  if (j >= c) { j -= c; pos += 8; m >>= 8; }
  c = __popc(m & 0xfu);
  if (j >= c) { j -= c; pos += 4; m >>= 4; }
  c = __popc(m & 0x3u);
  if (j >= c) { j -= c; pos += 2; m >>= 2; }
  return pos + (j >= (int)(m & 1u) ? 1 : 0);
}

// ---- scene mode prologue: where each compacted tile starts in the full stream
// bit i = byte i of the 16 is kept (256-bit table, L1-cached)
__device__ __forceinline__ uint32_t keep16(const uint32_t* keepw, uint4 raw) {
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) {
    const uint32_t b = (w[i >> 2] >> (8 * (i & 3))) & 255u;
    m |= ((__ldg(keepw + (b >> 5)) >> (b & 31)) & 1u) << i;
  }
  return m;
}
// bytes < 4 of 16 (the hierarchy tags; keep03): bit 6 of ((x >> 2) & 0x3f) + 0x3f
// per byte is set iff x >= 4, gathered by one multiply per 8 bytes
__device__ __forceinline__ uint32_t lt4_16(uint4 raw) {
  auto hi4 = [](uint32_t x) { return ((((x >> 2) & 0x3f3f3f3fu) + 0x3f3f3f3fu) >> 6) & 0x01010101u; };
  return ~top_bytes(gather8(hi4(raw.x), hi4(raw.y)), gather8(hi4(raw.z), hi4(raw.w))) & 0xffffu;
}
// keep mask of the 64 full-stream elements [g, g + 64) (bits past n clear)
__device__ __forceinline__ uint64_t keep64(const Params& p, int64_t g) {
  uint64_t m = 0;
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const int64_t h = g + 16 * q;
    if (h >= p.n) break;
    const uint4 raw = h + 16 <= p.n ? __ldg(reinterpret_cast<const uint4*>(p.tags_in + h))
                                     : load_tags16(p.tags_in, p.n, h, false);
    const int64_t rem = p.n - h;
    const uint32_t v = rem >= 16 ? 0xffffu : ((1u << rem) - 1u);
    m |= (uint64_t)((p.keep03 ? lt4_16(raw) : keep16(p.keepw, raw)) & v) << (16 * q);
  }
  return m;
}
// kept elements of each full-stream tile (one warp per tile)
__global__ void __launch_bounds__(256) sc_count(Params p) {
  const int lane = threadIdx.x & 31;
  const int u = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (u >= p.ntiles) return;
  int c = __popcll(keep64(p, (int64_t)u * W + 64 * lane));
  c = __reduce_add_sync(0xffffffffu, c);
  if (lane == 0) p.kcin[u] = c;
}
// their exclusive prefix and the kept count: 1024 tiles per block (a block
// scan), the block totals scanned by one block, then added back
__device__ __forceinline__ long long block_scan_excl(long long v, long long& tot, long long* ws) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    long long t = ws[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, t, off);
      if (lane >= off) t += y;
    }
    ws[lane] = t;
  }
  __syncthreads();
  tot = ws[31];
  const long long r = (warp ? ws[warp - 1] : 0) + x - v;
  __syncthreads();
  return r;
}
__global__ void __launch_bounds__(1024) sc_scan1(Params p, long long* bsum) {
  __shared__ long long ws[32];
  const int u = blockIdx.x * 1024 + threadIdx.x;
  long long tot;
  const long long ex = block_scan_excl(u < p.ntiles ? __ldcg(p.kcin + u) : 0, tot, ws);
  if (u < p.ntiles) p.kpin[u] = ex;
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(1024) sc_scan2(Params p, long long* bsum, int nb) {
  __shared__ long long ws[32];
  long long tot;
  const int i = threadIdx.x;  // nb <= 1024 (ntiles <= 2^20)
  const long long ex = block_scan_excl(i < nb ? bsum[i] : 0, tot, ws);
  if (i < nb) bsum[i] = ex;
  if (i == 0) {
    p.kpin[p.ntiles] = tot;
    *p.nkp = tot;
  }
}
__global__ void __launch_bounds__(1024) sc_scan3(Params p, const long long* bsum) {
  const int u = blockIdx.x * 1024 + threadIdx.x;
  if (u < p.ntiles) p.kpin[u] += bsum[blockIdx.x];
}
// the kept elements' tags and full-stream indices at their compacted positions
// (one warp per full-stream tile from its prefix kpin; 32 consecutive elements
// per ballot step -- coalesced loads and stores)
__global__ void __launch_bounds__(256) sc_compact(Params p) {
  const int lane = threadIdx.x & 31;
  const int u = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (u >= p.ntiles) return;
  const int64_t base = (int64_t)u * W;
  int64_t co = __ldcg(p.kpin + u);
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t kt[8];
#pragma unroll
  for (int i = 0; i < 8; i++) kt[i] = __ldg(p.keepw + i);
  for (int c0 = 0; c0 < W && base + c0 < p.n; c0 += 512) {
    uint32_t bytes[16];  // 16 coalesced byte loads in flight: lane l takes element c0 + 32 b + l
#pragma unroll
    for (int b = 0; b < 16; b++) {
      const int64_t g = base + c0 + 32 * b + lane;
      bytes[b] = g < p.n ? (uint32_t)__ldg(p.tags_in + g) : 255u;
    }
#pragma unroll
    for (int b = 0; b < 16; b++) {
      const uint32_t byte = bytes[b];
      const int64_t g = base + c0 + 32 * b + lane;
      bool kept;
      if (p.keep03) {
        kept = byte < 4u;
      } else {
        uint32_t kw = kt[0];
#pragma unroll
        for (int i = 1; i < 8; i++) kw = (byte >> 5) == (uint32_t)i ? kt[i] : kw;
        kept = (kw >> (byte & 31)) & 1u;
      }
      kept = kept && g < p.n;
      const uint32_t bal = __ballot_sync(0xffffffffu, kept);
      if (kept) {
        const int64_t k = co + __popc(bal & lt);
        p.tags_out[k] = (uint8_t)byte;
        p.index_out[k] = (int32_t)g;
      }
      co += __popc(bal);
    }
  }
}

constexpr int RL = W / 32;  // 64 elements per lane
// scene mode: per warp, the compacted tile's tags and full-stream indices

template <bool SC>
__global__ void __launch_bounds__(256) fz_reduce(Params p) {
  __shared__ uint8_t bic4[256];  // Bic of 4 elements: index = open nibble | close nibble << 4; value a | b << 4
  __shared__ __align__(16) uint8_t unm4[UNM4_ENTRIES];
  const int lane = threadIdx.x & 31;
  {
    const int t = threadIdx.x;
    Bic v{0, 0};
#pragma unroll
    for (int j = 0; j < 4; j++) v = bic_combine(v, Bic{(t >> (4 + j)) & 1, (t >> j) & 1});
    bic4[t] = (uint8_t)(v.a | (v.b << 4));
    if (t < UNM4_ENTRIES / 16)
      reinterpret_cast<uint4*>(unm4)[t] = reinterpret_cast<const uint4*>(g_unm4)[t];
  }
  __syncthreads();
  const int T = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (T >= p.ntiles) return;
  const int64_t base = (int64_t)T * W, lbase = base + (int64_t)lane * RL;
  // scene mode: the compacted stream (tags_out, written by sc_compact); its
  // length is on the device, tiles past it are empty
  const int64_t nn = SC ? __ldcg(p.nkp) : p.n;
  if (SC && base >= nn) {
    if (lane == 0) p.ctrl.agg[T] = make_int2(0, 0);
    return;
  }
  uint32_t om[2], cm[2], bk[2];
  {
    uint4 raw[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int64_t g = lbase + 16 * q;
      raw[q] = g + 16 <= nn ? __ldg(reinterpret_cast<const uint4*>(p.tags + g)) : load_tags16(p.tags, nn, g, false);
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      uint32_t o, c, b;
      classify16b(raw[q], o, c, b);
      if (q & 1) {
        om[q >> 1] |= o << 16;
        cm[q >> 1] |= c << 16;
        bk[q >> 1] |= b << 16;
      } else {
        om[q >> 1] = o;
        cm[q >> 1] = c;
        bk[q >> 1] = b;
      }
    }
  }
  Bic lb{0, 0};
#pragma unroll
  for (int w = 0; w < 2; w++) {
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const uint32_t e = bic4[((om[w] >> (4 * q)) & 15u) | (((cm[w] >> (4 * q)) & 15u) << 4)];
      lb = bic_combine(lb, Bic{(int)(e & 15u), (int)(e >> 4)});
    }
  }
  Bic incl = lb, suf = lb;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const Bic a{__shfl_up_sync(0xffffffffu, incl.a, off), __shfl_up_sync(0xffffffffu, incl.b, off)};
    if (lane >= off) incl = bic_combine(a, incl);
    const Bic b{__shfl_down_sync(0xffffffffu, suf.a, off), __shfl_down_sync(0xffffffffu, suf.b, off)};
    if (lane + off < 32) suf = bic_combine(suf, b);
  }
  const Bic tot{__shfl_sync(0xffffffffu, incl.a, 31), __shfl_sync(0xffffffffu, incl.b, 31)};
  Bic ex{__shfl_up_sync(0xffffffffu, incl.a, 1), __shfl_up_sync(0xffffffffu, incl.b, 1)};
  Bic sx{__shfl_down_sync(0xffffffffu, suf.a, 1), __shfl_down_sync(0xffffffffu, suf.b, 1)};
  if (lane == 0) ex = Bic{0, 0};
  if (lane == 31) sx = Bic{0, 0};
  if (lane == 0) p.ctrl.agg[T] = make_int2(tot.a, tot.b);
  // the lane's unmatched opens that survive to the tile end: its bottom s_l,
  // at tile-relative heights l + k, slice positions [l + a_T, l + a_T + s_l)
  const int l = ex.b - ex.a - lb.a;
  const int s_l = max(lb.b - sx.a, 0);
  uint32_t sv0 = 0u, sv1 = 0u;
  if (s_l > 0) {
    int P = 0;
    const uint32_t um1 = unm32(unm4, om[1], cm[1], P);
    const uint32_t um0 = unm32(unm4, om[0], cm[0], P);
    const int c0 = __popc(um0);
    if (s_l <= c0) {
      sv0 = um0 & ((2u << select_bit32(um0, s_l - 1)) - 1u);
    } else {
      sv0 = um0;
      sv1 = um1 & ((2u << select_bit32(um1, s_l - c0 - 1)) - 1u);
    }
  }
  // lc = ∩ of the clip boxes of the slice entries at and below each entry
  // (blend opens pass the clip through, R7), 32 slice positions at a time:
  // position -> owning lane (the lanes' ranges are contiguous, in lane order)
  // -> element, one gather per lane, an inclusive ∩-scan over the lanes
  const int start = l + tot.a;
  int endm = s_l > 0 ? start + s_l : 0;  // running max of the range ends
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, endm, off);
    if (lane >= off) endm = max(endm, y);
  }
  float4 carry = bINF();
  for (int p0 = 0; p0 < tot.b; p0 += 32) {
    const int pos = p0 + lane;
    int L = 0;  // first lane with endm > pos
#pragma unroll
    for (int k = 4; k >= 0; k--) {
      const int e = __shfl_sync(0xffffffffu, endm, L + (1 << k) - 1);
      if (e <= pos) L += 1 << k;
    }
    L = min(L, 31);
    const int ostart = __shfl_sync(0xffffffffu, start, L);
    const uint32_t o0 = __shfl_sync(0xffffffffu, sv0, L), o1 = __shfl_sync(0xffffffffu, sv1, L);
    const uint32_t b0 = __shfl_sync(0xffffffffu, bk[0], L), b1 = __shfl_sync(0xffffffffu, bk[1], L);
    const bool act = pos < tot.b;
    float4 v = bINF();
    uint32_t e = 0u, blend = 0u;
    if (act) {
      const int k = pos - ostart, c0 = __popc(o0);
      const int j = k < c0 ? select_bit32(o0, k) : 32 + select_bit32(o1, k - c0);
      blend = ((j < 32 ? b0 : b1) >> (j & 31)) & 1u;
      e = (uint32_t)(base + L * RL + j);
      if (!blend && !p.nobox) v = SC ? __ldg(p.boxes_in + __ldg(p.index_out + e)) : __ldg(p.boxes + e);
      e += (uint32_t)p.goff;
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const float4 o = shfl_up_box(v, off);
      if (lane >= off) v = isect(v, o);
    }
    v = isect(v, carry);
    carry = make_float4(__shfl_sync(0xffffffffu, v.x, 31), __shfl_sync(0xffffffffu, v.y, 31),
                        __shfl_sync(0xffffffffu, v.z, 31), __shfl_sync(0xffffffffu, v.w, 31));
    if (act) {
      p.slice_idx[base + pos] = (int)(e | (blend << 31));
      if (!p.nobox) p.slice_box[base + pos] = v;
      else p.match[e - (uint32_t)p.goff] = -1;  // matching alone: a later tile writes the partner (fz_match E)
    }
  }
}

// ----------------------------------------------------------------------------
// fz_ctrl (cooperative): tile scan, low-water hierarchy, TC by pointer jumping,
// slice contexts
// ----------------------------------------------------------------------------
// Bic value of a run of tiles (§3) and the sum of their a
struct Agg {
  int a, b;
  long long s;
};
__device__ __forceinline__ Agg agg_combine(Agg x, Agg y) {
  const Bic c = bic_combine(Bic{x.a, x.b}, Bic{y.a, y.b});
  return Agg{c.a, c.b, x.s + y.s};
}
__device__ __forceinline__ Agg shfl_up_agg(Agg v, int d) {
  return Agg{__shfl_up_sync(0xffffffffu, v.a, d), __shfl_up_sync(0xffffffffu, v.b, d),
             (long long)__shfl_up_sync(0xffffffffu, (unsigned long long)v.s, d)};
}
constexpr int NTC = 1024;  // fz_ctrl threads per block (one block per SM: cheap grid barriers)
constexpr int NWC = NTC / 32;
// exclusive scan of v over the block's threads in thread order
__device__ __forceinline__ void block_excl(Agg v, Agg& ex, Agg& tot, Agg* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Agg incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const Agg o = shfl_up_agg(incl, off);
    if (lane >= off) incl = agg_combine(o, incl);
  }
  if (lane == 31) sh[warp] = incl;
  __syncthreads();
  if (warp == 0) {  // scan of the warp totals
    Agg x = sh[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const Agg o = shfl_up_agg(x, off);
      if (lane >= off) x = agg_combine(o, x);
    }
    sh[lane] = x;  // inclusive
  }
  __syncthreads();
  const Agg wpre = warp ? sh[warp - 1] : Agg{0, 0, 0};
  Agg e = shfl_up_agg(incl, 1);
  if (lane == 0) e = Agg{0, 0, 0};
  ex = agg_combine(wpre, e);
  tot = sh[NWC - 1];
  __syncthreads();
}
__device__ __forceinline__ int block_min(int v, int* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = __reduce_min_sync(0xffffffffu, v);
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  const int m = __reduce_min_sync(0xffffffffu, sh[lane]);
  __syncthreads();
  return m;
}

// owner rule F1 over the low-water hierarchy written by this kernel (L2 loads)
__device__ __forceinline__ int owner_search_cg(const Ctrl& c, int from, int X, int& Lout) {
  const int lane = threadIdx.x & 31;
  const uint32_t ux = (uint32_t)X;
  {
    const int t = from - 1 - lane;
    const uint32_t v = t >= 0 ? __ldcg(c.lw + t) - 1u : 0xffffffffu;
    const unsigned m = __ballot_sync(0xffffffffu, t >= 0 && v <= ux);
    if (m) {
      const int k = __ffs(m) - 1;
      Lout = (int)__shfl_sync(0xffffffffu, v, k);
      return from - 1 - k;
    }
    if (from <= 32) return -1;
    from -= 32;
  }
  int idx = from;
#pragma unroll 1
  for (int k = 0; k < HLEVELS; k++) {
    const int g = idx >> 5, r = idx & 31;
    const uint32_t v = lane < r ? __ldcg(c.lv[k] + ((size_t)g << 5) + lane) - 1u : 0xffffffffu;
    const unsigned m = __ballot_sync(0xffffffffu, lane < r && v <= ux);
    if (m) {
      int E = (g << 5) + (31 - __clz(m));
      uint32_t L = __shfl_sync(0xffffffffu, v, 31 - __clz(m));
#pragma unroll 1
      for (int j = k - 1; j >= 0; j--) {
        const uint32_t v2 = __ldcg(c.lv[j] + ((size_t)E << 5) + lane) - 1u;
        const unsigned m2 = __ballot_sync(0xffffffffu, v2 <= ux);
        const int top = 31 - __clz(m2);
        L = __shfl_sync(0xffffffffu, v2, top);
        E = (E << 5) + top;
      }
      Lout = (int)L;
      return E;
    }
    idx = g;
    if (idx == 0) break;
  }
  return -1;
}

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define FZ_TRACE(k)                                                              \
  do {                                                                           \
    if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) p.trace[(k)] = gtimer(); \
  } while (0)

constexpr int CMAX = 1024;  // tiles per fz_ctrl block kept in shared memory (larger chunks: no in-block ANSV)
constexpr int CLOG = 10;

__global__ void __launch_bounds__(NTC, 1) fz_ctrl(Params p) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ Agg sh[NWC];
  __shared__ int shm[NWC];
  __shared__ __align__(16) int mw[CLOG][CMAX];  // ANSV windows over the chunk (levels >= 1); then P3's local jumps
  __shared__ int nun;
  __shared__ int unres[CMAX];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // (scene mode: only the tiles of the compacted stream, whose length is on the device)
  const int nt = p.scene ? (int)((__ldcg(p.nkp) + W - 1) / W) : p.ntiles, G = gridDim.x, bx = blockIdx.x;
  const int C = p.chunk;  // tiles per block, a multiple of 32 (level-1 groups stay inside a block)
  const int t0 = min(bx * C, nt), t1 = min(t0 + C, nt);
  const int per = (C + NTC - 1) / NTC;
  const int ta = min(t0 + tid * per, t1), tb = min(ta + per, t1);  // this thread's tiles
  FZ_TRACE(0);

  // P0: Bic value and a-sum of the block's tiles
  Agg v{0, 0, 0};
  for (int T = ta; T < tb; T++) {
    const int2 g = __ldcg(p.ctrl.agg + T);
    v = agg_combine(v, Agg{g.x, g.y, g.x});
  }
  Agg ex, tot;
  block_excl(v, ex, tot, sh);
  if (tid == 0) {
    p.blk[bx] = make_int4(tot.a, tot.b, (int)(unsigned)(tot.s & 0xffffffffll), (int)(tot.s >> 32));
    if (bx == 0) {
      p.flag[0] = p.flag[1] = p.flag[2] = p.flag[3] = 0;  // [3]: fz_hier's arrival counter
    }
  }
  grid.sync();
  FZ_TRACE(1);

  // P1: prefix over earlier blocks; start heights H, low-water marks L = max(H - a, 0),
  // pop offsets; level 1 of the low-water hierarchy (32-tile groups inside the block)
  Agg pre;
  {
    const int perb = (bx + NTC - 1) / NTC;
    const int ba = min(tid * perb, bx), bb = min(ba + perb, bx);
    Agg u{0, 0, 0};
    for (int j = ba; j < bb; j++) {
      const int4 x = __ldcg(p.blk + j);
      u = agg_combine(u, Agg{x.x, x.y, (long long)(((unsigned long long)(unsigned)x.w << 32) | (unsigned)x.z)});
    }
    Agg ux, ut;
    block_excl(u, ux, ut, sh);
    pre = ut;
  }
  int lmin = INT_MAX;
  {
    Agg cur = agg_combine(pre, ex);
    for (int T = ta; T < tb; T++) {
      const int2 g = __ldcg(p.ctrl.agg + T);
      // one device: the height is the prefix's b (its a closes popped the root);
      // shard mode: h0 imported entries below, the prefix's a of them popped
      const int H = p.h0 ? p.h0 - cur.a + cur.b : cur.b;
      const int L = max(H - g.x, 0);
      p.ctrl.hstart[T] = H;
      p.ctrl.lw[T] = (uint32_t)L + 1u;
      p.aoff[T] = cur.s;
      lmin = min(lmin, L);
      cur = agg_combine(cur, Agg{g.x, g.y, g.x});
    }
    if (tb == nt && ta < tb) {
      *p.ctrl.total = make_int2(cur.a, cur.b);
      p.aoff[nt] = cur.s;
    }
  }
  lmin = block_min(lmin, shm);
  if (tid == 0) p.blkmin[bx] = lmin;
  for (int g = (t0 >> 5) + warp; g < ((t1 + 31) >> 5); g += NWC) {
    const int i = g * 32 + lane;
    uint32_t x = i < nt ? __ldcg(p.ctrl.lw + i) : 0xffffffffu;
    x = __reduce_min_sync(0xffffffffu, x);
    if (lane == 0) p.ctrl.lv[1][g] = x;
  }
  grid.sync();
  FZ_TRACE(2);

  // P2: smin (min L over the later tiles: which slice entries survive to the
  // end, F1); the upper levels of the hierarchy (block 0)
  {
    int after = INT_MAX;
    for (int j = bx + 1 + tid; j < G; j += NTC) after = min(after, __ldcg(p.blkmin + j));
    after = block_min(after, shm);
    int mine = INT_MAX;
    for (int T = ta; T < tb; T++) mine = min(mine, (int)__ldcg(p.ctrl.lw + T) - 1);
    // exclusive suffix min over the threads after this one
    int x = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_down_sync(0xffffffffu, x, off);
      if (lane + off < 32) x = min(x, y);
    }
    if (lane == 0) shm[warp] = x;
    __syncthreads();
    int later = after;
    for (int w = warp + 1; w < NWC; w++) later = min(later, shm[w]);
    int sx = __shfl_down_sync(0xffffffffu, x, 1);
    if (lane == 31) sx = INT_MAX;
    int run = min(later, sx);
    for (int T = tb - 1; T >= ta; T--) {
      p.ctrl.smin[T] = run;
      run = min(run, (int)__ldcg(p.ctrl.lw + T) - 1);
    }
    __syncthreads();
  }
  if (bx == 0) {
    int m = (nt + 31) / 32;  // nodes at level 1
    for (int k = 2; k < HLEVELS; k++) {
      __syncthreads();
      const int groups = (m + 31) / 32;
      for (int g = warp; g < groups; g += NWC) {
        const int i = g * 32 + lane;
        uint32_t x = i < m ? __ldcg(p.ctrl.lv[k - 1] + i) : 0xffffffffu;
        x = __reduce_min_sync(0xffffffffu, x);
        if (lane == 0) p.ctrl.lv[k][g] = x;
      }
      m = groups;
    }
  }
  grid.sync();
  FZ_TRACE(3);

  // P3: the link owner of each tile = the tile that pushed the entry at height
  // L_T - 1 (F1: the last tile U < T with L_U < L_T, a previous-smaller value)
  // and TC's initial pointer.  Inside the block's chunk by binary lifting over
  // window minima in shared memory; tiles with no smaller value earlier in the
  // chunk ask the global hierarchy (one warp each).
  const bool local = C <= CMAX;
  if (tid == 0) nun = 0;
  if (local) {
    // mw[k][i] = min L over chunk tiles [i - 2^k + 1, i] (k >= 1; level 0 read from lw)
    const int cn = t1 - t0;
    __syncthreads();
    for (int k = 1; k < CLOG && (1 << k) <= cn; k++) {
      for (int i = tid; i < cn; i += NTC) {
        const int h = 1 << (k - 1);
        const int a = k == 1 ? (int)__ldcg(p.ctrl.lw + t0 + i) - 1 : mw[k - 1][i];
        const int b = i - h >= 0 ? (k == 1 ? (int)__ldcg(p.ctrl.lw + t0 + i - h) - 1 : mw[k - 1][i - h]) : INT_MAX;
        mw[k][i] = min(a, b);
      }
      __syncthreads();
    }
    for (int T = t0 + tid; T < t1; T += NTC) {
      const int L = (int)__ldcg(p.ctrl.lw + T) - 1;
      int U = -1;
      if (L >= 1) {
        int pos = T - 1 - t0;  // chunk-local
        for (int k = CLOG - 1; k >= 1; k--) {
          if ((1 << k) <= cn && pos - (1 << k) + 1 >= 0 && mw[k][pos] >= L) pos -= 1 << k;
        }
        if (pos >= 0 && (int)__ldcg(p.ctrl.lw + t0 + pos) - 1 >= L) pos--;
        if (pos >= 0) {
          U = t0 + pos;
        } else {
          unres[atomicAdd(&nun, 1)] = T;
          continue;
        }
      }
      float4 acc = bINF();
      if (U >= 0 && !p.nobox) acc = __ldcg(p.slice_box + (int64_t)U * W + (L - 1 - ((int)__ldcg(p.ctrl.lw + U) - 1)));
      p.pj_acc[T] = acc;
      p.pj_ptr[T] = U >= 0 || L < 1 ? U : -2 - (L - 1);  // no local owner: imported height L - 1
      p.pj_own[T] = U;
    }
    __syncthreads();
  }
  FZ_TRACE(9);
  {
    // unresolved tiles (or every tile when the chunk is too long for shared memory)
    const int cnt = local ? nun : (t1 - t0);
    for (int j = warp; j < cnt; j += NWC) {
      const int T = local ? unres[j] : t0 + j;
      const int L = (int)__ldcg(p.ctrl.lw + T) - 1;
      float4 acc = bINF();
      int U = -1;
      if (L >= 1) {
        int LU = 0;
        U = owner_search_cg(p.ctrl, T, L - 1, LU);
        if (U >= 0 && !p.nobox) acc = __ldcg(p.slice_box + (int64_t)U * W + (L - 1 - LU));
      }
      if (lane == 0) {
        p.pj_acc[T] = acc;
        p.pj_ptr[T] = U >= 0 || L < 1 ? U : -2 - (L - 1);
        p.pj_own[T] = U;
      }
    }
  }
  FZ_TRACE(10);
  if (local && !p.nobox) {
    // pointer jumping inside the chunk first (block barriers, shared memory):
    // the grid rounds of P4 then only follow pointers that leave the chunk
    static_assert(sizeof(mw) >= 2 * CMAX * (sizeof(float4) + sizeof(int)), "local jump buffers");
    float4* la = reinterpret_cast<float4*>(&mw[0][0]);
    int* lp = reinterpret_cast<int*>(la + 2 * CMAX);
    const int cn = t1 - t0;
    __syncthreads();  // the chunk's pj values (this block's global writes) and mw dead
    int more = 0;
    for (int i = tid; i < cn; i += NTC) {
      la[i] = __ldcg(p.pj_acc + t0 + i);
      lp[i] = __ldcg(p.pj_ptr + t0 + i);
      more |= lp[i] >= t0;
    }
    int cb = 0;
    bool any = __syncthreads_or(more);
    while (any) {
      more = 0;
      for (int i = tid; i < cn; i += NTC) {
        float4 a = la[cb * CMAX + i];
        int q = lp[cb * CMAX + i];
        if (q >= t0) {
          a = isect(a, la[cb * CMAX + q - t0]);
          q = lp[cb * CMAX + q - t0];
          more |= q >= t0;
        }
        la[(cb ^ 1) * CMAX + i] = a;
        lp[(cb ^ 1) * CMAX + i] = q;
      }
      cb ^= 1;
      any = __syncthreads_or(more);
    }
    for (int i = tid; i < cn; i += NTC) {
      p.pj_acc[t0 + i] = la[cb * CMAX + i];
      p.pj_ptr[t0 + i] = lp[cb * CMAX + i];
    }
  }
  grid.sync();
  FZ_TRACE(4);

  // P4: TC(T) = acc ∩ TC(ptr) by pointer jumping (thread per tile), one grid
  // barrier per round; flag r % 3 collects round r's "not done", flag
  // (r + 1) % 3 is cleared in round r
  const int gt = (int)(bx * (int64_t)blockDim.x + tid);
  const int nthr = (int)(G * (int64_t)blockDim.x);
  // the incoming stack of each tile (its a_T + 1 top entries) as runs of one
  // owner each: T - 1 owns heights [L_{T-1}, H_T); below a run of U the owner
  // is U's link owner (F1) -- a walk along the link-owner pointers
  for (int T = gt; T < nt; T += nthr) {
    const int H = __ldcg(p.ctrl.hstart + T);
    const int aT = __ldcg(p.ctrl.agg + T).x;
    const int lo = max(H - 1 - aT, 0);
    int hi = H - 1, U = T - 1, k = 0;
    while (hi >= lo && U >= 0) {
      const int LU = (int)__ldcg(p.ctrl.lw + U) - 1;
      const int nxt = __ldcg(p.pj_own + U);
      if (LU <= hi) {
        if (k < RMAX) p.runs[(int64_t)T * RMAX + k] = make_int2(U, LU);
        k++;
        hi = LU - 1;
      }
      U = nxt;
    }
    p.nruns[T] = k;
  }
  FZ_TRACE(8);
  if (p.nobox) return;  // matching only: no tile contexts
  // the two buffers of each array by selects (a runtime index into a pointer
  // array would place it in local memory)
  auto accb = [&](int b) { return b ? p.pj_acc + nt : p.pj_acc; };
  auto ptrb = [&](int b) { return b ? p.pj_ptr + nt : p.pj_ptr; };
  // at most one tile per thread (nt <= threads of the grid, n <= 3.1e8 on a
  // B200): its value and pointer stay in registers across the rounds
  const bool one = nt <= nthr;
  float4 ra = bINF();
  int rq = -1;
  if (one && gt < nt) {
    ra = __ldcg(accb(0) + gt);
    rq = __ldcg(ptrb(0) + gt);
  }
  int cb = 0;
  for (int round = 0; round < 64; round++) {
    if (gt == 0) p.flag[(round + 1) % 3] = 0;
    int any = 0;
    if (one) {
      if (rq >= 0) {
        ra = isect(ra, __ldcg(accb(cb) + rq));
        rq = __ldcg(ptrb(cb) + rq);
        any = rq >= 0;
      }
      if (gt < nt) {
        accb(cb ^ 1)[gt] = ra;
        ptrb(cb ^ 1)[gt] = rq;
      }
    } else {
      for (int V = gt; V < nt; V += nthr) {
        float4 a = __ldcg(accb(cb) + V);
        int q = __ldcg(ptrb(cb) + V);
        if (q >= 0) {
          a = isect(a, __ldcg(accb(cb) + q));
          q = __ldcg(ptrb(cb) + q);
          any |= q >= 0;
        }
        accb(cb ^ 1)[V] = a;
        ptrb(cb ^ 1)[V] = q;
      }
    }
    any = __syncthreads_or(any);
    if (any && tid == 0) atomicOr(p.flag + round % 3, 1);
    cb ^= 1;
    grid.sync();
    if (__ldcg(p.flag + round % 3) == 0) {
      if (p.trace && bx == 0 && tid == 0) p.trace[6] = (uint64_t)round + 1;
      break;
    }
  }
  FZ_TRACE(5);
  // P5: TC for the main pass (slice context = lc ∩ TC of the slice's tile)
  if (one) {
    if (gt < nt) {
      p.tc[gt] = ra;
      p.tcend[gt] = rq;  // -1, or -2 - h: TC still lacks imported height h's context
    }
  } else {
    for (int V = gt; V < nt; V += nthr) {
      p.tc[V] = __ldcg(accb(cb) + V);
      p.tcend[V] = __ldcg(ptrb(cb) + V);
    }
  }
  FZ_TRACE(7);
}

// ----------------------------------------------------------------------------
// fz_main
// ----------------------------------------------------------------------------
struct Walk {
  uint32_t om, cm, bm, lm;  // opens, closes, blend opens, leaves (valid elements only)
  uint32_t S;               // opens still on the thread stack at its end (thread-unmatched)
  uint32_t plo, phi;        // nibble i: in-thread parent of element i (a matched close: its open)
  uint32_t ext;             // elements whose parent lies before the thread
  uint32_t ucm;             // closes with no in-thread open (they pop the stack at the thread start)
};

// Fig. 1 over the thread's 16 elements with a bitmask stack (four
// groups of four elements: a rolled outer loop keeps the code small).  An
// in-thread open's match is stored at its pop (mrow[i] = element i's match
// slot: gtb + its close); BM: the blend-open mask too (fz_main; the matching
// alone has no boxes)
template <bool BM>
__device__ __forceinline__ Walk walk_m(uint4 raw, uint32_t valid, int32_t* mrow, int gtb) {
  Walk w;
  if (BM) {
    classify16b(raw, w.om, w.cm, w.bm);
  } else {
    classify16(raw, w.om, w.cm);
    w.bm = 0u;
  }
  w.om &= valid;
  w.cm &= valid;
  w.bm &= valid;
  w.lm = valid & ~(w.om | w.cm);
  uint32_t S = 0, plo = 0, phi = 0, ext = 0;
#pragma unroll 1
  for (int q = 0; q < K / 4; q++) {
    const int i0 = 4 * q;
    const uint32_t oq = w.om >> i0, cq = w.cm >> i0;
    uint32_t gp = 0, gx = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int i = i0 + j;
      const int top = 31 - __clz(S);  // -1 when the thread stack is empty
      gp |= (uint32_t)(top & 15) << (4 * j);
      gx |= S ? 0u : (1u << j);
      const bool pop = ((cq >> j) & 1u) && S;
      if (pop) mrow[top] = gtb + i;
      S = ((oq >> j) & 1u) ? (S | (1u << i)) : (pop ? (S ^ (1u << top)) : S);
    }
    const int sh = 16 * (q & 1);
    if (q < 2) plo |= gp << sh;
    else phi |= gp << sh;
    ext |= gx << i0;
  }
  w.S = S;
  w.plo = plo;
  w.phi = phi;
  w.ext = ext;
  w.ucm = w.cm & ext;
  return w;
}

constexpr int RCAP = 7;      // segment unions kept per thread (more unmatched opens: recomputed in H1)
constexpr int INCCAP = 192;  // incoming entries cached in shared memory (deeper ones: read from global)

// Shared memory of fz_main (<= 56 KB: four CTAs per SM).  The scratch region u
// is reused phase by phase: B-C owner windows; D link contexts; (l, uo, link
// kept through E); F-H1 segment unions; G-H2 the range table over threads.
struct Smem {
  float4 val[W];                    // boxes -> lc / contexts / clips / unions (swizzled slots)
  int32_t matchS[W + W / K];        // match values (global indices), padded: element e at e + e / K
  union {
    struct {
      int lwin[NW][5][32];          // low-water windows (thread owner lookups)
      int lwmin[NW];
    } ref;
    struct {
      float4 acc[2][NT];            // thread link contexts by pointer jumping
      int ptr[2][NT];
      int l[NT];                    // kept B-E
      uint32_t uo[NT];
      int link[NT];
      int inc_idx[INCCAP];          // A-E: incoming entries at depth D < INCCAP (cp.async): slice_idx value (-1: root)
      int inc_ref[INCCAP];          //      slice reference
      float4 inc_box[INCCAP];       //      lc
      float4 inc_tc[INCCAP];        //      TC of the owner tile
    } pj;
    float4 rbuf[RCAP][NT];          // F-H1: the accumulator at each thread-unmatched open (k < RCAP)
    struct {
      float4 win[5][NT];            // win[k][t] = union of threads [t - 2^k + 1, t] within t's warp (k = 0: t)
      float4 pre[NT];               // inclusive prefix within the warp
      float4 suf[NT];               // inclusive suffix within the warp
    } rt;
  } u;
  int2 runs[RMAX];
  uint64_t mbar;                    // TMA completion of the box tile
  uint32_t bmS[NT];                 // blend opens of each thread
  float4 wtu[NW];                   // warp unions
  float4 wmid[NW][NW];              // union of the warps strictly between
  Bic wtot[NW];
};
static_assert(sizeof(Smem) <= 56 * 1024, "four CTAs per SM");
// rbuf addressed as val[RB0 + k * NT + t] (both arrays of float4 in one shared block)
constexpr int RB0 = (int)((offsetof(Smem, u) - offsetof(Smem, val)) / sizeof(float4));
static_assert((offsetof(Smem, u) - offsetof(Smem, val)) % sizeof(float4) == 0, "rbuf alignment");

// Box slots: the tile as two halves (elements 0-7 and 8-15 of every thread),
// each NT rows of 128 bytes with the TMA 128-byte swizzle: element i of thread
// t lives at slot (i / 8) * 8 NT + 8 t + ((i mod 8) ^ (t mod 8)).  One TMA box
// per half moves a whole tile; the per-thread accesses are conflict-free (8
// lanes, distinct t mod 8).
__device__ __forceinline__ int slot_of(int e) {
  const int t = e >> LOGK, i = e & (K - 1);
  return ((i & 8) << 7) | (t << 3) | ((i & 7) ^ (t & 7));
}
static_assert(NT * 8 == 1024 && K == 16, "slot layout");
__device__ __forceinline__ int mpad(int e) { return e + (int)((unsigned)e >> LOGK); }

// union of the clipped leaves of whole threads [a, b] (F4): inside one warp two
// overlapping backward windows (min/max are idempotent); across warps the
// suffix of a's warp, the warps between, the prefix of b's warp
__device__ __forceinline__ float4 range_threads(const Smem& s, int a, int b) {
  if (a > b) return bEMPTY();
  const int wa = a >> 5, wb = b >> 5;
  if (wa == wb) {
    const int len = b - a + 1;
    if (len == 32) return s.wtu[wa];
    const int k = 31 - __clz(len);
    return unite(s.u.rt.win[k][b], s.u.rt.win[k][a + (1 << k) - 1]);
  }
  return unite(unite(s.u.rt.suf[a], s.u.rt.pre[b]), s.wmid[wa][wb]);
}

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) { return (uint32_t)__cvta_generic_to_shared(ptr); }
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred pr; mbarrier.try_wait.parity.shared::cta.b64 pr, [%1], %2; selp.u32 %0, 1, 0, pr; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(c0),
               "r"(c1), "r"(src)
               : "memory");
}

// slice reference (owner tile * W + slice position) of the entry at height h
// (>= 0) of the tile's incoming stack: the first run whose low-water mark is
// <= h; past the stored runs, the walk along the link owners continues
template <class S>
__device__ __forceinline__ int inc_ref(const Params& p, const S& s, int nruns, int h) {
  const int nr = min(nruns, RMAX);
  for (int k = 0; k < nr; k++) {
    const int2 r = s.runs[k];
    if (r.y <= h) return r.x * W + (h - r.y);
  }
  if (nruns > RMAX) {  // the incoming stack has more than RMAX runs
    int U = __ldg(p.pj_own + s.runs[RMAX - 1].x);
    while (U >= 0) {
      const int LU = (int)__ldg(p.ctrl.lw + U) - 1;
      if (LU <= h) return U * W + (h - LU);
      U = __ldg(p.pj_own + U);
    }
  }
  return p.vbase + h;  // below every run of this chunk: the imported stack (shard mode)
}

#ifndef FZ_MINB
#define FZ_MINB 4
#endif
template <bool PM, bool SC>
__global__ void __launch_bounds__(NT, FZ_MINB) fz_main(Params p, const __grid_constant__ Maps maps) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockIdx.x;
  const int64_t base = (int64_t)T * W;
  const int64_t nn = SC ? __ldg(p.nkp) : p.n;  // scene mode: the compacted stream's length
  if (SC && base >= nn) {                       // a tile past it: no leaves
    if (tid == 0) p.tu[0][T] = bEMPTY();
    return;
  }
  const int nvalid = (int)(nn - base < W ? nn - base : W);
  const int gbase = p.goff + (int)base;  // global indices fit in int32 (n <= 2^31 - 1)
  const int tl0 = tid * K;      // tile-local index of the thread's first element
  const int gtb = gbase + tl0;
  const int sb = (tid << 3) | (tid & 7);  // slot(tid, i) = ((i & 8) << 7) | (sb ^ (i & 7))
  auto sl = [sb](int i) { return sb ^ ((i * 129) & 0x407); };  // (i & 7) | (i & 8) << 7, one IMAD + LOP3
  const int mb = mpad(tl0);                  // matchS index of element i = mb + i

  // ---- A. loads, register walk -------------------------------------------------
  const uint4 raw = load_tags16(p.tags, nn, base + tl0, nvalid == W);
  if (tid < W / 128) {  // the tags of the tile that will take this CTA's place (about one residency later) into L2
    const int64_t pf = base + (int64_t)p.pf_tiles * W + tid * 128;
    if (pf < nn) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.tags + pf));
  }
  const int H = __ldg(p.ctrl.hstart + T);
  const int aT = __ldg(p.ctrl.agg + T).x;
  const int64_t poff = __ldg(p.aoff + T);  // pop records of this tile: [poff, poff + a_T)
  // the boxes of a full tile arrive by TMA (two 16 KB boxes, one per half of
  // the thread rows); the last, partial tile is copied by the threads
  const uint32_t val_sa = smem_u32(&s.val[0]), mbar = smem_u32(&s.mbar);
  const bool tma = p.use_tma && nvalid == W && (val_sa & 1023u) == 0u;  // TMA store (and load, off scene mode)
  if (tma && !SC) {
    if (tid == 0) {
      mbar_init(mbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(mbar, 2 * NT * 128);
      tma_load_2d(val_sa, &maps.in[0], 0, T * NT, mbar);
      tma_load_2d(val_sa + NT * 128, &maps.in[1], 0, T * NT, mbar);
    }
  } else if (SC) {  // the kept elements' boxes, through their full-stream indices (all in flight)
    int gi[K];
#pragma unroll
    for (int j = 0; j < K; j++) {
      const int e = j * NT + tid;
      gi[j] = e < nvalid ? __ldg(p.index_out + base + e) : -1;
    }
#pragma unroll
    for (int j = 0; j < K; j++) s.val[slot_of(j * NT + tid)] = gi[j] >= 0 ? __ldg(p.boxes_in + gi[j]) : bEMPTY();
  } else {
#pragma unroll 1
    for (int j = 0; j < K; j++) {
      const int e = j * NT + tid;
      s.val[slot_of(e)] = e < nvalid ? __ldg(p.boxes + base + e) : bEMPTY();
    }
  }
  // the tile's incoming stack as runs of one owner tile each (fz_ctrl)
  if (tid < RMAX) {
    cp_async8(smem_u32(&s.runs[tid]), p.runs + (int64_t)T * RMAX + tid);
    cp_async_commit();
  }
  const int nruns = __ldg(p.nruns + T);
  const int nv_t = nvalid - tl0;
  const uint32_t valid = nv_t >= K ? 0xffffu : (nv_t <= 0 ? 0u : ((1u << nv_t) - 1u));
  const Walk w = walk_m<true>(raw, valid, s.matchS + mb, gtb);  // an in-thread open's close: matchS[mb + i] - gtb
  const int a_t = __popc(w.ucm), b_t = __popc(w.S);

  // ---- B. block Bic scan: relative height at the thread start, low-water mark
  if (tid < RMAX) cp_async_wait_all();
  Bic ex, sx, tot;
  block_bic_scans<NW>(Bic{a_t, b_t}, s.wtot, ex, sx, tot, false);
  const int r_t = ex.b - ex.a;
  const int l_t = r_t - a_t;
#pragma unroll
  for (int i = 0; i < K; i++)  // closed by another thread / tile (a fixed predicated loop)
    if ((w.S >> i) & 1u) s.matchS[mb + i] = -1;
  int wl[5];
  lane_windows(l_t, wl);
#pragma unroll
  for (int k = 0; k < 5; k++) s.u.ref.lwin[warp][k][lane] = wl[k];
  {
    const int o = __shfl_sync(0xffffffffu, wl[4], 15);
    if (lane == 31) s.u.ref.lwmin[warp] = min(wl[4], o);
  }
  s.u.pj.l[tid] = l_t;
  s.u.pj.uo[tid] = w.S;
  s.bmS[tid] = w.bm;
  __syncthreads();

  // ---- C. thread-level owner lookups (F2); lc of the thread-unmatched opens --
  // the incoming entries at depths D < INCCAP, fetched asynchronously (used in D-E)
  const int ninc = min(aT + 1, INCCAP);
  for (int D = tid; D < ninc; D += NT) {
    const int h = H - 1 - D;
    if (h < 0) {
      s.u.pj.inc_idx[D] = -1;
      s.u.pj.inc_ref[D] = -1;
      s.u.pj.inc_box[D] = bINF();
      s.u.pj.inc_tc[D] = bINF();
    } else {
      const int ref = inc_ref(p, s, nruns, h);
      s.u.pj.inc_ref[D] = ref;
      cp_async4(smem_u32(&s.u.pj.inc_idx[D]), p.slice_idx + ref);
      cp_async16(smem_u32(&s.u.pj.inc_box[D]), p.slice_box + ref);
      cp_async16(smem_u32(&s.u.pj.inc_tc[D]), p.tc + (ref >> LOGW));
    }
  }
  cp_async_commit();
  int top_ref = 0, lk = 0;
#pragma unroll 1
  for (int qq = 0; qq < 2; qq++) {  // one inlined copy of the lookup
    const int r = thread_ref<NW, K>(wl, l_t, w.S, qq ? l_t - 1 : r_t - 1, s.u.ref.lwin, s.u.ref.lwmin, s.u.pj.l,
                                    s.u.pj.uo);
    if (qq) lk = r;
    else top_ref = r;
  }
  s.u.pj.link[tid] = lk;
  if (tma && !SC) mbar_wait(mbar, 0);
  {
    float4 acc = bINF();
    for (uint32_t q = w.S; q; q &= q - 1) {
      const int i = __ffs(q) - 1;
      float4& v = s.val[sl(i)];
      if (!((w.bm >> i) & 1u)) acc = isect(acc, v);
      v = acc;
    }
  }
  cp_async_wait_all();
  __syncthreads();

  // ---- D. context of each thread's link: TL(t) = lc(link) ∩ TL(thread of link)
  //      (pointer jumping over threads); the link's global index
  int giLast, cbf;
  float4 TL;
  {
    float4 acc = bINF();
    int ptr = -1;
    if (lk >= 0) {
      acc = s.val[slot_of(lk)];
      ptr = lk >> LOGK;
      giLast = gbase + lk;
    } else {
      const int D = -lk - 1;
      giLast = -1;
      if (H - 1 - D >= 0) {
        int si;
        if (D < INCCAP) {
          si = s.u.pj.inc_idx[D];
          acc = isect(s.u.pj.inc_box[D], s.u.pj.inc_tc[D]);
        } else {
          const int ref = inc_ref(p, s, nruns, H - 1 - D);
          si = __ldg(p.slice_idx + ref);
          acc = isect(__ldg(p.slice_box + ref), __ldg(p.tc + (ref >> LOGW)));
        }
        giLast = si == -1 ? -1 : si & 0x7fffffff;  // -1: an imported slot below the global root (INF)
      }
    }
    int cb = 0;
    s.u.pj.acc[0][tid] = acc;
    s.u.pj.ptr[0][tid] = ptr;
    int any = __syncthreads_or(ptr >= 0);
    while (any) {
      if (ptr >= 0) {
        acc = isect(acc, s.u.pj.acc[cb][ptr]);
        ptr = s.u.pj.ptr[cb][ptr];
      }
      s.u.pj.acc[cb ^ 1][tid] = acc;
      s.u.pj.ptr[cb ^ 1][tid] = ptr;
      cb ^= 1;
      any = __syncthreads_or(ptr >= 0);
    }
    TL = acc;
    cbf = cb;  // pj.acc[cbf] holds every thread's TL
  }

  // ---- E. entries popped by this thread's unmatched closes c_0 .. c_{a_t - 1}
  //      (c_d pops the entry at depth d of the thread's start stack): c_d's
  //      match (= its parent and that of the elements before it at depth d) in
  //      matchS[c_d]; the partner of a popped in-tile open; the context at
  //      depth d where a leaf or open sits there, in c_d's slot (depth a_t:
  //      the link, TL(t))
  uint32_t xcm = 0;  // closes popping an entry of an earlier tile
  uint32_t icm = 0;  // closes popping an open of an earlier thread of this tile
  {
    int ref = top_ref, d = 0, prevc = -1;
    uint32_t q = w.ucm;
    const uint32_t needm = w.ext & (w.lm | w.om);
    if (d < a_t && ref >= 0) {
      // the owner thread's unmatched-open mask stays in a register; shared
      // memory is read again only when the chain moves to another thread
      int V = ref >> LOGK, bp = ref & (K - 1);
      uint32_t uV = s.u.pj.uo[V];
      float4 tV = s.u.pj.acc[cbf][V];
      while (true) {
        const int e = (V << LOGK) | bp;  // the entry at depth d: a tile-local open
        const int ci = __ffs(q) - 1;
        q &= q - 1;
        const uint32_t seg = ((1u << ci) - 1u) & ~((1u << (prevc + 1)) - 1u);  // elements at depth d
        prevc = ci;
        icm |= 1u << ci;
        s.matchS[mb + ci] = gbase + e;
        s.matchS[mpad(e)] = gtb + ci;
        {  // the context at depth d (loads unconditional, the store predicated)
          const float4 cx = isect(s.val[slot_of(e)], tV);
          if (seg & needm) s.val[sl(ci)] = cx;
        }
        if (++d >= a_t) break;
        const uint32_t below = uV & ((1u << bp) - 1u);
        if (below) {
          bp = 31 - __clz(below);
        } else {
          ref = s.u.pj.link[V];
          if (ref < 0) break;  // the rest is in the incoming stack
          V = ref >> LOGK;
          bp = ref & (K - 1);
          uV = s.u.pj.uo[V];
          tV = s.u.pj.acc[cbf][V];
        }
      }
    }
    // the rest are consecutive entries of the incoming stack (a chain that
    // leaves the tile never returns into it)
    for (; d < a_t; d++, ref--) {
      const int ci = __ffs(q) - 1;
      q &= q - 1;
      const uint32_t seg = ((1u << ci) - 1u) & ~((1u << (prevc + 1)) - 1u);
      prevc = ci;
      const int D = -ref - 1;
      int gi = -1;
      float4 cx = bINF();
      if (H - 1 - D >= 0) {
        int rf, si;
        if (D < INCCAP) {
          rf = s.u.pj.inc_ref[D];
          si = s.u.pj.inc_idx[D];
          cx = isect(s.u.pj.inc_box[D], s.u.pj.inc_tc[D]);
        } else {
          rf = inc_ref(p, s, nruns, H - 1 - D);
          si = __ldg(p.slice_idx + rf);
          if (seg & needm) cx = isect(__ldg(p.slice_box + rf), __ldg(p.tc + (rf >> LOGW)));
        }
        if (si != -1) {
          gi = si & 0x7fffffff;
          xcm |= 1u << ci;
          p.pop[poff + D] = make_int2(gtb + ci, rf);
        } else {
          p.pop[poff + D] = make_int2(-1, -1);  // an imported slot below the global root (R3)
        }
      } else {
        p.pop[poff + D] = make_int2(-1, -1);  // pops the root (R3)
      }
      s.matchS[mb + ci] = gi;
      if (seg & needm) s.val[sl(ci)] = cx;
    }
  }
  __syncthreads();

  // ---- F. one forward walk: clips (ctx(e) = box ∩ ctx(parent), blend opens
  //      pass it through, R6/R7), unions of in-thread nodes (an open saves the
  //      enclosing accumulator -- in its close's slot when the close is in the
  //      thread, else in rbuf -- and restarts it), parent / match.  By the Bic
  //      normal form all of a thread's unmatched closes precede its unmatched
  //      opens and the thread stack is empty at them, so there the
  //      accumulator holds the thread's prefix union.  Element 15's slot holds
  //      TL (the context after the last unmatched close) until 15 is reached:
  //      if 15 is an unmatched close nothing needs TL, if it is a matched
  //      close its open overwrites the slot after every reader of TL.
  float4 acc = bEMPTY();
  {
    const bool u15 = (w.ucm >> (K - 1)) & 1u;
    const float4 v15 = s.val[sl(K - 1)];
    if (!u15) s.val[sl(K - 1)] = TL;
#pragma unroll 1
    for (int q = 0; q < K / 4; q++) {
      // the masks shifted once per group: bit tests below use immediates
      const int i0 = 4 * q;
      const uint32_t Lq = w.lm >> i0, Bq = w.bm >> i0, Oq = w.om >> i0, Cq = w.cm >> i0, Uq = w.ucm >> i0;
      const uint32_t Sq = w.S >> i0, Xq = w.ext >> i0;
      const uint32_t pwq = (q < 2 ? w.plo : w.phi) >> (16 * (q & 1));
      const int kq = __popc(w.S & ((1u << i0) - 1u));      // thread-unmatched opens before the group
      const int sbq = ((q >> 1) << 10) | (sb ^ ((q & 1) << 2));  // slot of element i0 + jq = sbq ^ jq
      int pv[4];
#pragma unroll
      for (int jq = 0; jq < 4; jq++) {
        const int i = i0 + jq;
        const bool isL = (Lq >> jq) & 1u, isB = (Bq >> jq) & 1u;
        const bool isO = (Oq >> jq) & 1u, isC = (Cq >> jq) & 1u, isU = (Uq >> jq) & 1u;
        const bool isUO = (Sq >> jq) & 1u;
        const bool isMC = isC && !isU;
        const int si = sbq ^ jq;
        float4 v = s.val[si];
        if (jq == 3 && q == K / 4 - 1 && !isMC) v = v15;
        const int pn = (int)((pwq >> (4 * jq)) & 15u);
        const int pt = isC ? pn : s.matchS[mb + i] - gtb;  // a close's partner is its parent; an open's, from the walk
        const bool isx = (Xq >> jq) & 1u;
        const uint32_t nc = Uq >> jq;                        // unmatched closes at or after i
        const int j = nc ? i + __ffs(nc) - 1 : K - 1;        // the next one: c_d of element i's depth d (none: TL)
        // a close takes nothing from its parent (clipped = v ∩ v = v)
        const int spn = sl(pn);
        const int cidx = isC ? si : sl(isx ? j : pn);
        const float4 cpar = s.val[cidx];
        const int mj = s.matchS[mb + j];
        const int par = isx ? (nc ? mj : giLast) : gtb + pn;
        const float4 clipped = isect(v, cpar);
        // own slot: leaf / clip open -> clipped; blend open -> parent context;
        // close -> union (in-thread node) / prefix (outer node) / EMPTY (R3)
        float4 o = isB ? cpar : clipped;
        o = isC ? ((isU && par < 0) ? bEMPTY() : acc) : o;
        s.val[si] = o;
        {  // an open saves the enclosing accumulator: into its close's slot, or rbuf when left open
          const int k = kq + __popc(Sq & ((1u << jq) - 1u));
          const int di = isUO ? RB0 + min(k, RCAP - 1) * NT + tid : sl(pt);
          if (isO && (!isUO || k < RCAP)) s.val[di] = acc;
        }
        if (isMC && ((w.bm >> pn) & 1u)) s.val[spn] = acc;  // the close of an in-thread blend open
        const float4 add = (isL || isMC) ? clipped : bEMPTY();
        acc = unite(acc, add);
        acc = isO ? bEMPTY() : acc;
        if (PM && !(isUO || isU || isO)) s.matchS[mb + i] = isL ? -1 : gtb + pt;  // in-thread opens: stored by the walk
        pv[jq] = par;
      }
      if (PM) {
        if (nv_t >= 4 * q + 4) {
          __stcs(reinterpret_cast<int4*>(p.parent + base + tl0) + q, make_int4(pv[0], pv[1], pv[2], pv[3]));
        } else {
#pragma unroll
          for (int jj = 0; jj < 4; jj++)
            if (4 * q + jj < nv_t) p.parent[base + tl0 + 4 * q + jj] = pv[jj];
        }
      }
    }
  }
  // the thread's union: the prefix at its first unmatched open ∪ the segments
  const bool ovf = b_t > RCAP;
  float4 tu = acc;
  if (!ovf) {
#pragma unroll
    for (int k = 0; k < RCAP; k++)  // a fixed trip count, predicated (no divergent loop)
      if (k < b_t) tu = unite(tu, s.u.rbuf[k][tid]);
  } else {
#pragma unroll 1
    for (int i = 0; i < K; i++)
      if ((w.lm >> i) & 1u) tu = unite(tu, s.val[sl(i)]);
  }
  // warp-level prefix / suffix of the thread unions, warp totals
  float4 pw = tu, sw = tu;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float4 a = shfl_up_box(pw, off);
    if (lane >= off) pw = unite(pw, a);
    const float4 b = make_float4(__shfl_down_sync(0xffffffffu, sw.x, off), __shfl_down_sync(0xffffffffu, sw.y, off),
                                 __shfl_down_sync(0xffffffffu, sw.z, off), __shfl_down_sync(0xffffffffu, sw.w, off));
    if (lane + off < 32) sw = unite(sw, b);
  }
  if (lane == 31) s.wtu[warp] = pw;
  __syncthreads();
  if (tid < NW * NW) {
    const int x = tid / NW, y = tid % NW;
    float4 m = bEMPTY();
#pragma unroll 1
    for (int w2 = x + 1; w2 < y; w2++) m = unite(m, s.wtu[w2]);
    s.wmid[x][y] = m;
  }
  // union of the threads before / after this one (tile prefix / suffix)
  float4 pre = bEMPTY(), after = bEMPTY();
  {
    const float4 pe = shfl_up_box(pw, 1);
    if (lane > 0) pre = pe;
    const float4 se = make_float4(__shfl_down_sync(0xffffffffu, sw.x, 1), __shfl_down_sync(0xffffffffu, sw.y, 1),
                                  __shfl_down_sync(0xffffffffu, sw.z, 1), __shfl_down_sync(0xffffffffu, sw.w, 1));
    if (lane < 31) after = se;
#pragma unroll
    for (int w2 = 0; w2 < NW; w2++) {
      if (w2 < warp) pre = unite(pre, s.wtu[w2]);
      if (w2 > warp) after = unite(after, s.wtu[w2]);
    }
  }

  // ---- H1. opens left open at the thread end, top down with R = union of the
  //      thread's leaves after them (the segment unions): closed by a later
  //      thread of the tile -> that close's slot takes R (the closer adds the
  //      threads between in H2); otherwise a slice entry: su = R ∪ the threads
  //      after.  Closes of earlier tiles' nodes: the tile prefix before them
  //      into their pop records (fz_close ends them)
  if (w.S) {
    auto handle = [&](int i, int k, const float4& R) {  // predicated both ways (no branch)
      const int mc = s.matchS[mb + i];
      const bool in_tile = mc >= 0;
      float4& cv = s.val[slot_of(in_tile ? mc - gbase : 0)];
      const float4 c0 = cv;
      if (in_tile) cv = unite(c0, R);
      if (!in_tile) p.slice_su[base + l_t + k + aT] = unite(R, after);
    };
    if (!ovf) {
      float4 R = acc;  // segment after the top open
      uint32_t q = w.S;
      for (int k = b_t - 1; k >= 0; k--) {
        const int i = 31 - __clz(q);
        q ^= 1u << i;
        handle(i, k, R);
        R = unite(R, s.u.rbuf[k][tid]);
      }
    } else {
      float4 R = bEMPTY();
      int k = b_t - 1;
      for (int i = K - 1; i >= 0; i--) {
        const uint32_t bit = 1u << i;
        if (w.S & bit) {
          handle(i, k, R);
          k--;
        } else if (w.lm & bit) {
          R = unite(R, s.val[sl(i)]);
        }
      }
    }
  }
  for (uint32_t q = xcm; q; q &= q - 1) {  // the tile prefix before the close (fz_close reads it back)
    float4& cv = s.val[sl(__ffs(q) - 1)];
    cv = unite(cv, pre);
  }
  if (tid == 0) {
    float4 t = s.wtu[0];
#pragma unroll
    for (int w2 = 1; w2 < NW; w2++) t = unite(t, s.wtu[w2]);
    p.tu[0][T] = t;
  }
  __syncthreads();

  // ---- G. range table over threads (the segment buffer is dead) --------------
  {
    float4 wv = tu;
    s.u.rt.win[0][tid] = wv;
#pragma unroll
    for (int k = 1; k < 5; k++) {
      const int off = 1 << (k - 1);
      const float4 a = shfl_up_box(wv, off);
      if (lane >= off) wv = unite(wv, a);
      s.u.rt.win[k][tid] = wv;
    }
    s.u.rt.pre[tid] = pw;
    s.u.rt.suf[tid] = sw;
  }
  __syncthreads();

  // ---- H2. closes of nodes opened in an earlier thread of the tile: add the
  //      threads between; a blend open receives the union
  for (uint32_t q = icm; q; q &= q - 1) {
    const int ci = __ffs(q) - 1;
    const int o = s.matchS[mb + ci] - gbase;
    const int to = o >> LOGK;
    float4& cv = s.val[sl(ci)];
    const float4 U = unite(cv, range_threads(s, to + 1, tid - 1));
    cv = U;
    if ((s.bmS[to] >> (o & (K - 1))) & 1u) s.val[slot_of(o)] = U;
  }
  if (tma) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> the TMA store
  __syncthreads();

  // ---- I. copy-out: node boxes by TMA (full tiles), match coalesced ---------
  if (tma) {
    if (tid == 0) {
      tma_store_2d(&maps.out[0], 0, T * NT, val_sa);
      tma_store_2d(&maps.out[1], 0, T * NT, val_sa + NT * 128);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  } else {
#pragma unroll 1
    for (int j = 0; j < K; j++) {
      const int e = j * NT + tid;
      if (e < nvalid) __stcs(p.out + base + e, s.val[slot_of(e)]);
    }
  }
  if (PM) {
#pragma unroll
    for (int j = 0; j < W / 4 / NT; j++) {
      const int e = 4 * (j * NT + tid);
      const int pe = mpad(e);
      const int4 v4 = make_int4(s.matchS[pe], s.matchS[pe + 1], s.matchS[pe + 2], s.matchS[pe + 3]);
      if (e + 4 <= nvalid) {
        __stcs(reinterpret_cast<int4*>(p.match + base + e), v4);
      } else {
        if (e < nvalid) p.match[base + e] = v4.x;
        if (e + 1 < nvalid) p.match[base + e + 1] = v4.y;
        if (e + 2 < nvalid) p.match[base + e + 2] = v4.z;
      }
    }
  }
  if (tma && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ----------------------------------------------------------------------------
// fz_match: paren_match alone -- fz_main's matching phases
// only (no boxes, contexts or unions): 15 KB of shared memory per tile instead
// of 56, so four times the tiles per SM
// ----------------------------------------------------------------------------
struct SmemM {
  int32_t matchS[W + W / K];
  int lwin[NW][5][32];
  int lwmin[NW];
  int l[NT];
  uint32_t uo[NT];
  int link[NT];
  int inc_idx[INCCAP];
  int inc_ref[INCCAP];
  int2 runs[RMAX];
  Bic wtot[NW];
};

__global__ void __launch_bounds__(NT) fz_match(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmemM& s = *reinterpret_cast<SmemM*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockIdx.x;
  const int64_t base = (int64_t)T * W;
  const int nvalid = (int)(p.n - base < W ? p.n - base : W);
  const int gbase = p.goff + (int)base;  // shard mode: global indices
  const int tl0 = tid * K;
  const int gtb = gbase + tl0;
  const int mb = mpad(tl0);
  const uint4 raw = load_tags16(p.tags, p.n, base + tl0, nvalid == W);
  const int H = __ldg(p.ctrl.hstart + T);
  const int aT = __ldg(p.ctrl.agg + T).x;
  const int64_t poff = __ldg(p.aoff + T);
  if (tid < RMAX) {
    cp_async8(smem_u32(&s.runs[tid]), p.runs + (int64_t)T * RMAX + tid);
    cp_async_commit();
  }
  const int nruns = __ldg(p.nruns + T);
  const int nv_t = nvalid - tl0;
  const uint32_t valid = nv_t >= K ? 0xffffu : (nv_t <= 0 ? 0u : ((1u << nv_t) - 1u));
  const Walk w = walk_m<false>(raw, valid, s.matchS + mb, gtb);  // in-thread opens' matches stored here
  const int a_t = __popc(w.ucm);

  // B. block Bic scan; thread low-water windows
  if (tid < RMAX) cp_async_wait_all();
  Bic ex, sx, tot;
  block_bic_scans<NW>(Bic{a_t, __popc(w.S)}, s.wtot, ex, sx, tot, false);
  const int r_t = ex.b - ex.a;
  const int l_t = r_t - a_t;
  for (uint32_t q = w.S; q; q &= q - 1) s.matchS[mb + __ffs(q) - 1] = -1;
  int wl[5];
  lane_windows(l_t, wl);
#pragma unroll
  for (int k = 0; k < 5; k++) s.lwin[warp][k][lane] = wl[k];
  {
    const int o = __shfl_sync(0xffffffffu, wl[4], 15);
    if (lane == 31) s.lwmin[warp] = min(wl[4], o);
  }
  s.l[tid] = l_t;
  s.uo[tid] = w.S;
  __syncthreads();

  // C. incoming entries (global index only); the thread's top entry and link
  const int ninc = min(aT + 1, INCCAP);
  for (int D = tid; D < ninc; D += NT) {
    const int h = H - 1 - D;
    if (h < 0) {
      s.inc_idx[D] = -1;
      s.inc_ref[D] = -1;
    } else {
      const int ref = inc_ref(p, s, nruns, h);
      s.inc_ref[D] = ref;
      cp_async4(smem_u32(&s.inc_idx[D]), p.slice_idx + ref);
    }
  }
  cp_async_commit();
  int top_ref = 0, lk = 0;
#pragma unroll 1
  for (int qq = 0; qq < 2; qq++) {
    const int r = thread_ref<NW, K>(wl, l_t, w.S, qq ? l_t - 1 : r_t - 1, s.lwin, s.lwmin, s.l, s.uo);
    if (qq) lk = r;
    else top_ref = r;
  }
  s.link[tid] = lk;
  cp_async_wait_all();
  __syncthreads();
  // D. the link's global index (the parent of the thread's outer elements after its last unmatched close)
  int giLast = -1;
  if (lk >= 0) {
    giLast = gbase + lk;
  } else {
    const int D = -lk - 1;
    if (H - 1 - D >= 0) {
      const int si = D < INCCAP ? s.inc_idx[D] : __ldg(p.slice_idx + inc_ref(p, s, nruns, H - 1 - D));
      giLast = si == -1 ? -1 : si & 0x7fffffff;
    }
  }
  // E. the entries popped by the thread's unmatched closes
  {
    int ref = top_ref, d = 0;
    uint32_t q = w.ucm;
    if (d < a_t && ref >= 0) {
      int V = ref >> LOGK, bp = ref & (K - 1);
      uint32_t uV = s.uo[V];
      while (true) {
        const int e = (V << LOGK) | bp;
        const int ci = __ffs(q) - 1;
        q &= q - 1;
        s.matchS[mb + ci] = gbase + e;
        s.matchS[mpad(e)] = gtb + ci;
        if (++d >= a_t) break;
        const uint32_t below = uV & ((1u << bp) - 1u);
        if (below) {
          bp = 31 - __clz(below);
        } else {
          ref = s.link[V];
          if (ref < 0) break;
          V = ref >> LOGK;
          bp = ref & (K - 1);
          uV = s.uo[V];
        }
      }
    }
    for (; d < a_t; d++, ref--) {
      const int ci = __ffs(q) - 1;
      q &= q - 1;
      const int D = -ref - 1;
      int gi = -1;
      if (H - 1 - D >= 0) {
        const int rf = D < INCCAP ? s.inc_ref[D] : inc_ref(p, s, nruns, H - 1 - D);
        const int si = D < INCCAP ? s.inc_idx[D] : __ldg(p.slice_idx + rf);
        if (si != -1) {  // the open's match directly (its tile leaves that slot alone; fz_reduce wrote -1)
          gi = si & 0x7fffffff;
          if (rf >= p.vbase) p.exc[rf - p.vbase] = gtb + ci;  // an imported entry (shard mode)
          else p.match[gi - p.goff] = gtb + ci;
        }
      }
      s.matchS[mb + ci] = gi;
    }
  }
  __syncthreads();
  // F. parent of every element, match of the in-thread pairs and leaves
#pragma unroll 1
  for (int q = 0; q < K / 4; q++) {
    const int i0 = 4 * q;
    const uint32_t Lq = w.lm >> i0, Uq = w.ucm >> i0, Sq = w.S >> i0, Xq = w.ext >> i0;
    const uint32_t pwq = (q < 2 ? w.plo : w.phi) >> (16 * (q & 1)), Oq = w.om >> i0;
    int pv[4];
#pragma unroll
    for (int jq = 0; jq < 4; jq++) {
      const int i = i0 + jq;
      const bool isL = (Lq >> jq) & 1u, isU = (Uq >> jq) & 1u, isUO = (Sq >> jq) & 1u, isx = (Xq >> jq) & 1u;
      const int pn = (int)((pwq >> (4 * jq)) & 15u);
      const bool isO = (Oq >> jq) & 1u;  // an in-thread open's match was stored by the walk
      const uint32_t nc = Uq >> jq;
      const int j = nc ? i + __ffs(nc) - 1 : K - 1;
      pv[jq] = isx ? (nc ? s.matchS[mb + j] : giLast) : gtb + pn;
      if (!(isUO || isU || isO)) s.matchS[mb + i] = isL ? -1 : gtb + pn;  // a close's partner is its parent
    }
    if (nv_t >= 4 * q + 4) {
      __stcs(reinterpret_cast<int4*>(p.parent + base + tl0) + q, make_int4(pv[0], pv[1], pv[2], pv[3]));
    } else {
#pragma unroll
      for (int jj = 0; jj < 4; jj++)
        if (4 * q + jj < nv_t) p.parent[base + tl0 + 4 * q + jj] = pv[jj];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < W / 4 / NT; j++) {  // match out, coalesced; the tile's surviving opens are skipped
    const int e = 4 * (j * NT + tid);
    const int pe = mpad(e);
    const int4 v4 = make_int4(s.matchS[pe], s.matchS[pe + 1], s.matchS[pe + 2], s.matchS[pe + 3]);
    // survivors: thread-unmatched opens no later thread of the tile closed (matchS still -1)
    const uint32_t uo4 = (s.uo[e >> LOGK] >> (e & (K - 1))) & 15u;
    const uint32_t sk = uo4 & ((v4.x < 0 ? 1u : 0u) | (v4.y < 0 ? 2u : 0u) | (v4.z < 0 ? 4u : 0u) | (v4.w < 0 ? 8u : 0u));
    if (e + 4 <= nvalid && !sk) {
      __stcs(reinterpret_cast<int4*>(p.match + base + e), v4);
    } else {
      if (e < nvalid && !(sk & 1u)) p.match[base + e] = v4.x;
      if (e + 1 < nvalid && !(sk & 2u)) p.match[base + e + 1] = v4.y;
      if (e + 2 < nvalid && !(sk & 4u)) p.match[base + e + 2] = v4.z;
      if (e + 3 < nvalid && !(sk & 8u)) p.match[base + e + 3] = v4.w;
    }
  }
}


// ----------------------------------------------------------------------------
// fz_hier: level k of the tile-union hierarchy (one warp per group of 32)
// ----------------------------------------------------------------------------
// one launch: every block reduces its level-1 groups; the last block to finish
// (arrival counter flag[3], zeroed by fz_ctrl) builds the upper levels
__global__ void __launch_bounds__(256) fz_hier(Params p) {
  __shared__ int last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int m = p.ntiles;  // nodes at level 0
  {
    const int g = blockIdx.x * 8 + warp;
    if ((g << 5) < m) {
      const int c = (g << 5) + lane;
      const float4 v = warp_unite_all(c < m ? __ldcg(p.tu[0] + c) : bEMPTY());
      if (lane == 0) p.tu[1][g] = v;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(p.flag + 3, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  m = (m + 31) / 32;  // nodes at level 1
  for (int k = 2; k < LV && m > 1; k++) {
    const int groups = (m + 31) / 32;
    for (int g = warp; g < groups; g += 8) {
      const int c = (g << 5) + lane;
      const float4 v = warp_unite_all(c < m ? __ldcg(p.tu[k - 1] + c) : bEMPTY());
      if (lane == 0) p.tu[k][g] = v;
    }
    __threadfence_block();
    __syncthreads();
    m = groups;
  }
}

// union over tiles [a, b] by one warp (a, b warp-uniform): per level of the
// 32-ary hierarchy the partial groups at both ends, every load issued at once
__device__ __forceinline__ float4 range_tiles(const Params& p, int a, int b) {
  const int lane = threadIdx.x & 31;
  float4 acc = bEMPTY();
#pragma unroll
  for (int k = 0; k < LV; k++) {
    int i1 = -1, i2 = -1;
    if (a <= b) {
      if ((a >> 5) == (b >> 5) || k == LV - 1) {
        if (a + lane <= b) i1 = a + lane;
        a = 1;
        b = 0;
      } else {
        if (a & 31) {
          const int e = a | 31;
          if (a + lane <= e) i1 = a + lane;
          a = e + 1;
        }
        if ((b & 31) != 31) {
          const int s0 = b & ~31;
          if (s0 + lane <= b) i2 = s0 + lane;
          b = s0 - 1;
        }
        if (a <= b) {
          a >>= 5;
          b = ((b + 1) >> 5) - 1;
        }
      }
    }
    const float4 v1 = i1 >= 0 ? __ldcg(p.tu[k] + i1) : bEMPTY();
    const float4 v2 = i2 >= 0 ? __ldcg(p.tu[k] + i2) : bEMPTY();
    acc = unite(acc, unite(v1, v2));
  }
  return warp_unite_all(acc);
}

// ----------------------------------------------------------------------------
// fz_close: nodes opened in an earlier tile (one warp per tile, 32 pops at a time)
// ----------------------------------------------------------------------------
template <bool PM>
__global__ void __launch_bounds__(128) fz_close(Params p) {
  const int lane = threadIdx.x & 31;
  const int T = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (T >= (p.scene ? (int)((__ldg(p.nkp) + W - 1) / W) : p.ntiles)) return;  // scene: past the compacted stream
  const int64_t poff = __ldg(p.aoff + T);
  const int npop = (int)(__ldg(p.aoff + T + 1) - poff);
  const int bT = __ldg(p.ctrl.agg + T).y;
  const int L = (int)__ldg(p.ctrl.lw + T) - 1;
  const int sm = __ldg(p.ctrl.smin + T);
  int cto = INT_MIN;  // warp cache: the last tile range resolved
  float4 cR = bEMPTY();
  for (int j0 = 0; j0 < npop; j0 += 32) {
    const int j = j0 + lane;
    int2 r = make_int2(-1, -1);
    if (j < npop) r = __ldcg(p.pop + poff + j);
    const bool valid = r.x >= 0;  // root pops (R3) have no node
    int To = T, si = 0;
    float4 P = bEMPTY(), su = bEMPTY();
    const bool imp = r.y >= p.vbase;  // pops an imported entry (shard mode): opened on another chunk
    if (valid) {
      To = imp ? -1 : r.y >> LOGW;
      P = __ldcg(p.out + (r.x - p.goff));  // the tile prefix before the close (fz_main)
      if (!imp) {
        su = __ldg(p.slice_su + r.y);
        si = __ldg(p.slice_idx + r.y);
      }
    }
    float4 R = bEMPTY();
    bool pending = valid && To < T - 1;
    if (pending && To == cto) {
      R = cR;
      pending = false;
    }
    uint32_t mask;
    while ((mask = __ballot_sync(0xffffffffu, pending)) != 0u) {
      const int tl = __shfl_sync(0xffffffffu, To, __ffs(mask) - 1);
      const float4 Rl = range_tiles(p, tl + 1, T - 1);
      if (pending && To == tl) {
        R = Rl;
        pending = false;
      }
      cto = tl;
      cR = Rl;
    }
    if (valid) {
      const float4 U = unite(unite(P, su), R);
      p.out[r.x - p.goff] = U;
      if (imp) {  // this chunk's part of the node; the rest after the exchange (fused_shard.cuh)
        const int h = r.y - p.vbase;
        p.exc[h] = r.x;
        p.exu[h] = U;
      } else {
        const int o = (si & 0x7fffffff) - p.goff;
        if (si < 0) p.out[o] = U;  // a blend open
        if (PM) p.match[o] = r.x;
      }
    }
  }
  if (p.h0) return;  // shard mode: the chunk's final stack is finished after the exchange
  // blend opens never closed (R4): the tile's slice entries that survive to
  // the end of the stream (F1: its bottom min(b_T, smin_T - L_T))
  const int surv = min(bT, sm == INT_MAX ? bT : max(sm - L, 0));
  if (surv > 0) {
    bool anyb = false;
    for (int k = lane; k < surv; k += 32) anyb |= __ldg(p.slice_idx + (int64_t)T * W + k) < 0;
    if (__any_sync(0xffffffffu, anyb)) {
      const float4 after = range_tiles(p, T + 1, p.ntiles - 1);
      for (int k = lane; k < surv; k += 32) {
        const int64_t ref = (int64_t)T * W + k;
        const int si = __ldg(p.slice_idx + ref);
        if (si < 0) p.out[(si & 0x7fffffff) - p.goff] = unite(__ldg(p.slice_su + ref), after);
      }
    }
  }
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)f;
  }
  return fn;
}

// the four maps of fz_main over boxes / node_bbox (full thread rows only: the
// partial last tile never uses them); false: TMA unavailable
static bool make_maps(const float* boxes, float* out, int64_t n, Maps& m) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = encode_fn();
  const uint64_t rows = (uint64_t)(n / K);
  if (!enc || rows < (uint64_t)NT) return false;
  const cuuint64_t dims[2] = {32, rows};
  const cuuint64_t strides[1] = {(cuuint64_t)K * 16};
  const cuuint32_t box[2] = {32, NT};
  const cuuint32_t estr[2] = {1, 1};
  for (int h = 0; h < 2; h++) {
    CUresult r = enc(&m.in[h], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)(boxes + 32 * h), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    r = enc(&m.out[h], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)(out + 32 * h), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
  }
  return true;
}

static int main_ctas() {  // resident CTAs of fz_main on the device (4 per SM: shared memory)
  static int cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& c = cache[dev & 63];
  if (c == 0) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fz_main<true, false>, NT, sizeof(Smem));
    c = sm_count() * std::max(occ, 1);
  }
  return c;
}

static int ctrl_blocks() {  // co-resident CTAs of the cooperative kernel
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fz_ctrl, NTC, 0);
  return std::min(MAXCTRL, sms * std::min(occ > 0 ? occ : 1, 1));
}

static cudaError_t setup() {
  if (once_per_device(3)) {
    cudaError_t e = cudaSuccess;
    for (const void* f : {(const void*)fz_main<true, false>, (const void*)fz_main<false, false>,
                          (const void*)fz_main<true, true>, (const void*)fz_main<false, true>}) {
      if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
      if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(fz_match, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmemM));
    uint8_t tab[UNM4_ENTRIES];
    for (int i = 0; i < UNM4_ENTRIES; i++) tab[i] = unm4_entry(i);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_unm4, tab, sizeof tab);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace fz

static uint64_t* g_fz_trace = nullptr;  // debug hook (tb_debug_fz_trace)
void fused_set_trace(uint64_t* dev) { g_fz_trace = dev; }
static int g_fz_tma = 1;  // debug hook (tb_debug_fz_tma): 0 = the threads copy every tile
static int g_fz_ctrl_cap = 0;  // debug hook (tb_debug_fz_ctrl_blocks): at most this many fz_ctrl blocks (0: all)
int fused_set_ctrl_blocks(int g) {
  const int old = g_fz_ctrl_cap;
  if (g >= 0) g_fz_ctrl_cap = g;
  return old;
}
int fused_set_tma(int on) {
  const int old = g_fz_tma;
  if (on >= 0) g_fz_tma = on;
  return old;
}

size_t fused_workspace_bytes(int64_t n) { return n > 0 ? fz::Layout(n).bytes : 0; }
size_t fused_match_workspace_bytes(int64_t n) { return n > 0 ? fz::Layout(n, 0, true).bytes : 0; }
int fused_tile_elems() { return fz::W; }

// debug: TB_FZ_SYNC=1 synchronises after every launch and names the failing one
static cudaError_t dbg_sync(cudaStream_t s, const char* what) {
  static const bool on = getenv("TB_FZ_SYNC") != nullptr;
  if (!on) return cudaSuccess;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) fprintf(stderr, "fused: %s failed: %s\n", what, cudaGetErrorString(e));
  return e;
}

// the passes before the main pass: tile Bic values and slices, then the
// cooperative control kernel (tile scan, link owners, TC)
static cudaError_t launch_front(fz::Params& p, cudaStream_t stream) {
  const int nt = p.ntiles;
  if (p.scene) {
    TB_LAUNCH(stream, "sc_count", (fz::sc_count<<<(unsigned)((nt + 7) / 8), 256, 0, stream>>>(p)));
    const int nb = (nt + 1023) / 1024;
    long long* bsum = (long long*)p.blk;  // fz_ctrl's block aggregates: free until fz_ctrl
    TB_LAUNCH(stream, "sc_scan", (fz::sc_scan1<<<nb, 1024, 0, stream>>>(p, bsum)));
    TB_LAUNCH(stream, "sc_scan", (fz::sc_scan2<<<1, 1024, 0, stream>>>(p, bsum, nb)));
    TB_LAUNCH(stream, "sc_scan", (fz::sc_scan3<<<nb, 1024, 0, stream>>>(p, bsum)));
    TB_LAUNCH(stream, "sc_compact", (fz::sc_compact<<<(unsigned)((nt + 7) / 8), 256, 0, stream>>>(p)));
    TB_LAUNCH(stream, "fz_reduce", (fz::fz_reduce<true><<<(unsigned)((nt + 7) / 8), 256, 0, stream>>>(p)));
  } else {
    TB_LAUNCH(stream, "fz_reduce", (fz::fz_reduce<false><<<(unsigned)((nt + 7) / 8), 256, 0, stream>>>(p)));
  }
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = dbg_sync(stream, "fz_reduce");
  if (e != cudaSuccess) return e;
  // enough blocks for the per-tile warps of P3 / P5, at most the co-resident
  // count; chunks of whole 32-tile groups
  const int cbk = g_fz_ctrl_cap > 0 ? std::min(g_fz_ctrl_cap, fz::ctrl_blocks()) : fz::ctrl_blocks();
  const int G = std::max(1, std::min((nt + 31) / 32, cbk));
  p.chunk = (((nt + G - 1) / G) + 31) & ~31;
  void* args[] = {(void*)&p};
  void* tok;
  prof_begin(stream, "fz_ctrl", &tok);
  e = cudaLaunchCooperativeKernel((const void*)fz::fz_ctrl, dim3(G), dim3(fz::NTC), args, 0, stream);
  prof_end(stream, tok);
  if (e == cudaSuccess) e = dbg_sync(stream, "fz_ctrl");
  return e;
}

// the main pass, the tile-union hierarchy and the close pass
static cudaError_t launch_back(fz::Params& p, const float* leaf_bbox, float* node_bbox, bool pm, cudaStream_t stream) {
  const int nt = p.ntiles;
  fz::Maps maps;
  memset(&maps, 0, sizeof maps);
  p.use_tma = g_fz_tma && fz::make_maps(leaf_bbox, node_bbox, p.n, maps) ? 1 : 0;
  p.pf_tiles = fz::main_ctas();
  const unsigned g = (unsigned)nt;
  const size_t sm = sizeof(fz::Smem);
  if (p.scene) {
    if (pm)
      TB_LAUNCH(stream, "fz_main", (fz::fz_main<true, true><<<g, fz::NT, sm, stream>>>(p, maps)));
    else
      TB_LAUNCH(stream, "fz_main", (fz::fz_main<false, true><<<g, fz::NT, sm, stream>>>(p, maps)));
  } else {
    if (pm)
      TB_LAUNCH(stream, "fz_main", (fz::fz_main<true, false><<<g, fz::NT, sm, stream>>>(p, maps)));
    else
      TB_LAUNCH(stream, "fz_main", (fz::fz_main<false, false><<<g, fz::NT, sm, stream>>>(p, maps)));
  }
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = dbg_sync(stream, "fz_main");
  if (e != cudaSuccess) return e;
  if (nt > 1) {
    const int groups = (nt + 31) / 32;
    TB_LAUNCH(stream, "fz_hier", (fz::fz_hier<<<(unsigned)((groups + 7) / 8), 256, 0, stream>>>(p)));
    e = dbg_sync(stream, "fz_hier");
    if (e != cudaSuccess) return e;
  }
  if (pm)
    TB_LAUNCH(stream, "fz_close", (fz::fz_close<true><<<(unsigned)((nt + 3) / 4), 128, 0, stream>>>(p)));
  else
    TB_LAUNCH(stream, "fz_close", (fz::fz_close<false><<<(unsigned)((nt + 3) / 4), 128, 0, stream>>>(p)));
  e = cudaGetLastError();
  if (e == cudaSuccess) e = dbg_sync(stream, "fz_close");
  return e;
}

cudaError_t fused_launch(const uint8_t* tags, const float* leaf_bbox, int64_t n, int32_t* match, int32_t* parent,
                         float* node_bbox, void* ws, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  cudaError_t e = fz::setup();
  if (e != cudaSuccess) return e;
  fz::Params p = fz::make_params(tags, leaf_bbox, n, match, parent, node_bbox, ws);
  p.trace = g_fz_trace;
  e = launch_front(p, stream);
  if (e != cudaSuccess) return e;
  return launch_back(p, leaf_bbox, node_bbox, match != nullptr, stream);
}

// the matching main pass and its close pass (no boxes)
static cudaError_t launch_back_match(fz::Params& p, cudaStream_t stream) {
  const int nt = p.ntiles;
  TB_LAUNCH(stream, "fz_match", (fz::fz_match<<<(unsigned)nt, fz::NT, sizeof(fz::SmemM), stream>>>(p)));
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = dbg_sync(stream, "fz_match");
  if (e != cudaSuccess) return e;
  return e;
}

// paren_match alone by the fused machinery (no boxes): match and parent
cudaError_t fused_match_launch(const uint8_t* tags, int64_t n, int32_t* match, int32_t* parent, void* ws,
                               cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  cudaError_t e = fz::setup();
  if (e != cudaSuccess) return e;
  fz::Params p = fz::make_params(tags, nullptr, n, match, parent, nullptr, ws, 0, 0, true);
  p.nobox = 1;
  e = launch_front(p, stream);
  if (e != cudaSuccess) return e;
  return launch_back_match(p, stream);
}

// scene mode (stream compaction fused into the loaders): the full stream in,
// the kept elements' outputs at their compacted indices; *d_n_out = the kept count
cudaError_t fused_scene_launch(const uint8_t* tags, const float* boxes, int64_t n, const uint8_t* h_keep_map,
                               uint8_t* tags_out, int32_t* index_out, int32_t* match, int32_t* parent,
                               float* node_bbox, int64_t* d_n_out, void* ws, cudaStream_t stream) {
  if (n <= 0) return cudaMemsetAsync(d_n_out, 0, sizeof(int64_t), stream);
  cudaError_t e = fz::setup();
  if (e != cudaSuccess) return e;
  fz::Params p = fz::make_params(tags_out, boxes, n, match, parent, node_bbox, ws);  // the passes read the compacted tags
  p.scene = 1;
  p.tags_in = tags;
  p.boxes_in = (const float4*)boxes;
  p.tags_out = tags_out;
  p.index_out = index_out;
  uint32_t kw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int b = 0; b < 256; b++)
    if (h_keep_map[b]) kw[b >> 5] |= 1u << (b & 31);
  p.keep03 = kw[0] == 0xfu && !(kw[1] | kw[2] | kw[3] | kw[4] | kw[5] | kw[6] | kw[7]);
  e = cudaMemcpyAsync((void*)p.keepw, kw, sizeof kw, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = launch_front(p, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_n_out, p.nkp, sizeof(int64_t), cudaMemcpyDeviceToDevice, stream);
  if (e != cudaSuccess) return e;
  return launch_back(p, boxes, node_bbox, match != nullptr, stream);
}

#include "fused_shard.cuh"

}  // namespace tb
