// Multi-GPU sharding of paren_match.
//
// The global stream is split into contiguous chunks, one per rank.  The
// stack-monoid structure (§4) makes the exchange small: a chunk is
// summarised by its Bic value (a_g, b_g) and its unmatched opens
// (the chunk's stack slice), b_g global indices.
//   phase 1: chunk-local reduce pass; summary kernel -> header + open list.
//   exchange 1: all-gather headers, then open lists (padded to the max b).
//   phase 2: the top a_g + 1 entries of the stack at the chunk start are
//            composed from earlier chunks' lists by the owner rule over chunks
//            (the entry at height X belongs to the last chunk h < g with
//            L_h <= X, at position X - L_h); reduce + finish passes run with
//            that initial stack; closes that pop an entry of an earlier chunk
//            record (open, close) pairs instead of writing into another GPU.
//   exchange 2: all-gather the pair lists; each rank writes match[open] for
//            its own opens.
// Two drivers share the protocol: NCCL (one chunk per process; the
// `*_shard` C entry points) and an in-process "virtual" driver that runs G
// chunks of one buffer on one GPU in lockstep (tests; no peer traffic).
#include <algorithm>
#include <cstring>
#include <vector>

#include "kernels.h"
#include "stackscan.cuh"
#include "treebbox.h"
#ifdef TB_WITH_NCCL
#include <nccl.h>
#endif

namespace tb {

__global__ void compose_stack_k(const int32_t* allopens, int maxb, const int* L, int g, int lo, int H,
                                int32_t* out) {
  for (int X = lo + blockIdx.x * blockDim.x + threadIdx.x; X < H; X += gridDim.x * blockDim.x) {
    int h = g - 1;
    while (h > 0 && L[h] > X) h--;
    out[X - lo] = allopens[(int64_t)h * maxb + (X - L[h])];
  }
}

__global__ void apply_pairs_k(const int2* pairs, int64_t total, int64_t off, int64_t n, int32_t* match) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int2 pr = pairs[i];
    if (pr.x >= off && pr.x < off + n) match[pr.x - off] = pr.y;
  }
}

namespace {

struct Bic2 {
  int64_t a, b;
};
Bic2 combine(Bic2 x, Bic2 y) {
  const int64_t m = std::min(x.b, y.a);
  return Bic2{x.a + y.a - m, x.b + y.b - m};
}

// Per-chunk state of the paren_match shard protocol.
struct PmChunk {
  const uint8_t* tags;
  int64_t n, off;
  int32_t* match;
  int32_t* parent;
  cudaStream_t s;
  // device buffers (one allocation)
  void* mem = nullptr;
  void* ws;           // pm workspace
  int32_t* hdr;       // [2] a, b
  int32_t* opens;     // [n] unmatched opens (send)
  int32_t* stack;     // [n + 1] composed initial stack
  int2* pairs;        // [n] (open, close) send
  int* Ldev;          // [G]
  size_t bytes = 0;

  cudaError_t alloc(int G) {
    const size_t wsb = pm_workspace_bytes(std::max<int64_t>(n, 1));
    const size_t nn = (size_t)std::max<int64_t>(n, 1);
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    bytes = al(wsb) + al(8) + al(4 * nn) + al(4 * (nn + 1)) + al(8 * nn) + al(4 * (size_t)G);
    cudaError_t e = cudaMalloc(&mem, bytes);
    if (e != cudaSuccess) return e;
    char* b = (char*)mem;
    ws = b; b += al(wsb);
    hdr = (int32_t*)b; b += al(8);
    opens = (int32_t*)b; b += al(4 * nn);
    stack = (int32_t*)b; b += al(4 * (nn + 1));
    pairs = (int2*)b; b += al(8 * nn);
    Ldev = (int*)b;
    return cudaSuccess;
  }
  void release() {
    if (mem) cudaFree(mem);
    mem = nullptr;
  }

  // phase 1: chunk-local reduce + summary
  cudaError_t phase1() {
    ShardInit local{0, 0, nullptr, 0, off, nullptr};  // chunk-local frame, global indices
    cudaError_t e = pm_reduce_launch(tags, n, match, ws, &local, s);
    if (e == cudaSuccess) e = pm_summary_launch(tags, n, ws, hdr, opens, s);
    return e;
  }

  // phase 2: compose the initial stack, run reduce + finish with it.
  // hdrs: all chunks' (a, b); allopens: G x maxb.
  cudaError_t phase2(int g, const std::vector<Bic2>& hdrs, const int32_t* allopens, int maxb, int64_t* npairs) {
    const int G = (int)hdrs.size();
    std::vector<int> L(G);
    Bic2 pre{0, 0};
    Bic2 mine{0, 0};
    for (int h = 0; h < G; h++) {
      if (h == g) mine = pre;
      L[h] = (int)std::max<int64_t>(pre.b - hdrs[h].a, 0);
      pre = combine(pre, hdrs[h]);
    }
    const int H = (int)mine.b;
    const int ag = (int)hdrs[g].a;
    const int lo = std::max(H - 1 - ag, 0);
    cudaError_t e = cudaMemcpyAsync(Ldev, L.data(), sizeof(int) * G, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    if (H > lo) {
      const int cnt = H - lo;
      compose_stack_k<<<std::min((cnt + 255) / 256, 1024), 256, 0, s>>>(allopens, maxb, Ldev, g, lo, H, stack);
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    *npairs = std::min<int64_t>(ag, H);
    e = cudaMemsetAsync(pairs, 0xff, sizeof(int2) * (size_t)std::max<int64_t>(n, 1), s);
    if (e != cudaSuccess) return e;
    ShardInit init{(int)mine.a, H, stack, lo, off, pairs};
    e = pm_reduce_launch(tags, n, match, ws, &init, s);
    if (e == cudaSuccess) e = pm_finish_launch(tags, n, match, parent, ws, &init, s);
    return e;
  }

  cudaError_t phase3(const int2* allpairs, int64_t total) {
    if (total <= 0) return cudaSuccess;
    apply_pairs_k<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, s>>>(allpairs, total, off, n,
                                                                                       match);
    return cudaGetLastError();
  }
};

// ---- tree_bbox --------------------------------------------------------------
// Same protocol with box payloads:
//   phase 1: chunk-local reduce; header (a_g, b_g) read back; summary = the
//            chunk's final stack with chunk-local cumulative clips.
//   exchange 1: headers, summaries.
//   phase 2: true clips of the provided stack entries (clip chain over
//            chunks); reduce + finish with them; closes popping an entry of an
//            earlier chunk record their partial union; export the chunk's
//            union and the union after each final-stack entry.
//   exchange 2: chunk unions, suffix unions, pop records.
//   phase 3: fix-up of nodes spanning chunks and of blend nodes open at the
//            end of the stream.
struct BbChunk {
  const uint8_t* tags;
  const float* leaf;
  int64_t n, off;
  float* out;
  cudaStream_t s;
  void* ws = nullptr;  // tree_bbox workspace (owned)
  void* buf = nullptr;  // summary / exchange buffers (owned)
  int32_t* hdr = nullptr;
  void* recs = nullptr;     // [b] SumRec
  int4* runs = nullptr;     // [b + 1]
  float4* suf_tiles = nullptr;
  float4* tu = nullptr;     // [1]
  float4* su = nullptr;     // [b]
  float4* init_clip = nullptr;
  int4* init_meta = nullptr;
  void* pops = nullptr;     // [a] BbPop
  int* Ldev = nullptr;
  int64_t a = 0, b = 0;

  cudaError_t alloc_ws() {
    cudaError_t e = cudaMalloc(&ws, bb_workspace_bytes(std::max<int64_t>(n, 1)));
    if (e == cudaSuccess) e = cudaMalloc(&hdr, 256);
    return e;
  }
  cudaError_t phase1a() {  // chunk-local reduce; header into hdr (device)
    BbShard local{off, 0, 0, nullptr, nullptr, nullptr};
    return bb_reduce_launch(tags, leaf, n, ws, &local, s);
  }
  cudaError_t alloc_buffers(int G) {
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const int64_t ntiles = (n + bb_tile_elems() - 1) / bb_tile_elems() + 1;
    const size_t bb1 = (size_t)std::max<int64_t>(b, 1), ab1 = (size_t)std::max<int64_t>(a, 1);
    const size_t bytes = al(bb_sumrec_bytes() * bb1) + al(16 * (bb1 + 1)) + al(16 * (size_t)ntiles) + al(16) +
                         al(16 * bb1) + al(16 * (ab1 + 1)) + al(16 * (ab1 + 1)) + al(bb_pop_bytes() * ab1) +
                         al(4 * (size_t)G);
    cudaError_t e = cudaMalloc(&buf, bytes);
    if (e != cudaSuccess) return e;
    char* c = (char*)buf;
    recs = c; c += al(bb_sumrec_bytes() * bb1);
    runs = (int4*)c; c += al(16 * (bb1 + 1));
    suf_tiles = (float4*)c; c += al(16 * (size_t)ntiles);
    tu = (float4*)c; c += al(16);
    su = (float4*)c; c += al(16 * bb1);
    init_clip = (float4*)c; c += al(16 * (ab1 + 1));
    init_meta = (int4*)c; c += al(16 * (ab1 + 1));
    pops = c; c += al(bb_pop_bytes() * ab1);
    Ldev = (int*)c;
    return cudaSuccess;
  }
  cudaError_t phase1b() { return bb_summary_launch(tags, leaf, n, ws, hdr, recs, runs, s); }
  cudaError_t phase2(int g, const std::vector<Bic2>& hdrs, const void* allrecs, int maxb) {
    const int G = (int)hdrs.size();
    std::vector<int> L(G);
    Bic2 pre{0, 0}, mine{0, 0};
    for (int h = 0; h < G; h++) {
      if (h == g) mine = pre;
      L[h] = (int)std::max<int64_t>(pre.b - hdrs[h].a, 0);
      pre = combine(pre, hdrs[h]);
    }
    const int H = (int)mine.b;
    const int lo = std::max(H - 1 - (int)a, 0);
    cudaError_t e = cudaMemcpyAsync(Ldev, L.data(), sizeof(int) * G, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && H > lo) e = bb_compose_launch(allrecs, maxb, Ldev, g, lo, H, init_clip, init_meta, s);
    if (e != cudaSuccess) return e;
    BbShard sh{off, H, lo, init_clip, init_meta, pops};
    e = bb_reduce_launch(tags, leaf, n, ws, &sh, s);
    if (e == cudaSuccess) e = bb_finish_launch(tags, leaf, n, out, ws, &sh, s);
    if (e == cudaSuccess) e = bb_export_launch(tags, leaf, n, ws, recs, (int)b, suf_tiles, tu, su, s);
    return e;
  }
  cudaError_t phase3(int g, const std::vector<Bic2>& hdrs, const float4* alltu, const float4* allsu, int maxb,
                     const void* allpops, int maxp, const int* npops_dev) {
    const int G = (int)hdrs.size();
    std::vector<int> L(G);
    Bic2 pre{0, 0};
    for (int h = 0; h < G; h++) {
      L[h] = (int)std::max<int64_t>(pre.b - hdrs[h].a, 0);
      pre = combine(pre, hdrs[h]);
    }
    int min_after = 0x7fffffff;
    for (int h = g + 1; h < G; h++) min_after = std::min(min_after, L[h]);
    return bb_fixup_launch(G, g, off, (int)b, min_after, L[g], alltu, allsu, maxb, allpops, maxp, npops_dev, recs,
                           reinterpret_cast<float4*>(out), s);
  }
  void release() {
    if (ws) cudaFree(ws);
    if (buf) cudaFree(buf);
    if (hdr) cudaFree(hdr);
    ws = buf = nullptr;
    hdr = nullptr;
  }
};

// header (a, b) of a chunk after phase 1a: the inclusive descriptor of its last tile
cudaError_t read_bb_header(BbChunk& c) {
  const size_t ctrl = 0;
  (void)ctrl;
  const int64_t ntiles = (c.n + bb_tile_elems() - 1) / bb_tile_elems();
  if (ntiles == 0) {
    c.a = c.b = 0;
    return cudaSuccess;
  }
  // Bic value of the chunk, written by the tile scan into the control block
  int2 t{0, 0};
  cudaError_t e = cudaMemcpyAsync(&t, (char*)c.ws + CtrlLayout(ntiles).off_total, 8, cudaMemcpyDeviceToHost, c.s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c.s);
  c.a = t.x;
  c.b = t.y;
  return e;
}

}  // namespace

cudaError_t bb_vshard(const uint8_t* tags, const float* leaf, int64_t n, int G, float* out, cudaStream_t s) {
  std::vector<BbChunk> ch(G);
  cudaError_t e = cudaSuccess;
  for (int g = 0; g < G && e == cudaSuccess; g++) {
    const int64_t a = (g == 0) ? 0 : (n * g / G) & ~int64_t(63);
    const int64_t b = (g == G - 1) ? n : (n * (g + 1) / G) & ~int64_t(63);
    ch[g].tags = tags + a;
    ch[g].leaf = leaf + 4 * a;
    ch[g].n = b - a;
    ch[g].off = a;
    ch[g].out = out + 4 * a;
    ch[g].s = s;
    e = ch[g].alloc_ws();
  }
  for (int g = 0; g < G && e == cudaSuccess; g++) e = ch[g].phase1a();
  for (int g = 0; g < G && e == cudaSuccess; g++) e = read_bb_header(ch[g]);
  for (int g = 0; g < G && e == cudaSuccess; g++) e = ch[g].alloc_buffers(G);
  for (int g = 0; g < G && e == cudaSuccess; g++) e = ch[g].phase1b();
  std::vector<Bic2> hdrs(G);
  int maxb = 1, maxp = 1;
  for (int g = 0; g < G; g++) {
    hdrs[g] = Bic2{ch[g].a, ch[g].b};
    maxb = std::max<int>(maxb, (int)ch[g].b);
  }
  std::vector<int> np(G);
  {
    Bic2 pre{0, 0};
    for (int g = 0; g < G; g++) {
      np[g] = (int)std::min<int64_t>(hdrs[g].a, pre.b);
      maxp = std::max(maxp, np[g]);
      pre = combine(pre, hdrs[g]);
    }
  }
  const size_t rs = bb_sumrec_bytes(), ps = bb_pop_bytes();
  char* allrecs = nullptr;
  float4 *alltu = nullptr, *allsu = nullptr;
  char* allpops = nullptr;
  int* npops_dev = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&allrecs, rs * (size_t)maxb * G);
  if (e == cudaSuccess) e = cudaMalloc(&alltu, 16 * (size_t)G);
  if (e == cudaSuccess) e = cudaMalloc(&allsu, 16 * (size_t)maxb * G);
  if (e == cudaSuccess) e = cudaMalloc(&allpops, ps * (size_t)maxp * G);
  if (e == cudaSuccess) e = cudaMalloc(&npops_dev, 4 * (size_t)G);
  if (e == cudaSuccess) e = cudaMemcpyAsync(npops_dev, np.data(), 4 * (size_t)G, cudaMemcpyHostToDevice, s);
  for (int g = 0; g < G && e == cudaSuccess; g++)
    if (ch[g].b > 0) e = cudaMemcpyAsync(allrecs + rs * (size_t)maxb * g, ch[g].recs, rs * ch[g].b, cudaMemcpyDeviceToDevice, s);
  for (int g = 0; g < G && e == cudaSuccess; g++) e = ch[g].phase2(g, hdrs, allrecs, maxb);
  for (int g = 0; g < G && e == cudaSuccess; g++) {
    e = cudaMemcpyAsync(alltu + g, ch[g].tu, 16, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && ch[g].b > 0)
      e = cudaMemcpyAsync(allsu + (size_t)maxb * g, ch[g].su, 16 * ch[g].b, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && np[g] > 0)
      e = cudaMemcpyAsync(allpops + ps * (size_t)maxp * g, ch[g].pops, ps * np[g], cudaMemcpyDeviceToDevice, s);
  }
  for (int g = 0; g < G && e == cudaSuccess; g++)
    e = ch[g].phase3(g, hdrs, alltu, allsu, maxb, allpops, maxp, npops_dev);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  cudaFree(allrecs);
  cudaFree(alltu);
  cudaFree(allsu);
  cudaFree(allpops);
  cudaFree(npops_dev);
  for (auto& c : ch) c.release();
  return e;
}

#ifdef TB_WITH_NCCL
cudaError_t bb_nccl_shard(const uint8_t* tags, const float* leaf, int64_t n, int64_t off, float* out,
                          ncclComm_t comm, cudaStream_t s, int* nccl_err) {
  *nccl_err = 0;
  int G = 0, g = 0;
  if (ncclCommCount(comm, &G) != ncclSuccess || ncclCommUserRank(comm, &g) != ncclSuccess) {
    *nccl_err = 1;
    return cudaSuccess;
  }
  auto ok = [&](ncclResult_t r) {
    if (r != ncclSuccess) *nccl_err = (int)r;
    return r == ncclSuccess;
  };
  BbChunk c;
  c.tags = tags;
  c.leaf = leaf;
  c.n = n;
  c.off = off;
  c.out = out;
  c.s = s;
  cudaError_t e = c.alloc_ws();
  if (e == cudaSuccess) e = c.phase1a();
  if (e == cudaSuccess) e = read_bb_header(c);
  if (e == cudaSuccess) e = c.alloc_buffers(G);
  if (e == cudaSuccess) e = c.phase1b();
  // exchange 1: headers then summaries
  int32_t* dh = nullptr;
  std::vector<Bic2> hdrs(G);
  int maxb = 1, maxp = 1;
  std::vector<int> np(G);
  if (e == cudaSuccess) e = cudaMalloc(&dh, 16 * (size_t)G);
  if (e == cudaSuccess) {
    int32_t mine[2] = {(int32_t)c.a, (int32_t)c.b};
    e = cudaMemcpyAsync(dh + 2 * G, mine, 8, cudaMemcpyHostToDevice, s);
  }
  if (e == cudaSuccess && ok(ncclAllGather(dh + 2 * G, dh, 2, ncclInt32, comm, s))) {
    std::vector<int32_t> h(2 * G);
    e = cudaMemcpyAsync(h.data(), dh, 8 * (size_t)G, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    Bic2 pre{0, 0};
    for (int r = 0; r < G; r++) {
      hdrs[r] = Bic2{h[2 * r], h[2 * r + 1]};
      maxb = std::max(maxb, h[2 * r + 1]);
      np[r] = (int)std::min<int64_t>(hdrs[r].a, pre.b);
      maxp = std::max(maxp, np[r]);
      pre = combine(pre, hdrs[r]);
    }
  }
  const size_t rs = bb_sumrec_bytes(), ps = bb_pop_bytes();
  char *allrecs = nullptr, *allpops = nullptr;
  float4 *alltu = nullptr, *allsu = nullptr;
  int* npops_dev = nullptr;
  if (e == cudaSuccess && !*nccl_err) e = cudaMalloc(&allrecs, rs * (size_t)maxb * (G + 1));
  if (e == cudaSuccess && !*nccl_err) e = cudaMalloc(&alltu, 16 * (size_t)(G + 1));
  if (e == cudaSuccess && !*nccl_err) e = cudaMalloc(&allsu, 16 * (size_t)maxb * (G + 1));
  if (e == cudaSuccess && !*nccl_err) e = cudaMalloc(&allpops, ps * (size_t)maxp * (G + 1));
  if (e == cudaSuccess && !*nccl_err) e = cudaMalloc(&npops_dev, 4 * (size_t)G);
  if (e == cudaSuccess && !*nccl_err)
    e = cudaMemcpyAsync(npops_dev, np.data(), 4 * (size_t)G, cudaMemcpyHostToDevice, s);
  char* sendrecs = allrecs + rs * (size_t)maxb * G;
  if (e == cudaSuccess && !*nccl_err && c.b > 0)
    e = cudaMemcpyAsync(sendrecs, c.recs, rs * c.b, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && !*nccl_err) ok(ncclAllGather(sendrecs, allrecs, rs * (size_t)maxb, ncclUint8, comm, s));
  if (e == cudaSuccess && !*nccl_err) e = c.phase2(g, hdrs, allrecs, maxb);
  // exchange 2
  float4* sendsu = allsu + (size_t)maxb * G;
  char* sendpops = allpops + ps * (size_t)maxp * G;
  if (e == cudaSuccess && !*nccl_err && c.b > 0)
    e = cudaMemcpyAsync(sendsu, c.su, 16 * c.b, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && !*nccl_err && np[g] > 0)
    e = cudaMemcpyAsync(sendpops, c.pops, ps * np[g], cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && !*nccl_err) ok(ncclAllGather(c.tu, alltu, 16, ncclUint8, comm, s));
  if (e == cudaSuccess && !*nccl_err) ok(ncclAllGather(sendsu, allsu, 16 * (size_t)maxb, ncclUint8, comm, s));
  if (e == cudaSuccess && !*nccl_err) ok(ncclAllGather(sendpops, allpops, ps * (size_t)maxp, ncclUint8, comm, s));
  if (e == cudaSuccess && !*nccl_err) e = c.phase3(g, hdrs, alltu, allsu, maxb, allpops, maxp, npops_dev);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  cudaFree(dh);
  cudaFree(allrecs);
  cudaFree(alltu);
  cudaFree(allsu);
  cudaFree(allpops);
  cudaFree(npops_dev);
  c.release();
  return e;
}
#endif

// Virtual shards: G contiguous chunks of one device buffer, lockstep on one
// stream; the all-gathers are device copies.  Results must equal the
// unsharded call (tests).
cudaError_t pm_vshard(const uint8_t* tags, int64_t n, int G, int32_t* match, int32_t* parent, cudaStream_t s) {
  std::vector<PmChunk> ch(G);
  cudaError_t e = cudaSuccess;
  for (int g = 0; g < G && e == cudaSuccess; g++) {
    // split points on 64-element boundaries keep every chunk's pointers 16-byte aligned
    const int64_t a = (g == 0) ? 0 : (n * g / G) & ~int64_t(63);
    const int64_t b = (g == G - 1) ? n : (n * (g + 1) / G) & ~int64_t(63);
    ch[g].tags = tags + a;
    ch[g].n = b - a;
    ch[g].off = a;
    ch[g].match = match + a;
    ch[g].parent = parent + a;
    ch[g].s = s;
    e = ch[g].alloc(G);
  }
  for (int g = 0; g < G && e == cudaSuccess; g++) e = ch[g].phase1();
  // exchange 1
  std::vector<Bic2> hdrs(G);
  int maxb = 1;
  if (e == cudaSuccess) {
    std::vector<int32_t> h(2 * G);
    for (int g = 0; g < G && e == cudaSuccess; g++)
      e = cudaMemcpyAsync(&h[2 * g], ch[g].hdr, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    for (int g = 0; g < G; g++) {
      hdrs[g] = Bic2{h[2 * g], h[2 * g + 1]};
      maxb = std::max(maxb, h[2 * g + 1]);
    }
  }
  int32_t* allopens = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&allopens, sizeof(int32_t) * (size_t)maxb * G);
  for (int g = 0; g < G && e == cudaSuccess; g++)
    if (hdrs[g].b > 0)
      e = cudaMemcpyAsync(allopens + (size_t)g * maxb, ch[g].opens, 4 * (size_t)hdrs[g].b, cudaMemcpyDeviceToDevice,
                          s);
  std::vector<int64_t> np(G, 0);
  for (int g = 0; g < G && e == cudaSuccess; g++) e = ch[g].phase2(g, hdrs, allopens, maxb, &np[g]);
  // exchange 2
  int64_t maxp = 1;
  for (int g = 0; g < G; g++) maxp = std::max(maxp, np[g]);
  int2* allpairs = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&allpairs, sizeof(int2) * (size_t)maxp * G);
  if (e == cudaSuccess) e = cudaMemsetAsync(allpairs, 0xff, sizeof(int2) * (size_t)maxp * G, s);
  for (int g = 0; g < G && e == cudaSuccess; g++)
    if (np[g] > 0)
      e = cudaMemcpyAsync(allpairs + (size_t)g * maxp, ch[g].pairs, sizeof(int2) * (size_t)np[g],
                          cudaMemcpyDeviceToDevice, s);
  for (int g = 0; g < G && e == cudaSuccess; g++) e = ch[g].phase3(allpairs, maxp * G);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  cudaFree(allopens);
  cudaFree(allpairs);
  for (auto& c : ch) c.release();
  return e;
}

#ifdef TB_WITH_NCCL
// One chunk per process over NCCL.  Returns a cudaError_t-like status; NCCL
// failures are reported through *nccl_err.
cudaError_t pm_nccl_shard(const uint8_t* tags, int64_t n, int64_t off, int32_t* match, int32_t* parent,
                          ncclComm_t comm, cudaStream_t s, int* nccl_err) {
  *nccl_err = 0;
  int G = 0, g = 0;
  if (ncclCommCount(comm, &G) != ncclSuccess || ncclCommUserRank(comm, &g) != ncclSuccess) {
    *nccl_err = 1;
    return cudaSuccess;
  }
  PmChunk c;
  c.tags = tags;
  c.n = n;
  c.off = off;
  c.match = match;
  c.parent = parent;
  c.s = s;
  cudaError_t e = c.alloc(G);
  if (e == cudaSuccess) e = c.phase1();
  int32_t* allhdr = nullptr;
  int32_t* allopens = nullptr;
  int2* allpairs = nullptr;
  std::vector<Bic2> hdrs(G);
  int maxb = 1;
  auto nccl_ok = [&](ncclResult_t r) {
    if (r != ncclSuccess) *nccl_err = (int)r;
    return r == ncclSuccess;
  };
  if (e == cudaSuccess) e = cudaMalloc(&allhdr, 8 * (size_t)G);
  if (e == cudaSuccess && nccl_ok(ncclAllGather(c.hdr, allhdr, 2, ncclInt32, comm, s))) {
    std::vector<int32_t> h(2 * G);
    e = cudaMemcpyAsync(h.data(), allhdr, 8 * (size_t)G, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    for (int r = 0; r < G; r++) {
      hdrs[r] = Bic2{h[2 * r], h[2 * r + 1]};
      maxb = std::max(maxb, h[2 * r + 1]);
    }
  }
  // send buffers padded to the largest contribution (NCCL all-gather counts are uniform)
  int32_t* sendopens = nullptr;
  int2* sendpairs = nullptr;
  if (e == cudaSuccess && !*nccl_err) e = cudaMalloc(&allopens, sizeof(int32_t) * (size_t)maxb * (G + 1));
  if (e == cudaSuccess && !*nccl_err) {
    sendopens = allopens + (size_t)maxb * G;
    if (hdrs[g].b > 0)
      e = cudaMemcpyAsync(sendopens, c.opens, 4 * (size_t)hdrs[g].b, cudaMemcpyDeviceToDevice, s);
  }
  if (e == cudaSuccess && !*nccl_err)
    nccl_ok(ncclAllGather(sendopens, allopens, (size_t)maxb, ncclInt32, comm, s));
  int64_t np = 0;
  if (e == cudaSuccess && !*nccl_err) e = c.phase2(g, hdrs, allopens, maxb, &np);
  // every rank's pair count follows from the headers
  int64_t maxp = 1;
  if (!*nccl_err) {
    Bic2 pre{0, 0};
    for (int r = 0; r < G; r++) {
      maxp = std::max<int64_t>(maxp, std::min<int64_t>(hdrs[r].a, pre.b));
      pre = combine(pre, hdrs[r]);
    }
  }
  if (e == cudaSuccess && !*nccl_err) e = cudaMalloc(&allpairs, sizeof(int2) * (size_t)maxp * (G + 1));
  if (e == cudaSuccess && !*nccl_err) {
    sendpairs = allpairs + (size_t)maxp * G;
    e = cudaMemsetAsync(sendpairs, 0xff, sizeof(int2) * (size_t)maxp, s);
    if (e == cudaSuccess && np > 0)
      e = cudaMemcpyAsync(sendpairs, c.pairs, sizeof(int2) * (size_t)np, cudaMemcpyDeviceToDevice, s);
  }
  if (e == cudaSuccess && !*nccl_err)
    nccl_ok(ncclAllGather(sendpairs, allpairs, 2 * (size_t)maxp, ncclInt32, comm, s));
  if (e == cudaSuccess && !*nccl_err) e = c.phase3(allpairs, maxp * G);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  cudaFree(allhdr);
  cudaFree(allopens);
  cudaFree(allpairs);
  c.release();
  return e;
}
#endif

}  // namespace tb
