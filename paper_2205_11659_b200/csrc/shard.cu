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
// Two drivers share each protocol: NCCL (one chunk per process; the
// `*_shard` C entry points) and an in-process "virtual" driver that runs G
// chunks of one buffer on one GPU in lockstep (tests; no peer traffic).
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
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

// Device scratch of the shard protocols, reused across calls per (device,
// stream) so that a steady-state call allocates nothing: a bump arena.  A call
// that outgrows it gets extra blocks, merged into one block at the start of
// the next call.  Calls on one stream are issued by one host thread at a time.
struct Arena {
  std::vector<std::pair<char*, size_t>> blocks;
  int cur = 0;      // block being filled
  size_t used = 0;  // its fill
};
std::mutex g_arena_mu;
std::map<std::pair<int, cudaStream_t>, Arena> g_arenas;
}  // namespace

// tb_release_workspaces: free every shard arena of the current device (the
// caller guarantees no call is in flight on any stream of it)
void fz_forget_last(int dev);
int shard_release_arenas(int dev) {
  fz_forget_last(dev);
  std::lock_guard<std::mutex> lk(g_arena_mu);
  int freed = 0;
  for (auto it = g_arenas.begin(); it != g_arenas.end();) {
    if (it->first.first / 8 == dev) {
      for (auto& b : it->second.blocks) cudaFree(b.first);
      it = g_arenas.erase(it);
      freed++;
    } else {
      ++it;
    }
  }
  return freed;
}
namespace {

class Scratch {
 public:
  // slot: one arena per protocol (a driver holding buffers calls others)
  Scratch(cudaStream_t s, int slot) : s_(s), slot_(slot) {}
  cudaError_t begin() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_arena_mu);
    a_ = &g_arenas[{dev * 8 + slot_, s_}];
    if (a_->blocks.size() > 1) {
      size_t total = 0;
      for (auto& b : a_->blocks) total += b.second;
      e = cudaStreamSynchronize(s_);
      for (auto& b : a_->blocks) cudaFree(b.first);
      a_->blocks.clear();
      char* q = nullptr;
      if (e == cudaSuccess) e = cudaMalloc(&q, total);
      if (e != cudaSuccess) return e;
      a_->blocks.push_back({q, total});
    }
    a_->cur = 0;
    a_->used = 0;
    return cudaSuccess;
  }
  template <class T>
  cudaError_t get(size_t bytes, T** out) {
    bytes = std::max<size_t>((bytes + 255) & ~size_t(255), 256);
    Arena& a = *a_;
    while (a.cur < (int)a.blocks.size() && a.used + bytes > a.blocks[a.cur].second) {
      a.cur++;
      a.used = 0;
    }
    if (a.cur == (int)a.blocks.size()) {
      char* q = nullptr;
      const size_t sz = std::max(bytes, (size_t)64 << 20);
      cudaError_t e = cudaMalloc(&q, sz);
      if (e != cudaSuccess) return e;
      a.blocks.push_back({q, sz});
      a.used = 0;
    }
    *out = reinterpret_cast<T*>(a.blocks[a.cur].first + a.used);
    a.used += bytes;
    return cudaSuccess;
  }

 private:
  cudaStream_t s_;
  int slot_;
  Arena* a_ = nullptr;
};

// Per-chunk state of the paren_match shard protocol.
struct PmChunk {
  const uint8_t* tags;
  int64_t n, off;
  int32_t* match;
  int32_t* parent;
  cudaStream_t s;
  // device buffers (shard scratch)
  void* ws;           // pm workspace
  int32_t* hdr;       // [2] a, b
  int32_t* opens;     // [n] unmatched opens (send)
  int32_t* stack;     // [n + 1] composed initial stack
  int2* pairs;        // [n] (open, close) send
  int* Ldev;          // [G]

  cudaError_t alloc(int G, Scratch& sc) {
    const size_t wsb = pm_workspace_bytes(std::max<int64_t>(n, 1));
    const size_t nn = (size_t)std::max<int64_t>(n, 1);
    cudaError_t e = sc.get(wsb, &ws);
    if (e == cudaSuccess) e = sc.get(8, &hdr);
    if (e == cudaSuccess) e = sc.get(4 * nn, &opens);
    if (e == cudaSuccess) e = sc.get(4 * (nn + 1), &stack);
    if (e == cudaSuccess) e = sc.get(8 * nn, &pairs);
    if (e == cudaSuccess) e = sc.get(4 * (size_t)G, &Ldev);
    return e;
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
    *npairs = std::min<int64_t>(ag, H);  // the d-th pop of the incoming stack writes pairs[d]
    if (*npairs > 0) {
      e = cudaMemsetAsync(pairs, 0xff, sizeof(int2) * (size_t)*npairs, s);
      if (e != cudaSuccess) return e;
    }
    ShardInit init{(int)mine.a, H, stack, lo, off, pairs};
    e = pm_rescan_launch(n, match, ws, &init, s);  // phase 1's per-tile aggregates and slices stand
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

}  // namespace

// ---- tree_bbox ----------------------------------------------------------------
// The boxes from the matching (tree_bbox_m.cu) over contiguous chunks.  Each
// chunk has paren_match's GLOBAL match / parent for its elements.
//   phase 1: chunk-local slice clips and tile chains (contexts of earlier
//            chunks unknown = INF); the chunk's final stack (its opens closed
//            after it or never) with chunk-local cumulative clips, and its link
//            (the parent of its bottom entry, in an earlier chunk or the root).
//   exchange 1: {off, n, b, link} per chunk, then the final-stack lists.
//   compose: TCc(h) = ctx(link_h) chained over chunks in order; the import
//            table of chunk g = the final-stack opens of chunks h < g with their
//            true contexts (lcc ∩ TCc(h)).
//   phase 2: the full local passes with the import table; closes of nodes
//            opened in an earlier chunk report (close, open, this chunk's prefix).
//   exchange 2: chunk unions, the union after each final-stack open, reports.
//   fix-up: those closes, blend opens closed in a later chunk, blend opens
//            never closed (F4 over chunks).
namespace {

struct BbmChunk {
  const uint8_t* tags;
  const float* leaf;
  const int32_t* match;
  const int32_t* parent;
  int64_t n, off;
  float* out;
  cudaStream_t s;
  void* ws = nullptr;
  ShardOpen* fs = nullptr;   // [n] final stack (send 1)
  ShardOpen* suc = nullptr;  // [n] union after each final-stack open (send 2)
  ShardPop* pops = nullptr;  // [n] closes of earlier chunks' nodes (send 2)
  uint32_t* npops = nullptr;
  int* link = nullptr;
  float4* tu = nullptr;      // chunk union (send 2)
  int* bdev = nullptr;
  int32_t* ext_idx = nullptr;
  float4* ext_ctx = nullptr;
  int b = 0, linkh = -1, np = 0, n_ext = 0;

  BbmShard sh() const { return BbmShard{off, ext_idx, ext_ctx, n_ext, pops, npops}; }

  cudaError_t alloc(Scratch& sc) {
    const size_t nn = (size_t)std::max<int64_t>(n, 1);
    char* c = nullptr;
    cudaError_t e = sc.get(bbm_workspace_bytes((int64_t)nn), &ws);
    if (e == cudaSuccess) e = sc.get(32 * nn, &fs);
    if (e == cudaSuccess) e = sc.get(32 * nn, &suc);
    if (e == cudaSuccess) e = sc.get(32 * nn, &pops);
    if (e == cudaSuccess) e = sc.get(64, &c);
    if (e != cudaSuccess) return e;
    tu = (float4*)c;
    npops = (uint32_t*)(c + 16);
    link = (int*)(c + 20);
    return cudaMemsetAsync(npops, 0, 4, s);
  }
  cudaError_t phase1() { return bbm_shard_phase1(tags, leaf, match, parent, n, off, out, ws, fs, &bdev, link, s); }
  cudaError_t read_header() {
    cudaError_t e = cudaMemcpyAsync(&b, bdev, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&linkh, link, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return e;
  }
  cudaError_t compose(const int4* hdr, int G, int g, const ShardOpen* allfs, int maxb, int cnt, Scratch& sc) {
    n_ext = cnt;
    const size_t c1 = (size_t)std::max(cnt, 1);
    cudaError_t e = sc.get(16 * c1, &ext_ctx);
    if (e == cudaSuccess) e = sc.get(4 * c1, &ext_idx);
    if (e != cudaSuccess) return e;
    if (cnt == 0) return cudaSuccess;
    return bbm_compose_launch(hdr, G, g, allfs, maxb, cnt, ext_idx, ext_ctx, s);
  }
  cudaError_t phase2() {
    const BbmShard x = sh();
    return bbm_shard_phase2(tags, leaf, match, parent, n, out, ws, &x, s);
  }
  cudaError_t read_npops() {
    cudaError_t e = cudaMemcpyAsync(&np, npops, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return e;
  }
  cudaError_t export_unions() {
    const BbmShard x = sh();
    return bbm_export_launch(tags, leaf, match, parent, n, out, ws, &x, fs, b, suc, tu, s);
  }
  cudaError_t fixup(const int4* hdr, int G, int g, const ShardOpen* allsuc, int maxb, const float4* alltu,
                    const ShardPop* allpops, const int* npops_all, int maxp) {
    const BbmShard x = sh();
    return bbm_fixup_launch(tags, leaf, match, parent, n, out, ws, &x, hdr, G, g, allsuc, maxb, alltu, allpops,
                            npops_all, maxp, s);
  }
};

}  // namespace

// Virtual shards of one buffer (tests): the matching of the whole buffer comes
// from the single-device paren_match (its sharded protocol is tested apart).
cudaError_t bb_vshard(const uint8_t* tags, const float* leaf, int64_t n, int G, float* out, cudaStream_t s) {
  Scratch sc(s, 3);
  {
    const cudaError_t e0 = sc.begin();
    if (e0 != cudaSuccess) return e0;
  }
  int32_t* mp = nullptr;
  void* pmws = nullptr;
  const int64_t n64 = (n + 63) & ~int64_t(63);  // keeps parent 16-byte aligned
  cudaError_t e = sc.get(8 * (size_t)n64, &mp);
  if (e == cudaSuccess) e = sc.get(pm_workspace_bytes(n), &pmws);
  int32_t* match = mp;
  int32_t* parent = mp + n64;
  if (e == cudaSuccess) e = pm_launch(tags, n, match, parent, pmws, nullptr, s);
  std::vector<BbmChunk> ch(G);
  for (int g = 0; g < G && e == cudaSuccess; g++) {
    const int64_t a = (g == 0) ? 0 : (n * g / G) & ~int64_t(63);
    const int64_t b = (g == G - 1) ? n : (n * (g + 1) / G) & ~int64_t(63);
    BbmChunk& c = ch[g];
    c.tags = tags + a;
    c.leaf = leaf + 4 * a;
    c.match = match + a;
    c.parent = parent + a;
    c.n = b - a;
    c.off = a;
    c.out = out + 4 * a;
    c.s = s;
    e = c.alloc(sc);
  }
  for (int g = 0; g < G && e == cudaSuccess; g++) e = ch[g].phase1();
  for (int g = 0; g < G && e == cudaSuccess; g++) e = ch[g].read_header();
  // exchange 1
  std::vector<int4> hdr(G);
  int maxb = 1;
  for (int g = 0; g < G; g++) {
    hdr[g] = make_int4((int)ch[g].off, (int)ch[g].n, ch[g].b, ch[g].linkh);
    maxb = std::max(maxb, ch[g].b);
  }
  int4* hdr_dev = nullptr;
  ShardOpen *allfs = nullptr, *allsuc = nullptr;
  float4* alltu = nullptr;
  if (e == cudaSuccess) e = sc.get(sizeof(int4) * G, &hdr_dev);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hdr_dev, hdr.data(), sizeof(int4) * G, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = sc.get(sizeof(ShardOpen) * (size_t)maxb * G, &allfs);
  if (e == cudaSuccess) e = sc.get(sizeof(ShardOpen) * (size_t)maxb * G, &allsuc);
  if (e == cudaSuccess) e = sc.get(sizeof(float4) * G, &alltu);
  for (int g = 0; g < G && e == cudaSuccess; g++)
    if (ch[g].b > 0)
      e = cudaMemcpyAsync(allfs + (size_t)g * maxb, ch[g].fs, sizeof(ShardOpen) * ch[g].b, cudaMemcpyDeviceToDevice,
                          s);
  // compose + phase 2
  int before = 0;
  for (int g = 0; g < G && e == cudaSuccess; g++) {
    e = ch[g].compose(hdr_dev, G, g, allfs, maxb, before, sc);
    if (e == cudaSuccess) e = ch[g].phase2();
    before += ch[g].b;
  }
  for (int g = 0; g < G && e == cudaSuccess; g++) e = ch[g].read_npops();
  // exchange 2
  int maxp = 1;
  std::vector<int> np(G);
  for (int g = 0; g < G; g++) {
    np[g] = ch[g].np;
    maxp = std::max(maxp, np[g]);
  }
  ShardPop* allpops = nullptr;
  int* np_dev = nullptr;
  if (e == cudaSuccess) e = sc.get(sizeof(ShardPop) * (size_t)maxp * G, &allpops);
  if (e == cudaSuccess) e = sc.get(sizeof(int) * G, &np_dev);
  if (e == cudaSuccess) e = cudaMemcpyAsync(np_dev, np.data(), sizeof(int) * G, cudaMemcpyHostToDevice, s);
  for (int g = 0; g < G && e == cudaSuccess; g++) e = ch[g].export_unions();
  for (int g = 0; g < G && e == cudaSuccess; g++) {
    if (np[g] > 0)
      e = cudaMemcpyAsync(allpops + (size_t)g * maxp, ch[g].pops, sizeof(ShardPop) * np[g], cudaMemcpyDeviceToDevice,
                          s);
    if (e == cudaSuccess && ch[g].b > 0)
      e = cudaMemcpyAsync(allsuc + (size_t)g * maxb, ch[g].suc, sizeof(ShardOpen) * ch[g].b,
                          cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(alltu + g, ch[g].tu, sizeof(float4), cudaMemcpyDeviceToDevice, s);
  }
  for (int g = 0; g < G && e == cudaSuccess; g++) e = ch[g].fixup(hdr_dev, G, g, allsuc, maxb, alltu, allpops, np_dev, maxp);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  return e;
}

#ifdef TB_WITH_NCCL
cudaError_t pm_nccl_shard(const uint8_t* tags, int64_t n, int64_t off, int32_t* match, int32_t* parent,
                          ncclComm_t comm, cudaStream_t s, int* nccl_err);

// One rank: the boxes from the global matching (match / parent of the chunk).
cudaError_t bbm_nccl_shard(const uint8_t* tags, const float* leaf, const int32_t* match, const int32_t* parent,
                           int64_t n, int64_t off, float* out, ncclComm_t comm, cudaStream_t s, int* nccl_err) {
  *nccl_err = 0;
  Scratch sc(s, 1);
  {
    const cudaError_t e0 = sc.begin();
    if (e0 != cudaSuccess) return e0;
  }
  int G = 0, g = 0;
  if (ncclCommCount(comm, &G) != ncclSuccess || ncclCommUserRank(comm, &g) != ncclSuccess) {
    *nccl_err = 1;
    return cudaSuccess;
  }
  auto ok = [&](ncclResult_t r) {
    if (r != ncclSuccess) *nccl_err = (int)r;
    return r == ncclSuccess;
  };
  cudaError_t e = cudaSuccess;
  BbmChunk c;
  c.tags = tags;
  c.leaf = leaf;
  c.match = match;
  c.parent = parent;
  c.n = n;
  c.off = off;
  c.out = out;
  c.s = s;
  if (e == cudaSuccess && !*nccl_err) e = c.alloc(sc);
  if (e == cudaSuccess && !*nccl_err) e = c.phase1();
  if (e == cudaSuccess && !*nccl_err) e = c.read_header();
  // exchange 1: headers, then final-stack lists padded to the largest
  int4* hdr_dev = nullptr;
  std::vector<int4> hdr(G);
  int maxb = 1, before = 0;
  if (e == cudaSuccess && !*nccl_err) e = sc.get(sizeof(int4) * (G + 1), &hdr_dev);
  if (e == cudaSuccess && !*nccl_err) {
    const int4 mine = make_int4((int)off, (int)n, c.b, c.linkh);
    e = cudaMemcpyAsync(hdr_dev + G, &mine, sizeof(int4), cudaMemcpyHostToDevice, s);
  }
  if (e == cudaSuccess && !*nccl_err && ok(ncclAllGather(hdr_dev + G, hdr_dev, 4, ncclInt32, comm, s))) {
    e = cudaMemcpyAsync(hdr.data(), hdr_dev, sizeof(int4) * G, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    for (int r = 0; r < G; r++) {
      maxb = std::max(maxb, hdr[r].z);
      if (r < g) before += hdr[r].z;
    }
  }
  ShardOpen *allfs = nullptr, *allsuc = nullptr;
  if (e == cudaSuccess && !*nccl_err) e = sc.get(sizeof(ShardOpen) * (size_t)maxb * (G + 1), &allfs);
  if (e == cudaSuccess && !*nccl_err) e = sc.get(sizeof(ShardOpen) * (size_t)maxb * (G + 1), &allsuc);
  ShardOpen* sendfs = allfs + (size_t)maxb * G;
  if (e == cudaSuccess && !*nccl_err && c.b > 0)
    e = cudaMemcpyAsync(sendfs, c.fs, sizeof(ShardOpen) * c.b, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && !*nccl_err)
    ok(ncclAllGather(sendfs, allfs, sizeof(ShardOpen) * (size_t)maxb, ncclUint8, comm, s));
  if (e == cudaSuccess && !*nccl_err) e = c.compose(hdr_dev, G, g, allfs, maxb, before, sc);
  if (e == cudaSuccess && !*nccl_err) e = c.phase2();
  if (e == cudaSuccess && !*nccl_err) e = c.read_npops();
  // exchange 2
  int* np_dev = nullptr;
  std::vector<int> np(G, 0);
  int maxp = 1;
  if (e == cudaSuccess && !*nccl_err) e = sc.get(sizeof(int) * (G + 1), &np_dev);
  if (e == cudaSuccess && !*nccl_err) e = cudaMemcpyAsync(np_dev + G, &c.np, sizeof(int), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && !*nccl_err && ok(ncclAllGather(np_dev + G, np_dev, 1, ncclInt32, comm, s))) {
    e = cudaMemcpyAsync(np.data(), np_dev, sizeof(int) * G, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    for (int r = 0; r < G; r++) maxp = std::max(maxp, np[r]);
  }
  ShardPop* allpops = nullptr;
  float4* alltu = nullptr;
  if (e == cudaSuccess && !*nccl_err) e = sc.get(sizeof(ShardPop) * (size_t)maxp * (G + 1), &allpops);
  if (e == cudaSuccess && !*nccl_err) e = sc.get(sizeof(float4) * G, &alltu);
  if (e == cudaSuccess && !*nccl_err) e = c.export_unions();
  ShardPop* sendpops = allpops + (size_t)maxp * G;
  ShardOpen* sendsuc = allsuc + (size_t)maxb * G;
  if (e == cudaSuccess && !*nccl_err && c.np > 0)
    e = cudaMemcpyAsync(sendpops, c.pops, sizeof(ShardPop) * c.np, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && !*nccl_err && c.b > 0)
    e = cudaMemcpyAsync(sendsuc, c.suc, sizeof(ShardOpen) * c.b, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && !*nccl_err) ok(ncclAllGather(c.tu, alltu, sizeof(float4), ncclUint8, comm, s));
  if (e == cudaSuccess && !*nccl_err)
    ok(ncclAllGather(sendsuc, allsuc, sizeof(ShardOpen) * (size_t)maxb, ncclUint8, comm, s));
  if (e == cudaSuccess && !*nccl_err)
    ok(ncclAllGather(sendpops, allpops, sizeof(ShardPop) * (size_t)maxp, ncclUint8, comm, s));
  if (e == cudaSuccess && !*nccl_err) e = c.fixup(hdr_dev, G, g, allsuc, maxb, alltu, allpops, np_dev, maxp);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  return e;
}

// One rank: paren_match over the shards (global match / parent), then the boxes.
cudaError_t bb_nccl_shard(const uint8_t* tags, const float* leaf, int64_t n, int64_t off, float* out,
                          ncclComm_t comm, cudaStream_t s, int* nccl_err) {
  *nccl_err = 0;
  Scratch sc(s, 2);
  {
    const cudaError_t e0 = sc.begin();
    if (e0 != cudaSuccess) return e0;
  }
  int32_t* mp = nullptr;
  const int64_t n64 = (std::max<int64_t>(n, 1) + 63) & ~int64_t(63);  // keeps parent 16-byte aligned
  cudaError_t e = sc.get(8 * (size_t)n64, &mp);
  int32_t* match = mp;
  int32_t* parent = mp + n64;
  if (e == cudaSuccess) e = pm_nccl_shard(tags, n, off, match, parent, comm, s, nccl_err);
  if (e == cudaSuccess && !*nccl_err) e = bbm_nccl_shard(tags, leaf, match, parent, n, off, out, comm, s, nccl_err);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  return e;
}
#endif

// Virtual shards: G contiguous chunks of one device buffer, lockstep on one
// stream; the all-gathers are device copies.  Results must equal the
// unsharded call (tests).
cudaError_t pm_vshard(const uint8_t* tags, int64_t n, int G, int32_t* match, int32_t* parent, cudaStream_t s) {
  Scratch sc(s, 4);
  {
    const cudaError_t e0 = sc.begin();
    if (e0 != cudaSuccess) return e0;
  }
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
    e = ch[g].alloc(G, sc);
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
  if (e == cudaSuccess) e = sc.get(sizeof(int32_t) * (size_t)maxb * G, &allopens);
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
  if (e == cudaSuccess) e = sc.get(sizeof(int2) * (size_t)maxp * G, &allpairs);
  if (e == cudaSuccess) e = cudaMemsetAsync(allpairs, 0xff, sizeof(int2) * (size_t)maxp * G, s);
  for (int g = 0; g < G && e == cudaSuccess; g++)
    if (np[g] > 0)
      e = cudaMemcpyAsync(allpairs + (size_t)g * maxp, ch[g].pairs, sizeof(int2) * (size_t)np[g],
                          cudaMemcpyDeviceToDevice, s);
  for (int g = 0; g < G && e == cudaSuccess; g++) e = ch[g].phase3(allpairs, maxp * G);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  return e;
}

#ifdef TB_WITH_NCCL
// One chunk per process over NCCL.  Returns a cudaError_t-like status; NCCL
// failures are reported through *nccl_err.
cudaError_t pm_nccl_shard(const uint8_t* tags, int64_t n, int64_t off, int32_t* match, int32_t* parent,
                          ncclComm_t comm, cudaStream_t s, int* nccl_err) {
  *nccl_err = 0;
  Scratch sc(s, 0);
  {
    const cudaError_t e0 = sc.begin();
    if (e0 != cudaSuccess) return e0;
  }
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
  cudaError_t e = c.alloc(G, sc);
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
  if (e == cudaSuccess) e = sc.get(8 * (size_t)G, &allhdr);
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
  if (e == cudaSuccess && !*nccl_err) e = sc.get(sizeof(int32_t) * (size_t)maxb * (G + 1), &allopens);
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
  if (e == cudaSuccess && !*nccl_err) e = sc.get(sizeof(int2) * (size_t)maxp * (G + 1), &allpairs);
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
  return e;
}
#endif

// ---- the fused pass over shards (fused_shard.cuh) -------------------------------
// Buffers of one rank: workspace, its two slots and the two gathered copies,
// from the per-(device, stream) arena (no allocation in a steady state).
namespace {
struct FzBufs {
  char* ws = nullptr;
  char* slot1 = nullptr;
  char* recv1 = nullptr;
  char* slot2 = nullptr;
  char* recv2 = nullptr;
};
cudaError_t fz_bufs(Scratch& sc, int64_t n, int cap, int G, int nws, bool nobox, FzBufs& b) {
  const size_t wsb = fused_shard_workspace_bytes(std::max<int64_t>(n, 1), cap, nobox);
  const size_t s1 = fused_shard_slot1_bytes(cap), s2 = fused_shard_slot2_bytes(cap);
  cudaError_t e = sc.get(wsb * (size_t)nws, &b.ws);
  if (e == cudaSuccess) e = sc.get(s1, &b.slot1);
  if (e == cudaSuccess) e = sc.get(s1 * (size_t)G, &b.recv1);
  if (e == cudaSuccess) e = sc.get(s2, &b.slot2);
  if (e == cudaSuccess) e = sc.get(s2 * (size_t)G, &b.recv2);
  return e;
}
std::mutex g_fzlast_mu;
struct FzLast {
  int64_t n;
  int cap;
  char* ws;
};
std::map<std::pair<int, cudaStream_t>, FzLast> g_fzlast;  // the last call's workspace (status)
}  // namespace

// Virtual shards (tests): G contiguous chunks of one buffer, the phases in
// lockstep on one stream; chunk k's slots ARE the k-th parts of the gathered
// buffers, so the exchanges are no-ops.
cudaError_t fz_vshard(const uint8_t* tags, const float* leaf, int64_t n, int G, int cap, int32_t* match,
                      int32_t* parent, float* out, cudaStream_t s, int* overflow) {
  Scratch sc(s, 3);
  cudaError_t e = sc.begin();
  if (e != cudaSuccess) return e;
  // chunk borders at multiples of 16 elements (the kernels' 16-byte alignment of
  // every array); chunks may be empty
  auto off = [&](int k) { return k >= G ? n : (n * k / G) & ~int64_t(15); };
  int64_t nmax = 0;
  for (int k = 0; k < G; k++) nmax = std::max(nmax, off(k + 1) - off(k));
  FzBufs b;
  const bool nobox = leaf == nullptr;
  e = fz_bufs(sc, nmax, cap, G, G, nobox, b);
  if (e != cudaSuccess) return e;
  const size_t wsb = fused_shard_workspace_bytes(std::max<int64_t>(nmax, 1), cap, nobox);
  const size_t s1 = fused_shard_slot1_bytes(cap), s2 = fused_shard_slot2_bytes(cap);
  for (int k = 0; k < G && e == cudaSuccess; k++)
    e = fused_shard_phase1(tags + off(k), leaf ? leaf + 4 * off(k) : nullptr, off(k + 1) - off(k), off(k), cap,
                           match ? match + off(k) : nullptr, b.ws + wsb * k, b.recv1 + s1 * k, s);
  for (int k = 0; k < G && e == cudaSuccess; k++)
    e = fused_shard_phase2(tags + off(k), leaf ? leaf + 4 * off(k) : nullptr, off(k + 1) - off(k), off(k), cap, G, k,
                           match ? match + off(k) : nullptr, parent ? parent + off(k) : nullptr,
                           out ? out + 4 * off(k) : nullptr, b.ws + wsb * k, b.recv1, b.recv2 + s2 * k, s);
  for (int k = 0; k < G && e == cudaSuccess; k++)
    e = fused_shard_phase3(off(k + 1) - off(k), off(k), cap, G, k, match ? match + off(k) : nullptr,
                           out ? out + 4 * off(k) : nullptr, b.ws + wsb * k, b.recv1, b.recv2, s);
  if (e == cudaSuccess && overflow) {
    cudaError_t e2 = cudaSuccess;
    *overflow = 0;
    for (int k = 0; k < G && e2 == cudaSuccess; k++)
      *overflow |= fused_shard_status(std::max<int64_t>(nmax, 1), cap, b.ws + wsb * k, s, &e2);
    e = e2;
  }
  return e;
}

#ifdef TB_WITH_NCCL
// One rank over NCCL: two all-gathers of fixed size, nothing waits on the host.
// NCCL failures (including asynchronous ones: ncclCommGetAsyncError after each
// collective is enqueued) are reported through *nccl_err.
cudaError_t fz_nccl_shard(const uint8_t* tags, const float* leaf, int64_t n, int64_t off, int cap, int32_t* match,
                          int32_t* parent, float* out, ncclComm_t comm, cudaStream_t s, int* nccl_err) {
  *nccl_err = 0;
  int G = 0, g = 0;
  if (ncclCommCount(comm, &G) != ncclSuccess || ncclCommUserRank(comm, &g) != ncclSuccess) {
    *nccl_err = 1;
    return cudaSuccess;
  }
  Scratch sc(s, 3);
  cudaError_t e = sc.begin();
  if (e != cudaSuccess) return e;
  FzBufs b;
  e = fz_bufs(sc, n, cap, G, 1, leaf == nullptr, b);
  if (e != cudaSuccess) return e;
  auto nccl_ok = [&](ncclResult_t r) {
    ncclResult_t ar = ncclSuccess;
    if (r == ncclSuccess) r = ncclCommGetAsyncError(comm, &ar);
    if (r != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress)) *nccl_err = 1;
    return !*nccl_err;
  };
  const size_t s1 = fused_shard_slot1_bytes(cap), s2 = fused_shard_slot2_bytes(cap);
  e = fused_shard_phase1(tags, leaf, n, off, cap, match, b.ws, b.slot1, s);
  if (e != cudaSuccess || !nccl_ok(ncclAllGather(b.slot1, b.recv1, s1, ncclUint8, comm, s))) return e;
  e = fused_shard_phase2(tags, leaf, n, off, cap, G, g, match, parent, out, b.ws, b.recv1, b.slot2, s);
  if (e != cudaSuccess || !nccl_ok(ncclAllGather(b.slot2, b.recv2, s2, ncclUint8, comm, s))) return e;
  e = fused_shard_phase3(n, off, cap, G, g, match, out, b.ws, b.recv1, b.recv2, s);
  if (e == cudaSuccess) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_fzlast_mu);
    g_fzlast[{dev, s}] = FzLast{n, cap, b.ws};
  }
  return e;
}
#endif

void fz_forget_last(int dev) {
  std::lock_guard<std::mutex> lk(g_fzlast_mu);
  for (auto it = g_fzlast.begin(); it != g_fzlast.end();) it = it->first.first == dev ? g_fzlast.erase(it) : std::next(it);
}

// overflow flag of the last sharded call on this (device, stream): waits for it
cudaError_t fz_shard_status(cudaStream_t s, int* overflow) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  FzLast last{-1, 0, nullptr};
  {
    std::lock_guard<std::mutex> lk(g_fzlast_mu);
    auto it = g_fzlast.find({dev, s});
    if (it != g_fzlast.end()) last = it->second;
  }
  *overflow = 0;
  if (!last.ws) return cudaSuccess;
  *overflow = fused_shard_status(std::max<int64_t>(last.n, 1), last.cap, last.ws, s, &e);
  return e;
}

}  // namespace tb
