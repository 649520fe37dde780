// C ABI (include/treebbox.h): argument validation, workspace cache, launches.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "kernels.h"
#include "treebbox.h"
#ifdef TB_WITH_NCCL
#include <nccl.h>
namespace tb {
int shard_release_arenas(int dev);
cudaError_t fz_vshard(const uint8_t* tags, const float* leaf, int64_t n, int G, int cap, int32_t* match,
                      int32_t* parent, float* out, cudaStream_t s, int* overflow);
cudaError_t fz_shard_status(cudaStream_t s, int* overflow);
cudaError_t pm_nccl_shard(const uint8_t* tags, int64_t n, int64_t off, int32_t* match, int32_t* parent,
                          ncclComm_t comm, cudaStream_t s, int* nccl_err);
cudaError_t bbm_nccl_shard(const uint8_t* tags, const float* leaf, const int32_t* match, const int32_t* parent,
                           int64_t n, int64_t off, float* out, ncclComm_t comm, cudaStream_t s, int* nccl_err);
cudaError_t bb_nccl_shard(const uint8_t* tags, const float* leaf, int64_t n, int64_t off, float* out,
                          ncclComm_t comm, cudaStream_t s, int* nccl_err);
cudaError_t fz_nccl_shard(const uint8_t* tags, const float* leaf, int64_t n, int64_t off, int cap, int32_t* match,
                          int32_t* parent, float* out, ncclComm_t comm, cudaStream_t s, int* nccl_err);
}
#endif

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(TB_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

constexpr int64_t kMaxN = 2147483647LL;

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + nb && y < x + na;
}

int check_n(int64_t n) {
  if (n < 0 || n > kMaxN) return fail(TB_ERR_ARG, "n = %lld out of range [0, 2^31-1]", (long long)n);
  return TB_OK;
}

// ---- per-(device, stream) scratch cache ---------------------------------
struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};
std::mutex g_mu;
std::map<std::pair<int, void*>, Buf> g_ws;

int get_ws(void* stream, int slot, size_t need, void** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_mu);
  Buf& b = g_ws[{dev * 16 + slot, stream}];
  if (b.bytes < need) {
    if (b.p) {
      e = cudaStreamSynchronize((cudaStream_t)stream);
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
      cudaFree(b.p);
      b.p = nullptr;
      b.bytes = 0;
    }
    size_t sz = need + need / 8 + 4096;
    e = cudaMalloc(&b.p, sz);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(workspace)");
    b.bytes = sz;
  }
  *out = b.p;
  return TB_OK;
}

// Side streams / events of the host pipeline, one set per device (never freed).
constexpr int kMaxChunks = 16;  // chunks of the pipelined host path
int g_chunk_shift = 23;         // at least 2^shift elements per chunk (tests lower it)
struct AuxStreams {
  cudaStream_t in = nullptr, out = nullptr;
  cudaEvent_t start = nullptr, in_done = nullptr, pm_done = nullptr, out_done = nullptr;
  cudaEvent_t chunk_in[kMaxChunks] = {}, chunk_done[kMaxChunks] = {};
  cudaStream_t side = nullptr;  // paren_match_tree_bbox: the box reduce pass beside paren_match
  cudaEvent_t fork = nullptr, join = nullptr;
};
std::map<int, AuxStreams> g_aux;
// Serialises the enqueue sequences that use the shared side streams and events
// (a record / wait pair of one caller must not interleave with another's).
std::mutex g_aux_enqueue_mu;

int get_aux(AuxStreams** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_mu);
  AuxStreams& a = g_aux[dev];
  if (!a.in) {
    e = cudaStreamCreateWithFlags(&a.in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&a.out, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&a.start, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&a.in_done, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&a.pm_done, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&a.out_done, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&a.side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming);
    for (int c = 0; c < kMaxChunks && e == cudaSuccess; c++) {
      e = cudaEventCreateWithFlags(&a.chunk_in[c], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&a.chunk_done[c], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
      a = AuxStreams{};
      return cuda_fail(e, "side streams");
    }
  }
  *out = &a;
  return TB_OK;
}

// The fused single-device path (fused.cu) runs paren_match + tree_bbox from one
// tile pass; tb_debug_use_fused(0) selects the earlier two-call path
// (paren_match, then the boxes from its match / parent) for comparisons.
static int g_use_fused = 1;

int pm_checks(const uint8_t* tags, int64_t n, int32_t* match, int32_t* parent) {
  int r = check_n(n);
  if (r) return r;
  if (n == 0) return TB_OK;
  if (!tags || !match || !parent) return fail(TB_ERR_ARG, "null pointer with n > 0");
  if (!aligned16(tags) || !aligned16(match) || !aligned16(parent))
    return fail(TB_ERR_ALIGN, "tags, match and parent must be 16-byte aligned");
  const size_t n4 = (size_t)n * 4;
  if (overlap(match, n4, parent, n4) || overlap(match, n4, tags, (size_t)n) ||
      overlap(parent, n4, tags, (size_t)n))
    return fail(TB_ERR_ALIAS, "outputs overlap each other or the input");
  return TB_OK;
}

int bb_checks(const uint8_t* tags, const float* leaf, int64_t n, float* out) {
  int r = check_n(n);
  if (r) return r;
  if (n == 0) return TB_OK;
  if (!tags || !leaf || !out) return fail(TB_ERR_ARG, "null pointer with n > 0");
  if (!aligned16(tags) || !aligned16(leaf) || !aligned16(out))
    return fail(TB_ERR_ALIGN, "tags, leaf_bbox and node_bbox must be 16-byte aligned");
  const size_t nb = (size_t)n * 16;
  if (overlap(out, nb, leaf, nb) || overlap(out, nb, tags, (size_t)n))
    return fail(TB_ERR_ALIAS, "node_bbox overlaps an input");
  return TB_OK;
}

}  // namespace

extern "C" {

const char* tb_last_error(void) { return g_err; }

int tb_release_workspaces(void) {
  g_err[0] = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "tb_release_workspaces");
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto it = g_ws.begin(); it != g_ws.end();) {
      if (it->first.first / 16 == dev) {
        cudaFree(it->second.p);
        it = g_ws.erase(it);
      } else {
        ++it;
      }
    }
  }
#ifdef TB_WITH_NCCL
  tb::shard_release_arenas(dev);
#endif
  return TB_OK;
}
const char* tb_version(void) { return "treebbox-b200 0.1 (sm_100a)"; }

size_t paren_match_workspace_bytes(int64_t n) { return n > 0 ? tb::pm_workspace_bytes(n) : 0; }

int paren_match_ws(const uint8_t* d_tags, int64_t n, int32_t* d_match, int32_t* d_parent,
                   void* d_workspace, size_t workspace_bytes, void* stream) {
  g_err[0] = 0;
  int r = pm_checks(d_tags, n, d_match, d_parent);
  if (r || n == 0) return r;
  if (!d_workspace || workspace_bytes < tb::pm_workspace_bytes(n))
    return fail(TB_ERR_ARG, "workspace too small: need %zu bytes", tb::pm_workspace_bytes(n));
  cudaError_t e = tb::pm_launch(d_tags, n, d_match, d_parent, d_workspace, nullptr, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "paren_match launch");
  return TB_OK;
}

int paren_match(const uint8_t* d_tags, int64_t n, int32_t* d_match, int32_t* d_parent, void* stream) {
  g_err[0] = 0;
  int r = pm_checks(d_tags, n, d_match, d_parent);
  if (r || n == 0) return r;
  void* ws = nullptr;
  if (g_use_fused) {  // the fused tile pass without boxes (fz_match)
    r = get_ws(stream, 14, tb::fused_match_workspace_bytes(n), &ws);
    if (r) return r;
    cudaError_t e = tb::fused_match_launch(d_tags, n, d_match, d_parent, ws, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "paren_match launch");
    return TB_OK;
  }
  const size_t need = tb::pm_workspace_bytes(n);
  r = get_ws(stream, 0, need, &ws);
  if (r) return r;
  return paren_match_ws(d_tags, n, d_match, d_parent, ws, need, stream);
}

int paren_match_host(const uint8_t* h_tags, int64_t n, int32_t* h_match, int32_t* h_parent,
                     void* stream) {
  g_err[0] = 0;
  int r = check_n(n);
  if (r || n == 0) return r;
  if (!h_tags || !h_match || !h_parent) return fail(TB_ERR_ARG, "null pointer with n > 0");
  const size_t nb_t = ((size_t)n + 255) & ~(size_t)255;
  const size_t nb_i = ((size_t)n * 4 + 255) & ~(size_t)255;
  void* io = nullptr;
  r = get_ws(stream, 1, nb_t + 2 * nb_i, &io);
  if (r) return r;
  uint8_t* d_tags = (uint8_t*)io;
  int32_t* d_match = (int32_t*)((char*)io + nb_t);
  int32_t* d_parent = (int32_t*)((char*)io + nb_t + nb_i);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(d_tags, h_tags, (size_t)n, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "H2D tags");
  r = paren_match(d_tags, n, d_match, d_parent, stream);
  if (r) return r;
  e = cudaMemcpyAsync(h_match, d_match, (size_t)n * 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h_parent, d_parent, (size_t)n * 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "D2H results");
  return TB_OK;
}

// tree_bbox = paren_match into the workspace, then the boxes from the matching
struct BbWs {
  size_t pm_off, match_off, parent_off, bbm_off, bytes;
  explicit BbWs(int64_t n) {
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    size_t o = 0;
    pm_off = o; o = al(o + tb::pm_workspace_bytes(n));
    match_off = o; o = al(o + 4 * (size_t)n);
    parent_off = o; o = al(o + 4 * (size_t)n);
    bbm_off = o; o = al(o + tb::bbm_workspace_bytes(n));
    bytes = o;
  }
};

static int bbm_checks(const uint8_t* tags, const float* leaf, const int32_t* match, const int32_t* parent, int64_t n,
               float* out) {
  int r = bb_checks(tags, leaf, n, out);
  if (r || n == 0) return r;
  if (!match || !parent) return fail(TB_ERR_ARG, "null pointer with n > 0");
  if (!aligned16(match) || !aligned16(parent)) return fail(TB_ERR_ALIGN, "match and parent must be 16-byte aligned");
  const size_t nb = (size_t)n * 16, n4 = (size_t)n * 4;
  if (overlap(out, nb, match, n4) || overlap(out, nb, parent, n4))
    return fail(TB_ERR_ALIAS, "node_bbox overlaps an input");
  return TB_OK;
}

size_t tree_bbox_workspace_bytes(int64_t n) {
  if (n <= 0) return 0;
  return std::max(BbWs(n).bytes, tb::fused_workspace_bytes(n));
}

static int tree_bbox_ws_impl(const uint8_t* d_tags, const float* d_leaf_bbox, int64_t n, float* d_node_bbox,
                             void* d_workspace, size_t workspace_bytes, void* stream, uint64_t* trace) {
  g_err[0] = 0;
  int r = bb_checks(d_tags, d_leaf_bbox, n, d_node_bbox);
  if (r || n == 0) return r;
  const BbWs L(n);
  if (!d_workspace || workspace_bytes < L.bytes)
    return fail(TB_ERR_ARG, "workspace too small: need %zu bytes", L.bytes);
  if (g_use_fused && trace == nullptr) {
    if (workspace_bytes < tb::fused_workspace_bytes(n))
      return fail(TB_ERR_ARG, "workspace too small: need %zu bytes", tb::fused_workspace_bytes(n));
    cudaError_t e = tb::fused_launch(d_tags, d_leaf_bbox, n, nullptr, nullptr, d_node_bbox, d_workspace,
                                     (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "tree_bbox launch");
    return TB_OK;
  }
  char* w = (char*)d_workspace;
  int32_t* match = (int32_t*)(w + L.match_off);
  int32_t* parent = (int32_t*)(w + L.parent_off);
  cudaError_t e = tb::pm_launch(d_tags, n, match, parent, w + L.pm_off, nullptr, (cudaStream_t)stream);
  if (e == cudaSuccess)
    e = tb::bbm_launch(d_tags, d_leaf_bbox, match, parent, n, d_node_bbox, w + L.bbm_off, (cudaStream_t)stream,
                       trace);
  if (e != cudaSuccess) return cuda_fail(e, "tree_bbox launch");
  return TB_OK;
}

int tree_bbox_ws(const uint8_t* d_tags, const float* d_leaf_bbox, int64_t n, float* d_node_bbox,
                 void* d_workspace, size_t workspace_bytes, void* stream) {
  return tree_bbox_ws_impl(d_tags, d_leaf_bbox, n, d_node_bbox, d_workspace, workspace_bytes, stream, nullptr);
}

int tree_bbox(const uint8_t* d_tags, const float* d_leaf_bbox, int64_t n, float* d_node_bbox, void* stream) {
  g_err[0] = 0;
  int r = bb_checks(d_tags, d_leaf_bbox, n, d_node_bbox);
  if (r || n == 0) return r;
  void* ws = nullptr;
  const size_t need = tree_bbox_workspace_bytes(n);
  r = get_ws(stream, 3, need, &ws);
  if (r) return r;
  return tree_bbox_ws(d_tags, d_leaf_bbox, n, d_node_bbox, ws, need, stream);
}

size_t tree_bbox_matched_workspace_bytes(int64_t n) { return n > 0 ? tb::bbm_workspace_bytes(n) : 0; }

int tree_bbox_matched_ws(const uint8_t* d_tags, const float* d_leaf_bbox, const int32_t* d_match,
                         const int32_t* d_parent, int64_t n, float* d_node_bbox, void* d_workspace,
                         size_t workspace_bytes, void* stream) {
  g_err[0] = 0;
  int r = bbm_checks(d_tags, d_leaf_bbox, d_match, d_parent, n, d_node_bbox);
  if (r || n == 0) return r;
  if (!d_workspace || workspace_bytes < tb::bbm_workspace_bytes(n))
    return fail(TB_ERR_ARG, "workspace too small: need %zu bytes", tb::bbm_workspace_bytes(n));
  cudaError_t e = tb::bbm_launch(d_tags, d_leaf_bbox, d_match, d_parent, n, d_node_bbox, d_workspace,
                                 (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "tree_bbox_matched launch");
  return TB_OK;
}

int tree_bbox_matched(const uint8_t* d_tags, const float* d_leaf_bbox, const int32_t* d_match,
                      const int32_t* d_parent, int64_t n, float* d_node_bbox, void* stream) {
  g_err[0] = 0;
  int r = bbm_checks(d_tags, d_leaf_bbox, d_match, d_parent, n, d_node_bbox);
  if (r || n == 0) return r;
  void* ws = nullptr;
  const size_t need = tb::bbm_workspace_bytes(n);
  r = get_ws(stream, 5, need, &ws);
  if (r) return r;
  return tree_bbox_matched_ws(d_tags, d_leaf_bbox, d_match, d_parent, n, d_node_bbox, ws, need, stream);
}

int paren_match_tree_bbox(const uint8_t* d_tags, const float* d_leaf_bbox, int64_t n, int32_t* d_match,
                          int32_t* d_parent, float* d_node_bbox, void* stream) {
  g_err[0] = 0;
  int r = pm_checks(d_tags, n, d_match, d_parent);
  if (r || n == 0) return r;
  r = bbm_checks(d_tags, d_leaf_bbox, d_match, d_parent, n, d_node_bbox);
  if (r) return r;
  const size_t nb = (size_t)n * 16, n4 = (size_t)n * 4;
  if (overlap(d_match, n4, d_leaf_bbox, nb) || overlap(d_parent, n4, d_leaf_bbox, nb))
    return fail(TB_ERR_ALIAS, "match / parent overlap leaf_bbox");
  if (g_use_fused) {
    void* fws = nullptr;
    r = get_ws(stream, 7, tb::fused_workspace_bytes(n), &fws);
    if (r) return r;
    cudaError_t e = tb::fused_launch(d_tags, d_leaf_bbox, n, d_match, d_parent, d_node_bbox, fws,
                                     (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "paren_match_tree_bbox launch");
    return TB_OK;
  }
  void* pmws = nullptr;
  void* bws = nullptr;
  r = get_ws(stream, 0, tb::pm_workspace_bytes(n), &pmws);
  if (r) return r;
  r = get_ws(stream, 5, tb::bbm_workspace_bytes(n), &bws);
  if (r) return r;
  AuxStreams* ax = nullptr;
  r = get_aux(&ax);
  if (r) return r;
  // The box path's reduce pass reads only tags and boxes: it runs on a side
  // stream beside paren_match's tile scan (one CTA) and finish pass, forked
  // after paren_match's reduce pass and joined before the passes that need
  // match / parent.
  cudaStream_t s = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lk(g_aux_enqueue_mu);
  cudaError_t e = tb::pm_reduce_only_launch(d_tags, n, d_match, pmws, nullptr, s);
  if (e == cudaSuccess) e = cudaEventRecord(ax->fork, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ax->side, ax->fork, 0);
  if (e == cudaSuccess) e = tb::bbm_launch_reduce(d_tags, d_leaf_bbox, n, d_node_bbox, bws, ax->side);
  if (e == cudaSuccess) e = cudaEventRecord(ax->join, ax->side);
  if (e == cudaSuccess) e = tb::pm_rescan_launch(n, d_match, pmws, nullptr, s);
  if (e == cudaSuccess) e = tb::pm_finish_launch(d_tags, n, d_match, d_parent, pmws, nullptr, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ax->join, 0);
  if (e == cudaSuccess) e = tb::bbm_launch_rest(d_tags, d_leaf_bbox, d_match, d_parent, n, d_node_bbox, bws, s);
  if (e != cudaSuccess) return cuda_fail(e, "paren_match_tree_bbox launch");
  return TB_OK;
}

int tree_bbox_host(const uint8_t* h_tags, const float* h_leaf_bbox, int64_t n, float* h_node_bbox,
                   void* stream) {
  g_err[0] = 0;
  int r = check_n(n);
  if (r || n == 0) return r;
  if (!h_tags || !h_leaf_bbox || !h_node_bbox) return fail(TB_ERR_ARG, "null pointer with n > 0");
  const size_t nb_t = ((size_t)n + 255) & ~(size_t)255;
  const size_t nb_b = ((size_t)n * 16 + 255) & ~(size_t)255;
  void* io = nullptr;
  r = get_ws(stream, 4, nb_t + 2 * nb_b, &io);
  if (r) return r;
  uint8_t* d_tags = (uint8_t*)io;
  float* d_in = (float*)((char*)io + nb_t);
  float* d_out = (float*)((char*)io + nb_t + nb_b);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(d_tags, h_tags, (size_t)n, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_in, h_leaf_bbox, (size_t)n * 16, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "H2D inputs");
  r = tree_bbox(d_tags, d_in, n, d_out, stream);
  if (r) return r;
  e = cudaMemcpyAsync(h_node_bbox, d_out, (size_t)n * 16, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "D2H results");
  return TB_OK;
}

// The chunked schedule of paren_match_tree_bbox_host (host result mapped):
// tags in, paren_match, match / parent out (side stream `out`); boxes in by
// chunks of tiles (side stream `in`); per chunk, once its boxes are in, the box
// passes over its tiles (they read only earlier tiles) and its result out;
// finally the never-closed blend opens, and the entries written after their
// chunk went out are stored into the mapped host result by a kernel.
static int pm_tb_host_pipelined(const uint8_t* h_tags, const float* h_leaf_bbox, int64_t n, int32_t* h_match,
                                int32_t* h_parent, float* h_node_bbox, float* hmap, uint8_t* d_tags,
                                int32_t* d_match, int32_t* d_parent, float* d_in, float* d_out, cudaStream_t s,
                                AuxStreams* ax) {
  const int nt = tb::bbm_tiles(n);
  const int64_t tile = tb::bbm_tile_elems();
  int C = (int)std::min<int64_t>(kMaxChunks, std::max<int64_t>(1, n >> g_chunk_shift));
  const int ct = (nt + C - 1) / C;
  C = (nt + ct - 1) / ct;
  void* bws = nullptr;
  int r = get_ws(s, 5, tb::bbm_workspace_bytes(n), &bws);
  if (r) return r;
  auto lo = [&](int c) { return std::min<int64_t>(n, (int64_t)c * ct * tile); };
  std::unique_lock<std::mutex> lk(g_aux_enqueue_mu);
  cudaError_t e = cudaEventRecord(ax->start, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ax->in, ax->start, 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_tags, h_tags, (size_t)n, cudaMemcpyHostToDevice, s);
  for (int c = 0; c < C && e == cudaSuccess; c++) {
    const int64_t a = lo(c), b = lo(c + 1);
    e = cudaMemcpyAsync(d_in + 4 * a, h_leaf_bbox + 4 * a, (size_t)(b - a) * 16, cudaMemcpyHostToDevice, ax->in);
    if (e == cudaSuccess) e = cudaEventRecord(ax->chunk_in[c], ax->in);
  }
  if (e != cudaSuccess) return cuda_fail(e, "H2D inputs");
  r = paren_match(d_tags, n, d_match, d_parent, s);
  if (r) return r;
  e = cudaEventRecord(ax->pm_done, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ax->out, ax->pm_done, 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h_match, d_match, (size_t)n * 4, cudaMemcpyDeviceToHost, ax->out);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h_parent, d_parent, (size_t)n * 4, cudaMemcpyDeviceToHost, ax->out);
  if (e == cudaSuccess) e = tb::bbm_begin(bws, n, s);
  for (int c = 0; c < C && e == cudaSuccess; c++) {
    const int64_t a = lo(c), b = lo(c + 1);
    e = cudaStreamWaitEvent(s, ax->chunk_in[c], 0);
    if (e == cudaSuccess)
      e = tb::bbm_tiles_launch(d_tags, d_in, d_match, d_parent, n, d_out, bws, c * ct, std::min(nt, (c + 1) * ct), s);
    if (e == cudaSuccess) e = cudaEventRecord(ax->chunk_done[c], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ax->out, ax->chunk_done[c], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h_node_bbox + 4 * a, d_out + 4 * a, (size_t)(b - a) * 16, cudaMemcpyDeviceToHost, ax->out);
  }
  if (e == cudaSuccess) e = tb::bbm_end(d_tags, d_in, d_match, d_parent, n, d_out, bws, s);
  if (e == cudaSuccess) e = cudaEventRecord(ax->out_done, ax->out);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ax->out_done, 0);
  if (e == cudaSuccess) e = tb::bbm_patch_host_launch(d_tags, d_match, n, d_out, bws, hmap, ct, s);
  lk.unlock();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "pipelined host path");
  return TB_OK;
}

int paren_match_tree_bbox_host(const uint8_t* h_tags, const float* h_leaf_bbox, int64_t n, int32_t* h_match,
                               int32_t* h_parent, float* h_node_bbox, void* stream) {
  g_err[0] = 0;
  int r = check_n(n);
  if (r || n == 0) return r;
  if (!h_tags || !h_leaf_bbox || !h_match || !h_parent || !h_node_bbox)
    return fail(TB_ERR_ARG, "null pointer with n > 0");
  const size_t nb_t = ((size_t)n + 255) & ~(size_t)255;
  const size_t nb_i = ((size_t)n * 4 + 255) & ~(size_t)255;
  const size_t nb_b = ((size_t)n * 16 + 255) & ~(size_t)255;
  void* io = nullptr;
  r = get_ws(stream, 6, nb_t + 2 * nb_i + 2 * nb_b, &io);
  if (r) return r;
  char* c = (char*)io;
  uint8_t* d_tags = (uint8_t*)c;
  int32_t* d_match = (int32_t*)(c + nb_t);
  int32_t* d_parent = (int32_t*)(c + nb_t + nb_i);
  float* d_in = (float*)(c + nb_t + 2 * nb_i);
  float* d_out = (float*)(c + nb_t + 2 * nb_i + nb_b);
  // Copies overlap the kernels and each other (PCIe is full duplex): the boxes
  // go in on a side stream while paren_match runs, match/parent come out on a
  // second side stream while the boxes are still going in.
  cudaStream_t s = (cudaStream_t)stream;
  AuxStreams* ax = nullptr;
  r = get_aux(&ax);
  if (r) return r;
  // Pinned (device-mapped) result: the box passes run chunk by chunk as the
  // boxes arrive and each chunk's result goes out while later chunks compute.
  float* hmap = nullptr;
  {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, h_node_bbox) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
        pa.devicePointer)
      hmap = (float*)pa.devicePointer;
    (void)cudaGetLastError();
  }
  if (hmap) return pm_tb_host_pipelined(h_tags, h_leaf_bbox, n, h_match, h_parent, h_node_bbox, hmap, d_tags,
                                        d_match, d_parent, d_in, d_out, s, ax);
  std::unique_lock<std::mutex> lk(g_aux_enqueue_mu);
  cudaError_t e = cudaEventRecord(ax->start, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ax->in, ax->start, 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_tags, h_tags, (size_t)n, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_in, h_leaf_bbox, (size_t)n * 16, cudaMemcpyHostToDevice, ax->in);
  if (e == cudaSuccess) e = cudaEventRecord(ax->in_done, ax->in);
  if (e != cudaSuccess) return cuda_fail(e, "H2D inputs");
  r = paren_match(d_tags, n, d_match, d_parent, stream);
  if (r) return r;
  e = cudaEventRecord(ax->pm_done, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ax->out, ax->pm_done, 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h_match, d_match, (size_t)n * 4, cudaMemcpyDeviceToHost, ax->out);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h_parent, d_parent, (size_t)n * 4, cudaMemcpyDeviceToHost, ax->out);
  if (e == cudaSuccess) e = cudaEventRecord(ax->out_done, ax->out);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ax->in_done, 0);
  if (e != cudaSuccess) return cuda_fail(e, "D2H match/parent");
  r = tree_bbox_matched(d_tags, d_in, d_match, d_parent, n, d_out, stream);
  if (r) return r;
  e = cudaMemcpyAsync(h_node_bbox, d_out, (size_t)n * 16, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ax->out_done, 0);
  lk.unlock();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "D2H results");
  return TB_OK;
}

int paren_match_bytes(const uint8_t* d_bytes, int64_t n, const uint8_t* h_class_map, int32_t* d_match,
                      int32_t* d_parent, void* stream) {
  g_err[0] = 0;
  int r = pm_checks(d_bytes, n, d_match, d_parent);
  if (r || n == 0) return r;
  if (!h_class_map) return fail(TB_ERR_ARG, "null class map");
  const size_t nb_t = ((size_t)n + 255) & ~(size_t)255;
  const size_t need = nb_t + tb::pm_workspace_bytes(n);
  void* ws = nullptr;
  r = get_ws(stream, 7, need, &ws);
  if (r) return r;
  uint8_t* tags = (uint8_t*)ws;
  cudaError_t e = tb::classify_bytes_launch(d_bytes, n, h_class_map, tags, (cudaStream_t)stream);
  if (e == cudaSuccess)
    e = tb::pm_launch(tags, n, d_match, d_parent, (char*)ws + nb_t, nullptr, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "paren_match_bytes launch");
  return TB_OK;
}

int tree_transform(const uint8_t* d_tags, const float* d_local, const int32_t* d_match, const int32_t* d_parent,
                   int64_t n, float* d_world, void* stream) {
  g_err[0] = 0;
  int r = check_n(n);
  if (r || n == 0) return r;
  if (!d_tags || !d_local || !d_match || !d_parent || !d_world) return fail(TB_ERR_ARG, "null pointer with n > 0");
  if (!aligned16(d_tags) || !aligned16(d_local) || !aligned16(d_match) || !aligned16(d_parent) ||
      !aligned16(d_world))
    return fail(TB_ERR_ALIGN, "tags, local, match, parent and world must be 16-byte aligned");
  const size_t nb = (size_t)n * 24, n4 = (size_t)n * 4;
  if (overlap(d_world, nb, d_local, nb) || overlap(d_world, nb, d_tags, (size_t)n) ||
      overlap(d_world, nb, d_match, n4) || overlap(d_world, nb, d_parent, n4))
    return fail(TB_ERR_ALIAS, "world overlaps an input");
  void* ws = nullptr;
  r = get_ws(stream, 8, tb::tt_workspace_bytes(n), &ws);
  if (r) return r;
  cudaError_t e = tb::tt_launch(d_tags, d_local, d_match, d_parent, n, d_world, ws, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "tree_transform launch");
  return TB_OK;
}

int tree_fold(const uint8_t* d_tags, const uint32_t* d_x, const int32_t* d_match, int64_t n, uint32_t* d_out,
              void* stream) {
  g_err[0] = 0;
  int r = check_n(n);
  if (r || n == 0) return r;
  if (!d_tags || !d_x || !d_match || !d_out) return fail(TB_ERR_ARG, "null pointer with n > 0");
  if (!aligned16(d_tags) || !aligned16(d_x) || !aligned16(d_match) || !aligned16(d_out))
    return fail(TB_ERR_ALIGN, "tags, x, match and out must be 16-byte aligned");
  const size_t nb = (size_t)n * 16, n4 = (size_t)n * 4;
  if (overlap(d_out, nb, d_x, nb) || overlap(d_out, nb, d_tags, (size_t)n) || overlap(d_out, nb, d_match, n4))
    return fail(TB_ERR_ALIAS, "out overlaps an input");
  void* ws = nullptr;
  r = get_ws(stream, 12, tb::tf_workspace_bytes(n), &ws);
  if (r) return r;
  cudaError_t e = tb::tf_launch(d_tags, d_x, d_match, n, d_out, ws, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "tree_fold launch");
  return TB_OK;
}

int bin_leaves(const uint8_t* d_tags, const float* d_node_bbox, int64_t n, int grid_w, int grid_h, float bin_size,
               int32_t* d_counts, int32_t* d_offsets, int32_t* d_items, int64_t capacity, int64_t* h_total,
               void* stream) {
  g_err[0] = 0;
  int r = check_n(n);
  if (r) return r;
  if (grid_w <= 0 || grid_h <= 0 || (int64_t)grid_w * grid_h > (1 << 26) || !(bin_size > 0.f))
    return fail(TB_ERR_ARG, "bad bin grid");
  if (!d_counts || !d_offsets || !h_total || (n > 0 && (!d_tags || !d_node_bbox)) || (capacity > 0 && !d_items))
    return fail(TB_ERR_ARG, "null pointer");
  if (n > 0 && !aligned16(d_node_bbox)) return fail(TB_ERR_ALIGN, "node_bbox must be 16-byte aligned");
  void* ws = nullptr;
  r = get_ws(stream, 9, tb::bins_workspace_bytes(grid_w * grid_h), &ws);
  if (r) return r;
  cudaError_t e = tb::bins_launch(d_tags, d_node_bbox, n, grid_w, grid_h, bin_size, d_counts, d_offsets,
                                  (int32_t*)ws, d_items, capacity, h_total, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "bin_leaves");
  return TB_OK;
}

int compact_scene(const uint8_t* d_tags, const float* d_boxes, int64_t n, const uint8_t* h_keep_map,
                  uint8_t* d_tags_out, float* d_boxes_out, int32_t* d_index_out, int64_t* h_n_out, void* stream) {
  g_err[0] = 0;
  int r = check_n(n);
  if (r) return r;
  if (!h_keep_map || !h_n_out) return fail(TB_ERR_ARG, "null pointer");
  if (n > 0 && (!d_tags || !d_tags_out || !d_index_out || (d_boxes && !d_boxes_out)))
    return fail(TB_ERR_ARG, "null pointer with n > 0");
  if (n > 0 && (!aligned16(d_tags) || (d_boxes && (!aligned16(d_boxes) || !aligned16(d_boxes_out)))))
    return fail(TB_ERR_ALIGN, "tags and boxes must be 16-byte aligned");
  void* ws = nullptr;
  r = get_ws(stream, 10, tb::compact_workspace_bytes(n), &ws);
  if (r) return r;
  cudaError_t e = tb::compact_launch(d_tags, d_boxes, n, h_keep_map, d_tags_out, d_boxes_out, d_index_out, h_n_out,
                                     ws, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "compact_scene");
  return TB_OK;
}

int paren_match_tree_bbox_scene(const uint8_t* d_scene, const float* d_boxes, int64_t n, const uint8_t* h_keep_map,
                                uint8_t* d_tags_out, int32_t* d_index_out, int32_t* d_match, int32_t* d_parent,
                                float* d_node_bbox, int64_t* d_n_out, void* stream) {
  g_err[0] = 0;
  int r = check_n(n);
  if (r) return r;
  if (!h_keep_map || !d_n_out) return fail(TB_ERR_ARG, "null pointer");
  if (n > 0 && (!d_scene || !d_boxes || !d_tags_out || !d_index_out || !d_node_bbox || !d_match != !d_parent))
    return fail(TB_ERR_ARG, "null pointer with n > 0");
  if (n > 0 && (!aligned16(d_scene) || !aligned16(d_boxes) || !aligned16(d_node_bbox) ||
                (d_match && (!aligned16(d_match) || !aligned16(d_parent)))))
    return fail(TB_ERR_ALIGN, "scene, boxes, node_bbox, match and parent must be 16-byte aligned");
  const size_t nb = (size_t)n * 16, n4 = (size_t)n * 4;
  if (overlap(d_node_bbox, nb, d_boxes, nb) || overlap(d_node_bbox, nb, d_scene, (size_t)n) ||
      overlap(d_tags_out, (size_t)n, d_scene, (size_t)n) || overlap(d_index_out, n4, d_boxes, nb) ||
      (d_match && (overlap(d_match, n4, d_boxes, nb) || overlap(d_parent, n4, d_boxes, nb) ||
                   overlap(d_match, n4, d_parent, n4))))
    return fail(TB_ERR_ALIAS, "an output overlaps an input or another output");
  void* ws = nullptr;
  r = get_ws(stream, 13, n > 0 ? tb::fused_workspace_bytes(n) : 256, &ws);
  if (r) return r;
  cudaError_t e = tb::fused_scene_launch(d_scene, d_boxes, n, h_keep_map, d_tags_out, d_index_out, d_match, d_parent,
                                         d_node_bbox, d_n_out, ws, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "paren_match_tree_bbox_scene launch");
  return TB_OK;
}

/* Debug (not in the public header): tree_bbox with per-tile phase timestamps
 * (globaltimer ns) of the finish pass in d_trace[tile * 16 + slot]. */
int tb_debug_bb_tile(void) { return tb::bbm_tile_elems(); }

int tb_debug_fz_tma(int on) { return tb::fused_set_tma(on); }

/* Debug: cap the fused control kernel's blocks at g (0 = the co-resident count); returns the old cap.
 * Few blocks make long chunks: more than 1024 tiles per block takes the global owner-search path. */
int tb_debug_fz_ctrl_blocks(int g) { return tb::fused_set_ctrl_blocks(g); }

/* Debug: fz_ctrl phase timestamps (globaltimer ns, block 0) into dev_buf[0..10] (16 int64 slots); NULL turns it off. */
int tb_debug_fz_trace(void* dev_buf) {
  tb::fused_set_trace((uint64_t*)dev_buf);
  return 0;
}

int tb_debug_use_fused(int on) {
  const int old = g_use_fused;
  if (on >= 0) g_use_fused = on ? 1 : 0;
  return old;
}

/* Debug: capacity of bin_leaves' list of binned leaves (returns the previous
 * one); tests lower it to reach the streaming fill. */
int64_t tb_debug_bins_cap(int64_t cap) { return tb::bins_debug_cap(cap); }

/* Debug: minimum chunk size (log2 elements) of the pipelined host path;
 * returns the previous value (tests use small chunks on small inputs). */
int tb_debug_host_chunk_shift(int shift) {
  const int old = g_chunk_shift;
  if (shift >= 10 && shift <= 40) g_chunk_shift = shift;
  return old;
}

int tb_debug_tree_bbox_trace(const uint8_t* d_tags, const float* d_leaf_bbox, int64_t n, float* d_node_bbox,
                             uint64_t* d_trace, void* stream) {
  g_err[0] = 0;
  int r = bb_checks(d_tags, d_leaf_bbox, n, d_node_bbox);
  if (r || n == 0) return r;
  void* ws = nullptr;
  const size_t need = tree_bbox_workspace_bytes(n);
  r = get_ws(stream, 3, need, &ws);
  if (r) return r;
  return tree_bbox_ws_impl(d_tags, d_leaf_bbox, n, d_node_bbox, ws, need, stream, d_trace);
}

/* ---- sharding ------------------------------------------------------------ */

int tb_get_unique_id(uint8_t* out) {
  g_err[0] = 0;
  if (!out) return fail(TB_ERR_ARG, "null pointer");
#ifdef TB_WITH_NCCL
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(TB_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  static_assert(sizeof(id) == TB_UNIQUE_ID_BYTES, "NCCL unique id size");
  memcpy(out, &id, sizeof(id));
  return TB_OK;
#else
  return fail(TB_ERR_NCCL, "built without NCCL");
#endif
}

int tb_comm_init(const uint8_t* id, int nranks, int rank, void** comm) {
  g_err[0] = 0;
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return fail(TB_ERR_ARG, "bad communicator arguments");
#ifdef TB_WITH_NCCL
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclCommInitRank(&c, nranks, uid, rank);
  if (r != ncclSuccess) return fail(TB_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  *comm = c;
  return TB_OK;
#else
  return fail(TB_ERR_NCCL, "built without NCCL");
#endif
}

int tb_comm_destroy(void* comm) {
  g_err[0] = 0;
#ifdef TB_WITH_NCCL
  if (comm) ncclCommDestroy((ncclComm_t)comm);
  return TB_OK;
#else
  return fail(TB_ERR_NCCL, "built without NCCL");
#endif
}

int paren_match_shard(const uint8_t* d_tags, int64_t n_local, int64_t offset, int32_t* d_match, int32_t* d_parent,
                      void* comm, void* stream) {
  g_err[0] = 0;
  int r = pm_checks(d_tags, n_local, d_match, d_parent);
  if (r) return r;
  if (offset < 0 || offset + n_local > kMaxN) return fail(TB_ERR_ARG, "offset + n_local out of range");
  if (!comm) return fail(TB_ERR_ARG, "null communicator");
#ifdef TB_WITH_NCCL
  // the sharded fused pass without boxes (two fixed-size all-gathers); its
  // capacity from the largest chunk (an all-reduce), then the status check
  int nranks = 0;
  if (ncclCommCount((ncclComm_t)comm, &nranks) != ncclSuccess) return fail(TB_ERR_NCCL, "ncclCommCount");
  if (nranks > 256) return fail(TB_ERR_ARG, "paren_match_shard supports at most 256 ranks");
  void* nmx = nullptr;
  r = get_ws(stream, 11, 256, &nmx);
  if (r) return r;
  int64_t nl = n_local;
  cudaError_t e = cudaMemcpyAsync(nmx, &nl, sizeof nl, cudaMemcpyHostToDevice, (cudaStream_t)stream);
  if (e == cudaSuccess &&
      ncclAllReduce(nmx, nmx, 1, ncclInt64, ncclMax, (ncclComm_t)comm, (cudaStream_t)stream) != ncclSuccess)
    return fail(TB_ERR_NCCL, "ncclAllReduce");
  if (e == cudaSuccess) e = cudaMemcpyAsync(&nl, nmx, sizeof nl, cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "paren_match_shard");
  int nerr = 0;
  e = tb::fz_nccl_shard(d_tags, nullptr, n_local, offset, (int)tb_shard_default_cap(nl), d_match, d_parent, nullptr,
                        (ncclComm_t)comm, (cudaStream_t)stream, &nerr);
  if (nerr) return fail(TB_ERR_NCCL, "NCCL error");
  if (e != cudaSuccess) return cuda_fail(e, "paren_match_shard");
  return tb_shard_status(stream);
#else
  return fail(TB_ERR_NCCL, "built without NCCL");
#endif
}

int tree_bbox_shard(const uint8_t* d_tags, const float* d_leaf_bbox, int64_t n_local, int64_t offset,
                    float* d_node_bbox, void* comm, void* stream) {
  g_err[0] = 0;
  int r = bb_checks(d_tags, d_leaf_bbox, n_local, d_node_bbox);
  if (r) return r;
  if (offset < 0 || offset + n_local > kMaxN) return fail(TB_ERR_ARG, "offset + n_local out of range");
  if (!comm) return fail(TB_ERR_ARG, "null communicator");
#ifdef TB_WITH_NCCL
  // the fused protocol without match / parent, checked; its capacity must be
  // equal on every rank: the default for the largest chunk (an all-reduce)
  int nranks = 0;
  if (ncclCommCount((ncclComm_t)comm, &nranks) != ncclSuccess) return fail(TB_ERR_NCCL, "ncclCommCount");
  if (nranks > 256) return fail(TB_ERR_ARG, "tree_bbox_shard supports at most 256 ranks");
  void* nmx = nullptr;
  r = get_ws(stream, 11, 256, &nmx);
  if (r) return r;
  int64_t nl = n_local;
  cudaError_t e = cudaMemcpyAsync(nmx, &nl, sizeof nl, cudaMemcpyHostToDevice, (cudaStream_t)stream);
  if (e == cudaSuccess &&
      ncclAllReduce(nmx, nmx, 1, ncclInt64, ncclMax, (ncclComm_t)comm, (cudaStream_t)stream) != ncclSuccess)
    return fail(TB_ERR_NCCL, "ncclAllReduce");
  if (e == cudaSuccess) e = cudaMemcpyAsync(&nl, nmx, sizeof nl, cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "tree_bbox_shard");
  int nerr = 0;
  e = tb::fz_nccl_shard(d_tags, d_leaf_bbox, n_local, offset, (int)tb_shard_default_cap(nl), nullptr, nullptr,
                        d_node_bbox, (ncclComm_t)comm, (cudaStream_t)stream, &nerr);
  if (nerr) return fail(TB_ERR_NCCL, "NCCL error");
  if (e != cudaSuccess) return cuda_fail(e, "tree_bbox_shard");
  return tb_shard_status(stream);
#else
  return fail(TB_ERR_NCCL, "built without NCCL");
#endif
}

int64_t tb_shard_default_cap(int64_t n_local) {
  if (n_local < 0) n_local = 0;
  int64_t r = (int64_t)std::sqrt((double)n_local);
  while (r * r < n_local) r++;
  return std::min<int64_t>(4 * r + 4096, n_local + 2);
}

int paren_match_tree_bbox_shard(const uint8_t* d_tags, const float* d_leaf_bbox, int64_t n_local, int64_t offset,
                                int64_t cap, int32_t* d_match, int32_t* d_parent, float* d_node_bbox, void* comm,
                                void* stream) {
  g_err[0] = 0;
  int r = pm_checks(d_tags, n_local, d_match, d_parent);
  if (r) return r;
  r = bbm_checks(d_tags, d_leaf_bbox, d_match, d_parent, n_local, d_node_bbox);
  if (r) return r;
  const size_t nb = (size_t)n_local * 16, n4 = (size_t)n_local * 4;
  if (overlap(d_match, n4, d_leaf_bbox, nb) || overlap(d_parent, n4, d_leaf_bbox, nb))
    return fail(TB_ERR_ALIAS, "match / parent overlap leaf_bbox");
  if (offset < 0 || offset + n_local > kMaxN) return fail(TB_ERR_ARG, "offset + n_local out of range");
  if (cap < 1 || cap > kMaxN) return fail(TB_ERR_ARG, "cap out of range");
  if (!comm) return fail(TB_ERR_ARG, "null communicator");
#ifdef TB_WITH_NCCL
  int nranks = 0;
  if (ncclCommCount((ncclComm_t)comm, &nranks) != ncclSuccess) return fail(TB_ERR_NCCL, "ncclCommCount");
  if (nranks > 256) return fail(TB_ERR_ARG, "paren_match_tree_bbox_shard supports at most 256 ranks");
  int nerr = 0;
  cudaError_t e = tb::fz_nccl_shard(d_tags, d_leaf_bbox, n_local, offset, (int)cap, d_match, d_parent, d_node_bbox,
                                    (ncclComm_t)comm, (cudaStream_t)stream, &nerr);
  if (nerr) return fail(TB_ERR_NCCL, "NCCL error (ncclAllGather / ncclCommGetAsyncError)");
  if (e != cudaSuccess) return cuda_fail(e, "paren_match_tree_bbox_shard");
  return TB_OK;
#else
  return fail(TB_ERR_NCCL, "built without NCCL");
#endif
}

int tb_shard_status(void* stream) {
  g_err[0] = 0;
  int ovf = 0;
  cudaError_t e = tb::fz_shard_status((cudaStream_t)stream, &ovf);
  if (e != cudaSuccess) return cuda_fail(e, "tb_shard_status");
  if (ovf) return fail(TB_ERR_CAPACITY, "a chunk's Bic value exceeds the sharded call's capacity (a + 1 or b > cap)");
  return TB_OK;
}

int tb_debug_pair_vshard(const uint8_t* d_tags, const float* d_leaf_bbox, int64_t n, int nshards, int64_t cap,
                         int32_t* d_match, int32_t* d_parent, float* d_node_bbox, void* stream) {
  g_err[0] = 0;
  int r = 0;
  if (d_leaf_bbox || d_node_bbox) {
    r = bb_checks(d_tags, d_leaf_bbox, n, d_node_bbox);
    if (r || n == 0) return r;
  } else if (!d_match) {
    return fail(TB_ERR_ARG, "no outputs");
  }
  if (d_match || d_parent) {
    r = pm_checks(d_tags, n, d_match, d_parent);
    if (r || n == 0) return r;
  }
  if (nshards < 1 || nshards > 256) return fail(TB_ERR_ARG, "bad shard count");
  if (cap < 1 || cap > kMaxN) return fail(TB_ERR_ARG, "cap out of range");
  int ovf = 0;
  cudaError_t e = tb::fz_vshard(d_tags, d_leaf_bbox, n, nshards, (int)cap, d_match, d_parent, d_node_bbox,
                                (cudaStream_t)stream, &ovf);
  if (e != cudaSuccess) return cuda_fail(e, "pair vshard");
  if (ovf) return fail(TB_ERR_CAPACITY, "a chunk's Bic value exceeds cap");
  return TB_OK;
}

int tree_bbox_matched_shard(const uint8_t* d_tags, const float* d_leaf_bbox, const int32_t* d_match,
                            const int32_t* d_parent, int64_t n_local, int64_t offset, float* d_node_bbox, void* comm,
                            void* stream) {
  g_err[0] = 0;
  int r = bbm_checks(d_tags, d_leaf_bbox, d_match, d_parent, n_local, d_node_bbox);
  if (r) return r;
  if (offset < 0 || offset + n_local > kMaxN) return fail(TB_ERR_ARG, "offset + n_local out of range");
  if (!comm) return fail(TB_ERR_ARG, "null communicator");
#ifdef TB_WITH_NCCL
  int nranks = 0;
  if (ncclCommCount((ncclComm_t)comm, &nranks) != ncclSuccess) return fail(TB_ERR_NCCL, "ncclCommCount");
  if (nranks > 64) return fail(TB_ERR_ARG, "tree_bbox_matched_shard supports at most 64 ranks");
  int nerr = 0;
  cudaError_t e = tb::bbm_nccl_shard(d_tags, d_leaf_bbox, d_match, d_parent, n_local, offset, d_node_bbox,
                                     (ncclComm_t)comm, (cudaStream_t)stream, &nerr);
  if (nerr) return fail(TB_ERR_NCCL, "NCCL error %d", nerr);
  if (e != cudaSuccess) return cuda_fail(e, "tree_bbox_matched_shard");
  return TB_OK;
#else
  return fail(TB_ERR_NCCL, "built without NCCL");
#endif
}

int tb_debug_tree_bbox_vshard(const uint8_t* d_tags, const float* d_leaf_bbox, int64_t n, int nshards,
                              float* d_node_bbox, void* stream) {
  g_err[0] = 0;
  int r = bb_checks(d_tags, d_leaf_bbox, n, d_node_bbox);
  if (r || n == 0) return r;
  if (nshards < 1 || nshards > n || nshards > 64) return fail(TB_ERR_ARG, "bad shard count (1 .. min(n, 64))");
  cudaError_t e = tb::bb_vshard(d_tags, d_leaf_bbox, n, nshards, d_node_bbox, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "tree_bbox vshard");
  return TB_OK;
}

/* Debug / test (not in the public header): the shard protocol with G virtual
 * shards of one device buffer on one GPU; must equal paren_match. */
int tb_debug_paren_match_vshard(const uint8_t* d_tags, int64_t n, int nshards, int32_t* d_match, int32_t* d_parent,
                                void* stream) {
  g_err[0] = 0;
  int r = pm_checks(d_tags, n, d_match, d_parent);
  if (r || n == 0) return r;
  if (nshards < 1 || nshards > n) return fail(TB_ERR_ARG, "bad shard count");
  cudaError_t e = tb::pm_vshard(d_tags, n, nshards, d_match, d_parent, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "paren_match vshard");
  return TB_OK;
}

int tb_count_unmatched(const uint8_t* d_tags, int64_t n, int64_t* h_a, int64_t* h_b, void* stream) {
  g_err[0] = 0;
  int r = check_n(n);
  if (r) return r;
  if (!h_a || !h_b || (n > 0 && !d_tags)) return fail(TB_ERR_ARG, "null pointer");
  void* ws = nullptr;
  r = get_ws(stream, 2, tb::bic_count_workspace_bytes(n) + 256, &ws);
  if (r) return r;
  int64_t* d_out = (int64_t*)((char*)ws + tb::bic_count_workspace_bytes(n));
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = tb::bic_count_launch(d_tags, n, ws, d_out, s);
  if (e != cudaSuccess) return cuda_fail(e, "bic_count launch");
  int64_t h[2];
  e = cudaMemcpyAsync(h, d_out, sizeof h, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "bic_count readback");
  *h_a = h[0];
  *h_b = h[1];
  return TB_OK;
}

}  // extern "C"
