// Internal launch interface between the C ABI (api.cu) and the kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tb {

// Stack live before the first element of a (shard) launch: Bic prefix (a, h)
// and the entries at heights [lo, h) (global indices), device memory.
struct ShardInit {
  int a;
  int h;
  const int32_t* stack;
  int lo;
  int64_t offset;  // global index of the chunk's first element
  int2* pairs;     // paren_match: (open, close) for closes that pop stack entries
};

// One-time per-device setup (kernel attributes, occupancy-derived grid sizes):
// `slot` names the setup, the bit of the current device says it is done.
bool once_per_device(int slot);
int sm_count();  // SMs of the current device (grid sizing: multiples of it)

// Launch accounting / optional event timing around each kernel (prof.cu).
void prof_begin(cudaStream_t s, const char* name, void** token);
void prof_end(cudaStream_t s, void* token);
#define TB_LAUNCH(stream, name, ...)             \
  do {                                           \
    void* tb_tok_;                               \
    ::tb::prof_begin((stream), (name), &tb_tok_); \
    __VA_ARGS__;                                 \
    ::tb::prof_end((stream), tb_tok_);           \
  } while (0)

struct Ctrl;
// apre (optional, int64[ntiles + 1]): exclusive prefix sums of (a_T + 1), total last
cudaError_t tile_scan_launch(const Ctrl& c, int64_t ntiles, int init_a, int init_h, cudaStream_t stream,
                             int64_t* apre = nullptr);

size_t pm_workspace_bytes(int64_t n);
size_t pm_ctrl_bytes(int64_t n);
cudaError_t pm_launch(const uint8_t* tags, int64_t n, int32_t* match, int32_t* parent, void* ws,
                      const ShardInit* init, cudaStream_t stream);
cudaError_t pm_reduce_launch(const uint8_t* tags, int64_t n, int32_t* match, void* ws, const ShardInit* init,
                             cudaStream_t stream);
cudaError_t pm_reduce_only_launch(const uint8_t* tags, int64_t n, int32_t* match, void* ws, const ShardInit* init,
                                  cudaStream_t stream);
cudaError_t pm_rescan_launch(int64_t n, int32_t* match, void* ws, const ShardInit* init, cudaStream_t stream);
cudaError_t pm_finish_launch(const uint8_t* tags, int64_t n, int32_t* match, int32_t* parent, void* ws,
                             const ShardInit* init, cudaStream_t stream);
cudaError_t pm_summary_launch(const uint8_t* tags, int64_t n, void* ws, int32_t* hdr, int32_t* opens,
                              cudaStream_t stream);

// A close whose node was opened in an earlier chunk (shard mode): its global
// index, the open's global index and the union of this chunk's clipped leaves
// before the close.
struct ShardPop {
  float4 pre;
  int c, o, pad0, pad1;
};
// One open of a chunk's final stack: global index and a box (its chunk-local
// cumulative clip in exchange 1, the union of the chunk's leaves after it in
// exchange 2).
struct ShardOpen {
  float4 v;
  int idx, pad0, pad1, pad2;
};

// paren_match + tree_bbox in one tile pass (fused.cu): the single-device path.
// match / parent may be null (tree_bbox alone: only node_bbox is written).
size_t fused_workspace_bytes(int64_t n);
void fused_set_trace(uint64_t* dev);  // debug: fz_ctrl phase timestamps (8 x u64 device buffer) or null
int fused_set_tma(int on);
int fused_set_ctrl_blocks(int g);
// the fused pass over one chunk of a sharded stream (fused_shard.cuh): three
// phases around two fixed-size exchanges of slot1 / slot2 (cap: the largest
// Bic a + 1 and b of a chunk; equal on every rank)
size_t fused_shard_workspace_bytes(int64_t n, int cap, bool nobox);  // nobox: matching only (leaf_bbox null)
size_t fused_shard_slot1_bytes(int cap);
size_t fused_shard_slot2_bytes(int cap);
cudaError_t fused_shard_phase1(const uint8_t* tags, const float* leaf_bbox, int64_t n, int64_t goff, int cap,
                               int32_t* match, void* ws, void* slot1, cudaStream_t stream);
cudaError_t fused_shard_phase2(const uint8_t* tags, const float* leaf_bbox, int64_t n, int64_t goff, int cap, int G,
                               int g, int32_t* match, int32_t* parent, float* node_bbox, void* ws, const void* recv1,
                               void* slot2, cudaStream_t stream);
cudaError_t fused_shard_phase3(int64_t n, int64_t goff, int cap, int G, int g, int32_t* match, float* node_bbox,
                               void* ws, const void* recv1, const void* recv2, cudaStream_t stream);
int fused_shard_status(int64_t n, int cap, void* ws, cudaStream_t stream, cudaError_t* err);
int fused_tile_elems();
size_t fused_match_workspace_bytes(int64_t n);
cudaError_t fused_match_launch(const uint8_t* tags, int64_t n, int32_t* match, int32_t* parent, void* ws,
                               cudaStream_t stream);
cudaError_t fused_scene_launch(const uint8_t* tags, const float* boxes, int64_t n, const uint8_t* h_keep_map,
                               uint8_t* tags_out, int32_t* index_out, int32_t* match, int32_t* parent,
                               float* node_bbox, int64_t* d_n_out, void* ws, cudaStream_t stream);
cudaError_t fused_launch(const uint8_t* tags, const float* leaf_bbox, int64_t n, int32_t* match, int32_t* parent,
                         float* node_bbox, void* ws, cudaStream_t stream);

// tree_bbox from matching (tree_bbox_m.cu)
size_t bbm_workspace_bytes(int64_t n);
int bbm_tile_elems();
cudaError_t bbm_launch(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                       int64_t n, float* node_bbox, void* ws, cudaStream_t stream, uint64_t* trace = nullptr);
// bbm_launch in two parts: the reduce pass reads only tags and boxes (it can
// run while paren_match computes match / parent), the rest needs both.
cudaError_t bbm_launch_reduce(const uint8_t* tags, const float* leaf_bbox, int64_t n, float* node_bbox, void* ws,
                              cudaStream_t stream);
cudaError_t bbm_launch_rest(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                            int64_t n, float* node_bbox, void* ws, cudaStream_t stream, uint64_t* trace = nullptr);
// The same passes split over tile ranges in order (chunked host pipeline):
// bbm_begin once, bbm_tiles_launch for [t0, t1) as each range's boxes arrive
// (every pass reads only its own and earlier tiles), bbm_end (never-closed
// blend opens), then bbm_patch_host stores the entries written after their
// chunk was copied out (blend opens closed in a later chunk, never-closed
// ones) into the mapped host result.
int bbm_tiles(int64_t n);
cudaError_t bbm_begin(void* ws, int64_t n, cudaStream_t stream);
cudaError_t bbm_tiles_launch(const uint8_t* tags, const float* leaf_bbox, const int32_t* match,
                             const int32_t* parent, int64_t n, float* node_bbox, void* ws, int t0, int t1,
                             cudaStream_t stream);
cudaError_t bbm_end(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                    int64_t n, float* node_bbox, void* ws, cudaStream_t stream);
cudaError_t bbm_patch_host_launch(const uint8_t* tags, const int32_t* match, int64_t n, const float* node_bbox,
                                  void* ws, float* host_mapped, int chunk_tiles, cudaStream_t stream);

// Shard mode of the same kernels: match / parent hold global indices, the
// chunk's element 0 is global index `off`; contexts of earlier chunks' opens
// come from an imported table; closes of earlier chunks' nodes are reported.
struct BbmShard {
  int64_t off;
  const int32_t* ext_idx;  // ascending global indices
  const float4* ext_ctx;   // true contexts
  int n_ext;
  ShardPop* pops;
  uint32_t* npops;
};
cudaError_t bbm_shard_phase1(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                             int64_t n, int64_t off, float* node_bbox, void* ws, ShardOpen* fs, int** b_dev,
                             int* link_dev, cudaStream_t stream);
cudaError_t bbm_compose_launch(const int4* hdr, int G, int g, const ShardOpen* allfs, int maxb, int n_ext,
                               int32_t* ext_idx, float4* ext_ctx, cudaStream_t stream);
cudaError_t bbm_shard_phase2(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                             int64_t n, float* node_bbox, void* ws, const BbmShard* sh, cudaStream_t stream);
cudaError_t bbm_export_launch(const uint8_t* tags, const float* leaf_bbox, const int32_t* match,
                              const int32_t* parent, int64_t n, float* node_bbox, void* ws, const BbmShard* sh,
                              const ShardOpen* fs, int b, ShardOpen* suc, float4* tu, cudaStream_t stream);
cudaError_t bbm_fixup_launch(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                             int64_t n, float* node_bbox, void* ws, const BbmShard* sh, const int4* hdr, int G, int g,
                             const ShardOpen* allsuc, int maxb, const float4* alltu, const ShardPop* allpops,
                             const int* npops, int maxp, cudaStream_t stream);

cudaError_t bb_vshard(const uint8_t* tags, const float* leaf, int64_t n, int G, float* out, cudaStream_t s);
cudaError_t pm_vshard(const uint8_t* tags, int64_t n, int G, int32_t* match, int32_t* parent, cudaStream_t s);

// 2D affine transforms composed down the tree (tree_transform.cu)
size_t tt_workspace_bytes(int64_t n);
cudaError_t tt_launch(const uint8_t* tags, const float* local, const int32_t* match, const int32_t* parent,
                      int64_t n, float* world, void* ws, cudaStream_t stream);

// 2x2 matrices mod 2^32 multiplied up the tree (tree_fold.cu)
size_t tf_workspace_bytes(int64_t n);
cudaError_t tf_launch(const uint8_t* tags, const uint32_t* x, const int32_t* match, int64_t n, uint32_t* out,
                      void* ws, cudaStream_t stream);

// culling + binning of clipped leaf boxes (bins.cu); synchronises to read the total
size_t bins_workspace_bytes(int nb);
int64_t bins_debug_cap(int64_t cap);
cudaError_t bins_launch(const uint8_t* tags, const float* node_bbox, int64_t n, int gw, int gh, float bs,
                        int32_t* counts, int32_t* offsets, int32_t* cursor, int32_t* items, int64_t capacity,
                        int64_t* total, cudaStream_t stream);

// exclusive prefix sum of a small int32 array in one CTA: out[0..n) and out[n] = total
cudaError_t excl_scan_launch(const int* in, int n, int* out, const char* name, cudaStream_t stream);

// stream compaction front end (compact.cu); synchronises to read the count
size_t compact_workspace_bytes(int64_t n);
cudaError_t compact_launch(const uint8_t* tags, const float* boxes, int64_t n, const uint8_t* keep_map,
                           uint8_t* tags_out, float* boxes_out, int32_t* index_out, int64_t* n_out, void* ws,
                           cudaStream_t stream);

// raw bytes -> tag bytes through a 256-entry class map (host pointer)
cudaError_t classify_bytes_launch(const uint8_t* in, int64_t n, const uint8_t* class_map, uint8_t* out,
                                  cudaStream_t stream);

size_t bic_count_workspace_bytes(int64_t n);
cudaError_t bic_count_launch(const uint8_t* tags, int64_t n, void* ws, int64_t* d_out2,
                             cudaStream_t stream);

}  // namespace tb
