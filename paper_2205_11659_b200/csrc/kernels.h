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
cudaError_t tile_scan_launch(const Ctrl& c, int64_t ntiles, int init_a, int init_h, cudaStream_t stream);

size_t pm_workspace_bytes(int64_t n);
size_t pm_ctrl_bytes(int64_t n);
cudaError_t pm_launch(const uint8_t* tags, int64_t n, int32_t* match, int32_t* parent, void* ws,
                      const ShardInit* init, cudaStream_t stream);
cudaError_t pm_reduce_launch(const uint8_t* tags, int64_t n, int32_t* match, void* ws, const ShardInit* init,
                             cudaStream_t stream);
cudaError_t pm_finish_launch(const uint8_t* tags, int64_t n, int32_t* match, int32_t* parent, void* ws,
                             const ShardInit* init, cudaStream_t stream);
cudaError_t pm_summary_launch(const uint8_t* tags, int64_t n, void* ws, int32_t* hdr, int32_t* opens,
                              cudaStream_t stream);

// tree_bbox from matching (tree_bbox_m.cu): the single-device path
size_t bbm_workspace_bytes(int64_t n);
int bbm_tile_elems();
cudaError_t bbm_launch(const uint8_t* tags, const float* leaf_bbox, const int32_t* match, const int32_t* parent,
                       int64_t n, float* node_bbox, void* ws, cudaStream_t stream, uint64_t* trace = nullptr);

// tree_bbox by stack slices (tree_bbox.cu): the shard path
size_t bb_workspace_bytes(int64_t n);
cudaError_t bb_launch(const uint8_t* tags, const float* leaf_bbox, int64_t n, float* node_bbox, void* ws,
                      cudaStream_t stream, uint64_t* trace = nullptr);

// tree_bbox shard mode: the stack live before the chunk, with true clips.
struct BbShard {
  int64_t offset;  // global index of the chunk's first element
  int H0;          // stack height at the chunk start
  int init_lo;     // entries provided for heights [init_lo, H0)
  const float4* init_clip;
  const int4* init_meta;  // {global index, kind, source chunk, slice position}
  void* pops;             // BbPop records of closes popping provided entries
};
int bb_tile_elems();
size_t bb_sumrec_bytes();
size_t bb_pop_bytes();
cudaError_t bb_reduce_launch(const uint8_t* tags, const float* leaf_bbox, int64_t n, void* ws, const BbShard* sh,
                             cudaStream_t stream);
cudaError_t bb_finish_launch(const uint8_t* tags, const float* leaf_bbox, int64_t n, float* node_bbox, void* ws,
                             const BbShard* sh, cudaStream_t stream, uint64_t* trace = nullptr);
cudaError_t bb_summary_launch(const uint8_t* tags, const float* leaf_bbox, int64_t n, void* ws, int32_t* hdr,
                              void* recs, int4* runs, cudaStream_t stream);
cudaError_t bb_export_launch(const uint8_t* tags, const float* leaf_bbox, int64_t n, void* ws, const void* recs,
                             int b, float4* suf_tiles, float4* out_tu, float4* out_su, cudaStream_t stream);
cudaError_t bb_compose_launch(const void* allrecs, int maxb, const int* L, int g, int lo, int H, float4* init_clip,
                              int4* init_meta, cudaStream_t stream);
cudaError_t bb_fixup_launch(int G, int g, int64_t off, int b_g, int min_L_after, int L_g, const float4* tu,
                            const float4* allsu, int maxb, const void* allpops, int maxp, const int* npops,
                            const void* myrecs, float4* out, cudaStream_t stream);

cudaError_t bb_vshard(const uint8_t* tags, const float* leaf, int64_t n, int G, float* out, cudaStream_t s);
cudaError_t pm_vshard(const uint8_t* tags, int64_t n, int G, int32_t* match, int32_t* parent, cudaStream_t s);

size_t bic_count_workspace_bytes(int64_t n);
cudaError_t bic_count_launch(const uint8_t* tags, int64_t n, void* ws, int64_t* d_out2,
                             cudaStream_t stream);

}  // namespace tb
