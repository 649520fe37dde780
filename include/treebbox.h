/*
 * treebbox.h — C ABI of the B200 (sm_100a) hot path of
 *   R. Levien, "Fast GPU bounding boxes on tree-structured scenes",
 *   arXiv 2205.11659.
 * Citations: P:n = PAPER.md line n (section in brackets); R<k> = reading k of
 * DESIGN.md §3 (points the paper leaves open).
 *
 * Input model (§1.1): a flattened tree, one byte per element:
 *     1 = open of a clip node, 2 = open of a blend node, 3 = close,
 *     every other byte value = leaf (R2).
 *
 * Conventions shared by every entry point
 *   - Pointers named d_* are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *     on the current CUDA device; h_* are HOST pointers.  All arrays are
 *     caller-owned; the library never frees them.  Inputs must stay alive and
 *     unmodified until `stream` has passed the call.
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *     Everything is enqueued on it; device entry points never synchronise the
 *     host.  Outputs are valid once the stream has reached the call.
 *   - Return value: 0 on success, otherwise a negative TB_ERR_* code; the
 *     message is available from tb_last_error() (thread-local).  Only
 *     host-checkable conditions are errors.  Data-dependent situations
 *     (unmatched closes, opens left open at the end) are NOT errors and have
 *     defined outputs (R3, R4).
 *   - n == 0 is a successful no-op.  n must be <= 2^31 - 1 (int32 indices,
 *     -1 sentinel; R5).
 *   - Alignment: d_tags, d_match, d_parent, d_leaf_bbox, d_node_bbox must be
 *     16-byte aligned (TB_ERR_ALIGN otherwise).  Outputs must not overlap
 *     inputs or each other (TB_ERR_ALIAS).
 *   - Workspace: the library keeps a per-(device, stream) scratch cache grown
 *     on demand (the growth itself synchronises the device once).  The *_ws
 *     variants take caller-provided scratch instead (no allocation; suitable
 *     for CUDA-graph capture); size it with *_workspace_bytes(n).
 *   - Results are deterministic and bit-identical to the sequential
 *     definitions (Fig. 1), whatever the tiling.
 *   - Threads: entry points may be called from several host threads at once
 *     on different streams (the library's side streams and events are used
 *     under a lock while enqueuing); calls on one stream are issued by one
 *     host thread at a time.
 */
#ifndef TREEBBOX_H
#define TREEBBOX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TB_OK 0
#define TB_ERR_ARG -1    /* n < 0, n > 2^31-1, null pointer with n > 0, bad size */
#define TB_ERR_ALIGN -2  /* a pointer is not 16-byte aligned */
#define TB_ERR_ALIAS -3  /* an output overlaps an input or another output */
#define TB_ERR_CUDA -4   /* CUDA launch / allocation / copy error */
#define TB_ERR_NCCL -5   /* NCCL error (sharded entry points) */
#define TB_ERR_CAPACITY -6 /* sharded call: a chunk's Bic value exceeds the fixed capacity (a + 1 or b > cap) */

/* Tag byte values (R2). */
#define TB_LEAF 0
#define TB_OPEN_CLIP 1
#define TB_OPEN_BLEND 2
#define TB_CLOSE 3

/* Message for the last nonzero return on this host thread ("" if none). */
const char *tb_last_error(void);

/* Library version string. */
const char *tb_version(void);

/* Free the library's cached device workspaces of the current device (the
 * per-(device, stream) caches of the calls below and the shard protocols'
 * arenas).  Synchronizes the device first; no call may be in flight on any
 * stream of it.  The next call re-allocates what it needs.  Returns 0 or
 * TB_ERR_CUDA. */
int tb_release_workspaces(void);

/* ------------------------------------------------------------------------
 * paren_match — parentheses matching (§2; §3; §4)
 *
 * d_tags   : device uint8[n], tag bytes as above.
 * d_parent : device int32[n] out.  parent[i] = Fig. 1's out[i]: the
 *            index of the innermost open enclosing element i, -1 at the root.
 *            For a matched close this is its matching open ("stronger
 *            version").
 * d_match  : device int32[n] out.  Classical partner: matched opens and
 *            closes point at each other; leaves, opens never closed (R4) and
 *            closes with nothing to close (R3) get -1.
 * Computation (the fused machinery without boxes, csrc/fused.cu): a reduce
 * pass over the tags (each 2048-element tile's value in the bicyclic monoid,
 * P:96-102, and its stack slice; the tile's surviving opens get
 * match -1), a cooperative control kernel (the scan of the tile values,
 * low-water marks and their 32-ary min hierarchy, link owners and incoming
 * runs) and the matching pass (in-tile resolution, cross-tile lookup by the
 * owner rule = the suffix relation; the closes of earlier tiles'
 * opens write those opens' match).  HBM traffic ~10 bytes/element (+ slices).
 * ------------------------------------------------------------------------ */
int paren_match(const uint8_t *d_tags, int64_t n, int32_t *d_match, int32_t *d_parent,
                void *stream);

size_t paren_match_workspace_bytes(int64_t n);
/* With caller workspace: round 1's three passes (a reduce over 4096-element
 * tiles, a one-CTA scan of the tile values, a finish pass; csrc/paren_match.cu),
 * same outputs.  d_workspace: device scratch of >= paren_match_workspace_bytes(n)
 * bytes, 256-byte aligned, not used concurrently by another call. */
int paren_match_ws(const uint8_t *d_tags, int64_t n, int32_t *d_match, int32_t *d_parent,
                   void *d_workspace, size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------
 * paren_match_bytes — parenthesis matching over raw text (SURVEY §8(f) NEXT
 * row 3; the parsing use of the method)
 *
 * d_bytes     : device uint8[n] text (16-byte aligned).
 * h_class_map : HOST uint8[256]; byte value -> tag class (1 or 2 = open,
 *               3 = close, anything else = leaf; e.g. '{' '[' -> 1,
 *               '}' ']' -> 3 for JSON brackets).  Read during the call.
 * d_match, d_parent: as paren_match, for the classified stream.  Brackets are
 * classified per byte (string literals and escapes are not special).
 * ------------------------------------------------------------------------ */
int paren_match_bytes(const uint8_t *d_bytes, int64_t n, const uint8_t *h_class_map, int32_t *d_match,
                      int32_t *d_parent, void *stream);

/* ------------------------------------------------------------------------
 * tree_bbox — clip intersections and blend unions (§6; §9)
 *
 * d_tags      : device uint8[n] as above.
 * d_leaf_bbox : device float32[n][4] (x0, y0, x1, y1).  Read for leaves and
 *               clip opens only (blend opens and closes are ignored, R7).
 * d_node_bbox : device float32[n][4] out:
 *     leaf          own box ∩ every clip node on its root path
 *     clip open     own box ∩ every clip ancestor (effective clip)   (R6)
 *     close         raw union of the clipped leaves strictly inside
 *                   the node, for clip and blend nodes alike          (R8, R10)
 *     blend open    the same union, scattered to the open
 *     unmatched     close -> EMPTY; an open never closed spans to the end (R3, R4)
 * INF = (-inf,-inf,+inf,+inf), EMPTY = (+inf,+inf,-inf,-inf) (R11).  min/max
 * order -0 below +0 and ignore NaN operands (R12; the measured semantics of
 * PTX min/max.f32), so results are unique bit patterns.  Boxes are never
 * canonicalised (R9).
 * The matching structure is re-derived inside the same tile pass that
 * computes the boxes (the fused pass of paren_match_tree_bbox, without its
 * match / parent stores): ~36 bytes/element of HBM traffic (+ slices).
 * ------------------------------------------------------------------------ */
int tree_bbox(const uint8_t *d_tags, const float *d_leaf_bbox, int64_t n, float *d_node_bbox,
              void *stream);

size_t tree_bbox_workspace_bytes(int64_t n);
int tree_bbox_ws(const uint8_t *d_tags, const float *d_leaf_bbox, int64_t n, float *d_node_bbox,
                 void *d_workspace, size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------
 * tree_bbox_matched — the same boxes from a matching already computed
 *
 * d_match, d_parent: device int32[n], exactly paren_match's outputs for
 * d_tags (16-byte aligned; not checked for consistency — other values give
 * undefined node_bbox but never out-of-bounds accesses only if they are
 * paren_match's).  With the parent of every element known, an element's clip is
 * box ∩ clip(parent) and a node's union is the union of the clipped
 * leaves strictly between its open and its close; both are
 * evaluated per tile with the cross-tile parts taken from the tiles' slices
 * (tile-unmatched opens) and a hierarchy of tile unions.
 * ------------------------------------------------------------------------ */
int tree_bbox_matched(const uint8_t *d_tags, const float *d_leaf_bbox, const int32_t *d_match,
                      const int32_t *d_parent, int64_t n, float *d_node_bbox, void *stream);
size_t tree_bbox_matched_workspace_bytes(int64_t n);
int tree_bbox_matched_ws(const uint8_t *d_tags, const float *d_leaf_bbox, const int32_t *d_match,
                         const int32_t *d_parent, int64_t n, float *d_node_bbox, void *d_workspace,
                         size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------
 * paren_match_tree_bbox — the whole hot path in one device call: d_match and
 * d_parent as paren_match, d_node_bbox as tree_bbox_matched on them (same
 * arguments, layouts and error codes as those two; match / parent must not
 * overlap leaf_bbox either).  One fused tile pass (csrc/fused.cu): a reduce
 * pass (tile Bic values and slices with their clips), a
 * cooperative control kernel (tile scan, link owners, tile contexts), the
 * main pass (matching, clips and unions of each 2048-element tile; tags and
 * boxes read once, match / parent / node_bbox written once) and a close pass
 * for nodes that span tiles.  Stream-ordered on `stream`; capturable in a
 * CUDA graph.
 * ------------------------------------------------------------------------ */
int paren_match_tree_bbox(const uint8_t *d_tags, const float *d_leaf_bbox, int64_t n, int32_t *d_match,
                          int32_t *d_parent, float *d_node_bbox, void *stream);

/* ------------------------------------------------------------------------
 * tree_transform — a generic monoid payload down the tree (SURVEY §8(f) NEXT
 * row 2; "it can compute any monoid"): 2D affine transforms,
 * composition being neither commutative nor idempotent (reading R15).
 *
 * d_local : device float32[n][6] (a, b, c, d, tx, ty): p -> [[a,b],[c,d]] p + t.
 *           Read for leaves and opens (clip and blend alike); ignored for closes.
 * d_match, d_parent: paren_match's outputs for d_tags.
 * d_world : device float32[n][6] out: leaf / open: world(enclosing open) ∘ local
 *           (root: identity); close: the world of the node it closes;
 *           unmatched close: identity.  fp32 with fused multiply-adds; the
 *           association order differs from the sequential walk, so results
 *           match it exactly only when every product is exact (DESIGN R15).
 * All device pointers 16-byte aligned; world must not overlap an input.
 * ------------------------------------------------------------------------ */
int tree_transform(const uint8_t *d_tags, const float *d_local, const int32_t *d_match, const int32_t *d_parent,
                   int64_t n, float *d_world, void *stream);

/* ------------------------------------------------------------------------
 * tree_fold — a generic monoid payload UP the tree (SURVEY §8(f) NEXT row 2,
 * the "up" half: blends are upward flow; unions run in reverse, P:298;
 * "any monoid"; reading R17).
 *
 * d_x     : device uint32[n][4], a 2x2 matrix (a, b, c, d) = [[a, b], [c, d]]
 *           per element; products are taken mod 2^32 (exactly associative,
 *           neither commutative nor idempotent).  Read for leaves only.
 * d_match : paren_match's match for d_tags.
 * d_out   : device uint32[n][4] out: a node's value — the product, in stream
 *           order, of the payloads of the leaves strictly between its open and
 *           its close — at its open and its close; an open never closed: the
 *           leaves after it to the stream end (R4); a leaf: its own payload; an
 *           unmatched close: the identity (R3).  Bit-exact at any size.
 * All device pointers 16-byte aligned; out must not overlap an input.
 * ------------------------------------------------------------------------ */
int tree_fold(const uint8_t *d_tags, const uint32_t *d_x, const int32_t *d_match, int64_t n, uint32_t *d_out,
              void *stream);

/* ------------------------------------------------------------------------
 * bin_leaves — culling and binning of the clipped leaf boxes (SURVEY §8(f)
 * NEXT row 4; "input to visibility culling and binning"; R16)
 *
 * d_node_bbox : tree_bbox's output (device float32[n][4], 16-byte aligned).
 * A leaf whose box is non-empty (x0 < x1, y0 < y1) and overlaps the viewport
 * [0, grid_w*bin_size) x [0, grid_h*bin_size) is listed in every bin (bx, by)
 * whose square [bx*bin_size, (bx+1)*bin_size) x [...] overlaps its box.
 * d_counts  : device int32[grid_w*grid_h] out (bin index = by*grid_w + bx).
 * d_offsets : device int32[grid_w*grid_h + 1] out, exclusive prefix of counts.
 * d_items   : device int32[capacity] out: leaf indices, bin after bin; the
 *             order inside a bin is unspecified.  Filled only if the total
 *             fits in capacity.
 * *h_total  : HOST out, the number of (bin, leaf) items.  The call synchronises
 * `stream` (the total is read on the host).
 * ------------------------------------------------------------------------ */
int bin_leaves(const uint8_t *d_tags, const float *d_node_bbox, int64_t n, int grid_w, int grid_h, float bin_size,
               int32_t *d_counts, int32_t *d_offsets, int32_t *d_items, int64_t capacity, int64_t *h_total,
               void *stream);

/* ------------------------------------------------------------------------
 * compact_scene — stream compaction front end (the
 * step upstream of the path)
 *
 * d_tags      : device uint8[n] full scene stream (16-byte aligned).
 * d_boxes     : device float32[n][4] or NULL (then no boxes are moved).
 * h_keep_map  : HOST uint8[256]: nonzero = keep elements with that byte value.
 * d_tags_out, d_boxes_out, d_index_out: device [n] out (capacity n); the kept
 *               elements in stream order, their boxes, their index in the
 *               full stream.
 * *h_n_out    : HOST out, the number kept.  The call synchronises `stream`.
 * ------------------------------------------------------------------------ */
/* ------------------------------------------------------------------------
 * paren_match_tree_bbox_scene — stream compaction fused into the hot path's
 * tile loader: the FULL scene stream in,
 * the bench step's outputs for its kept elements out, with no compaction
 * pass over HBM.  Elements whose byte has h_keep_map[byte] == 0 are dropped:
 * null for the matching and the boxes (no Bic, no box, no output).  Kept
 * element k (k-th in stream order) gets:
 *   d_tags_out[k], d_index_out[k] (its index in the full stream),
 *   d_match[k], d_parent[k] (compacted indices, as paren_match on the
 *   compacted stream), d_node_bbox[k] (as tree_bbox on the compacted stream);
 * *d_n_out (device int64) = the kept count.  Capacity n for every output.
 * d_match and d_parent may both be null (boxes only).  Stream-ordered; no
 * host synchronisation.  Same results as compact_scene followed by
 * paren_match_tree_bbox on its output, bit for bit.
 * ------------------------------------------------------------------------ */
int paren_match_tree_bbox_scene(const uint8_t *d_scene, const float *d_boxes, int64_t n, const uint8_t *h_keep_map,
                                uint8_t *d_tags_out, int32_t *d_index_out, int32_t *d_match, int32_t *d_parent,
                                float *d_node_bbox, int64_t *d_n_out, void *stream);
int compact_scene(const uint8_t *d_tags, const float *d_boxes, int64_t n, const uint8_t *h_keep_map,
                  uint8_t *d_tags_out, float *d_boxes_out, int32_t *d_index_out, int64_t *h_n_out, void *stream);

/* ------------------------------------------------------------------------
 * Host-buffer variants (end-to-end API): h_* are host pointers (pinned or
 * pageable).  Inputs are copied to library-owned device buffers on `stream`,
 * the device call runs, outputs are copied back, and the call synchronises
 * `stream` before returning.
 * ------------------------------------------------------------------------ */
int paren_match_host(const uint8_t *h_tags, int64_t n, int32_t *h_match, int32_t *h_parent,
                     void *stream);
int tree_bbox_host(const uint8_t *h_tags, const float *h_leaf_bbox, int64_t n, float *h_node_bbox,
                   void *stream);
/* The whole hot path from host buffers: copy tags and boxes in, paren_match,
 * tree_bbox_matched on its outputs, copy match, parent and node_bbox out.  The
 * box upload and the match/parent download run on library side streams,
 * overlapped with the kernels (pass pinned host memory for real overlap).
 * When h_node_bbox is pinned (device-mapped under unified addressing) the box
 * passes run in up to 16 chunks of tiles as the boxes arrive (each pass reads
 * only its own and earlier tiles, §6 P:192-221 clips top-down, unions of
 * closed nodes), each chunk's node_bbox is copied out while later chunks
 * compute, and the few entries finished later (blend opens closed in a later
 * chunk or never, R4) are then stored into h_node_bbox by a kernel through
 * the mapping.  Same results as the unchunked path, bit for bit. */
int paren_match_tree_bbox_host(const uint8_t *h_tags, const float *h_leaf_bbox, int64_t n, int32_t *h_match,
                               int32_t *h_parent, float *h_node_bbox, void *stream);

/* ------------------------------------------------------------------------
 * Multi-GPU sharding: one process per GPU, the global stream
 * split into contiguous chunks in rank order.  Each rank passes its chunk:
 * d_tags / d_match / d_parent hold n_local elements whose global indices are
 * [offset, offset + n_local); outputs hold GLOBAL indices and are identical
 * to the single-GPU call on the whole stream.  The chunks are summarised by
 * their Bic value and unmatched-open list (§3-§4), exchanged with
 * NCCL all-gathers on `comm`, and each rank finishes locally; a close whose
 * open lies in an earlier chunk is reported to that chunk in a second small
 * all-gather.  `comm` is an ncclComm_t (from tb_comm_init).  Collective: all
 * ranks must call with their chunks.  paren_match_tree_bbox_shard (the bench
 * step) enqueues two fixed-size all-gathers and does not synchronise;
 * paren_match_shard and tree_bbox_shard run the same protocol (matching alone
 * / boxes alone) with a capacity from the largest chunk (an all-reduce) and
 * check it, so they synchronise `stream`; tree_bbox_matched_shard (round 1's
 * protocol, at most 64 ranks) synchronises too.
 * ------------------------------------------------------------------------ */
#define TB_UNIQUE_ID_BYTES 128
/* Rank 0 creates an id; broadcast its 128 bytes to the other ranks. */
int tb_get_unique_id(uint8_t *out);
/* Create / destroy the library's NCCL communicator (*comm = ncclComm_t). */
int tb_comm_init(const uint8_t *id, int nranks, int rank, void **comm);
int tb_comm_destroy(void *comm);
int paren_match_shard(const uint8_t *d_tags, int64_t n_local, int64_t offset, int32_t *d_match,
                      int32_t *d_parent, void *comm, void *stream);
/* tree_bbox over contiguous chunks: d_leaf_bbox / d_node_bbox hold the chunk's
 * n_local boxes.  paren_match_tree_bbox_shard below without match / parent,
 * capacity tb_shard_default_cap of the largest chunk (an all-reduce over the
 * ranks), then tb_shard_status (synchronises `stream`; TB_ERR_CAPACITY when a
 * chunk is deeper than that capacity). */
int tree_bbox_shard(const uint8_t *d_tags, const float *d_leaf_bbox, int64_t n_local, int64_t offset,
                    float *d_node_bbox, void *comm, void *stream);
/* The bench step sharded: paren_match + tree_bbox of the fused one-device pass
 * (fused.cu) over contiguous chunks with TWO fixed-size NCCL all-gathers and no
 * host synchronisation (csrc/fused_shard.cuh):
 *   exchange 1: each chunk's Bic value (a, b) and its final stack
 *     (the b opens it leaves open, bottom to top: global index | blend << 31,
 *     context inside the chunk), cap entries per rank;
 *   exchange 2: each chunk's union, the union after each final-stack open to
 *     the chunk end, and the closes of earlier chunks' opens with this
 *     chunk's part of their union (cap entries per rank).
 * Every rank composes the top of its incoming stack from the headers (the
 * owner rule over chunks, F1) before its main pass and finishes the nodes
 * that span chunks after exchange 2.  `cap` must be equal on every rank and
 * bound every chunk's a + 1 and b (tb_shard_default_cap(n_local) = 4 sqrt(n)
 * + 4096 suits random streams; a deep stream needs up to n_local + 2).  The
 * call returns once the work is enqueued; an overflow of cap is detected on
 * the device (every rank sees the headers) and reported by tb_shard_status,
 * which waits for the stream: TB_ERR_CAPACITY, outputs undefined.
 * d_match / d_parent may both be null (tree_bbox alone). */
int64_t tb_shard_default_cap(int64_t n_local);
int paren_match_tree_bbox_shard(const uint8_t *d_tags, const float *d_leaf_bbox, int64_t n_local, int64_t offset,
                                int64_t cap, int32_t *d_match, int32_t *d_parent, float *d_node_bbox, void *comm,
                                void *stream);
/* TB_ERR_CAPACITY if the last paren_match_tree_bbox_shard call on `stream`
 * overflowed its capacity, else 0.  Synchronises `stream`. */
int tb_shard_status(void *stream);
/* The same from a matching already computed by paren_match_shard (d_match /
 * d_parent: the chunk's n_local entries, GLOBAL indices). */
int tree_bbox_matched_shard(const uint8_t *d_tags, const float *d_leaf_bbox, const int32_t *d_match,
                            const int32_t *d_parent, int64_t n_local, int64_t offset, float *d_node_bbox, void *comm,
                            void *stream);

/* ------------------------------------------------------------------------
 * Validation helper: the global Bic of the stream: a = closes with
 * nothing to close, b = opens left open at the end.  Synchronises `stream`.
 * ------------------------------------------------------------------------ */
int tb_count_unmatched(const uint8_t *d_tags, int64_t n, int64_t *h_a, int64_t *h_b, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TREEBBOX_H */
