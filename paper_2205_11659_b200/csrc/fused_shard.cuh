// Sharded fused pass: one contiguous chunk of the global stream
// per rank, two fixed-capacity exchanges, no host synchronisation.
// Included by fused.cu (inside namespace tb).
//
// A chunk runs the one-device passes with its heights offset by h0 (= cap):
// heights 0 .. h0 - 1 are the top of the global stack at the chunk start (the
// "imported" entries, a virtual slice at slice reference vbase + h).  Nothing
// of a chunk depends on the imported entries until the main pass, so
//   phase 1  fz_reduce, fz_ctrl (TC chains that leave the chunk end at an
//            imported height, tcend); the chunk's final stack (its opens
//            closed after it or never) with their contexts inside the chunk
//            (lcc: slice lc ∩ the chunk-local TC)            -> slot 1
//   exchange 1 (all-gather of slot 1: Bic header, final stack)
//   phase 2  compose (every rank the same, from the headers): chunk start
//            heights H_k and low-water marks L_k (the Bic prefix over chunks,
//            P:96-102), the context below each chunk's final stack (TCc,
//            F1 over chunks), the imported entries of this chunk with their
//            true contexts (lcc ∩ TCc of the owning chunk) and TC's missing
//            factor; then fz_main / fz_hier / fz_close -- closes of imported
//            entries record (close, this chunk's part of the union); the
//            union after each final-stack open to the chunk end (su)
//                                                           -> slot 2
//   exchange 2 (all-gather of slot 2: chunk union, su, the recorded closes)
//   phase 3  fix-up: a node opened on chunk j and closed on chunk k gets
//            su_j ∪ (chunks j+1 .. k-1) ∪ k's part (R8-R9); blend opens take
//            it (R9), never-closed blend opens the union to the stream end (R4).
// A chunk whose Bic value has a + 1 > cap or b > cap overflows the fixed
// slots: every rank sees it in the headers and reports it (fused_shard_status).
namespace fz {

constexpr int GMAX = 256;  // chunks (ranks) of one sharded call

__host__ __device__ inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
// slot 1: [hdr int4 (a, b, overflow, 0)][lcc float4 * cap][idx int * cap]
__host__ __device__ inline size_t x1_bytes(int cap) { return al256(16 + 20 * (size_t)cap); }
// slot 2: [chunk union float4][su float4 * cap][exu float4 * cap][exc int * cap]
__host__ __device__ inline size_t x2_bytes(int cap) { return al256(16 + 36 * (size_t)cap); }

struct X1 {
  int4* hdr;
  float4* lcc;
  int32_t* idx;
};
__host__ __device__ inline X1 x1_view(char* slot, int cap) {
  return X1{(int4*)slot, (float4*)(slot + 16), (int32_t*)(slot + 16 + 16 * (size_t)cap)};
}
struct X2 {
  float4* cu;
  float4* su;
  float4* exu;
  int32_t* exc;
};
__host__ __device__ inline X2 x2_view(char* slot, int cap) {
  return X2{(float4*)slot, (float4*)(slot + 16), (float4*)(slot + 16 + 16 * (size_t)cap),
            (int32_t*)(slot + 16 + 32 * (size_t)cap)};
}

// shard workspace beyond the one-device layout: chunk table, chunk contexts,
// slice references of the final stack
struct ShardLayout {
  size_t tab, tcc, svref, bytes;
  ShardLayout(int64_t n, int cap, bool nobox) {
    size_t o = al256(Layout(n, cap, nobox).bytes);
    tab = o; o = al256(o + 16 * (size_t)GMAX);
    tcc = o; o = al256(o + 16 * (size_t)GMAX);
    svref = o; o = al256(o + 4 * (size_t)cap);
    bytes = o;
  }
};

// phase 1 tail: the chunk's final stack, bottom to top (heights L_g .. L_g + b - 1
// in chunk coordinates, L_g = h0 - a): entry = F1 owner over all the chunk's tiles
__global__ void __launch_bounds__(256) sh_export1(Params p, int cap, char* slot, int32_t* svref) {
  const int lane = threadIdx.x & 31;
  const int2 tot = __ldcg(p.ctrl.total);
  const bool ovf = tot.y > cap || tot.x + 1 > p.h0;
  X1 x = x1_view(slot, cap);
  if (blockIdx.x == 0 && threadIdx.x == 0) *x.hdr = make_int4(tot.x, tot.y, ovf ? 1 : 0, 0);
  if (ovf) return;
  const int Lg = p.h0 - tot.x;
  const int nw = gridDim.x * 8;
  for (int j = blockIdx.x * 8 + (threadIdx.x >> 5); j < tot.y; j += nw) {
    int LU = 0;
    const int X = Lg + j;
    const int U = owner_search_cg(p.ctrl, p.ntiles, X, LU);
    if (lane == 0) {
      const int ref = U * W + (X - LU);
      x.idx[j] = __ldcg(p.slice_idx + ref);
      x.lcc[j] = p.nobox ? bINF() : isect(__ldcg(p.slice_box + ref), __ldcg(p.tc + U));
      svref[j] = ref;
    }
  }
}

// chunk table (every rank computes the same): start height, low-water mark,
// Bic value; the context below each chunk's final stack
struct ChunkRow {
  int H, L, a, b;
};
__device__ __forceinline__ int owner_chunk(const ChunkRow* tab, int k, int X) {  // F1 over chunks < k
  for (int j = k - 1; j >= 0; j--)
    if (tab[j].L <= X) return j;
  return -1;
}
__global__ void sh_table(Params p, int G, int g, int cap, const char* recv1, ChunkRow* tab, float4* tcc) {
  if (threadIdx.x != 0) return;
  const size_t s1 = x1_bytes(cap);
  int H = 0, ovf = 0;
  for (int k = 0; k < G; k++) {
    const int4 h = *(const int4*)(recv1 + s1 * k);
    const int L = max(H - h.x, 0);
    tab[k] = ChunkRow{H, L, h.x, h.y};
    ovf |= h.z;
    H = L + h.y;
  }
  for (int k = 0; k < G; k++) {
    float4 c = bINF();
    const int X = tab[k].L - 1;
    if (!ovf && X >= 0) {
      const int j = owner_chunk(tab, k, X);
      const X1 x = x1_view((char*)recv1 + s1 * j, cap);
      c = isect(x.lcc[X - tab[j].L], tcc[j]);
    }
    tcc[k] = c;
  }
  p.shd[1] = ovf;
}

// the context of imported height h; below the global stack's bottom (X < 0)
// a root slot: idx -1, context INF (a close popping it pops the root, R3)
__device__ __forceinline__ float4 imported_ctx(const Params& p, const ChunkRow* tab, const float4* tcc, int g,
                                               const char* recv1, int cap, int h, int& idx) {
  idx = -1;
  const int X = tab[g].H - p.h0 + h;
  if (X < 0 || p.shd[1]) return bINF();
  const int j = owner_chunk(tab, g, X);
  const int pos = X - tab[j].L;
  if (j < 0 || pos >= min(tab[j].b, cap)) return bINF();
  const X1 x = x1_view((char*)recv1 + x1_bytes(cap) * j, cap);
  idx = x.idx[pos];
  return isect(x.lcc[pos], tcc[j]);
}

// phase 2 head: the imported slice, TC's missing factor, empty close records
__global__ void __launch_bounds__(256) sh_compose(Params p, int g, int cap, const char* recv1, const ChunkRow* tab,
                                                  const float4* tcc) {
  const int nthr = gridDim.x * blockDim.x;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  for (int h = gt; h < p.h0; h += nthr) {
    int idx;
    const float4 c = imported_ctx(p, tab, tcc, g, recv1, cap, h, idx);
    p.slice_idx[p.vbase + h] = idx;
    p.exc[h] = -1;
    if (p.nobox) continue;
    p.slice_box[p.vbase + h] = c;
    p.exu[h] = bEMPTY();
  }
  if (p.nobox) return;  // matching only: no tile contexts
  const int ntv = (p.h0 + W - 1) / W;
  for (int j = gt; j < ntv; j += nthr) p.tc[p.ntiles + j] = bINF();
  for (int T = gt; T < p.ntiles; T += nthr) {
    const int code = __ldcg(p.tcend + T);
    if (code <= -2) {
      int idx;
      const float4 c = imported_ctx(p, tab, tcc, g, recv1, cap, -2 - code, idx);
      p.tc[T] = isect(__ldcg(p.tc + T), c);
    }
  }
}

// phase 2 tail: the chunk union; su of each final-stack open (the union after
// it to the chunk end)
__global__ void __launch_bounds__(256) sh_export2(Params p, int cap, char* slot, const int32_t* svref) {
  const int lane = threadIdx.x & 31;
  if (p.nobox) return;  // matching only: the recorded closes are all slot 2 carries
  X2 x = x2_view(slot, cap);
  const int2 tot = __ldcg(p.ctrl.total);
  const int nb = tot.y > cap || tot.x + 1 > p.h0 ? 0 : tot.y;
  const int nw = gridDim.x * 8;
  const int w0 = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (w0 == 0) {
    const float4 u = range_tiles(p, 0, p.ntiles - 1);
    if (lane == 0) *x.cu = u;
  }
  for (int j = w0; j < nb; j += nw) {
    const int ref = __ldcg(svref + j);
    const float4 r = range_tiles(p, (ref >> LOGW) + 1, p.ntiles - 1);
    if (lane == 0) x.su[j] = unite(__ldcg(p.slice_su + ref), r);
  }
}

// union of the chunk unions a .. b
__device__ __forceinline__ float4 chunks_union(const char* recv2, int cap, int a, int b) {
  float4 u = bEMPTY();
  for (int k = a; k <= b; k++) u = unite(u, *x2_view((char*)recv2 + x2_bytes(cap) * k, cap).cu);
  return u;
}

// phase 3: nodes that span chunks
template <bool PM>
__global__ void __launch_bounds__(256) sh_fixup(Params p, int G, int g, int cap, const char* recv1, const char* recv2,
                                                const ChunkRow* tab) {
  if (p.shd[1]) return;  // overflow: reported, outputs undefined
  const size_t s1 = x1_bytes(cap), s2 = x2_bytes(cap);
  const int h0 = p.h0;
  const int nA = h0, nB = (G - 1 - g) * h0, nC = min(tab[g].b, cap);
  const int64_t tot = (int64_t)nA + nB + nC;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const X1 mine = x1_view((char*)recv1 + s1 * g, cap);
  const X2 mine2 = x2_view((char*)recv2 + s2 * g, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += nthr) {
    if (i < nA) {
      // A: this chunk's close of an imported entry (opened on chunk j)
      if (p.nobox) continue;
      const int h = (int)i;
      const int c = mine2.exc[h];
      if (c < 0) continue;
      const int X = tab[g].H - h0 + h;
      const int j = owner_chunk(tab, g, X);
      const X2 xj = x2_view((char*)recv2 + s2 * j, cap);
      const float4 U = unite(unite(mine2.exu[h], xj.su[X - tab[j].L]), chunks_union(recv2, cap, j + 1, g - 1));
      p.out[c - p.goff] = U;
    } else if (i < nA + nB) {
      // B: a later chunk k closed one of this chunk's final-stack opens
      const int k = g + 1 + (int)((i - nA) / h0), h = (int)((i - nA) % h0);
      const X2 xk = x2_view((char*)recv2 + s2 * k, cap);
      const int c = xk.exc[h];
      if (c < 0) continue;
      const int X = tab[k].H - h0 + h;
      if (owner_chunk(tab, k, X) != g) continue;
      const int pos = X - tab[g].L;
      const int si = mine.idx[pos];
      const int o = (si & 0x7fffffff) - p.goff;
      if (PM) p.match[o] = c;
      if (si < 0 && !p.nobox)  // a blend open takes its node's union
        p.out[o] = unite(unite(xk.exu[h], mine2.su[pos]), chunks_union(recv2, cap, g + 1, k - 1));
    } else {
      // C: final-stack opens no later chunk closes (R4): blend opens take the union to the end
      if (p.nobox) continue;
      const int pos = (int)(i - nA - nB);
      const int X = tab[g].L + pos;
      int later = INT_MAX;
      for (int k = g + 1; k < G; k++) later = min(later, tab[k].L);
      if (X < later) {
        const int si = mine.idx[pos];
        if (si < 0) p.out[(si & 0x7fffffff) - p.goff] = unite(mine2.su[pos], chunks_union(recv2, cap, g + 1, G - 1));
      }
    }
  }
}

}  // namespace fz

// ---- host side of the sharded pass --------------------------------------------
size_t fused_shard_workspace_bytes(int64_t n, int cap, bool nobox) { return fz::ShardLayout(n, cap, nobox).bytes; }
size_t fused_shard_slot1_bytes(int cap) { return fz::x1_bytes(cap); }
size_t fused_shard_slot2_bytes(int cap) { return fz::x2_bytes(cap); }

static int sh_grid(int64_t work, int per_block) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + per_block - 1) / per_block, sm_count() * 16));
}

cudaError_t fused_shard_phase1(const uint8_t* tags, const float* leaf_bbox, int64_t n, int64_t goff, int cap,
                               int32_t* match, void* ws, void* slot1, cudaStream_t stream) {
  if (n <= 0) return cudaMemsetAsync(slot1, 0, 16, stream);  // header (0, 0): an empty chunk
  cudaError_t e = fz::setup();
  if (e != cudaSuccess) return e;
  const bool nobox = leaf_bbox == nullptr;  // paren_match alone
  // (the matching alone: fz_reduce marks the chunk's surviving opens in match)
  fz::Params p = fz::make_params(tags, leaf_bbox, n, nobox ? match : nullptr, nullptr, nullptr, ws, cap, (int)goff, nobox);
  p.nobox = nobox;
  e = launch_front(p, stream);
  if (e != cudaSuccess) return e;
  const fz::ShardLayout SL(n, cap, nobox);
  TB_LAUNCH(stream, "sh_export1",
            (fz::sh_export1<<<sh_grid(cap, 8), 256, 0, stream>>>(p, cap, (char*)slot1, (int32_t*)((char*)ws + SL.svref))));
  return cudaGetLastError();
}

cudaError_t fused_shard_phase2(const uint8_t* tags, const float* leaf_bbox, int64_t n, int64_t goff, int cap, int G,
                               int g, int32_t* match, int32_t* parent, float* node_bbox, void* ws, const void* recv1,
                               void* slot2, cudaStream_t stream) {
  const bool nobox = leaf_bbox == nullptr;
  const fz::ShardLayout SL(n > 0 ? n : 1, cap, nobox);
  cudaError_t e = fz::setup();
  if (e != cudaSuccess) return e;
  fz::Params p = fz::make_params(tags, leaf_bbox, n > 0 ? n : 1, match, parent, node_bbox, ws, cap, (int)goff, nobox);
  p.nobox = nobox;
  fz::X2 x = fz::x2_view((char*)slot2, cap);
  p.exc = x.exc;
  p.exu = x.exu;
  auto* tab = (fz::ChunkRow*)((char*)ws + SL.tab);
  auto* tcc = (float4*)((char*)ws + SL.tcc);
  TB_LAUNCH(stream, "sh_table", (fz::sh_table<<<1, 32, 0, stream>>>(p, G, g, cap, (const char*)recv1, tab, tcc)));
  if (n <= 0) {
    // an empty chunk: union EMPTY, no closes (the table above: its status)
    const float4 em = make_float4(INFINITY, INFINITY, -INFINITY, -INFINITY);
    e = cudaMemcpyAsync(x.cu, &em, sizeof em, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(x.exc, 0xff, 4 * (size_t)cap, stream);
    return e;
  }
  TB_LAUNCH(stream, "sh_compose",
            (fz::sh_compose<<<sh_grid(std::max<int64_t>(cap, p.ntiles), 256), 256, 0, stream>>>(
                p, g, cap, (const char*)recv1, tab, tcc)));
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = nobox ? launch_back_match(p, stream) : launch_back(p, leaf_bbox, node_bbox, match != nullptr, stream);
  if (e != cudaSuccess) return e;
  TB_LAUNCH(stream, "sh_export2",
            (fz::sh_export2<<<sh_grid(cap, 8), 256, 0, stream>>>(p, cap, (char*)slot2,
                                                                  (const int32_t*)((char*)ws + SL.svref))));
  return cudaGetLastError();
}

cudaError_t fused_shard_phase3(int64_t n, int64_t goff, int cap, int G, int g, int32_t* match, float* node_bbox,
                               void* ws, const void* recv1, const void* recv2, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;  // an empty chunk has no final stack and no closes
  const bool nobox = node_bbox == nullptr;
  const fz::ShardLayout SL(n, cap, nobox);
  fz::Params p = fz::make_params(nullptr, nullptr, n, match, nullptr, node_bbox, ws, cap, (int)goff, nobox);
  p.nobox = nobox;
  auto* tab = (const fz::ChunkRow*)((char*)ws + SL.tab);
  const int64_t work = (int64_t)cap * (G - g) + cap;
  if (match)
    TB_LAUNCH(stream, "sh_fixup", (fz::sh_fixup<true><<<sh_grid(work, 256), 256, 0, stream>>>(
                                      p, G, g, cap, (const char*)recv1, (const char*)recv2, tab)));
  else
    TB_LAUNCH(stream, "sh_fixup", (fz::sh_fixup<false><<<sh_grid(work, 256), 256, 0, stream>>>(
                                      p, G, g, cap, (const char*)recv1, (const char*)recv2, tab)));
  return cudaGetLastError();
}

// overflow of the fixed slots in the last sharded call on this workspace (reads
// the device flag: synchronises the stream); 1 = outputs undefined
int fused_shard_status(int64_t n, int cap, void* ws, cudaStream_t stream, cudaError_t* err) {
  const fz::Layout L(n > 0 ? n : 1, cap);
  int v[2] = {0, 0};
  cudaError_t e = cudaMemcpyAsync(v, (char*)ws + L.shd, sizeof v, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (err) *err = e;
  return v[1];
}
