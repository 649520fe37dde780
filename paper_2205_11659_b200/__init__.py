"""paper_2205_11659_b200 — B200 (sm_100a) hot path of Levien's tree bounding boxes.

Thin Python binding over the C ABI in ``include/treebbox.h``
(``libtreebbox.so``, built in-tree from ``csrc/``).  This module only
marshals arguments (torch CUDA tensors -> device pointers + current stream);
every step of the computation runs in the CUDA kernels.  There is no CPU or
PyTorch fallback: if the extension cannot be loaded, calls raise.

    match, parent = paren_match(tags)               # §2-§8 of the paper
    node_bbox     = tree_bbox(tags, leaf_bbox)      # §6, §9
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import build as _build

__all__ = ["release_workspaces", "paren_match", "paren_match_bytes", "tree_bbox", "tree_transform", "tree_fold", "bin_leaves", "compact_scene", "paren_match_tree_bbox_scene", "tree_bbox_matched", "paren_match_tree_bbox_host", "paren_match_host", "tree_bbox_host", "count_unmatched",
           "load", "TreeBBoxError", "LIB_PATH", "workspace_bytes", "ShardContext", "paren_match_vshard",
           "tree_bbox_vshard", "pair_vshard", "shard_default_cap"]

LIB_PATH = _build.LIB
_lock = threading.Lock()
_lib = None


class TreeBBoxError(RuntimeError):
    pass


def load():
    """Load (building first if the sources are newer) libtreebbox.so."""
    global _lib
    with _lock:
        if _lib is None:
            if _build.needs_build():
                _build.build()
            lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
            P, I64, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t
            sigs = {
                "tb_last_error": ([], ctypes.c_char_p),
                "tb_version": ([], ctypes.c_char_p),
                "tb_release_workspaces": ([], ctypes.c_int),
                "paren_match": ([P, I64, P, P, P], ctypes.c_int),
                "paren_match_ws": ([P, I64, P, P, P, SZ, P], ctypes.c_int),
                "paren_match_workspace_bytes": ([I64], SZ),
                "paren_match_host": ([P, I64, P, P, P], ctypes.c_int),
                "tree_bbox": ([P, P, I64, P, P], ctypes.c_int),
                "tree_bbox_ws": ([P, P, I64, P, P, SZ, P], ctypes.c_int),
                "tree_bbox_workspace_bytes": ([I64], SZ),
                "tree_bbox_host": ([P, P, I64, P, P], ctypes.c_int),
                "tree_bbox_matched": ([P, P, P, P, I64, P, P], ctypes.c_int),
                "paren_match_tree_bbox_host": ([P, P, I64, P, P, P, P], ctypes.c_int),
                "paren_match_bytes": ([P, I64, P, P, P, P], ctypes.c_int),
                "tree_transform": ([P, P, P, P, I64, P, P], ctypes.c_int),
                "tree_fold": ([P, P, P, I64, P, P], ctypes.c_int),
                "paren_match_tree_bbox_scene": ([P, P, I64, P, P, P, P, P, P, P, P], ctypes.c_int),
                "compact_scene": ([P, P, I64, P, P, P, P, P, P], ctypes.c_int),
                "bin_leaves": ([P, P, I64, ctypes.c_int, ctypes.c_int, ctypes.c_float, P, P, P, I64, P, P],
                               ctypes.c_int),
                "tree_bbox_matched_ws": ([P, P, P, P, I64, P, P, SZ, P], ctypes.c_int),
                "paren_match_tree_bbox": ([P, P, I64, P, P, P, P], ctypes.c_int),
                "tree_bbox_matched_workspace_bytes": ([I64], SZ),
                "tb_count_unmatched": ([P, I64, P, P, P], ctypes.c_int),
                "tb_get_unique_id": ([P], ctypes.c_int),
                "tb_comm_init": ([P, ctypes.c_int, ctypes.c_int, P], ctypes.c_int),
                "tb_comm_destroy": ([P], ctypes.c_int),
                "paren_match_shard": ([P, I64, I64, P, P, P, P], ctypes.c_int),
                "tb_debug_paren_match_vshard": ([P, I64, ctypes.c_int, P, P, P], ctypes.c_int),
                "tb_debug_tree_bbox_vshard": ([P, P, I64, ctypes.c_int, P, P], ctypes.c_int),
                "tb_debug_host_chunk_shift": ([ctypes.c_int], ctypes.c_int),
                "tb_debug_use_fused": ([ctypes.c_int], ctypes.c_int),
                "tb_debug_fz_trace": ([P], ctypes.c_int),
                "tb_debug_fz_tma": ([ctypes.c_int], ctypes.c_int),
                "tb_debug_fz_ctrl_blocks": ([ctypes.c_int], ctypes.c_int),
                "tb_debug_bins_cap": ([I64], I64),
                "tree_bbox_shard": ([P, P, I64, I64, P, P, P], ctypes.c_int),
                "paren_match_tree_bbox_shard": ([P, P, I64, I64, I64, P, P, P, P, P], ctypes.c_int),
                "tb_shard_status": ([P], ctypes.c_int),
                "tb_shard_default_cap": ([I64], I64),
                "tb_debug_pair_vshard": ([P, P, I64, ctypes.c_int, I64, P, P, P, P], ctypes.c_int),
                "tree_bbox_matched_shard": ([P, P, P, P, I64, I64, P, P, P], ctypes.c_int),
                "tb_launch_count": ([], ctypes.c_longlong),
                "tb_profile_enable": ([ctypes.c_int], ctypes.c_int),
                "tb_profile_read": ([ctypes.c_char_p, SZ], ctypes.c_int),
            }
            for name, (args, res) in sigs.items():
                fn = getattr(lib, name, None)
                if fn is None:
                    continue
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def _check(rc: int):
    if rc != 0:
        msg = load().tb_last_error().decode(errors="replace")
        raise TreeBBoxError(f"treebbox error {rc}: {msg}")


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _need_host(t: torch.Tensor, name: str, dtype, numel: int | None = None):
    """A CPU tensor of this dtype, contiguous, with `numel` elements."""
    if not isinstance(t, torch.Tensor) or t.is_cuda:
        raise TypeError(f"{name} must be a CPU (preferably pinned) tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} must have {numel} elements, got {t.numel()}")


def _need_size(t: torch.Tensor, name: str, numel: int):
    if t.numel() != numel:
        raise ValueError(f"{name} must have {numel} elements, got {t.numel()}")


def _need_cuda(t: torch.Tensor, name: str, dtype):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def paren_match(tags: torch.Tensor, match: torch.Tensor | None = None,
                parent: torch.Tensor | None = None):
    """Parentheses matching on the GPU.  tags: uint8 CUDA [n].

    Returns (match, parent), int32 CUDA [n] (see include/treebbox.h)."""
    lib = load()
    _need_cuda(tags, "tags", torch.uint8)
    n = tags.numel()
    if match is None:
        match = torch.empty(n, dtype=torch.int32, device=tags.device)
    if parent is None:
        parent = torch.empty(n, dtype=torch.int32, device=tags.device)
    _need_cuda(match, "match", torch.int32)
    _need_cuda(parent, "parent", torch.int32)
    with torch.cuda.device(tags.device):
        _check(lib.paren_match(tags.data_ptr(), n, match.data_ptr(), parent.data_ptr(),
                               _stream(tags.device)))
    return match, parent


def paren_match_bytes(text: torch.Tensor, class_map: bytes, match: torch.Tensor | None = None,
                      parent: torch.Tensor | None = None):
    """Parenthesis matching over raw text bytes (uint8 CUDA [n]); class_map: 256
    bytes mapping each byte value to a tag class (1/2 open, 3 close, else leaf)."""
    lib = load()
    _need_cuda(text, "text", torch.uint8)
    if len(class_map) != 256:
        raise ValueError("class_map must have 256 entries")
    n = text.numel()
    if match is None:
        match = torch.empty(n, dtype=torch.int32, device=text.device)
    if parent is None:
        parent = torch.empty(n, dtype=torch.int32, device=text.device)
    _need_cuda(match, "match", torch.int32)
    _need_cuda(parent, "parent", torch.int32)
    cm = (ctypes.c_uint8 * 256)(*bytes(class_map))
    with torch.cuda.device(text.device):
        _check(lib.paren_match_bytes(text.data_ptr(), n, cm, match.data_ptr(), parent.data_ptr(),
                                     _stream(text.device)))
    return match, parent


def tree_bbox(tags: torch.Tensor, leaf_bbox: torch.Tensor, node_bbox: torch.Tensor | None = None):
    """Clip intersections + blend unions on the GPU.

    tags: uint8 CUDA [n]; leaf_bbox: float32 CUDA [n, 4].  Returns float32 [n, 4]."""
    lib = load()
    _need_cuda(tags, "tags", torch.uint8)
    _need_cuda(leaf_bbox, "leaf_bbox", torch.float32)
    n = tags.numel()
    if leaf_bbox.numel() != 4 * n:
        raise ValueError("leaf_bbox must be [n, 4]")
    if node_bbox is None:
        node_bbox = torch.empty((n, 4), dtype=torch.float32, device=tags.device)
    _need_cuda(node_bbox, "node_bbox", torch.float32)
    with torch.cuda.device(tags.device):
        _check(lib.tree_bbox(tags.data_ptr(), leaf_bbox.data_ptr(), n, node_bbox.data_ptr(),
                             _stream(tags.device)))
    return node_bbox


def tree_bbox_matched(tags: torch.Tensor, leaf_bbox: torch.Tensor, match: torch.Tensor, parent: torch.Tensor,
                      node_bbox: torch.Tensor | None = None):
    """tree_bbox from paren_match's outputs (match, parent) for the same tags."""
    lib = load()
    _need_cuda(tags, "tags", torch.uint8)
    _need_cuda(leaf_bbox, "leaf_bbox", torch.float32)
    _need_cuda(match, "match", torch.int32)
    _need_cuda(parent, "parent", torch.int32)
    n = tags.numel()
    if leaf_bbox.numel() != 4 * n or match.numel() != n or parent.numel() != n:
        raise ValueError("leaf_bbox must be [n, 4], match and parent [n]")
    if node_bbox is None:
        node_bbox = torch.empty((n, 4), dtype=torch.float32, device=tags.device)
    _need_cuda(node_bbox, "node_bbox", torch.float32)
    with torch.cuda.device(tags.device):
        _check(lib.tree_bbox_matched(tags.data_ptr(), leaf_bbox.data_ptr(), match.data_ptr(), parent.data_ptr(), n,
                                     node_bbox.data_ptr(), _stream(tags.device)))
    return node_bbox


def paren_match_tree_bbox(tags: torch.Tensor, leaf_bbox: torch.Tensor, match: torch.Tensor | None = None,
                          parent: torch.Tensor | None = None, node_bbox: torch.Tensor | None = None):
    """The whole hot path in one device call: (match, parent, node_bbox), the
    box reduce pass overlapped with paren_match inside the library."""
    lib = load()
    _need_cuda(tags, "tags", torch.uint8)
    _need_cuda(leaf_bbox, "leaf_bbox", torch.float32)
    n = tags.numel()
    if leaf_bbox.numel() != 4 * n:
        raise ValueError("leaf_bbox must be [n, 4]")
    dev = tags.device
    match = torch.empty(n, dtype=torch.int32, device=dev) if match is None else match
    parent = torch.empty(n, dtype=torch.int32, device=dev) if parent is None else parent
    node_bbox = torch.empty((n, 4), dtype=torch.float32, device=dev) if node_bbox is None else node_bbox
    _need_cuda(match, "match", torch.int32)
    _need_cuda(parent, "parent", torch.int32)
    _need_cuda(node_bbox, "node_bbox", torch.float32)
    with torch.cuda.device(dev):
        _check(lib.paren_match_tree_bbox(tags.data_ptr(), leaf_bbox.data_ptr(), n, match.data_ptr(),
                                         parent.data_ptr(), node_bbox.data_ptr(), _stream(dev)))
    return match, parent, node_bbox


def tree_transform(tags: torch.Tensor, local: torch.Tensor, match: torch.Tensor, parent: torch.Tensor,
                   world: torch.Tensor | None = None):
    """2D affine transforms composed down the tree (local: float32 CUDA [n, 6])."""
    lib = load()
    _need_cuda(tags, "tags", torch.uint8)
    _need_cuda(local, "local", torch.float32)
    _need_cuda(match, "match", torch.int32)
    _need_cuda(parent, "parent", torch.int32)
    n = tags.numel()
    if local.numel() != 6 * n:
        raise ValueError("local must be [n, 6]")
    if world is None:
        world = torch.empty((n, 6), dtype=torch.float32, device=tags.device)
    _need_cuda(world, "world", torch.float32)
    with torch.cuda.device(tags.device):
        _check(lib.tree_transform(tags.data_ptr(), local.data_ptr(), match.data_ptr(), parent.data_ptr(), n,
                                  world.data_ptr(), _stream(tags.device)))
    return world


def tree_fold(tags: torch.Tensor, x: torch.Tensor, match: torch.Tensor, out: torch.Tensor | None = None):
    """2x2 matrices mod 2^32 multiplied UP the tree in stream order (R17).
    x: CUDA [n, 4] int32 or uint32 (a, b, c, d); match: paren_match's match.
    Returns [n, 4] of x's dtype: node values at opens and closes, leaves echo
    their payload, unmatched closes the identity."""
    lib = load()
    _need_cuda(tags, "tags", torch.uint8)
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype not in (torch.int32, torch.uint32):
        raise TypeError("x must be a CUDA int32 / uint32 tensor")
    if not x.is_contiguous():
        raise ValueError("x must be contiguous")
    _need_cuda(match, "match", torch.int32)
    n = tags.numel()
    if x.numel() != 4 * n or match.numel() != n:
        raise ValueError("x must be [n, 4], match [n]")
    if out is None:
        out = torch.empty((n, 4), dtype=x.dtype, device=tags.device)
    if not out.is_cuda or out.dtype != x.dtype or out.numel() != 4 * n or not out.is_contiguous():
        raise ValueError("out must be a contiguous CUDA [n, 4] tensor of x's dtype")
    with torch.cuda.device(tags.device):
        _check(lib.tree_fold(tags.data_ptr(), x.data_ptr(), match.data_ptr(), n, out.data_ptr(),
                             _stream(tags.device)))
    return out


def bin_leaves(tags: torch.Tensor, node_bbox: torch.Tensor, grid_w: int, grid_h: int, bin_size: float):
    """Culling + binning of clipped leaf boxes.  Returns (counts, offsets, items),
    int32 CUDA tensors; the order inside a bin is unspecified."""
    lib = load()
    _need_cuda(tags, "tags", torch.uint8)
    _need_cuda(node_bbox, "node_bbox", torch.float32)
    n = tags.numel()
    nb = grid_w * grid_h
    counts = torch.empty(nb, dtype=torch.int32, device=tags.device)
    offsets = torch.empty(nb + 1, dtype=torch.int32, device=tags.device)
    total = ctypes.c_int64(0)
    items = torch.empty(max(n, 1), dtype=torch.int32, device=tags.device)
    with torch.cuda.device(tags.device):
        for _ in range(2):  # a second call when the first guess of the capacity was too small
            _check(lib.bin_leaves(tags.data_ptr(), node_bbox.data_ptr(), n, grid_w, grid_h, float(bin_size),
                                  counts.data_ptr(), offsets.data_ptr(), items.data_ptr(), items.numel(),
                                  ctypes.byref(total), _stream(tags.device)))
            if total.value <= items.numel():
                break
            items = torch.empty(total.value, dtype=torch.int32, device=tags.device)
    return counts, offsets, items[:total.value]


def compact_scene(tags: torch.Tensor, boxes: torch.Tensor | None, keep_map: bytes):
    """Keep the elements whose byte value has keep_map[byte] != 0, in order.
    Returns (tags, boxes or None, index into the full stream)."""
    lib = load()
    _need_cuda(tags, "tags", torch.uint8)
    if len(keep_map) != 256:
        raise ValueError("keep_map must have 256 entries")
    n = tags.numel()
    t_out = torch.empty(max(n, 1), dtype=torch.uint8, device=tags.device)
    idx = torch.empty(max(n, 1), dtype=torch.int32, device=tags.device)
    b_out = None
    if boxes is not None:
        _need_cuda(boxes, "boxes", torch.float32)
        b_out = torch.empty((max(n, 1), 4), dtype=torch.float32, device=tags.device)
    km = (ctypes.c_uint8 * 256)(*bytes(keep_map))
    cnt = ctypes.c_int64(0)
    with torch.cuda.device(tags.device):
        _check(lib.compact_scene(tags.data_ptr(), boxes.data_ptr() if boxes is not None else None, n, km,
                                 t_out.data_ptr(), b_out.data_ptr() if b_out is not None else None, idx.data_ptr(),
                                 ctypes.byref(cnt), _stream(tags.device)))
    k = cnt.value
    return t_out[:k], (b_out[:k] if b_out is not None else None), idx[:k]


def paren_match_tree_bbox_scene(scene: torch.Tensor, boxes: torch.Tensor, keep_map: bytes | None = None,
                                pm: bool = True, sync: bool = True):
    """The bench step on a FULL scene stream with the compaction fused into the
    tile loader: elements whose byte has keep_map[byte] == 0 (default: keep
    bytes 0-3, the hierarchy tags) are dropped.  Returns (tags, index, match,
    parent, node_bbox, n_kept) for the kept elements in stream order; match /
    parent are compacted indices (None when pm=False).  sync=False returns the
    capacity-n tensors and n_kept as a device int64 tensor (no host sync)."""
    lib = load()
    _need_cuda(scene, "scene", torch.uint8)
    _need_cuda(boxes, "boxes", torch.float32)
    n = scene.numel()
    if boxes.numel() != 4 * n:
        raise ValueError("boxes must be [n, 4]")
    if keep_map is None:
        keep_map = bytes([1, 1, 1, 1] + [0] * 252)
    if len(keep_map) != 256:
        raise ValueError("keep_map must have 256 entries")
    dev = scene.device
    m = max(n, 1)
    t_out = torch.empty(m, dtype=torch.uint8, device=dev)
    idx = torch.empty(m, dtype=torch.int32, device=dev)
    out = torch.empty((m, 4), dtype=torch.float32, device=dev)
    match = torch.empty(m, dtype=torch.int32, device=dev) if pm else None
    parent = torch.empty(m, dtype=torch.int32, device=dev) if pm else None
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    km = (ctypes.c_uint8 * 256)(*bytes(keep_map))
    with torch.cuda.device(dev):
        _check(lib.paren_match_tree_bbox_scene(scene.data_ptr(), boxes.data_ptr(), n, km, t_out.data_ptr(),
                                               idx.data_ptr(), match.data_ptr() if pm else None,
                                               parent.data_ptr() if pm else None, out.data_ptr(), cnt.data_ptr(),
                                               _stream(dev)))
    if not sync:
        return t_out, idx, match, parent, out, cnt
    k = int(cnt.item())
    return (t_out[:k], idx[:k], match[:k] if pm else None, parent[:k] if pm else None, out[:k], k)


def release_workspaces(device=None):
    """Free the library's cached device workspaces of `device` (default: the
    current device); the next call re-allocates what it needs."""
    lib = load()
    with torch.cuda.device(device if device is not None else torch.cuda.current_device()):
        _check(lib.tb_release_workspaces())


def workspace_bytes(n: int) -> dict:
    lib = load()
    return {"paren_match": int(lib.paren_match_workspace_bytes(n)),
            "tree_bbox": int(lib.tree_bbox_workspace_bytes(n)),
            "tree_bbox_matched": int(lib.tree_bbox_matched_workspace_bytes(n))}


def paren_match_host(tags: torch.Tensor, match: torch.Tensor, parent: torch.Tensor,
                     device=None):
    """End-to-end host-buffer call (copies in, computes, copies out, syncs)."""
    lib = load()
    n = tags.numel()
    _need_host(tags, "tags", torch.uint8)
    _need_host(match, "match", torch.int32, n)
    _need_host(parent, "parent", torch.int32, n)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    with torch.cuda.device(dev):
        _check(lib.paren_match_host(tags.data_ptr(), tags.numel(), match.data_ptr(),
                                    parent.data_ptr(), _stream(dev)))
    return match, parent


def tree_bbox_host(tags: torch.Tensor, leaf_bbox: torch.Tensor, node_bbox: torch.Tensor,
                   device=None):
    lib = load()
    n = tags.numel()
    _need_host(tags, "tags", torch.uint8)
    _need_host(leaf_bbox, "leaf_bbox", torch.float32, 4 * n)
    _need_host(node_bbox, "node_bbox", torch.float32, 4 * n)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    with torch.cuda.device(dev):
        _check(lib.tree_bbox_host(tags.data_ptr(), leaf_bbox.data_ptr(), tags.numel(),
                                  node_bbox.data_ptr(), _stream(dev)))
    return node_bbox


def paren_match_tree_bbox_host(tags: torch.Tensor, leaf_bbox: torch.Tensor, match: torch.Tensor,
                               parent: torch.Tensor, node_bbox: torch.Tensor, device=None):
    """The whole hot path from (pinned) host tensors: copies in, paren_match,
    tree_bbox_matched, copies out, synchronises."""
    lib = load()
    n = tags.numel()
    _need_host(tags, "tags", torch.uint8)
    _need_host(leaf_bbox, "leaf_bbox", torch.float32, 4 * n)
    _need_host(match, "match", torch.int32, n)
    _need_host(parent, "parent", torch.int32, n)
    _need_host(node_bbox, "node_bbox", torch.float32, 4 * n)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    with torch.cuda.device(dev):
        _check(lib.paren_match_tree_bbox_host(tags.data_ptr(), leaf_bbox.data_ptr(), tags.numel(), match.data_ptr(),
                                              parent.data_ptr(), node_bbox.data_ptr(), _stream(dev)))
    return match, parent, node_bbox


def count_unmatched(tags: torch.Tensor):
    """Global Bic (a, b) of the stream, computed on the GPU (synchronises)."""
    lib = load()
    _need_cuda(tags, "tags", torch.uint8)
    a = ctypes.c_int64(0)
    b = ctypes.c_int64(0)
    with torch.cuda.device(tags.device):
        _check(lib.tb_count_unmatched(tags.data_ptr(), tags.numel(), ctypes.byref(a), ctypes.byref(b),
                                      _stream(tags.device)))
    return a.value, b.value


def paren_match_vshard(tags: torch.Tensor, nshards: int):
    """Test hook: the multi-GPU shard protocol run with `nshards` virtual shards
    of one device buffer on one GPU (device copies stand in for NCCL)."""
    lib = load()
    _need_cuda(tags, "tags", torch.uint8)
    n = tags.numel()
    match = torch.empty(n, dtype=torch.int32, device=tags.device)
    parent = torch.empty(n, dtype=torch.int32, device=tags.device)
    with torch.cuda.device(tags.device):
        _check(lib.tb_debug_paren_match_vshard(tags.data_ptr(), n, nshards, match.data_ptr(), parent.data_ptr(),
                                               _stream(tags.device)))
    return match, parent


def tree_bbox_vshard(tags: torch.Tensor, leaf_bbox: torch.Tensor, nshards: int):
    """Test hook: the tree_bbox shard protocol with `nshards` virtual shards."""
    lib = load()
    _need_cuda(tags, "tags", torch.uint8)
    _need_cuda(leaf_bbox, "leaf_bbox", torch.float32)
    out = torch.empty_like(leaf_bbox)
    with torch.cuda.device(tags.device):
        _check(lib.tb_debug_tree_bbox_vshard(tags.data_ptr(), leaf_bbox.data_ptr(), tags.numel(), nshards,
                                             out.data_ptr(), _stream(tags.device)))
    return out


def shard_default_cap(n_local: int) -> int:
    """Default capacity of a sharded call (every chunk's Bic a + 1 and b must
    fit): 4 sqrt(n_local) + 4096, at most n_local + 2."""
    return int(load().tb_shard_default_cap(int(n_local)))


def pair_vshard(tags: torch.Tensor, leaf_bbox: torch.Tensor, nshards: int, cap: int = None, pm: bool = True):
    """Test hook: paren_match_tree_bbox by the sharded fused protocol with
    `nshards` virtual shards of one device buffer on one GPU (the chunks run
    the three phases in lockstep; their slots are the gathered buffers).
    Returns (match, parent, node_bbox); match / parent are None when pm=False."""
    lib = load()
    _need_cuda(tags, "tags", torch.uint8)
    n = tags.numel()
    if leaf_bbox is not None:  # None: the matching alone (paren_match_shard's protocol)
        _need_cuda(leaf_bbox, "leaf_bbox", torch.float32)
        if leaf_bbox.shape != (n, 4):
            raise ValueError("leaf_bbox must be (n, 4)")
    elif not pm:
        raise ValueError("no outputs")
    if cap is None:
        cap = shard_default_cap((n + nshards - 1) // nshards + 16)  # chunk borders: multiples of 16
    out = torch.empty_like(leaf_bbox) if leaf_bbox is not None else None
    match = torch.empty(n, dtype=torch.int32, device=tags.device) if pm else None
    parent = torch.empty(n, dtype=torch.int32, device=tags.device) if pm else None
    with torch.cuda.device(tags.device):
        _check(lib.tb_debug_pair_vshard(tags.data_ptr(), leaf_bbox.data_ptr() if out is not None else None, n,
                                        nshards, int(cap), match.data_ptr() if pm else None,
                                        parent.data_ptr() if pm else None, out.data_ptr() if out is not None else None,
                                        _stream(tags.device)))
    return match, parent, out


class ShardContext:
    """One rank of a sharded run (one process per GPU, contiguous chunks in
    rank order).  Bootstraps the library's own NCCL communicator through the
    caller's torch.distributed process group (the 128-byte NCCL id is
    broadcast from rank 0), then exposes the sharded calls for this rank's
    chunk [offset, offset + n_local) of the global stream."""

    def __init__(self, world: int, rank: int, offset: int, n_local: int, device=None):
        import torch.distributed as dist
        lib = load()
        self.world, self.rank, self.offset, self.n = world, rank, offset, n_local
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        buf = (ctypes.c_uint8 * 128)()
        if rank == 0:
            _check(lib.tb_get_unique_id(buf))
        backend = dist.get_backend()
        t = torch.tensor(list(bytes(buf)), dtype=torch.uint8,
                         device=self.device if backend == "nccl" else "cpu")
        dist.broadcast(t, 0)
        # one capacity on every rank: from the largest chunk (once, at setup)
        nm = torch.tensor([int(n_local)], dtype=torch.int64, device=t.device)
        dist.all_reduce(nm, op=dist.ReduceOp.MAX)
        self.default_cap = shard_default_cap(int(nm.item()))
        ident = (ctypes.c_uint8 * 128)(*t.cpu().tolist())
        comm = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _check(lib.tb_comm_init(ident, world, rank, ctypes.byref(comm)))
        self.comm = comm

    def paren_match(self, tags: torch.Tensor, match: torch.Tensor, parent: torch.Tensor):
        lib = load()
        _need_cuda(tags, "tags", torch.uint8)
        for t, nm in ((match, "match"), (parent, "parent")):
            _need_cuda(t, nm, torch.int32)
            _need_size(t, nm, tags.numel())
        with torch.cuda.device(tags.device):
            _check(lib.paren_match_shard(tags.data_ptr(), tags.numel(), self.offset, match.data_ptr(),
                                         parent.data_ptr(), self.comm, _stream(tags.device)))
        return match, parent

    def tree_bbox(self, tags: torch.Tensor, leaf_bbox: torch.Tensor, node_bbox: torch.Tensor):
        lib = load()
        _need_cuda(tags, "tags", torch.uint8)
        for t, nm in ((leaf_bbox, "leaf_bbox"), (node_bbox, "node_bbox")):
            _need_cuda(t, nm, torch.float32)
            _need_size(t, nm, 4 * tags.numel())
        with torch.cuda.device(tags.device):
            _check(lib.tree_bbox_shard(tags.data_ptr(), leaf_bbox.data_ptr(), tags.numel(), self.offset,
                                       node_bbox.data_ptr(), self.comm, _stream(tags.device)))
        return node_bbox

    def paren_match_tree_bbox(self, tags: torch.Tensor, leaf_bbox: torch.Tensor, match: torch.Tensor,
                              parent: torch.Tensor, node_bbox: torch.Tensor, cap: int = None, check: bool = True):
        """The bench step on this rank's chunk: two fixed-size all-gathers, no
        host synchronisation.  `cap` must be equal on every rank (default:
        shard_default_cap of the largest chunk, ceil(n_total / world)).  With
        check=False the call only enqueues; call status() before trusting the
        outputs (an overflow of cap raises there)."""
        lib = load()
        _need_cuda(tags, "tags", torch.uint8)
        _need_cuda(leaf_bbox, "leaf_bbox", torch.float32)
        for t, nm in ((match, "match"), (parent, "parent")):
            _need_cuda(t, nm, torch.int32)
            if t.numel() != tags.numel():
                raise ValueError(f"{nm} must have n_local elements")
        _need_cuda(node_bbox, "node_bbox", torch.float32)
        if leaf_bbox.shape != (tags.numel(), 4) or node_bbox.shape != (tags.numel(), 4):
            raise ValueError("leaf_bbox / node_bbox must be (n_local, 4)")
        if cap is None:
            cap = self.default_cap
        with torch.cuda.device(tags.device):
            _check(lib.paren_match_tree_bbox_shard(tags.data_ptr(), leaf_bbox.data_ptr(), tags.numel(), self.offset,
                                                   int(cap), match.data_ptr(), parent.data_ptr(), node_bbox.data_ptr(),
                                                   self.comm, _stream(tags.device)))
            if check:
                _check(lib.tb_shard_status(_stream(tags.device)))
        return match, parent, node_bbox

    def status(self):
        """Wait for this rank's last sharded call; raises on a capacity overflow."""
        with torch.cuda.device(self.device):
            _check(load().tb_shard_status(_stream(self.device)))

    def tree_bbox_matched(self, tags: torch.Tensor, leaf_bbox: torch.Tensor, match: torch.Tensor,
                          parent: torch.Tensor, node_bbox: torch.Tensor):
        """Boxes from this rank's slice of the global matching (paren_match above)."""
        lib = load()
        _need_cuda(tags, "tags", torch.uint8)
        for t, nm in ((leaf_bbox, "leaf_bbox"), (node_bbox, "node_bbox")):
            _need_cuda(t, nm, torch.float32)
            _need_size(t, nm, 4 * tags.numel())
        for t, nm in ((match, "match"), (parent, "parent")):
            _need_cuda(t, nm, torch.int32)
            _need_size(t, nm, tags.numel())
        with torch.cuda.device(tags.device):
            _check(lib.tree_bbox_matched_shard(tags.data_ptr(), leaf_bbox.data_ptr(), match.data_ptr(),
                                               parent.data_ptr(), tags.numel(), self.offset, node_bbox.data_ptr(),
                                               self.comm, _stream(tags.device)))
        return node_bbox

    def close(self):
        if self.comm:
            load().tb_comm_destroy(self.comm)
            self.comm = None
