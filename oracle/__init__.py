"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain sequential CPU implementation of the hot path, written from the paper
(arXiv 2205.11659).  The arithmetic lives in ``oracle.c`` (plain C, one stack
walk per call, P:26 and Fig. 1); this module only compiles it with gcc
and marshals numpy arrays through ctypes.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_2205_11659_b200``) never imports it and shares no code
with it.

Pins (see tests/test_oracle_*.py and DESIGN.md §4): exhaustive equality with
an O(n^2) Bic brute force and with the stack-monoid characterisation
(P:121-125); the paper's worked examples and SPEC's
examples as golden fixtures; box results against an ancestor-walk / range-loop
brute force and closed forms (cummax/cummin chains, amin/amax, scatter_reduce).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc -O2, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            lib.oracle_paren_match.argtypes = [P, ctypes.c_int64, P, P]
            lib.oracle_paren_match.restype = ctypes.c_int
            lib.oracle_tree_bbox.argtypes = [P, P, ctypes.c_int64, P]
            lib.oracle_tree_bbox.restype = ctypes.c_int
            lib.oracle_count_unmatched.argtypes = [P, ctypes.c_int64, P, P]
            lib.oracle_count_unmatched.restype = ctypes.c_int
            lib.oracle_tree_transform.argtypes = [P, P, ctypes.c_int64, P]
            lib.oracle_tree_transform.restype = ctypes.c_int
            lib.oracle_tree_fold.argtypes = [P, P, ctypes.c_int64, P]
            lib.oracle_tree_fold.restype = ctypes.c_int
            lib.oracle_bin_leaves.argtypes = [P, P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_float,
                                              P, P, P, ctypes.c_int64]
            lib.oracle_bin_leaves.restype = ctypes.c_int64
            _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def paren_match(tags: np.ndarray, out_match: np.ndarray | None = None,
                out_parent: np.ndarray | None = None):
    """Fig. 1 stack walk.  Returns (match, parent) as int32 arrays."""
    tags = np.ascontiguousarray(tags, dtype=np.uint8)
    n = tags.shape[0]
    match = out_match if out_match is not None else np.empty(n, np.int32)
    parent = out_parent if out_parent is not None else np.empty(n, np.int32)
    if _load().oracle_paren_match(_ptr(tags), n, _ptr(match), _ptr(parent)) != 0:
        raise MemoryError("oracle_paren_match: allocation failed")
    return match, parent


def tree_bbox(tags: np.ndarray, leaf_bbox: np.ndarray, out: np.ndarray | None = None):
    """Two-box sequential stack walk.  leaf_bbox: float32 [n, 4]."""
    tags = np.ascontiguousarray(tags, dtype=np.uint8)
    boxes = np.ascontiguousarray(leaf_bbox, dtype=np.float32).reshape(-1, 4)
    n = tags.shape[0]
    if boxes.shape[0] != n:
        raise ValueError("leaf_bbox must have n rows")
    res = out if out is not None else np.empty((n, 4), np.float32)
    if _load().oracle_tree_bbox(_ptr(tags), _ptr(boxes), n, _ptr(res)) != 0:
        raise MemoryError("oracle_tree_bbox: allocation failed")
    return res


def tree_transform(tags: np.ndarray, local: np.ndarray):
    """Affine transforms composed down the tree (R15), fp64.  local: float32
    [n, 6] (a, b, c, d, tx, ty); returns float64 [n, 6]."""
    tags = np.ascontiguousarray(tags, dtype=np.uint8)
    loc = np.ascontiguousarray(local, dtype=np.float32).reshape(-1, 6)
    n = tags.shape[0]
    if loc.shape[0] != n:
        raise ValueError("local must have n rows")
    res = np.empty((n, 6), np.float64)
    if _load().oracle_tree_transform(_ptr(tags), _ptr(loc), n, _ptr(res)) != 0:
        raise MemoryError("oracle_tree_transform: allocation failed")
    return res


def tree_fold(tags: np.ndarray, x: np.ndarray):
    """2x2 matrices mod 2^32 multiplied UP the tree in stream order (R17):
    uint32 [n, 4] in (a, b, c, d); returns uint32 [n, 4] (node value at its
    open and close, leaves their own payload, unmatched closes the identity)."""
    tags = np.ascontiguousarray(tags, dtype=np.uint8)
    xx = np.ascontiguousarray(x, dtype=np.uint32).reshape(-1, 4)
    n = tags.shape[0]
    if xx.shape[0] != n:
        raise ValueError("x must have n rows")
    res = np.empty((n, 4), np.uint32)
    if _load().oracle_tree_fold(_ptr(tags), _ptr(xx), n, _ptr(res)) != 0:
        raise MemoryError("oracle_tree_fold: allocation failed")
    return res


def bin_leaves(tags: np.ndarray, node_bbox: np.ndarray, gw: int, gh: int, bs: float):
    """Culling + binning of clipped leaf boxes (R16).  Returns (counts, offsets,
    items) with items in leaf order inside each bin."""
    tags = np.ascontiguousarray(tags, dtype=np.uint8)
    box = np.ascontiguousarray(node_bbox, dtype=np.float32).reshape(-1, 4)
    counts = np.zeros(gw * gh, np.int32)
    offsets = np.zeros(gw * gh + 1, np.int32)
    total = _load().oracle_bin_leaves(_ptr(tags), _ptr(box), tags.shape[0], gw, gh, bs, _ptr(counts),
                                      _ptr(offsets), 0, 0)
    if total < 0:
        raise MemoryError("oracle_bin_leaves")
    items = np.zeros(max(total, 1), np.int32)
    _load().oracle_bin_leaves(_ptr(tags), _ptr(box), tags.shape[0], gw, gh, bs, _ptr(counts), _ptr(offsets),
                              _ptr(items), total)
    return counts, offsets, items[:total]


def count_unmatched(tags: np.ndarray):
    """Global Bic (unmatched closes a, unmatched opens b) of the stream."""
    tags = np.ascontiguousarray(tags, dtype=np.uint8)
    a = np.zeros(1, np.int64)
    b = np.zeros(1, np.int64)
    _load().oracle_count_unmatched(_ptr(tags), tags.shape[0], _ptr(a), _ptr(b))
    return int(a[0]), int(b[0])
