"""Seeded synthetic scene generators (shared by tests and bench).

This module holds NO arithmetic of the method (no Bic, no stack, no box
intersection/union).  It only draws element tags and leaf boxes with the
shapes of the paper's workloads, deterministically from ``seed`` and the
element index, so any shard can generate its own part and CPU/GPU draws are
bit-identical (all arithmetic is exact integer arithmetic on int64 tensors;
box coordinates are dyadic rationals exactly representable in fp32).

Tag bytes: 0 leaf, 1 open clip, 2 open blend, 3 close.

Workloads (DESIGN.md §5 "input recipe"):
* ``walk_tags``      — the paper's generator: push/pop equally likely
  unless underflow, realised as a reflected ±1 walk D = |S| (equal in law),
  with optional leaves (p_leaf) and clip/blend mix (p_clip).
* ``capped_tags``    — C1: tiny scene, nesting depth <= max_depth.
* ``deep_chain_tags``— C3: n/2 opens then n/2 closes (depth n/2); C3L puts two
  leaves in the middle.
* ``compacted_tags`` — C4: piet-gpu-like stream after stream compaction (no
  leaves), wide shallow groups plus rare bursts of deep clips.
* ``boxes``          — per-index counter-hash boxes (leaf: centre U[0,4096)^2,
  size 2^U[0,10); clip: size 2^U[6,12); others (0,0,0,0)).
"""
from __future__ import annotations

import numpy as np
import torch

M32 = 0xFFFFFFFF

LEAF, OPEN_CLIP, OPEN_BLEND, CLOSE = 0, 1, 2, 3


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for x in [0, 2^32) held in int64, without overflow."""
    lo = x & 0xFFFF
    hi = x >> 16
    return (lo * c + ((hi * (c & 0xFFFF)) << 16)) & M32


def _fmix32(x: torch.Tensor) -> torch.Tensor:
    x = x ^ (x >> 16)
    x = _mul32(x, 0x85EBCA6B)
    x = x ^ (x >> 13)
    x = _mul32(x, 0xC2B2AE35)
    x = x ^ (x >> 16)
    return x


def _fmix32_int(x: int) -> int:
    x &= M32
    x ^= x >> 16
    x = (x * 0x85EBCA6B) & M32
    x ^= x >> 13
    x = (x * 0xC2B2AE35) & M32
    x ^= x >> 16
    return x


def hash_u32(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """Counter-based 32-bit hash of (seed, stream, idx); idx int64 in [0, 2^32)."""
    k = _fmix32_int(_fmix32_int(seed * 0x9E3779B1 + 0x7F4A7C15) ^ (stream * 0x632BE5AB))
    return _fmix32(_fmix32((idx & M32) ^ k) ^ ((idx >> 32) & M32))


def _arange(start: int, n: int, device) -> torch.Tensor:
    return torch.arange(start, start + n, dtype=torch.int64, device=device)


def walk_tags(n: int, seed: int, p_leaf: float = 0.5, p_clip: float = 0.75,
              close_tail: bool = False, device="cpu", offset: int = 0) -> torch.Tensor:
    """Paper's random stream as a reflected walk; uint8 tensor.

    Element i (global index offset+i) is a leaf with probability p_leaf; other
    elements take a fair ±1 step of a free walk S and are an OPEN when |S|
    rises, a CLOSE when it falls — the same Markov chain as "push and pop
    equally probable unless it would underflow".  ``close_tail`` appends
    closes for every open left at the end (balanced variant, C2).
    Note: with offset>0 the walk restarts at 0, so shards are only generated
    with offset=0 here and sliced afterwards by the caller.
    """
    idx = _arange(offset, n, device)
    leaf = hash_u32(seed, 1, idx) < int(p_leaf * 2**32)
    step = (hash_u32(seed, 2, idx) & 1) * 2 - 1
    clip = hash_u32(seed, 3, idx) < int(p_clip * 2**32)
    step = torch.where(leaf, torch.zeros_like(step), step)
    s = torch.cumsum(step, 0)
    prev = s - step
    rise = s.abs() > prev.abs()
    tags = torch.full((n,), CLOSE, dtype=torch.uint8, device=device)
    tags[rise & clip] = OPEN_CLIP
    tags[rise & ~clip] = OPEN_BLEND
    tags[leaf] = LEAF
    if close_tail and n > 0:
        d = int(s[-1].abs().item())
        tags = torch.cat([tags, torch.full((d,), CLOSE, dtype=torch.uint8, device=device)])
    return tags


def capped_tags(n: int, seed: int, max_depth: int = 8, p_leaf: float = 0.5,
                p_clip: float = 0.75, close_tail: bool = True) -> torch.Tensor:
    """C1: random scene of n elements with nesting depth <= max_depth (CPU)."""
    idx = _arange(0, n, "cpu")
    u_leaf = hash_u32(seed, 1, idx).numpy()
    u_step = hash_u32(seed, 2, idx).numpy()
    u_kind = hash_u32(seed, 3, idx).numpy()
    out = np.empty(n, np.uint8)
    depth = 0
    for i in range(n):
        if u_leaf[i] < int(p_leaf * 2**32):
            out[i] = LEAF
            continue
        up = (u_step[i] & 1) == 1
        if depth == 0:
            up = True
        elif depth >= max_depth:
            up = False
        if up:
            out[i] = OPEN_CLIP if u_kind[i] < int(p_clip * 2**32) else OPEN_BLEND
            depth += 1
        else:
            out[i] = CLOSE
            depth -= 1
    if close_tail and depth:
        out = np.concatenate([out, np.full(depth, CLOSE, np.uint8)])
    return torch.from_numpy(out)


def deep_chain_tags(n: int, seed: int, p_clip: float = 0.75, leaves_mid: bool = False,
                    device="cpu") -> torch.Tensor:
    """C3: n//2 opens (clip w.p. p_clip) then n - n//2 closes; depth n/2.

    leaves_mid (C3L): the two middle elements become leaves, so every node's
    union is the hull of those two clipped leaves."""
    h = n // 2
    idx = _arange(0, h, device)
    clip = hash_u32(seed, 3, idx) < int(p_clip * 2**32)
    opens = torch.where(clip, torch.full_like(idx, OPEN_CLIP), torch.full_like(idx, OPEN_BLEND))
    tags = torch.cat([opens.to(torch.uint8),
                      torch.full((n - h,), CLOSE, dtype=torch.uint8, device=device)])
    if leaves_mid and h >= 1 and n - h >= 1:
        tags[h - 1] = LEAF
        tags[h] = LEAF
    return tags


def compacted_tags(n: int, seed: int, p_burst: float = 0.01, p_clip: float = 0.75,
                   burst_lo: int = 1024, burst_hi: int = 65536, max_depth: int = 4) -> torch.Tensor:
    """C4: stream-compacted piet-gpu-like scene (only clip/blend parens).

    Top-level groups: with prob 1-p_burst a shallow group (a walk of 2..64
    elements with depth <= max_depth, then closed); with prob p_burst a burst
    of D ~ U{burst_lo..burst_hi} clip opens followed by D closes.  Trimmed to n
    and closed (the last elements are replaced by closes for every open left).
    """
    parts = []
    total = 0
    g = 0
    while total < n:
        u = _fmix32_int(_fmix32_int(seed * 7919 + g) ^ 0xA5A5A5A5)
        if u < int(p_burst * 2**32):
            d = burst_lo + _fmix32_int(u ^ 0x1234567) % (burst_hi - burst_lo + 1)
            part = np.concatenate([np.full(d, OPEN_CLIP, np.uint8), np.full(d, CLOSE, np.uint8)])
        else:
            ln = 2 + _fmix32_int(u ^ 0x89ABCDE) % 63
            idx = _arange(g * 64, ln, "cpu")
            step = ((hash_u32(seed, 5, idx) & 1) * 2 - 1).numpy()
            kind = hash_u32(seed, 6, idx).numpy() < int(p_clip * 2**32)
            s = np.cumsum(step)
            period = 2 * max_depth
            tri = max_depth - np.abs(np.mod(s, period) - max_depth)     # reflected in [0, max_depth]
            prev = np.concatenate([[0], tri[:-1]])
            rise = tri > prev
            walk = np.where(rise, np.where(kind, OPEN_CLIP, OPEN_BLEND), CLOSE).astype(np.uint8)
            part = np.concatenate([walk, np.full(int(tri[-1]), CLOSE, np.uint8)])
        parts.append(part)
        total += part.shape[0]
        g += 1
    body = np.concatenate(parts[:-1]) if len(parts) > 1 else np.empty(0, np.uint8)
    if body.shape[0] > n:
        body = body[:0]
    # every group is balanced and of even length; fill the rest with "()" pairs
    rest = n - body.shape[0]
    pad = np.empty(rest, np.uint8)
    pad[0::2] = OPEN_CLIP
    pad[1::2] = CLOSE
    tags = np.concatenate([body, pad])
    return torch.from_numpy(tags)


def boxes(n: int, seed: int, tags: torch.Tensor | None = None, offset: int = 0,
          device="cpu") -> torch.Tensor:
    """float32 [n, 4] boxes (x0, y0, x1, y1) from a per-index hash.

    Leaf (and every index when tags is None): centre (cx, cy) in [0, 4096) in
    steps of 1/256, width/height (8 + f) * 2^(k-3), k in [0, 10), f in [0, 8).
    Clip opens: k in [6, 12).  Blend opens and closes: (0, 0, 0, 0).
    All coordinates are exact dyadic rationals, so CPU and GPU agree bitwise.
    """
    idx = _arange(offset, n, device)
    h1 = hash_u32(seed, 11, idx)
    h2 = hash_u32(seed, 12, idx)
    h3 = hash_u32(seed, 13, idx)
    cx = (h1 >> 12).double() / 256.0            # 20 bits -> [0, 4096)
    cy = (h2 >> 12).double() / 256.0
    kw = (h3 % 10)
    kh = ((h3 >> 8) % 10)
    fw = (h3 >> 16) & 7
    fh = (h3 >> 19) & 7
    if tags is not None:
        is_clip = (tags.to(device) == OPEN_CLIP)
        kw = torch.where(is_clip, 6 + ((h3 >> 22) % 6), kw)
        kh = torch.where(is_clip, 6 + ((h3 >> 26) % 6), kh)
    pw = torch.tensor([2.0 ** (k - 3) for k in range(12)], dtype=torch.float64, device=device)
    w = (8 + fw).double() * pw[kw]
    hh = (8 + fh).double() * pw[kh]
    out = torch.stack([cx - w / 2, cy - hh / 2, cx + w / 2, cy + hh / 2], dim=1).float()
    if tags is not None:
        t = tags.to(device)
        zero = (t == OPEN_BLEND) | (t == CLOSE)
        out[zero] = 0.0
    return out


def config(name: str, seed: int | None = None, device="cpu"):
    """Named workloads of BASELINE.json ``configs`` (sizes per DESIGN.md §5).

    Returns (tags uint8 tensor, description dict)."""
    name = name.upper()
    if name == "C1":
        s = 0 if seed is None else seed
        return capped_tags(1000, s), {"workload": "C1 tiny scene, depth<=8", "seed": s}
    if name == "C2":
        s = 1 if seed is None else seed
        return walk_tags(1 << 20, s, close_tail=True, device=device), \
            {"workload": "C2 balanced random tree 2^20 (+closing tail)", "seed": s}
    if name == "C3":
        s = 2 if seed is None else seed
        return deep_chain_tags(1 << 24, s, device=device), \
            {"workload": "C3 deep chain 2^24, depth n/2", "seed": s}
    if name == "C3L":
        s = 2 if seed is None else seed
        return deep_chain_tags(1 << 24, s, leaves_mid=True, device=device), \
            {"workload": "C3L deep chain 2^24 with two middle leaves", "seed": s}
    if name == "C4":
        s = 3 if seed is None else seed
        return compacted_tags(1 << 26, s).to(device), \
            {"workload": "C4 compacted piet-gpu-like 2^26", "seed": s}
    if name.startswith("C5"):
        s = 4 if seed is None else seed
        return walk_tags(1 << 27, s, device=device), \
            {"workload": "C5 random-depth walk 2^27 per GPU", "seed": s}
    raise ValueError(name)
