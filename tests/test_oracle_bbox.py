"""Pins for oracle.tree_bbox (CPU only).

The oracle is the two-box sequential stack walk of the introduction.
Pinned against: SPEC/paper examples (golden), an ancestor-walk + range-loop
brute force of the definitions exhaustively on small scenes,
special fp32 values, and closed forms that reduce to library routines
(identity, elementwise max/min, cummax/cummin, amin/amax, scatter_reduce).
"""
import itertools
import json
import os

import numpy as np
import pytest
import torch

import oracle
from brute import EMPTY_U, bbox_by_ancestors, f2u, parent_by_stk, match_from_parent

GOLD = os.path.join(os.path.dirname(__file__), "golden")
INF = float("inf")


def as_bits(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def run_oracle(tags, boxes):
    return oracle.tree_bbox(np.array(tags, np.uint8), np.array(boxes, np.float32).reshape(-1, 4))


def brute_bits(tags, boxes):
    bu = [tuple(f2u(float(v)) for v in row) for row in np.array(boxes, np.float32).reshape(-1, 4)]
    return np.array(bbox_by_ancestors(list(tags), bu), np.uint32).reshape(-1, 4)


@pytest.mark.parametrize("ex", json.load(open(os.path.join(GOLD, "bbox_examples.json")))["examples"],
                         ids=lambda e: e["cite"][:40])
def test_golden_examples(ex):
    tags = [r[0] for r in ex["scene"]]
    boxes = [r[1:] for r in ex["scene"]]
    out = run_oracle(tags, boxes)
    exp = np.array([[INF, INF, -INF, -INF] if e == "E" else e for e in ex["out"]], np.float32)
    assert np.array_equal(as_bits(out), as_bits(exp)), (out, ex["cite"])


def test_exhaustive_small_scenes_vs_brute():
    rng = np.random.default_rng(0)
    for n in range(0, 7):
        for combo in itertools.product((0, 1, 2, 3), repeat=n):
            for _ in range(2):
                lo = rng.integers(-8, 8, size=(n, 2))
                wh = rng.integers(-3, 9, size=(n, 2))        # negative => inverted boxes too
                boxes = np.concatenate([lo, lo + wh], 1).astype(np.float32)
                out = run_oracle(combo, boxes)
                assert np.array_equal(as_bits(out), brute_bits(combo, boxes)), (combo, boxes)


def test_random_scenes_vs_brute():
    rng = np.random.default_rng(1)
    for _ in range(300):
        n = int(rng.integers(1, 90))
        tags = rng.choice([0, 1, 2, 3], size=n, p=[0.4, 0.2, 0.15, 0.25])
        lo = rng.integers(-1000, 1000, size=(n, 2))
        wh = rng.integers(-50, 700, size=(n, 2))
        boxes = np.concatenate([lo, lo + wh], 1).astype(np.float32) / 8
        out = run_oracle(tags, boxes)
        assert np.array_equal(as_bits(out), brute_bits(tags, boxes))


SPECIALS = np.array([0.0, -0.0, INF, -INF, 1e-45, -1e-45, 1.1754942e-38, 3.4028235e38,
                     -3.4028235e38, 1.0, -1.0, 0.5], np.float32)


def test_special_values_vs_brute():
    """±0 (-0 < +0, DESIGN R12), ±inf, subnormals, extremes."""
    rng = np.random.default_rng(2)
    for _ in range(400):
        n = int(rng.integers(1, 30))
        tags = rng.choice([0, 1, 2, 3], size=n, p=[0.4, 0.25, 0.15, 0.2])
        boxes = rng.choice(SPECIALS, size=(n, 4))
        out = run_oracle(tags, boxes)
        assert np.array_equal(as_bits(out), brute_bits(tags, boxes))


def test_signed_zero_order():
    # max(-0,+0) = +0 and min(-0,+0) = -0 in either order (R12)
    for a, b in [(0.0, -0.0), (-0.0, 0.0)]:
        out = run_oracle([1, 0, 3], [[a, a, a, a], [b, b, b, b], [0, 0, 0, 0]])
        leaf = as_bits(out[1])
        assert leaf[0] == f2u(0.0) and leaf[1] == f2u(0.0)       # max -> +0
        assert leaf[2] == f2u(-0.0) and leaf[3] == f2u(-0.0)     # min -> -0


def test_nan_is_ignored():
    """NaN is outside the input domain; a NaN operand of min/max is ignored and
    two NaNs give the canonical NaN (DESIGN R12, the semantics of PTX
    min.f32/max.f32 measured on B200: tools/probe/minmax_probe.cu)."""
    qn = np.float32("nan")
    out = run_oracle([1, 0, 3], [[0, 0, 10, 10], [qn, 1, qn, 2], [0, 0, 0, 0]])
    b = as_bits(out[1])
    assert b[0] == f2u(0.0)                          # max(0, NaN) = 0
    assert b[2] == f2u(10.0)                         # min(10, NaN) = 10
    out = run_oracle([1, 0, 3], [[qn, 0, 10, 10], [qn, 1, 3, 2], [0, 0, 0, 0]])
    assert as_bits(out[0])[0] == f2u(-INF)           # NaN absorbed by the root's INF
    assert as_bits(out[1])[0] == f2u(-INF)
    rng = np.random.default_rng(5)
    vals = np.array([qn, -qn, 0.0, -0.0, 1.0, -1.0, np.inf, -np.inf], np.float32)
    for _ in range(300):
        n = int(rng.integers(1, 25))
        tags = rng.choice([0, 1, 2, 3], size=n)
        boxes = rng.choice(vals, size=(n, 4))
        assert np.array_equal(as_bits(run_oracle(tags, boxes)), brute_bits(tags, boxes))


# ---------------------------------------------------------------------------
# Closed forms -> library routines (torch CPU), at sizes brute force can't reach
# ---------------------------------------------------------------------------

def _rand_boxes(n, seed):
    g = torch.Generator().manual_seed(seed)
    lo = torch.randint(-4096, 4096, (n, 2), generator=g).float() / 4
    wh = torch.randint(0, 4096, (n, 2), generator=g).float() / 4
    return torch.cat([lo, lo + wh], 1)


def test_no_opens_is_identity():
    b = _rand_boxes(5000, 1)
    out = run_oracle([0] * 5000, b.numpy())
    assert np.array_equal(as_bits(out), as_bits(b.numpy()))


def test_one_clip_wrapping_all_is_elementwise():
    n = 4000
    b = _rand_boxes(n + 2, 2)
    tags = [1] + [0] * n + [3]
    out = torch.from_numpy(run_oracle(tags, b.numpy()))
    c = b[0]
    exp = torch.cat([torch.maximum(b[1:n + 1, :2], c[:2]), torch.minimum(b[1:n + 1, 2:], c[2:])], 1)
    assert torch.equal(out[1:n + 1], exp)
    hull = torch.cat([exp[:, :2].amin(0), exp[:, 2:].amax(0)])
    assert torch.equal(out[n + 1], hull)


def test_deep_chain_is_cummax_cummin():
    """C3-style chain (opens then closes) with two leaves in the middle (C3L):
    effective clips = cumulative max/min over clip opens' boxes (blend = INF);
    every node's union = raw hull of the two clipped middle leaves."""
    import scenegen
    n = 20000
    tags = scenegen.deep_chain_tags(n, 9, leaves_mid=True)
    b = _rand_boxes(n, 3)
    b[b[:, 0] > b[:, 2]] = 0
    out = torch.from_numpy(run_oracle(tags.numpy(), b.numpy()))
    h = n // 2
    opens = tags[: h - 1]
    eff = b[: h - 1].clone()
    eff[opens == 2] = torch.tensor([-INF, -INF, INF, INF])
    cmax = torch.cummax(eff[:, :2], 0).values
    cmin = torch.cummin(eff[:, 2:], 0).values
    clips = torch.cat([cmax, cmin], 1)
    is_clip = opens == 1
    assert torch.equal(out[: h - 1][is_clip], clips[is_clip])
    c_last = clips[-1]
    leaves = torch.stack([torch.cat([torch.maximum(b[i, :2], c_last[:2]), torch.minimum(b[i, 2:], c_last[2:])])
                          for i in (h - 1, h)])
    assert torch.equal(out[h - 1:h + 1], leaves)
    hull = torch.cat([leaves[:, :2].amin(0), leaves[:, 2:].amax(0)])
    closes = out[h + 1:]
    assert torch.equal(closes, hull.expand_as(closes))
    assert torch.equal(out[: h - 1][~is_clip], hull.expand(int((~is_clip).sum()), 4))


def test_one_level_of_groups_is_scatter_reduce():
    """Top-level blend groups of leaves: each group's box = amin/amax of its
    leaves (torch.scatter_reduce)."""
    g = torch.Generator().manual_seed(4)
    sizes = torch.randint(0, 12, (500,), generator=g).tolist()
    tags, gid = [], []
    for k, s in enumerate(sizes):
        tags += [2] + [0] * s + [3]
        gid += [k] * s
    n = len(tags)
    b = _rand_boxes(n, 5)
    out = torch.from_numpy(run_oracle(tags, b.numpy()))
    t = torch.tensor(tags)
    leafb = b[t == 0]
    gid = torch.tensor(gid)
    lo = torch.full((len(sizes), 2), INF).scatter_reduce(0, gid[:, None].expand(-1, 2), leafb[:, :2], "amin")
    hi = torch.full((len(sizes), 2), -INF).scatter_reduce(0, gid[:, None].expand(-1, 2), leafb[:, 2:], "amax")
    exp = torch.cat([lo, hi], 1)
    assert torch.equal(out[t == 3], exp)
    assert torch.equal(out[t == 2], exp)


def test_containment_invariants_on_generated_scene():
    """leaf box ⊆ every clip-ancestor box (even inverted); blend open == its close."""
    import scenegen
    tags = scenegen.walk_tags(30000, 21, p_leaf=0.5).numpy()
    b = scenegen.boxes(30000, 21, torch.from_numpy(tags)).numpy()
    out = run_oracle(tags, b)
    match, parent = oracle.paren_match(tags)
    for i in range(0, 30000, 37):
        if tags[i] not in (0, 1):
            continue
        p = parent[i]
        while p != -1:
            if tags[p] == 1:
                assert out[i, 0] >= out[p, 0] and out[i, 1] >= out[p, 1]
                assert out[i, 2] <= out[p, 2] and out[i, 3] <= out[p, 3]
            p = parent[p]
    bl = np.nonzero((tags == 2) & (match >= 0))[0]
    assert np.array_equal(as_bits(out[bl]), as_bits(out[match[bl]]))
