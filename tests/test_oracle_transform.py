"""Pins of oracle.tree_transform (reading R15): a
generic, non-commutative, non-idempotent monoid payload (2D affine transforms)
composed down the tree.  Independent of oracle.c: a brute-force ancestor walk
on the brute-force parent (tests/brute.py), closed forms for translation and
rotation chains, and a hand-computed example where the order matters."""
import numpy as np
import pytest

import oracle
import brute

ID = np.array([1, 0, 0, 1, 0, 0], np.float64)


def compose(A, B):  # (A ∘ B)(p) = A(B(p)), 6-vectors (a, b, c, d, tx, ty)
    a, b, c, d, tx, ty = A
    e, f, g, h, ux, uy = B
    return np.array([a * e + b * g, a * f + b * h, c * e + d * g, c * f + d * h,
                     a * ux + b * uy + tx, c * ux + d * uy + ty])


def brute_world(tags, local):
    parent = brute.parent_by_stk(list(tags))
    match = brute.match_from_parent(list(tags), parent)
    n = len(tags)
    out = np.empty((n, 6))
    for i in range(n):
        if tags[i] == 3:
            out[i] = out[match[i]] if match[i] >= 0 else ID
            continue
        chain = []
        j = parent[i]
        while j >= 0:
            chain.append(j)
            j = parent[j]
        w = ID
        for a in reversed(chain):          # root-most ancestor first
            w = compose(w, local[a])
        out[i] = compose(w, local[i])
    return out


def exact_locals(n, rng):
    """90-degree rotations, sign flips and small integer translations: exact in
    fp32 and fp64, and they do not commute."""
    mats = np.array([[1, 0, 0, 1], [0, -1, 1, 0], [-1, 0, 0, -1], [0, 1, -1, 0], [-1, 0, 0, 1], [1, 0, 0, -1]],
                    np.float32)
    m = mats[rng.integers(0, len(mats), n)]
    t = rng.integers(-3, 4, (n, 2)).astype(np.float32)
    return np.concatenate([m, t], 1)


def random_tags(n, rng):
    return rng.choice(np.array([0, 1, 2, 3], np.uint8), n, p=[0.4, 0.2, 0.1, 0.3])


@pytest.mark.parametrize("seed", range(20))
def test_brute_force_exact(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 120))
    tags = random_tags(n, rng)
    loc = exact_locals(n, rng)
    assert np.array_equal(oracle.tree_transform(tags, loc), brute_world(tags, loc.astype(np.float64)))


def test_brute_force_float():
    rng = np.random.default_rng(99)
    n = 300
    tags = random_tags(n, rng)
    ang = rng.uniform(-np.pi, np.pi, n)
    loc = np.stack([np.cos(ang), -np.sin(ang), np.sin(ang), np.cos(ang), rng.uniform(-1, 1, n),
                    rng.uniform(-1, 1, n)], 1).astype(np.float32)
    assert np.allclose(oracle.tree_transform(tags, loc), brute_world(tags, loc.astype(np.float64)), atol=1e-12)


def test_translation_chain_is_cumsum():
    rng = np.random.default_rng(1)
    k = 500
    tags = np.concatenate([np.ones(k, np.uint8), np.full(k, 3, np.uint8)])
    loc = np.tile(np.array([1, 0, 0, 1, 0, 0], np.float32), (2 * k, 1))
    loc[:k, 4:] = rng.integers(-5, 6, (k, 2))
    w = oracle.tree_transform(tags, loc)
    assert np.array_equal(w[:k, 4:], np.cumsum(loc[:k, 4:].astype(np.float64), 0))
    assert np.array_equal(w[k:], w[:k][::-1])     # each close echoes its node


def test_rotation_chain_period_four():
    k = 64
    tags = np.ones(k, np.uint8)
    loc = np.tile(np.array([0, -1, 1, 0, 0, 0], np.float32), (k, 1))   # +90 degrees
    w = oracle.tree_transform(tags, loc)
    R = [np.array([0, -1, 1, 0]), np.array([-1, 0, 0, -1]), np.array([0, 1, -1, 0]), np.array([1, 0, 0, 1])]
    for i in range(k):
        assert np.array_equal(w[i, :4], R[i % 4])


def test_order_matters():
    """( T(1,0) ( R90 leaf:T(0,1) ) ): world(leaf) = T(1,0) ∘ R90 ∘ T(0,1)."""
    tags = np.array([1, 1, 0, 3, 3], np.uint8)
    loc = np.array([[1, 0, 0, 1, 1, 0], [0, -1, 1, 0, 0, 0], [1, 0, 0, 1, 0, 1], [1, 0, 0, 1, 0, 0],
                    [1, 0, 0, 1, 0, 0]], np.float32)
    w = oracle.tree_transform(tags, loc)
    assert w[0].tolist() == [1, 0, 0, 1, 1, 0]
    assert w[1].tolist() == [0, -1, 1, 0, 1, 0]       # T(1,0) ∘ R90
    assert w[2].tolist() == [0, -1, 1, 0, 0, 0]       # R90·(0,1) + (1,0) = (0, 0)
    assert w[3].tolist() == w[1].tolist() and w[4].tolist() == w[0].tolist()
    # the other order differs: R90 ∘ T(1,0) puts the origin at (0, 1)
    loc2 = loc.copy()
    loc2[[0, 1]] = loc[[1, 0]]
    assert oracle.tree_transform(tags, loc2)[1].tolist() == [0, -1, 1, 0, 0, 1]


def test_underflow_and_unclosed():
    tags = np.array([3, 1, 0], np.uint8)               # R3 close, open never closed (R4)
    loc = np.array([[2, 0, 0, 2, 5, 5], [1, 0, 0, 1, 1, 1], [1, 0, 0, 1, 1, 1]], np.float32)
    w = oracle.tree_transform(tags, loc)
    assert w[0].tolist() == [1, 0, 0, 1, 0, 0]
    assert w[2].tolist() == [1, 0, 0, 1, 2, 2]
