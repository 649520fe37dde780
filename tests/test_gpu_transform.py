"""GPU parity of tree_transform (reading R15) vs the
oracle.  Exact subset (90-degree rotations, sign flips, integer translations:
every product is exact in fp32, and they do not commute): bit-exact.  General
rotations: within a bound derived from the arithmetic (DESIGN R15): with u =
2^-24, each fused composition of orthonormal matrices adds at most 4u per
entry, so an element at depth d is within 16 u (d + 1)^2 (1 + |world|)."""
import numpy as np
import pytest
import torch

import oracle
import scenegen
from test_oracle_transform import exact_locals

pytestmark = pytest.mark.gpu


def run(tags_np, loc_np):
    import paper_2205_11659_b200 as tb
    t = torch.from_numpy(np.ascontiguousarray(tags_np)).cuda()
    m, p = tb.paren_match(t)
    w = tb.tree_transform(t, torch.from_numpy(np.ascontiguousarray(loc_np)).cuda(), m, p)
    torch.cuda.synchronize()
    return w.cpu().numpy().astype(np.float64)


def check_exact(tags_np, seed):
    rng = np.random.default_rng(seed)
    loc = exact_locals(len(tags_np), rng)
    got = run(tags_np, loc)
    ref = oracle.tree_transform(tags_np, loc)
    bad = np.nonzero((got != ref).any(1))[0]
    assert len(bad) == 0, (bad[:10], len(bad), got[bad[:2]], ref[bad[:2]])


@pytest.mark.parametrize("n", [1, 7, 1023, 1024, 1025, 4097, 100_003, (1 << 20) + 5])
def test_exact_random_walks(n):
    check_exact(scenegen.walk_tags(n, n % 13, p_leaf=0.4).numpy(), n)


def test_exact_degenerate():
    for t in (np.full(70_000, 1, np.uint8), np.full(70_000, 2, np.uint8), np.full(9000, 3, np.uint8),
              np.zeros(5000, np.uint8), scenegen.deep_chain_tags(1 << 20, 3, leaves_mid=True).numpy()):
        check_exact(t, len(t))


def test_exact_underflow_heavy():
    g = torch.Generator().manual_seed(7)
    t = torch.multinomial(torch.tensor([0.3, 0.15, 0.1, 0.45]), 300_000, replacement=True, generator=g)
    check_exact(t.to(torch.uint8).numpy(), 7)


def depth_of(tags_np):
    _, parent = oracle.paren_match(tags_np)
    d = np.zeros(len(tags_np), np.int64)
    cur = parent.astype(np.int64)
    while (cur >= 0).any():
        d += cur >= 0
        cur = np.where(cur >= 0, parent[np.maximum(cur, 0)], -1)
    return d


@pytest.mark.parametrize("n", [50_000, 1 << 18])
def test_float_rotations_within_bound(n):
    rng = np.random.default_rng(n)
    tags = scenegen.walk_tags(n, 5, p_leaf=0.5).numpy()
    ang = rng.uniform(-np.pi, np.pi, n)
    loc = np.stack([np.cos(ang), -np.sin(ang), np.sin(ang), np.cos(ang), rng.uniform(-1, 1, n),
                    rng.uniform(-1, 1, n)], 1).astype(np.float32)
    got = run(tags, loc)
    ref = oracle.tree_transform(tags, loc)
    d = depth_of(tags)[:, None]
    bound = 16 * 2.0 ** -24 * (d + 1) ** 2 * (1 + np.abs(ref))
    assert (np.abs(got - ref) <= bound).all(), float((np.abs(got - ref) / bound).max())
