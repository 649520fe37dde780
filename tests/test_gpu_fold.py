"""GPU parity of tree_fold (csrc/tree_fold.cu, the "up"
half; reading R17) against oracle.tree_fold, bit for bit: 2x2 matrices mod
2^32 multiplied up the tree in stream order — exactly associative, neither
commutative nor idempotent, so any reordering or overlap in the GPU's range
products would show.  Shapes: nodes inside a thread / across threads / across
tiles (one and many tiles between), deep chains, opens never closed (R4),
unmatched closes (R3), junk bytes, ragged tails; the bench-size stream is
checked on a sample of nodes and by an invariant."""
import numpy as np
import pytest
import torch

import oracle
import scenegen

pytestmark = pytest.mark.gpu
W = 2048


def payload(n, seed):
    g = np.random.default_rng(seed)
    return g.integers(0, 1 << 32, size=(n, 4), dtype=np.uint64).astype(np.uint32)


def check(t, seed=1):
    import paper_2205_11659_b200 as tb
    t = np.ascontiguousarray(np.asarray(t, dtype=np.uint8))
    n = len(t)
    x = payload(n, seed)
    ref = oracle.tree_fold(t, x)
    tc = torch.from_numpy(t).cuda()
    m, _ = tb.paren_match(tc)
    got = tb.tree_fold(tc, torch.from_numpy(x.view(np.int32)).cuda(), m).cpu().numpy().view(np.uint32)
    if not np.array_equal(got, ref):
        bad = np.nonzero((got != ref).any(1))[0]
        raise AssertionError(f"{len(bad)} mismatches (n={n}), first {bad[:5].tolist()} tags {t[bad[:5]].tolist()}")


def walk(n, seed, **kw):
    return scenegen.walk_tags(n, seed, **kw).numpy()


def test_tiny():
    for v in (0, 1, 2, 3, 9):
        check([v])
    for n in (2, 5, 15, 16, 17, 33, 100):
        check(walk(n, n))
    check([1, 0, 0, 3])
    check([3, 3, 1, 1, 0, 0])


@pytest.mark.parametrize("n", [W - 1, W, W + 1, 3 * W + 7, 64 * W, 64 * W + 999])
def test_random_walks(n):
    check(walk(n, 1))
    check(walk(n, 2, p_leaf=0.2))
    check(walk(n, 3, p_leaf=0.9))


def test_deep_and_degenerate():
    check(scenegen.deep_chain_tags(40 * W, 5).numpy())
    check(scenegen.deep_chain_tags(40 * W + 3, 6, leaves_mid=True).numpy())
    t = np.zeros(10 * W, np.uint8)
    t[::2] = 1  # opens never closed, leaves between (R4)
    check(t)
    t = np.full(5 * W, 3, np.uint8)
    t[1::3] = 0  # unmatched closes (R3)
    check(t)
    # one node spanning many tiles: the hierarchy's disjoint pieces on both sides
    t = np.zeros(3000 * W, np.uint8)
    t[5] = 1
    t[-7] = 3
    check(t)


def test_junk_bytes():
    t = walk(20 * W + 5, 9)
    g = np.random.default_rng(4)
    sel = g.random(len(t)) < 0.1
    t[sel] = g.integers(4, 256, size=sel.sum())
    check(t)


def test_c5_sampled():
    """C5 size (2^27): nodes sampled, each checked against the product of its
    leaves computed on the host in int64 mod 2^32."""
    import paper_2205_11659_b200 as tb
    n = 1 << 27
    t = scenegen.walk_tags(n, 4, device="cuda")
    x = torch.randint(0, 1 << 31, (n, 4), dtype=torch.int32, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    m, _ = tb.paren_match(t)
    out = tb.tree_fold(t, x, m)
    torch.cuda.synchronize()
    mm = m.cpu().numpy()
    tt = t.cpu().numpy()
    opens = np.nonzero(((tt == 1) | (tt == 2)) & (mm >= 0))[0]
    g = np.random.default_rng(0)
    span = mm[opens] - opens
    small = opens[span < 5000]
    pick = np.concatenate([g.choice(small, 300, replace=False), opens[np.argsort(span)[-3:]]])
    MASK = (1 << 32) - 1
    xs = x.cpu().numpy().view(np.uint32).astype(np.uint64)
    leaf = ~np.isin(tt, [1, 2, 3])
    for o in pick[:303]:
        c = int(mm[o])
        if c - o > 200000:
            continue
        a, b, cc, d = 1, 0, 0, 1
        for j in np.nonzero(leaf[o + 1:c])[0] + o + 1:
            e, f, gg, h = (int(v) for v in xs[j])
            a, b, cc, d = (a * e + b * gg) & MASK, (a * f + b * h) & MASK, (cc * e + d * gg) & MASK, (cc * f + d * h) & MASK
        want = np.array([a, b, cc, d], np.uint64).astype(np.uint32)
        got = out[o].cpu().numpy().view(np.uint32)
        assert np.array_equal(got, want), o
        assert np.array_equal(out[c].cpu().numpy().view(np.uint32), want), c
