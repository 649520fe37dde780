"""Pins of oracle.tree_fold (R17: 2x2 matrices mod 2^32 multiplied up the
tree in stream order) against what the definition fixes, independently of the
oracle's stack walk:

* brute force: every node's value is the ordered product of the leaf payloads
  strictly between its open and its close (never closed: to the stream end,
  R4), with the bracket pairs found by a separate textbook matching and the
  products taken with Python integers mod 2^32;
* closed form: with one payload M on every leaf a node's value is M^k, k = its
  leaf count;
* order: swapping two leaves under one node changes its value (A B != B A)
  and equals the product in the new order;
* leaves echo their payload, unmatched closes get the identity (R3)."""
import numpy as np

import oracle

MASK = (1 << 32) - 1
I = (1, 0, 0, 1)


def mul(X, Y):
    a, b, c, d = X
    e, f, g, h = Y
    return ((a * e + b * g) & MASK, (a * f + b * h) & MASK, (c * e + d * g) & MASK, (c * f + d * h) & MASK)


def pairs(tags):
    st, m = [], {}
    for i, t in enumerate(tags):
        if t in (1, 2):
            st.append(i)
        elif t == 3 and st:
            o = st.pop()
            m[o] = i
    return m, st  # closed pairs, opens never closed


def brute(tags, x):
    n = len(tags)
    out = [None] * n
    leaf = [t not in (1, 2, 3) for t in tags]
    m, left = pairs(tags)
    closed = set(m.values())
    for i in range(n):
        if leaf[i]:
            out[i] = tuple(int(v) for v in x[i])
        elif tags[i] == 3 and i not in closed:
            out[i] = I
    for o, c in list(m.items()) + [(o, n) for o in left]:
        p = I
        for j in range(o + 1, c):
            if leaf[j]:
                p = mul(p, tuple(int(v) for v in x[j]))
        out[o] = p
        if c < n:
            out[c] = p
    return np.array(out, dtype=np.uint64).astype(np.uint32)


def test_brute_force_random():
    rng = np.random.default_rng(3)
    for trial in range(300):
        n = int(rng.integers(1, 40))
        tags = rng.choice([0, 0, 1, 2, 3, 3, 7], size=n).astype(np.uint8)
        x = rng.integers(0, 1 << 32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
        assert np.array_equal(oracle.tree_fold(tags, x), brute(list(tags), x)), trial


def test_power_closed_form():
    M = (3, 1, 4, 1)
    tags = np.array([1, 0, 2, 0, 0, 3, 0, 3, 0], np.uint8)  # outer node: 4 leaves, inner: 2
    x = np.tile(np.array(M, np.uint32), (9, 1))
    got = oracle.tree_fold(tags, x)
    P = I
    pw = [I]
    for _ in range(4):
        P = mul(P, M)
        pw.append(P)
    assert tuple(got[0]) == pw[4] and tuple(got[7]) == pw[4]   # outer open / close
    assert tuple(got[2]) == pw[2] and tuple(got[5]) == pw[2]   # inner
    assert tuple(got[8]) == M                                   # a root leaf echoes its payload


def test_order_matters():
    A, B = (1, 2, 0, 1), (1, 0, 3, 1)
    assert mul(A, B) != mul(B, A)
    tags = np.array([1, 0, 0, 3], np.uint8)
    ab = oracle.tree_fold(tags, np.array([I, A, B, I], np.uint32))
    ba = oracle.tree_fold(tags, np.array([I, B, A, I], np.uint32))
    assert tuple(ab[0]) == mul(A, B) and tuple(ba[0]) == mul(B, A) and tuple(ab[3]) == mul(A, B)


def test_unmatched_and_never_closed():
    A = (2, 0, 0, 5)
    tags = np.array([3, 0, 1, 0, 0], np.uint8)
    got = oracle.tree_fold(tags, np.array([A, A, I, A, A], np.uint32))
    assert tuple(got[0]) == I                       # R3
    assert tuple(got[2]) == mul(A, A)               # R4: leaves after the open to the end
