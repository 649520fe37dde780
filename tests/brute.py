"""Independent brute-force definitions used to PIN the oracle (tests only).

Nothing here is shared with oracle/ or with the CUDA path.  Each function is a
second, different definition of what the paper computes, chosen so that a
plausible slip in the oracle (a dropped term, a wrong index, a swapped min/max)
disagrees with one of them:

* ``bic_combine`` / ``bic_of``       — §3 P:96-102 (the ⊕ of the bicyclic semigroup)
* ``parent_by_bic``                  — §3: parenmatch[j] = max i with
                                        Bic(s[i..j]).b = 1 (O(n^2))
* ``stk_combine`` / ``parent_by_stk``— §4: last(Stk(enum(s)[..j]))
* ``bbox_by_ancestors``              — §1/§6: leaf = own ∩ all clip
                                        ancestors (ancestor walk); node union =
                                        range loop over clipped leaves
Elements: 1/2 = open (clip/blend), 3 = close, anything else = leaf.
"""
from __future__ import annotations

import struct

OPEN = (1, 2)
CLOSE = 3


def bic_elem(t):
    """open -> (0,1), close -> (1,0); leaf -> identity (DESIGN R2)."""
    if t in OPEN:
        return (0, 1)
    if t == CLOSE:
        return (1, 0)
    return (0, 0)


def bic_combine(x, y):
    """(a,b)⊕(c,d) = (a+c-min(b,c), b+d-min(b,c))."""
    a, b = x
    c, d = y
    m = min(b, c)
    return (a + c - m, b + d - m)


def bic_of(tags, i=0, j=None):
    """Bic(s[i..j]) — ⊕-reduction over the slice."""
    j = len(tags) if j is None else j
    acc = (0, 0)
    for k in range(i, j):
        acc = bic_combine(acc, bic_elem(tags[k]))
    return acc


def parent_by_bic(tags):
    """parent[j] = max i such that Bic(s[i..j]).b == 1, else -1."""
    n = len(tags)
    out = []
    for j in range(n):
        found = -1
        for i in range(j - 1, -1, -1):
            if bic_of(tags, i, j)[1] == 1:
                found = i
                break
        out.append(found)
    return out


def stk_elem(t, idx):
    """§4: open with value x -> (0,[x]); close -> (1,[]); leaf -> (0,[])."""
    if t in OPEN:
        return (0, [idx])
    if t == CLOSE:
        return (1, [])
    return (0, [])


def stk_combine(x, y):
    """(a0,l0)⊕(a1,l1) = (a0+a1-min(|l0|,a1), l0[..max(0,|l0|-a1)] + l1)."""
    a0, l0 = x
    a1, l1 = y
    return (a0 + a1 - min(len(l0), a1), l0[: max(0, len(l0) - a1)] + l1)


def stk_of(tags, i=0, j=None):
    j = len(tags) if j is None else j
    acc = (0, [])
    for k in range(i, j):
        acc = stk_combine(acc, stk_elem(tags[k], k))
    return acc


def parent_by_stk(tags):
    """parenmatch(s)[j] = last(Stk(enum(s)[..j])), -1 for the empty stack."""
    out = []
    acc = (0, [])
    for j, t in enumerate(tags):
        out.append(acc[1][-1] if acc[1] else -1)
        acc = stk_combine(acc, stk_elem(t, j))
    return out


def match_from_parent(tags, parent):
    """Classical partner: a close with parent p >= 0 is matched to p."""
    n = len(tags)
    m = [-1] * n
    for j in range(n):
        if tags[j] == CLOSE and parent[j] >= 0:
            m[j] = parent[j]
            m[parent[j]] = j
    return m


# ----------------------------------------------------------------------------
# Boxes.  Coordinates are handled as fp32 bit patterns; min/max order -0
# below +0 through an unsigned totalOrder key (a different mechanism from the
# oracle's comparisons and from the kernels' FMNMX); NaN operands are ignored
# (DESIGN R12).
# ----------------------------------------------------------------------------

def f2u(x: float) -> int:
    return struct.unpack("<I", struct.pack("<f", x))[0]


def u2f(u: int) -> float:
    return struct.unpack("<f", struct.pack("<I", u & 0xFFFFFFFF))[0]


def _key(u: int) -> int:
    return (~u) & 0xFFFFFFFF if u & 0x80000000 else u | 0x80000000


def _isnan(u: int) -> bool:
    return (u & 0x7FFFFFFF) > 0x7F800000


QNAN = 0x7FFFFFFF  # canonical NaN when both operands are NaN (DESIGN R12)


def umin(p: int, q: int) -> int:
    if _isnan(p) and _isnan(q):
        return QNAN
    if _isnan(p):
        return q
    if _isnan(q):
        return p
    return p if _key(p) <= _key(q) else q


def umax(p: int, q: int) -> int:
    if _isnan(p) and _isnan(q):
        return QNAN
    if _isnan(p):
        return q
    if _isnan(q):
        return p
    return q if _key(p) <= _key(q) else p


INF_U = (f2u(float("-inf")), f2u(float("-inf")), f2u(float("inf")), f2u(float("inf")))
EMPTY_U = (f2u(float("inf")), f2u(float("inf")), f2u(float("-inf")), f2u(float("-inf")))


def isect_u(p, q):
    return (umax(p[0], q[0]), umax(p[1], q[1]), umin(p[2], q[2]), umin(p[3], q[3]))


def union_u(p, q):
    return (umin(p[0], q[0]), umin(p[1], q[1]), umax(p[2], q[2]), umax(p[3], q[3]))


def bbox_by_ancestors(tags, boxes_u):
    """Brute force of P:24 from the tree structure given by parent_by_stk.

    boxes_u: list of 4-tuples of fp32 bit patterns.  Returns the same shape.
    leaf / clip open: own box ∩ boxes of all clip-open ancestors (ancestor walk)
    close c matched to o: raw union of clipped leaves strictly inside (o, c)
    blend open o: same union (matched) or union over (o, n) (unmatched, R4)
    unmatched close: EMPTY.
    """
    n = len(tags)
    parent = parent_by_stk(tags)
    match = match_from_parent(tags, parent)
    clipped = [None] * n
    out = [None] * n
    for i in range(n):
        t = tags[i]
        if t == CLOSE or t == 2:
            continue
        c = isect_u(boxes_u[i], INF_U)  # ∩ over an empty ancestor set = INF (R11)
        p = parent[i]
        while p != -1:
            if tags[p] == 1:
                c = isect_u(c, boxes_u[p])
            p = parent[p]
        clipped[i] = c
        out[i] = c

    def range_union(lo, hi):
        acc = EMPTY_U
        for k in range(lo, hi):
            if tags[k] not in OPEN and tags[k] != CLOSE:
                acc = union_u(acc, clipped[k])
        return acc

    for i in range(n):
        t = tags[i]
        if t == CLOSE:
            o = match[i]
            out[i] = EMPTY_U if o < 0 else range_union(o + 1, i)
        elif t == 2:
            c = match[i]
            out[i] = range_union(i + 1, n if c < 0 else c)
    return out
