"""Pins for oracle.paren_match (CPU only).

The oracle is Fig. 1 run literally.  It is pinned here against
things other than itself: the paper's printed values (golden fixtures), the
§3 Bic characterisation and the §4 stack-monoid characterisation
 by exhaustive enumeration, and structural invariants.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from brute import (bic_combine, bic_elem, bic_of, match_from_parent, parent_by_bic,
                   parent_by_stk, stk_combine, stk_of)

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SYM = {"(": 1, ")": 3, "x": 0}


def enc(s):
    return np.array([SYM[c] for c in s], np.uint8)


def test_bic_monoid_laws_and_examples():
    # P:98-100 examples from SPEC S:58-60, and associativity on random triples
    assert bic_combine((0, 0), (2, 1)) == (2, 1)
    assert bic_combine((0, 1), (1, 0)) == (0, 0)
    assert bic_combine((1, 0), (0, 1)) == (1, 1)
    rng = np.random.default_rng(0)
    for _ in range(5000):
        x, y, z = (tuple(int(v) for v in rng.integers(0, 6, 2)) for _ in range(3))
        assert bic_combine(bic_combine(x, y), z) == bic_combine(x, bic_combine(y, z))
        assert bic_combine((0, 0), x) == x == bic_combine(x, (0, 0))


def test_stk_monoid_laws_and_examples():
    # P:115-117 examples from SPEC S:84-86
    assert stk_combine((0, []), (1, [7])) == (1, [7])
    assert stk_combine((0, [1, 2]), (1, [])) == (0, [1])
    assert stk_combine((0, [3]), (2, [9])) == (1, [9])
    rng = np.random.default_rng(1)
    for _ in range(3000):
        vals = []
        for _ in range(3):
            a = int(rng.integers(0, 4))
            l = [int(v) for v in rng.integers(0, 100, int(rng.integers(0, 4)))]
            vals.append((a, l))
        x, y, z = vals
        assert stk_combine(stk_combine(x, y), z) == stk_combine(x, stk_combine(y, z))
        # projection to Bic is a homomorphism
        p = lambda v: (v[0], len(v[1]))
        assert p(stk_combine(x, y)) == bic_combine(p(x), p(y))


@pytest.mark.parametrize("ex", json.load(open(os.path.join(GOLD, "paren_examples.json")))["examples"],
                         ids=lambda e: repr(e["s"]))
def test_golden_examples(ex):
    s = ex["s"]
    tags = enc(s)
    match, parent = oracle.paren_match(tags)
    if "parent" in ex:
        assert parent.tolist() == ex["parent"], ex["cite"]
    if "match" in ex:
        assert match.tolist() == ex["match"], ex["cite"]
    if "bic" in ex:
        assert list(oracle.count_unmatched(tags)) == ex["bic"], ex["cite"]
        assert list(bic_of(list(tags))) == ex["bic"], ex["cite"]
    if "reverse_scan" in ex:
        t = list(tags)
        assert [list(bic_of(t, i)) for i in range(len(t))] == ex["reverse_scan"], ex["cite"]
    if "slice" in ex:
        unmatched_opens = [i for i in range(len(s)) if s[i] == "(" and match[i] == -1]
        assert unmatched_opens == ex["slice"], ex["cite"]
        assert stk_of(list(tags))[1] == ex["slice"]
    if "fig3" in ex:
        f = ex["fig3"]
        t = list(tags)
        assert len(t) == 16
        assert bic_of(t, f["i"], f["i1"])[1] == 0 and bic_of(t, f["i"] - 1, f["i1"])[1] == 1
        assert parent[f["i1"]] == f["parent_i1"] == f["i"] - 1, ex["cite"]


def _check_against_brute(tags_list):
    tags = np.array(tags_list, np.uint8)
    match, parent = oracle.paren_match(tags)
    pb = parent_by_bic(tags_list)
    ps = parent_by_stk(tags_list)
    assert parent.tolist() == pb, tags_list
    assert parent.tolist() == ps, tags_list
    assert match.tolist() == match_from_parent(tags_list, ps), tags_list


def test_exhaustive_parens_up_to_12():
    """All strings over {(,)} of length <= 12, underflowing ones included (R3)."""
    for n in range(0, 13):
        for combo in itertools.product((1, 3), repeat=n):
            _check_against_brute(list(combo))


def test_exhaustive_with_leaves_and_kinds_up_to_7():
    """All strings over {leaf, clip-open, blend-open, close} of length <= 7."""
    for n in range(0, 8):
        for combo in itertools.product((0, 1, 2, 3), repeat=n):
            _check_against_brute(list(combo))


def test_random_longer_strings():
    rng = np.random.default_rng(7)
    for trial in range(150):
        n = int(rng.integers(1, 120))
        p = rng.dirichlet([1, 1, 1, 1])
        t = rng.choice([0, 1, 2, 3, 7, 255], size=n, p=[p[0] / 3, p[1], p[2], p[3], p[0] / 3, p[0] / 3])
        _check_against_brute([int(v) for v in t])


def _invariants(tags, match, parent):
    n = tags.shape[0]
    idx = np.arange(n)
    assert np.all(parent < idx)
    has = match >= 0
    assert np.all(match[match[has]] == idx[has])                    # P:74 involution
    is_open = (tags == 1) | (tags == 2)
    is_close = tags == 3
    assert np.all(match[is_close & has] < idx[is_close & has])
    assert np.all(match[is_open & has] > idx[is_open & has])
    assert np.all(parent[is_close & has] == match[is_close & has])  # stronger version
    assert not np.any(has & ~is_open & ~is_close)
    # parents are -1 or opens
    pp = parent[parent >= 0]
    assert np.all(is_open[pp])
    # balanced span: every matched pair encloses a balanced string
    depth = np.concatenate([[0], np.cumsum(np.where(is_open, 1, np.where(is_close, -1, 0)))])
    c = idx[is_close & has]
    o = match[c]
    assert np.all(depth[o] == depth[c + 1])


def test_invariants_on_generated_configs():
    import scenegen
    for tags in [scenegen.config("C1")[0].numpy(),
                 scenegen.walk_tags(200_000, 11, p_leaf=0.3).numpy(),
                 scenegen.deep_chain_tags(100_000, 5).numpy(),
                 scenegen.walk_tags(50_000, 12, p_leaf=0.0).numpy()]:
        match, parent = oracle.paren_match(tags)
        _invariants(tags, match, parent)


def test_snapshots_recoverable_from_output():
    """every stack snapshot is recovered by following parent links to -1;
    it equals the §4 Stk reduction of the prefix."""
    rng = np.random.default_rng(3)
    t = [int(v) for v in rng.choice([0, 1, 3], size=300, p=[0.2, 0.45, 0.35])]
    match, parent = oracle.paren_match(np.array(t, np.uint8))
    for j in range(0, len(t), 7):
        chain = []
        p = parent[j]
        while p != -1:
            chain.append(int(p))
            p = parent[p]
        assert chain[::-1] == stk_of(t, 0, j)[1]
