"""Pins of oracle.bin_leaves (reading R16): culling +
binning of the clipped leaf boxes.  Independent of oracle.c: a brute-force
double loop over bins x leaves with the overlap definition written out, and a
hand-checked example."""
import numpy as np
import pytest

import oracle
import scenegen


def brute(tags, box, gw, gh, bs):
    lists = [[] for _ in range(gw * gh)]
    for e in range(len(tags)):
        if tags[e] in (1, 2, 3):
            continue
        x0, y0, x1, y1 = (float(v) for v in box[e])
        if not (x0 < x1 and y0 < y1):
            continue
        for by in range(gh):
            for bx in range(gw):
                if x0 < (bx + 1) * bs and x1 > bx * bs and y0 < (by + 1) * bs and y1 > by * bs:
                    lists[by * gw + bx].append(e)
    counts = np.array([len(l) for l in lists], np.int32)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    items = np.array([e for l in lists for e in l], np.int32)
    return counts, offsets, items


def test_hand_example():
    t = np.array([0, 1, 0, 3, 0], np.uint8)
    b = np.array([[1, 1, 20, 5], [0, 0, 0, 0], [30, 30, 10, 40], [0, 0, 0, 0], [-5, 15, 3, 17]], np.float32)
    c, o, it = oracle.bin_leaves(t, b, 4, 4, 16.0)
    assert c.tolist()[:5] == [2, 1, 0, 0, 1] and c.sum() == 4
    assert it.tolist() == [0, 4, 0, 4]          # bin 0: leaves 0 and 4; bin 1: 0; bin 4: 4


@pytest.mark.parametrize("seed", range(6))
def test_brute_force(seed):
    n = 400
    tags = scenegen.walk_tags(n, seed, p_leaf=0.5)
    boxes = scenegen.boxes(n, seed, tags).numpy()
    nb = oracle.tree_bbox(tags.numpy(), boxes)
    gw, gh, bs = 9, 7, 512.0
    got = oracle.bin_leaves(tags.numpy(), nb, gw, gh, bs)
    ref = brute(tags.numpy(), nb, gw, gh, bs)
    for g, r in zip(got, ref):
        assert np.array_equal(g, r)
