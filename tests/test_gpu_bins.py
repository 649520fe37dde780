"""GPU parity of bin_leaves vs the oracle:
counts and offsets exactly; the items of each bin as sets (their order inside
a bin is unspecified), which the oracle lists in leaf order."""
import numpy as np
import pytest
import torch

import oracle
import scenegen

pytestmark = pytest.mark.gpu


def check(tags, boxes, gw, gh, bs):
    import paper_2205_11659_b200 as tb
    nb_ref = oracle.tree_bbox(tags.numpy(), boxes.numpy())
    c_ref, o_ref, it_ref = oracle.bin_leaves(tags.numpy(), nb_ref, gw, gh, bs)
    t = tags.cuda()
    node = tb.tree_bbox(t, boxes.cuda())
    c, o, it = tb.bin_leaves(t, node, gw, gh, bs)
    torch.cuda.synchronize()
    c, o, it = c.cpu().numpy(), o.cpu().numpy(), it.cpu().numpy()
    assert np.array_equal(c, c_ref) and np.array_equal(o, o_ref)
    for k in range(gw * gh):
        seg = np.sort(it[o[k]:o[k + 1]])
        assert np.array_equal(seg, it_ref[o_ref[k]:o_ref[k + 1]]), k
    return len(it)


@pytest.mark.parametrize("n,gw,gh,bs", [(1, 4, 4, 64.0), (5000, 7, 5, 700.0), (300_001, 16, 16, 256.0),
                                        ((1 << 20) + 3, 64, 32, 100.0)])
def test_random_scenes(n, gw, gh, bs):
    tags = scenegen.walk_tags(n, n % 11, p_leaf=0.6)
    check(tags, scenegen.boxes(n, n % 5, tags), gw, gh, bs)


def test_special_boxes():
    """Inverted, infinite, off-screen and NaN-free edge boxes; bin edges exactly."""
    tags = torch.zeros(9, dtype=torch.uint8)
    inf = float("inf")
    boxes = torch.tensor([[0, 0, 64, 64], [64, 64, 128, 128], [63.999, 0, 64, 1], [-inf, -inf, inf, inf],
                          [10, 10, 5, 20], [-100, -100, -1, -1], [500, 500, 600, 600], [0, 0, 0, 10],
                          [1e30, 0, inf, 1]], dtype=torch.float32)
    check(tags, boxes, 4, 4, 64.0)


def test_grid_over_shared_histogram():
    """More bins than the per-CTA shared histogram holds (global-atomic counts)."""
    tags = scenegen.walk_tags(200_003, 3, p_leaf=0.6)
    check(tags, scenegen.boxes(200_003, 2, tags), 100, 60, 50.0)


def test_streaming_fill_fallback():
    """The list of binned leaves overflowing its capacity: the streaming fill."""
    import paper_2205_11659_b200 as tb
    lib = tb.load()
    old = lib.tb_debug_bins_cap(16)
    try:
        tags = scenegen.walk_tags(300_001, 4, p_leaf=0.6)
        assert check(tags, scenegen.boxes(300_001, 3, tags), 16, 16, 256.0) > 16  # the list overflowed
    finally:
        lib.tb_debug_bins_cap(old)
