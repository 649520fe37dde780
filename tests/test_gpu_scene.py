"""GPU parity of the fused stream-compaction front end
(paren_match_tree_bbox_scene): the FULL scene
stream goes into the tile pass, dropped elements are null there, and every
output of a kept element lands at its compacted index.  Reference: the kept
subsequence selected with numpy, then the oracle's paren_match / tree_bbox on
it — bit for bit (indices exactly, boxes as fp32 patterns); tags_out and
index_out are the kept bytes and their full-stream positions.  Shapes: the
S1 scene generator at several command densities (none, half, 90 %, all
dropped), tile boundaries and ragged tails, kept junk bytes (leaves), deep
chains broken up by commands, and the bench size checked against the
two-step path (compact_scene, then the fused call)."""
import numpy as np
import pytest
import torch

import oracle
import scenegen

pytestmark = pytest.mark.gpu
W = 2048
KEEP03 = bytes([1, 1, 1, 1] + [0] * 252)


def reference(scene, boxes, keep):
    km = np.frombuffer(keep, np.uint8).astype(bool)
    sel = km[scene]
    t = scene[sel]
    b = boxes[sel]
    m, p = oracle.paren_match(t)
    o = oracle.tree_bbox(t, b)
    return t, np.nonzero(sel)[0].astype(np.int32), m, p, o


def check(scene, boxes, keep=KEEP03):
    import paper_2205_11659_b200 as tb
    scene = np.ascontiguousarray(scene, np.uint8)
    boxes = np.ascontiguousarray(boxes, np.float32).reshape(-1, 4)
    t_r, i_r, m_r, p_r, o_r = reference(scene, boxes, keep)
    t, i, m, p, o, k = tb.paren_match_tree_bbox_scene(torch.from_numpy(scene).cuda(), torch.from_numpy(boxes).cuda(),
                                                     keep)
    assert k == len(t_r)
    for name, got, ref in (("tags", t, t_r), ("index", i, i_r), ("match", m, m_r), ("parent", p, p_r)):
        g = got.cpu().numpy()
        if not np.array_equal(g, ref):
            bad = np.nonzero(g != ref)[0]
            raise AssertionError(f"{name}: {len(bad)} mismatches of {k}, first {bad[:5].tolist()}: "
                                 f"got {g[bad[:3]].tolist()} want {ref[bad[:3]].tolist()}")
    g = o.cpu().numpy().view(np.uint32)
    if not np.array_equal(g, o_r.view(np.uint32)):
        bad = np.nonzero((g != o_r.view(np.uint32)).any(1))[0]
        raise AssertionError(f"node_bbox: {len(bad)} mismatches of {k}, first {bad[:5].tolist()}")
    _, _, _, _, o2, k2 = tb.paren_match_tree_bbox_scene(torch.from_numpy(scene).cuda(),
                                                       torch.from_numpy(boxes).cuda(), keep, pm=False)
    assert k2 == k and np.array_equal(o2.cpu().numpy().view(np.uint32), o_r.view(np.uint32))


@pytest.mark.parametrize("p_cmd", [0.0, 0.5, 0.9])
@pytest.mark.parametrize("n", [1, 17, W - 1, W, W + 5, 37 * W + 11])
def test_scene_streams(n, p_cmd):
    s, b = scenegen.scene_stream(n, 3, p_cmd=p_cmd)
    check(s.numpy(), b.numpy())


def test_all_dropped_and_empty():
    import paper_2205_11659_b200 as tb
    s = np.full(5 * W + 3, 9, np.uint8)
    b = np.zeros((len(s), 4), np.float32)
    check(s, b)
    _, _, _, _, _, k = tb.paren_match_tree_bbox_scene(torch.empty(0, dtype=torch.uint8, device="cuda"),
                                                     torch.empty((0, 4), device="cuda"))
    assert k == 0


def test_kept_junk_is_a_leaf():
    s, b = scenegen.scene_stream(20 * W + 9, 5, p_cmd=0.4)
    keep = bytearray(KEEP03)
    keep[7] = keep[200] = 1
    s = s.numpy().copy()
    s[::13] = 200
    check(s, b.numpy(), bytes(keep))


def test_deep_chain_with_commands():
    n = 64 * W
    t = scenegen.deep_chain_tags(n, 2).numpy()
    g = np.random.default_rng(1)
    cmd = g.random(2 * n) < 0.5
    s = np.empty(2 * n, np.uint8)
    s[cmd] = g.integers(4, 16, size=cmd.sum())
    s[~cmd] = np.resize(t, (~cmd).sum())
    b = g.normal(size=(2 * n, 4)).astype(np.float32) * 100
    check(s, b)


def test_bench_size_matches_two_step():
    """2^27 elements of S1: the fused call equals compact_scene + paren_match_tree_bbox."""
    import paper_2205_11659_b200 as tb
    n = 1 << 27
    s, b = scenegen.scene_stream(n, 4, p_cmd=0.5, device="cuda")
    t, i, m, p, o, k = tb.paren_match_tree_bbox_scene(s, b)
    t2, b2, i2 = tb.compact_scene(s, b, KEEP03)
    m2, p2, o2 = tb.paren_match_tree_bbox(t2.contiguous(), b2.contiguous())
    torch.cuda.synchronize()
    assert k == t2.numel()
    assert torch.equal(t, t2) and torch.equal(i, i2) and torch.equal(m, m2) and torch.equal(p, p2)
    assert torch.equal(o.view(torch.int32), o2.view(torch.int32))
