"""Stream compaction front end: compact_scene equals
the plain definition (a boolean-mask gather, numpy), keeps order, and the
compacted stream feeds the path.  The generator's kept subsequence is the
walk of walk_tags (CPU pin)."""
import numpy as np
import pytest
import torch

import oracle
import scenegen

KEEP = np.frombuffer(scenegen.SCENE_KEEP_MAP, np.uint8)


def test_scene_stream_kept_is_walk():
    s, b = scenegen.scene_stream(20_000, 3)
    m = KEEP[s.numpy()] != 0
    assert np.array_equal(s.numpy()[m], scenegen.walk_tags(int(m.sum()), 3).numpy())
    assert (s.numpy()[~m] >= 4).all()


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 4095, 4096, 4097, 300_001, (1 << 22) + 7])
def test_gpu_compaction_is_mask_gather(n):
    import paper_2205_11659_b200 as tb
    s, b = scenegen.scene_stream(n, n % 7 + 1)
    t_out, b_out, idx = tb.compact_scene(s.cuda(), b.cuda(), scenegen.SCENE_KEEP_MAP)
    torch.cuda.synchronize()
    m = KEEP[s.numpy()] != 0
    assert np.array_equal(idx.cpu().numpy(), np.nonzero(m)[0])
    assert np.array_equal(t_out.cpu().numpy(), s.numpy()[m])
    assert np.array_equal(b_out.cpu().numpy().view(np.uint32), b.numpy()[m].view(np.uint32))


@pytest.mark.gpu
def test_gpu_all_or_nothing():
    import paper_2205_11659_b200 as tb
    s = torch.full((10_000,), 9, dtype=torch.uint8)
    t_out, _, idx = tb.compact_scene(s.cuda(), None, scenegen.SCENE_KEEP_MAP)
    assert t_out.numel() == 0 and idx.numel() == 0
    s = torch.zeros(10_000, dtype=torch.uint8)
    t_out, _, idx = tb.compact_scene(s.cuda(), None, scenegen.SCENE_KEEP_MAP)
    assert torch.equal(idx.cpu(), torch.arange(10_000, dtype=torch.int32))


@pytest.mark.gpu
def test_gpu_pipeline_on_compacted_stream():
    """full stream -> compaction -> paren_match + tree_bbox_matched -> results
    scattered back to the full stream's positions."""
    import paper_2205_11659_b200 as tb
    s, b = scenegen.scene_stream(1_000_003, 5, p_cmd=0.6)
    t, bx, idx = tb.compact_scene(s.cuda(), b.cuda(), scenegen.SCENE_KEEP_MAP)
    m, p = tb.paren_match(t)
    out = tb.tree_bbox_matched(t, bx, m, p)
    full = torch.zeros((s.numel(), 4), dtype=torch.float32, device="cuda")
    full[idx.long()] = out
    torch.cuda.synchronize()
    mask = KEEP[s.numpy()] != 0
    ref = oracle.tree_bbox(s.numpy()[mask], b.numpy()[mask])
    assert np.array_equal(full.cpu().numpy()[mask].view(np.uint32), ref.view(np.uint32))
