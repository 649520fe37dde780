"""The Python binding rejects bad buffers before any library call touches them
(ADVICE r1): wrong dtype, size, device or layout of every host-buffer and
device-buffer argument raises TypeError / ValueError (CPU only: the checks
run before the first CUDA call)."""
import pytest
import torch

import paper_2205_11659_b200 as tb


def test_host_wrappers_validate():
    n = 64
    t = torch.zeros(n, dtype=torch.uint8)
    b = torch.zeros((n, 4), dtype=torch.float32)
    m = torch.zeros(n, dtype=torch.int32)
    p = torch.zeros(n, dtype=torch.int32)
    o = torch.zeros((n, 4), dtype=torch.float32)
    with pytest.raises(ValueError):
        tb.paren_match_host(t, m[:-1], p)
    with pytest.raises(TypeError):
        tb.paren_match_host(t, m.float(), p)
    with pytest.raises(ValueError):
        tb.tree_bbox_host(t, b[:-1], o)
    with pytest.raises(ValueError):
        tb.tree_bbox_host(t, b, o.t())  # not contiguous
    with pytest.raises(TypeError):
        tb.paren_match_tree_bbox_host(t.int(), b, m, p, o)
    with pytest.raises(ValueError):
        tb.paren_match_tree_bbox_host(t, b, m, p, o[:3])
    with pytest.raises(TypeError):
        tb.paren_match_tree_bbox_host(t, b, m, p, o.double())


def test_device_wrappers_reject_host_tensors():
    t = torch.zeros(8, dtype=torch.uint8)
    with pytest.raises(TypeError):
        tb.paren_match(t)
    with pytest.raises(TypeError):
        tb.paren_match_tree_bbox(t, torch.zeros((8, 4)))
