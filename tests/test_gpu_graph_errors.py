"""CUDA-graph capture of the workspace entry points (no allocation, no host
synchronisation inside: the header's promise) and the host-checkable error
codes of the newer entry points."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import scenegen

pytestmark = pytest.mark.gpu


def lib():
    import paper_2205_11659_b200 as tb
    L = tb.load()
    P, I64, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t
    L.paren_match_ws.argtypes = [P, I64, P, P, P, SZ, P]
    L.tree_bbox_matched_ws.argtypes = [P, P, P, P, I64, P, P, SZ, P]
    return L


def test_graph_capture_and_replay():
    L = lib()
    n = 300_007
    tags = scenegen.walk_tags(n, 17, p_leaf=0.5)
    boxes = scenegen.boxes(n, 17, tags)
    t, b = tags.cuda(), boxes.cuda()
    m = torch.empty(n, dtype=torch.int32, device="cuda")
    p = torch.empty_like(m)
    out = torch.empty_like(b)
    wpm = torch.empty(L.paren_match_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    wbb = torch.empty(L.tree_bbox_matched_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()

    def step(stream):
        h = stream.cuda_stream
        assert L.paren_match_ws(t.data_ptr(), n, m.data_ptr(), p.data_ptr(), wpm.data_ptr(), wpm.numel(), h) == 0
        assert L.tree_bbox_matched_ws(t.data_ptr(), b.data_ptr(), m.data_ptr(), p.data_ptr(), n, out.data_ptr(),
                                      wbb.data_ptr(), wbb.numel(), h) == 0

    with torch.cuda.stream(s):
        step(s)  # warm-up outside capture (one-time kernel attribute setup)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step(s)
    m.fill_(7)
    p.fill_(7)
    out.fill_(7)
    g.replay()
    torch.cuda.synchronize()
    m_ref, p_ref = oracle.paren_match(tags.numpy())
    ref = oracle.tree_bbox(tags.numpy(), boxes.numpy())
    assert np.array_equal(m.cpu().numpy(), m_ref) and np.array_equal(p.cpu().numpy(), p_ref)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))


def test_error_codes_new_entry_points():
    import paper_2205_11659_b200 as tb
    L = tb.load()
    n = 64
    t = torch.zeros(n, dtype=torch.uint8, device="cuda")
    i32 = torch.zeros(4 * n, dtype=torch.int32, device="cuda")
    f = torch.zeros(8 * n, dtype=torch.float32, device="cuda")
    P = lambda x, off=0: x.data_ptr() + off  # noqa: E731
    # tree_bbox_matched: misaligned match, aliasing output, negative n, null
    assert L.tree_bbox_matched(P(t), P(f), P(i32, 4), P(i32, 512), n, P(f, 4 * n * 4), 0) == -2
    assert L.tree_bbox_matched(P(t), P(f), P(i32), P(i32, 512), n, P(f), 0) == -3
    assert L.tree_bbox_matched(P(t), P(f), P(i32), P(i32, 512), -1, P(f, 4 * n * 4), 0) == -1
    assert L.tree_bbox_matched(P(t), P(f), 0, P(i32, 512), n, P(f, 4 * n * 4), 0) == -1
    # tree_transform: world overlapping local, misaligned local
    assert L.tree_transform(P(t), P(f), P(i32), P(i32, 512), n, P(f, 16), 0) == -3
    assert L.tree_transform(P(t), P(f, 4), P(i32), P(i32, 512), 8, P(f, 1024), 0) == -2
    # paren_match_bytes: null class map
    assert L.paren_match_bytes(P(t), n, None, P(i32), P(i32, 512), 0) == -1
    # n == 0 is a successful no-op everywhere
    assert L.tree_bbox_matched(0, 0, 0, 0, 0, 0, 0) == 0
    assert L.tree_transform(0, 0, 0, 0, 0, 0, 0) == 0


def test_graph_capture_fused_call():
    """paren_match_tree_bbox forks a side stream and joins it back: capturable
    (after one warm-up call on the same stream sized its workspace)."""
    import paper_2205_11659_b200 as tb
    n = 250_003
    tags = scenegen.walk_tags(n, 23, p_leaf=0.5)
    boxes = scenegen.boxes(n, 23, tags)
    t, b = tags.cuda(), boxes.cuda()
    m = torch.empty(n, dtype=torch.int32, device="cuda")
    p = torch.empty_like(m)
    out = torch.empty_like(b)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        tb.paren_match_tree_bbox(t, b, m, p, out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        tb.paren_match_tree_bbox(t, b, m, p, out)
    m.fill_(7)
    p.fill_(7)
    out.fill_(7)
    g.replay()
    torch.cuda.synchronize()
    m_ref, p_ref = oracle.paren_match(tags.numpy())
    ref = oracle.tree_bbox(tags.numpy(), boxes.numpy())
    assert np.array_equal(m.cpu().numpy(), m_ref) and np.array_equal(p.cpu().numpy(), p_ref)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))


def test_concurrent_callers_on_separate_streams():
    """Host threads driving the shared-side-stream entry points at once (ctypes
    releases the GIL), each on its own stream and input: every result stays
    bit-exact."""
    import threading
    import paper_2205_11659_b200 as tb
    lib = tb.load()
    old = lib.tb_debug_host_chunk_shift(12)
    cases = []
    for i in range(4):
        t = scenegen.walk_tags(120_000 + 1000 * i, 40 + i, p_leaf=0.5)
        b = scenegen.boxes(t.numel(), 40 + i, t)
        m_ref, p_ref = oracle.paren_match(t.numpy())
        cases.append((t, b, m_ref, p_ref, oracle.tree_bbox(t.numpy(), b.numpy())))
    errors = []

    def worker(i):
        try:
            t, b, m_ref, p_ref, ref = cases[i]
            s = torch.cuda.Stream()
            td, bd = t.cuda(), b.cuda()
            hb = b.pin_memory()
            hm = torch.empty(t.numel(), dtype=torch.int32).pin_memory()
            hp = torch.empty_like(hm).pin_memory()
            ho = torch.empty_like(hb).pin_memory()
            for _ in range(5):
                with torch.cuda.stream(s):
                    m, p, out = tb.paren_match_tree_bbox(td, bd)
                s.synchronize()
                assert np.array_equal(m.cpu().numpy(), m_ref) and np.array_equal(p.cpu().numpy(), p_ref)
                assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))
                with torch.cuda.stream(s):
                    tb.paren_match_tree_bbox_host(t.pin_memory(), hb, hm, hp, ho)
                assert np.array_equal(ho.numpy().view(np.uint32), ref.view(np.uint32))
        except Exception as e:  # noqa: BLE001
            errors.append((i, repr(e)))

    try:
        th = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
        for x in th:
            x.start()
        for x in th:
            x.join()
    finally:
        lib.tb_debug_host_chunk_shift(old)
    assert not errors, errors
