"""GPU parity: tree_bbox (CUDA, through the C ABI) vs the oracle, bit-exact.

Boxes are compared as raw fp32 bit patterns (0 ULP): min/max are
exact and totalOrder makes every result unique, including signed zeros.
Sizes span many tiles (1024 elements each) with ragged tails; edge corpora
hit tile boundaries, deep chains (C3/C3L), bursts (C4), unmatched closes
(R3), unmatched trailing opens (R4) and special fp32 values.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import scenegen

pytestmark = pytest.mark.gpu
TILE = 1024
INF = float("inf")


def gpu():
    import paper_2205_11659_b200 as tb
    return tb


def check(tags_cpu: torch.Tensor, boxes_cpu: torch.Tensor | None = None, seed: int = 0, matched: bool = False):
    tb = gpu()
    t = tags_cpu.to(torch.uint8).contiguous()
    n = t.numel()
    b = boxes_cpu if boxes_cpu is not None else scenegen.boxes(n, seed, t)
    b = b.float().contiguous().reshape(n, 4)
    ref = oracle.tree_bbox(t.numpy(), b.numpy())
    out = tb.tree_bbox(t.cuda(), b.cuda())
    torch.cuda.synchronize()
    same_bits(out, ref, t)
    if matched and n > 0:
        m, p = tb.paren_match(t.cuda())
        out2 = tb.tree_bbox_matched(t.cuda(), b.cuda(), m, p)
        torch.cuda.synchronize()
        same_bits(out2, ref, t)


def same_bits(out, ref, t):
    got = out.cpu().numpy()
    n = len(got)
    gb, rb = got.view(np.uint32), ref.view(np.uint32)
    if not np.array_equal(gb, rb):
        bad = np.nonzero((gb != rb).any(1))[0]
        raise AssertionError(f"node_bbox mismatch at {bad[:10]} of {len(bad)} (n={n}); tags {t[bad[:5]].tolist()} "
                             f"got {got[bad[:3]].tolist()} want {ref[bad[:3]].tolist()}")


def test_golden_examples():
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "bbox_examples.json")))
    for ex in gold["examples"]:
        tags = torch.tensor([r[0] for r in ex["scene"]], dtype=torch.uint8)
        boxes = torch.tensor([r[1:] for r in ex["scene"]], dtype=torch.float32)
        check(tags, boxes)


def test_empty_and_single():
    tb = gpu()
    out = tb.tree_bbox(torch.empty(0, dtype=torch.uint8, device="cuda"),
                       torch.empty((0, 4), dtype=torch.float32, device="cuda"))
    assert out.numel() == 0
    for v in (0, 1, 2, 3):
        check(torch.tensor([v], dtype=torch.uint8), torch.tensor([[1.0, 2.0, 3.0, 4.0]]))


@pytest.mark.parametrize("n", [7, 8, 9, 1023, 1024, 1025, 2047, 2048, 2049, 4095, 4096, 4097, 3 * 2048 + 5, 65 * 2048 - 1,
                               65 * 2048 + 3])
def test_tile_boundaries_random(n):
    for seed in range(3):
        check(scenegen.walk_tags(n, seed, p_leaf=0.5), seed=seed)
        check(scenegen.walk_tags(n, 100 + seed, p_leaf=0.2, p_clip=0.5), seed=seed + 1)


@pytest.mark.parametrize("n", [2048, 2049, 2 * 2048, 40 * 2048 + 3, 600 * 2048 + 9])
def test_degenerate(n):
    check(torch.full((n,), 1, dtype=torch.uint8))              # all clip opens (R4)
    check(torch.full((n,), 2, dtype=torch.uint8))              # all blend opens (R4)
    check(torch.full((n,), 3, dtype=torch.uint8))              # all closes (R3)
    check(torch.zeros(n, dtype=torch.uint8))                   # all leaves
    alt = torch.tensor([2, 0, 3], dtype=torch.uint8).repeat(n // 3 + 1)[:n]
    check(alt)
    check(scenegen.deep_chain_tags(n, 1))
    check(scenegen.deep_chain_tags(n, 2, leaves_mid=True))


def test_chain_with_leaves_everywhere():
    """Deep nesting with leaves at every level: long clip chains across tiles."""
    n = 300_000
    g = torch.Generator().manual_seed(3)
    opens = torch.where(torch.rand(n // 2, generator=g) < 0.7, 1, 2).to(torch.uint8)
    t = torch.stack([opens, torch.zeros(n // 2, dtype=torch.uint8)], 1).reshape(-1)
    t = torch.cat([t, torch.full((n // 2,), 3, dtype=torch.uint8)])
    check(t)


def test_staircases():
    parts = []
    for k in range(40):
        parts.append(torch.tensor([1, 0] * 1000, dtype=torch.uint8))
        parts.append(torch.tensor([3, 0] * 1050, dtype=torch.uint8))
    t = torch.cat([torch.tensor([2, 0] * 60_000, dtype=torch.uint8)] + parts)
    check(t)


def test_underflow_heavy_random():
    g = torch.Generator().manual_seed(5)
    for n in (1000, 50_000, 300_000):
        t = torch.multinomial(torch.tensor([0.3, 0.15, 0.1, 0.45]), n, replacement=True, generator=g)
        check(t.to(torch.uint8), seed=n)


SPECIALS = torch.tensor([0.0, -0.0, INF, -INF, 1e-45, -1e-45, 1.1754942e-38, 3.4028235e38,
                         -3.4028235e38, 1.0, -1.0, 0.5, float("nan"), -float("nan")])


def test_special_values():
    """±0, ±inf, subnormals, extremes and NaN (outside the domain; R12 rule)."""
    g = torch.Generator().manual_seed(9)
    n = 200_000
    t = scenegen.walk_tags(n, 9, p_leaf=0.4)
    idx = torch.randint(0, len(SPECIALS), (n, 4), generator=g)
    check(t, SPECIALS[idx])


def test_inverted_boxes():
    g = torch.Generator().manual_seed(11)
    n = 100_000
    t = scenegen.walk_tags(n, 11, p_leaf=0.5)
    lo = torch.randint(-100, 100, (n, 2), generator=g).float()
    wh = torch.randint(-30, 60, (n, 2), generator=g).float()
    check(t, torch.cat([lo, lo + wh], 1))


@pytest.mark.parametrize("seed", range(4))
def test_random_walks(seed):
    for n in (1 << 16, (1 << 20) + 12345):
        check(scenegen.walk_tags(n, seed, p_leaf=0.5 if seed % 2 else 0.25), seed=seed, matched=True)


def test_configs_c1_c2():
    check(scenegen.config("C1")[0], seed=0)
    check(scenegen.config("C2")[0], seed=1)


def test_config_c3_and_c3l_full():
    check(scenegen.config("C3")[0], seed=2)
    check(scenegen.config("C3L")[0], seed=2)


def test_config_c4_full():
    check(scenegen.config("C4")[0], seed=3)


def test_config_c5_bench_size():
    check(scenegen.config("C5")[0], seed=4)


def test_matched_entry_point():
    """tree_bbox_matched on paren_match's outputs: every corpus shape."""
    g = torch.Generator().manual_seed(21)
    cases = [scenegen.walk_tags(300_007, 21, p_leaf=0.5), scenegen.deep_chain_tags(50_000, 1),
             scenegen.deep_chain_tags(70_001, 2, leaves_mid=True), torch.full((5000,), 2, dtype=torch.uint8),
             torch.full((5000,), 3, dtype=torch.uint8),
             torch.multinomial(torch.tensor([0.3, 0.15, 0.1, 0.45]), 100_000, replacement=True,
                               generator=g).to(torch.uint8)]
    for i, t in enumerate(cases):
        check(t, seed=i, matched=True)


def test_deterministic_repeat():
    tb = gpu()
    t = scenegen.walk_tags(3_000_000, 9).cuda()
    b = scenegen.boxes(t.numel(), 9, t.cpu()).cuda()
    o1 = tb.tree_bbox(t, b).clone()
    o2 = tb.tree_bbox(t, b)
    assert torch.equal(o1.view(torch.int32), o2.view(torch.int32))


def test_host_api():
    tb = gpu()
    t = scenegen.walk_tags(400_000, 4).pin_memory()
    b = scenegen.boxes(t.numel(), 4, t).pin_memory()
    out = torch.empty_like(b).pin_memory()
    tb.tree_bbox_host(t, b, out)
    ref = oracle.tree_bbox(t.numpy(), b.numpy())
    assert np.array_equal(out.numpy().view(np.uint32), ref.view(np.uint32))


def test_pipeline_host_api():
    tb = gpu()
    t = scenegen.walk_tags(300_001, 5).pin_memory()
    b = scenegen.boxes(t.numel(), 5, t).pin_memory()
    m = torch.empty(t.numel(), dtype=torch.int32).pin_memory()
    p = torch.empty_like(m).pin_memory()
    out = torch.empty_like(b).pin_memory()
    tb.paren_match_tree_bbox_host(t, b, m, p, out)
    m_ref, p_ref = oracle.paren_match(t.numpy())
    ref = oracle.tree_bbox(t.numpy(), b.numpy())
    assert np.array_equal(m.numpy(), m_ref) and np.array_equal(p.numpy(), p_ref)
    assert np.array_equal(out.numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("nshards", [1, 2, 3, 5, 8])
def test_virtual_shards_equal_oracle(nshards):
    """tree_bbox shard protocol (clip chain over chunks, exchanged unions and
    pops, fix-up of nodes spanning chunks) with virtual shards on one GPU."""
    tb = gpu()
    g = torch.Generator().manual_seed(nshards)
    cases = [scenegen.walk_tags(1_000_003, 7, p_leaf=0.5),
             scenegen.walk_tags(200_000, 8, p_leaf=0.3, p_clip=0.5),
             scenegen.deep_chain_tags(300_000, 3, leaves_mid=True),
             torch.full((50_000,), 3, dtype=torch.uint8),
             torch.full((50_000,), 2, dtype=torch.uint8),
             torch.multinomial(torch.tensor([0.3, 0.15, 0.1, 0.45]), 400_000, replacement=True,
                               generator=g).to(torch.uint8)]
    chain = torch.stack([torch.where(torch.rand(60_000, generator=g) < 0.6, 1, 2).to(torch.uint8),
                         torch.zeros(60_000, dtype=torch.uint8)], 1).reshape(-1)
    cases.append(torch.cat([chain, torch.full((50_000,), 3, dtype=torch.uint8)]))
    for i, t in enumerate(cases):
        b = scenegen.boxes(t.numel(), 100 + i, t)
        ref = oracle.tree_bbox(t.numpy(), b.numpy())
        out = tb.tree_bbox_vshard(t.cuda(), b.cuda(), nshards)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        bad = np.nonzero((got.view(np.uint32) != ref.view(np.uint32)).any(1))[0]
        assert len(bad) == 0, (i, bad[:10], len(bad), t[bad[:5]].tolist(), got[bad[:3]].tolist(), ref[bad[:3]].tolist())


def _pipeline_cases():
    g = torch.Generator().manual_seed(77)
    chain = torch.stack([torch.where(torch.rand(40_000, generator=g) < 0.6, 1, 2).to(torch.uint8),
                         torch.zeros(40_000, dtype=torch.uint8)], 1).reshape(-1)
    return [scenegen.walk_tags(300_001, 5),
            scenegen.walk_tags(250_000, 8, p_leaf=0.3, p_clip=0.5),
            scenegen.deep_chain_tags(200_000, 3, leaves_mid=True),
            torch.cat([chain, torch.full((40_000,), 3, dtype=torch.uint8)]),  # blend opens closed chunks later
            torch.full((60_000,), 2, dtype=torch.uint8),                       # blend opens never closed (R4)
            torch.multinomial(torch.tensor([0.3, 0.15, 0.1, 0.45]), 300_000, replacement=True,
                              generator=g).to(torch.uint8)]


@pytest.mark.parametrize("shift", [12, 14])
def test_pipeline_host_api_chunked(shift):
    """The chunked schedule of paren_match_tree_bbox_host (pinned result): box
    passes over tile ranges as the boxes arrive, per-chunk copies out, late
    entries (blend opens closed in a later chunk, never-closed ones) stored
    through the host mapping -- bit-exact against the oracle."""
    tb = gpu()
    lib = tb.load()
    old = lib.tb_debug_host_chunk_shift(shift)
    try:
        for i, t in enumerate(_pipeline_cases()):
            t = t.pin_memory()
            b = scenegen.boxes(t.numel(), 40 + i, t).pin_memory()
            m = torch.empty(t.numel(), dtype=torch.int32).pin_memory()
            p = torch.empty_like(m).pin_memory()
            out = torch.full_like(b, float("nan")).pin_memory()
            tb.paren_match_tree_bbox_host(t, b, m, p, out)
            m_ref, p_ref = oracle.paren_match(t.numpy())
            ref = oracle.tree_bbox(t.numpy(), b.numpy())
            assert np.array_equal(m.numpy(), m_ref) and np.array_equal(p.numpy(), p_ref), i
            bad = np.nonzero((out.numpy().view(np.uint32) != ref.view(np.uint32)).any(1))[0]
            assert len(bad) == 0, (i, bad[:10], len(bad))
    finally:
        lib.tb_debug_host_chunk_shift(old)


def test_pipeline_host_api_pageable():
    """Pageable result buffer: the unchunked schedule, same results."""
    tb = gpu()
    t = scenegen.walk_tags(200_003, 6)
    b = scenegen.boxes(t.numel(), 6, t)
    m = torch.empty(t.numel(), dtype=torch.int32)
    p = torch.empty_like(m)
    out = torch.empty_like(b)
    tb.paren_match_tree_bbox_host(t, b, m, p, out)
    ref = oracle.tree_bbox(t.numpy(), b.numpy())
    assert np.array_equal(m.numpy(), oracle.paren_match(t.numpy())[0])
    assert np.array_equal(out.numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("n", [1, 7, 1023, 1024, 1025, 4097, 33_000])
def test_pipeline_host_api_ragged(n):
    """Chunked host path at the smallest chunk size on ragged sizes (one
    element, under one tile, exactly one tile, one tile + 1, many chunks);
    pageable inputs with a pinned result."""
    tb = gpu()
    lib = tb.load()
    old = lib.tb_debug_host_chunk_shift(10)
    try:
        t = scenegen.walk_tags(n, 90 + n % 7)
        b = scenegen.boxes(n, 91, t)
        m = torch.empty(n, dtype=torch.int32)
        p = torch.empty_like(m)
        out = torch.full((n, 4), float("nan")).pin_memory()
        tb.paren_match_tree_bbox_host(t, b, m, p, out)
        m_ref, p_ref = oracle.paren_match(t.numpy())
        ref = oracle.tree_bbox(t.numpy(), b.numpy())
        assert np.array_equal(m.numpy(), m_ref) and np.array_equal(p.numpy(), p_ref)
        assert np.array_equal(out.numpy().view(np.uint32), ref.view(np.uint32))
    finally:
        lib.tb_debug_host_chunk_shift(old)


def test_pipeline_host_api_c5_bench_size():
    """The e2e call bench.py times (C5, 2^27, pinned buffers, the default 16
    chunks) bit-exact against the oracle on the whole stream."""
    tb = gpu()
    t = scenegen.walk_tags(1 << 27, 4)
    b = scenegen.boxes(t.numel(), 4, t)
    tp, bp = t.pin_memory(), b.pin_memory()
    m = torch.empty(t.numel(), dtype=torch.int32).pin_memory()
    p = torch.empty_like(m).pin_memory()
    out = torch.empty_like(bp).pin_memory()
    tb.paren_match_tree_bbox_host(tp, bp, m, p, out)
    m_ref, p_ref = oracle.paren_match(t.numpy())
    assert np.array_equal(m.numpy(), m_ref) and np.array_equal(p.numpy(), p_ref)
    ref = oracle.tree_bbox(t.numpy(), b.numpy())
    assert np.array_equal(out.numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("cfg", ["C2", "C3L", "C5"])
def test_fused_device_call(cfg):
    """paren_match_tree_bbox (the bench step: box reduce pass beside
    paren_match on a side stream) equals the oracle on every output."""
    tb = gpu()
    t = scenegen.config(cfg)[0]
    b = scenegen.boxes(t.numel(), 13, t)
    m, p, out = tb.paren_match_tree_bbox(t.cuda(), b.cuda())
    torch.cuda.synchronize()
    m_ref, p_ref = oracle.paren_match(t.numpy())
    assert np.array_equal(m.cpu().numpy(), m_ref) and np.array_equal(p.cpu().numpy(), p_ref)
    ref = oracle.tree_bbox(t.numpy(), b.numpy())
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))
