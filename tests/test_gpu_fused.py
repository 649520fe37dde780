"""GPU parity of the fused single-device path (csrc/fused.cu) against the oracle.

paren_match_tree_bbox (the bench step) returns match, parent and node_bbox
from one tile pass; every output is compared with the oracle element by
element (indices exactly, boxes as fp32 bit patterns: 0 ULP).
Besides the shapes of test_gpu_paren / test_gpu_bbox the corpus aims at the
fused kernel's own mechanisms (tile = 2048 elements, 16 per thread):

* thread-level: more than RCAP = 7 unmatched opens in one thread (segment
  buffer overflow), link chains across all 128 threads, element 15 of a
  thread as an unmatched / matched close (its slot carries the link context);
* tile-level: incoming stacks deeper than INCCAP = 192 entries (read from
  global memory), and with more than RMAX = 8 owner runs (followed along the
  link owners), pops of the root (R3) mixed with real pops;
* transfers: full tiles by TMA, the last partial tile by the threads, and the
  thread-copy path for every tile (tb_debug_fz_tma(0));
* the two-call path (tb_debug_use_fused(0)) on the same corpus.
"""
import numpy as np
import pytest
import torch

import oracle
import scenegen

pytestmark = pytest.mark.gpu
W = 2048


def gpu():
    import paper_2205_11659_b200 as tb
    return tb


def check(t: torch.Tensor, boxes: torch.Tensor | None = None, seed: int = 7):
    tb = gpu()
    t = t.to(torch.uint8).contiguous()
    n = t.numel()
    b = (boxes if boxes is not None else scenegen.boxes(n, seed, t)).float().contiguous().reshape(n, 4)
    m_ref, p_ref = oracle.paren_match(t.numpy())
    o_ref = oracle.tree_bbox(t.numpy(), b.numpy()).view(np.uint32)
    m, p, o = tb.paren_match_tree_bbox(t.cuda(), b.cuda())
    torch.cuda.synchronize()
    for name, got, ref in (("parent", p.cpu().numpy(), p_ref), ("match", m.cpu().numpy(), m_ref)):
        if not np.array_equal(got, ref):
            bad = np.nonzero(got != ref)[0]
            raise AssertionError(f"{name}: {len(bad)} mismatches (n={n}), first {bad[:5].tolist()}: "
                                 f"got {got[bad[:5]].tolist()} want {ref[bad[:5]].tolist()}")
    got = o.cpu().numpy().view(np.uint32)
    if not np.array_equal(got, o_ref):
        bad = np.nonzero((got != o_ref).any(1))[0]
        raise AssertionError(f"node_bbox: {len(bad)} mismatches (n={n}), first {bad[:5].tolist()} "
                             f"tags {t.numpy()[bad[:5]].tolist()}")


def walk(n, seed, p_leaf=0.5, p_clip=0.75):
    return scenegen.walk_tags(n, seed, p_leaf=p_leaf, p_clip=p_clip)


def test_empty_and_tiny():
    tb = gpu()
    e = torch.empty(0, dtype=torch.uint8, device="cuda")
    m, p, o = tb.paren_match_tree_bbox(e, torch.empty((0, 4), device="cuda"))
    assert m.numel() == p.numel() == o.numel() == 0
    for v in (0, 1, 2, 3, 7):
        check(torch.tensor([v], dtype=torch.uint8))
    for n in (2, 15, 16, 17, 31, 33):
        check(walk(n, n))


@pytest.mark.parametrize("n", [W - 1, W, W + 1, 2 * W - 16, 2 * W + 15, 7 * W + 3, 129 * W, 129 * W + 1000])
def test_tile_boundaries(n):
    for seed in range(2):
        check(walk(n, seed))
        check(walk(n, 10 + seed, p_leaf=0.0, p_clip=0.5), seed=seed)
        check(walk(n, 20 + seed, p_leaf=0.8, p_clip=1.0), seed=seed)


@pytest.mark.parametrize("n", [W, 3 * W + 5, 64 * W + 1])
def test_degenerate(n):
    check(torch.full((n,), 1, dtype=torch.uint8))  # all clip opens (R4): b_t = 16 > RCAP in every thread
    check(torch.full((n,), 2, dtype=torch.uint8))  # all blend opens (R4)
    check(torch.full((n,), 3, dtype=torch.uint8))  # all closes: every pop takes the root (R3)
    check(torch.zeros(n, dtype=torch.uint8))       # all leaves
    check(torch.tensor([2, 0, 3], dtype=torch.uint8).repeat(n // 3 + 1)[:n])
    check(scenegen.deep_chain_tags(n, 1))          # incoming stacks of 2048 entries (> INCCAP)
    check(scenegen.deep_chain_tags(n, 2, leaves_mid=True))


def test_chain_with_leaves_everywhere():
    n = 300_000
    g = torch.Generator().manual_seed(3)
    opens = torch.where(torch.rand(n // 2, generator=g) < 0.7, 1, 2).to(torch.uint8)
    t = torch.stack([opens, torch.zeros(n // 2, dtype=torch.uint8)], 1).reshape(-1)
    check(torch.cat([t, torch.full((n // 2,), 3, dtype=torch.uint8)]))


def test_many_owner_runs():
    """Each tile leaves one unmatched open, a later close-heavy stretch pops
    them all: incoming stacks made of one entry per owner tile (> RMAX runs)."""
    unit = torch.cat([torch.tensor([1], dtype=torch.uint8), torch.tensor([1, 3] * (W // 2 - 1), dtype=torch.uint8),
                      torch.tensor([0], dtype=torch.uint8)])
    t = torch.cat([unit.repeat(40), torch.tensor([0, 3] * 45, dtype=torch.uint8), walk(5 * W, 5)])
    check(t)
    # leaves between the pops: contexts of the popped entries are needed
    t = torch.cat([unit.repeat(30), torch.tensor([0, 0, 3] * 35, dtype=torch.uint8)])
    check(t)


def test_thread_patterns():
    """Unmatched opens / closes at every position of a 16-element thread."""
    g = torch.Generator().manual_seed(8)
    for k in range(16):
        base = torch.multinomial(torch.tensor([0.4, 0.2, 0.1, 0.3]), 40 * W, replacement=True, generator=g)
        base = base.to(torch.uint8)
        base[k::16] = 3 if k % 2 else 1
        check(base, seed=k)


def test_underflow_and_junk():
    g = torch.Generator().manual_seed(5)
    for n in (1000, 50_000, 300_000):
        t = torch.multinomial(torch.tensor([0.3, 0.15, 0.1, 0.45]), n, replacement=True, generator=g)
        check(t.to(torch.uint8), seed=n)
    check(torch.randint(0, 256, (100_000,), generator=g, dtype=torch.int64).to(torch.uint8))


def test_special_values():
    specials = torch.tensor([0.0, -0.0, float("inf"), -float("inf"), 1e-45, -1e-45, 1.1754942e-38, 3.4028235e38,
                             -3.4028235e38, 1.0, -1.0, 0.5, float("nan"), -float("nan")])
    g = torch.Generator().manual_seed(9)
    n = 200_000
    check(walk(n, 9, p_leaf=0.4), specials[torch.randint(0, len(specials), (n, 4), generator=g)])


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C3L", "C4"])
def test_configs(name):
    check(scenegen.config(name)[0], seed=3)


def test_config_c5_bench_size():
    check(scenegen.config("C5")[0], seed=4)


def test_thread_copy_path():
    """Every tile through the threads' copies instead of TMA."""
    lib = gpu().load()
    old = lib.tb_debug_fz_tma(0)
    try:
        check(walk(50 * W + 77, 3))
        check(scenegen.deep_chain_tags(9 * W + 5, 4, leaves_mid=True))
    finally:
        lib.tb_debug_fz_tma(old)


def test_two_call_path():
    """The earlier two-call path (paren_match, then the boxes from its matching)."""
    lib = gpu().load()
    old = lib.tb_debug_use_fused(0)
    try:
        check(walk(300_007, 11))
        check(scenegen.deep_chain_tags(70_001, 2, leaves_mid=True))
    finally:
        lib.tb_debug_use_fused(old)


def test_tree_bbox_alone_equals_pair():
    """tree_bbox runs the same fused pass without match / parent outputs."""
    tb = gpu()
    t = walk(1_000_003, 12).cuda()
    b = scenegen.boxes(t.numel(), 12, t.cpu()).cuda()
    _, _, o = tb.paren_match_tree_bbox(t, b)
    o2 = tb.tree_bbox(t, b)
    torch.cuda.synchronize()
    assert torch.equal(o.view(torch.int32), o2.view(torch.int32))


def test_deterministic_repeat():
    tb = gpu()
    t = walk(3_000_000, 9).cuda()
    b = scenegen.boxes(t.numel(), 9, t.cpu()).cuda()
    r1 = [x.clone() for x in tb.paren_match_tree_bbox(t, b)]
    r2 = tb.paren_match_tree_bbox(t, b)
    for a, c in zip(r1, r2):
        assert torch.equal(a.view(torch.int32), c.view(torch.int32))
