"""GPU parity: paren_match (CUDA, through the C ABI) vs the oracle, bit-exact.

Integer outputs: equality is exact.  Sizes span many tiles (4096
elements each) with ragged tails; the edge corpora hit tile boundaries,
empty/single inputs, underflow (R3) and unmatched trailing opens (R4).
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import scenegen

pytestmark = pytest.mark.gpu
TILE = 4096
SYM = {"(": 1, ")": 3, "x": 0}


def gpu():
    import paper_2205_11659_b200 as tb
    return tb


def check(tags_cpu: torch.Tensor):
    tb = gpu()
    t = tags_cpu.to(torch.uint8).contiguous()
    m_ref, p_ref = oracle.paren_match(t.numpy())
    m, p = tb.paren_match(t.cuda())
    torch.cuda.synchronize()
    m = m.cpu().numpy()
    p = p.cpu().numpy()
    if not np.array_equal(p, p_ref):
        bad = np.nonzero(p != p_ref)[0]
        raise AssertionError(f"parent mismatch at {bad[:10]} of {len(bad)}; n={len(t)}; "
                             f"got {p[bad[:5]]} want {p_ref[bad[:5]]}")
    if not np.array_equal(m, m_ref):
        bad = np.nonzero(m != m_ref)[0]
        raise AssertionError(f"match mismatch at {bad[:10]} of {len(bad)}; n={len(t)}; "
                             f"got {m[bad[:5]]} want {m_ref[bad[:5]]}")


def test_golden_examples():
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paren_examples.json")))
    for ex in gold["examples"]:
        if ex["s"]:
            check(torch.tensor([SYM[c] for c in ex["s"]], dtype=torch.uint8))


def test_empty_and_single():
    tb = gpu()
    e = torch.empty(0, dtype=torch.uint8, device="cuda")
    m, p = tb.paren_match(e)
    assert m.numel() == 0 and p.numel() == 0
    for v in (0, 1, 2, 3, 9):
        check(torch.tensor([v], dtype=torch.uint8))


@pytest.mark.parametrize("n", [1, 15, 16, 17, 4095, 4096, 4097, 8191, 8192, 8193, 3 * 4096 + 5,
                               33 * 4096 - 1, 33 * 4096 + 7])
def test_tile_boundaries_random(n):
    for seed in range(3):
        check(scenegen.walk_tags(n, seed, p_leaf=0.3))
        check(scenegen.walk_tags(n, 100 + seed, p_leaf=0.0))


@pytest.mark.parametrize("n", [4096, 4097, 2 * 4096, 40 * 4096 + 3, 1100 * 4096 + 9])
def test_degenerate(n):
    check(torch.full((n,), 1, dtype=torch.uint8))            # all opens (R4)
    check(torch.full((n,), 3, dtype=torch.uint8))            # all closes (R3)
    alt = torch.tensor([1, 3], dtype=torch.uint8).repeat(n // 2 + 1)[:n]
    check(alt)                                               # ()()()...
    check(scenegen.deep_chain_tags(n, 1))                    # depth n/2
    check(scenegen.deep_chain_tags(n, 2, leaves_mid=True))


def test_pairs_straddling_boundaries():
    for off in (1, 2, 15, 16, 17, 4095, 4096, 4097, 5000):
        n = 4 * TILE
        t = torch.zeros(n, dtype=torch.uint8)
        for c in range(TILE - off % TILE, n, TILE):
            o = c - off
            if 0 <= o < c < n:
                t[o] = 1
                t[c] = 3
        check(t)


def test_staircases():
    """Low-water marks decreasing tile after tile (long owner chains)."""
    parts = []
    for k in range(60):
        parts.append(torch.full((2000,), 1, dtype=torch.uint8))
        parts.append(torch.full((2100,), 3, dtype=torch.uint8))
    t = torch.cat([torch.full((200_000,), 1, dtype=torch.uint8)] + parts)
    check(t)
    # each tile pops everything of the previous tile and pushes anew
    t2 = torch.cat([torch.full((TILE,), 1, dtype=torch.uint8)] +
                   [torch.cat([torch.full((TILE // 2,), 3, dtype=torch.uint8),
                               torch.full((TILE // 2,), 1, dtype=torch.uint8)]) for _ in range(200)])
    check(t2)


def test_many_incoming_runs():
    """One tile pops an incoming stack spread over more predecessor slices than
    pm_finish gathers per batch (RUNCAP = 32 runs), so the run search repeats."""
    for npred, per in ((40, 50), (70, 3), (33, 1)):
        pred = torch.cat([torch.full((per,), 1, dtype=torch.uint8),
                          torch.zeros(TILE - per, dtype=torch.uint8)])
        closes = torch.full((npred * per + 5,), 3, dtype=torch.uint8)  # pops everything, then underflows
        t = torch.cat([pred.repeat(npred), closes, torch.full((777,), 2, dtype=torch.uint8)])
        check(t)
        # the same closes one tile later, behind a tile of leaves
        check(torch.cat([pred.repeat(npred), torch.zeros(TILE + 17, dtype=torch.uint8), closes]))


def test_underflow_heavy_random():
    g = torch.Generator().manual_seed(5)
    for n in (1000, 50_000, 300_000):
        t = torch.multinomial(torch.tensor([0.2, 0.2, 0.1, 0.5]), n, replacement=True, generator=g)
        check(t.to(torch.uint8))
    # junk tag bytes are leaves (R2)
    t = torch.randint(0, 256, (100_000,), generator=g, dtype=torch.int64).to(torch.uint8)
    check(t)


@pytest.mark.parametrize("seed", range(6))
def test_random_walks(seed):
    for n in (1 << 16, (1 << 20) + 12345):
        check(scenegen.walk_tags(n, seed, p_leaf=0.5 if seed % 2 else 0.0))


def test_configs_c1_c2():
    check(scenegen.config("C1")[0])
    check(scenegen.config("C2")[0])


def test_config_c3_full():
    check(scenegen.config("C3")[0])


def test_config_c4_full():
    check(scenegen.config("C4")[0])


def test_config_c5_bench_size():
    """The size bench.py times (2^27, random walk, unbalanced tail)."""
    check(scenegen.config("C5")[0])


def test_deterministic_repeat():
    tb = gpu()
    t = scenegen.walk_tags(3_000_000, 9).cuda()
    m1, p1 = tb.paren_match(t)
    m2, p2 = tb.paren_match(t)
    assert torch.equal(m1, m2) and torch.equal(p1, p2)


def test_count_unmatched():
    tb = gpu()
    for t in (scenegen.walk_tags(1_000_003, 3), torch.full((9000,), 3, dtype=torch.uint8)):
        assert tb.count_unmatched(t.cuda()) == oracle.count_unmatched(t.numpy())


def test_host_api():
    tb = gpu()
    t = scenegen.walk_tags(500_000, 4).pin_memory()
    m = torch.empty(t.numel(), dtype=torch.int32).pin_memory()
    p = torch.empty(t.numel(), dtype=torch.int32).pin_memory()
    tb.paren_match_host(t, m, p)
    m_ref, p_ref = oracle.paren_match(t.numpy())
    assert np.array_equal(m.numpy(), m_ref) and np.array_equal(p.numpy(), p_ref)


def test_errors():
    tb = gpu()
    t = torch.zeros(64, dtype=torch.uint8, device="cuda")
    m = torch.empty(64, dtype=torch.int32, device="cuda")
    lib = tb.load()
    rc = lib.paren_match(t.data_ptr() + 1, 32, m.data_ptr(), m.data_ptr() + 128, 0)
    assert rc == -2
    rc = lib.paren_match(t.data_ptr(), 32, m.data_ptr(), m.data_ptr() + 16, 0)
    assert rc == -3
    rc = lib.paren_match(t.data_ptr(), -1, m.data_ptr(), m.data_ptr(), 0)
    assert rc == -1
    rc = lib.paren_match(0, 10, m.data_ptr(), m.data_ptr(), 0)
    assert rc == -1


@pytest.mark.parametrize("nshards", [1, 2, 3, 5, 8])
def test_virtual_shards_equal_oracle(nshards):
    """The multi-GPU protocol (chunk summaries, composed incoming stacks,
    (open, close) pairs across chunks) run with virtual shards on one GPU."""
    tb = gpu()
    cases = [scenegen.walk_tags(1_000_003, 7, p_leaf=0.5),
             scenegen.walk_tags(200_000, 8, p_leaf=0.0),
             scenegen.deep_chain_tags(300_000, 3),
             torch.full((50_000,), 3, dtype=torch.uint8),
             torch.full((50_000,), 1, dtype=torch.uint8),
             torch.cat([torch.full((30_000,), 1, dtype=torch.uint8), torch.full((45_000,), 3, dtype=torch.uint8),
                        torch.full((20_000,), 2, dtype=torch.uint8)])]
    g = torch.Generator().manual_seed(nshards)
    cases.append(torch.multinomial(torch.tensor([0.2, 0.2, 0.1, 0.5]), 400_000, replacement=True,
                                   generator=g).to(torch.uint8))
    for t in cases:
        m_ref, p_ref = oracle.paren_match(t.numpy())
        m, p = tb.paren_match_vshard(t.cuda(), nshards)
        torch.cuda.synchronize()
        assert np.array_equal(p.cpu().numpy(), p_ref)
        assert np.array_equal(m.cpu().numpy(), m_ref)
