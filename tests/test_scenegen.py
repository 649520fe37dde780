"""Input generators: determinism, shard-consistency and the paper's workload
statistics (push/pop equally likely unless underflow, depth ~ sqrt(n): P:315;
SPEC's acceptance band for mean max depth / sqrt(n) is [0.5, 2.5])."""
import numpy as np
import torch

import scenegen


def depth_profile(t):
    t = t.numpy().astype(np.int64)
    step = np.where((t == 1) | (t == 2), 1, np.where(t == 3, -1, 0))
    return np.cumsum(step)


def test_deterministic_and_shardable():
    a = scenegen.walk_tags(50_000, 3)
    assert torch.equal(a, scenegen.walk_tags(50_000, 3))
    s0 = scenegen.walk_step_sum(20_000, 3)
    b = torch.cat([scenegen.walk_tags(20_000, 3), scenegen.walk_tags(30_000, 3, offset=20_000, s_before=s0)])
    assert torch.equal(a, b)
    x = scenegen.boxes(1000, 5, a[:1000])
    y = torch.cat([scenegen.boxes(400, 5, a[:400]), scenegen.boxes(600, 5, a[400:1000], offset=400)])
    assert torch.equal(x, y)


def test_walk_never_underflows_and_depth_is_sqrt_n():
    ratios = []
    for seed in range(20):
        n = 1 << 16
        d = depth_profile(scenegen.walk_tags(n, seed, p_leaf=0.0))
        assert d.min() >= 0
        ratios.append(d.max() / np.sqrt(n))
    assert 0.5 <= float(np.mean(ratios)) <= 2.5


def test_push_pop_equally_likely_unless_underflow():
    t = scenegen.walk_tags(200_000, 1, p_leaf=0.0).numpy()
    d = np.concatenate([[0], depth_profile(torch.from_numpy(t))])[:-1]
    nz = d > 0
    frac_open = ((t == 1) | (t == 2))[nz].mean()
    assert abs(frac_open - 0.5) < 0.01
    assert (((t == 1) | (t == 2))[~nz]).all()   # at depth 0 the only move is a push


def test_configs_shapes():
    t, _ = scenegen.config("C1")
    d = depth_profile(t)
    assert d.max() <= 8 and d[-1] == 0 and d.min() >= 0
    t3 = scenegen.deep_chain_tags(1000, 0)
    assert depth_profile(t3).max() == 500


def test_boxes_exact_and_well_formed():
    t = scenegen.walk_tags(10_000, 2)
    b = scenegen.boxes(10_000, 2, t)
    leaf = t == 0
    assert (b[leaf, 2] > b[leaf, 0]).all() and (b[leaf, 3] > b[leaf, 1]).all()
    assert ((b[(t == 2) | (t == 3)]) == 0).all()
    # dyadic: exact in fp32 (round trip through fp64 unchanged)
    assert torch.equal(b.double().float(), b)
