"""GPU parity of the sharded fused protocol (csrc/fused_shard.cuh) on ONE GPU:
G virtual shards of one buffer run the three phases in lockstep, their slots
being the gathered buffers (what the NCCL all-gathers deliver on G ranks).

Every output must equal the oracle (small streams) and the unsharded fused
call bit for bit (match / parent exactly, node_bbox as fp32 bit patterns):
nodes that open on one chunk and close on a later one, chains of chunks
between, blend opens closed or never closed across chunks, pops of the global
root inside a later chunk, empty and one-element chunks, chunk borders inside
tiles, and the capacity check (TB_ERR_CAPACITY when a chunk's Bic a + 1 or b
exceeds cap)."""
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


def same(got, ref, name, n, G):
    got = got.cpu().numpy()
    ref = ref.cpu().numpy() if isinstance(ref, torch.Tensor) else ref
    if got.dtype == np.float32:
        got, ref = got.view(np.uint32), ref.view(np.uint32)
    if not np.array_equal(got, ref):
        bad = np.nonzero((got != ref).reshape(len(got), -1).any(1))[0]
        raise AssertionError(f"{name}: {len(bad)} mismatches (n={n}, G={G}), first {bad[:5].tolist()}: "
                             f"got {got[bad[:3]].tolist()} want {ref[bad[:3]].tolist()}")


def check(t: torch.Tensor, Gs=(1, 2, 3, 5, 8), cap=None, seed=5, use_oracle=False):
    tb = gpu()
    t = t.to(torch.uint8).contiguous()
    n = t.numel()
    b = scenegen.boxes(n, seed, t).float().contiguous().reshape(n, 4)
    tc, bc = t.cuda(), b.cuda()
    if use_oracle:
        m_ref, p_ref = oracle.paren_match(t.numpy())
        o_ref = oracle.tree_bbox(t.numpy(), b.numpy())
    else:
        m_ref, p_ref, o_ref = tb.paren_match_tree_bbox(tc, bc)
    for G in Gs:
        c = cap
        m, p, o = tb.pair_vshard(tc, bc, G, cap=c)
        torch.cuda.synchronize()
        same(p, p_ref, "parent", n, G)
        same(m, m_ref, "match", n, G)
        same(o, o_ref, "node_bbox", n, G)
        _, _, o2 = tb.pair_vshard(tc, bc, G, cap=c, pm=False)
        same(o2, o_ref, "node_bbox (tree_bbox alone)", n, G)
        m3, p3, _ = tb.pair_vshard(tc, None, G, cap=c)  # the matching alone (paren_match_shard)
        same(p3, p_ref, "parent (matching alone)", n, G)
        same(m3, m_ref, "match (matching alone)", n, G)


def walk(n, seed, p_leaf=0.5, p_clip=0.75):
    return scenegen.walk_tags(n, seed, p_leaf=p_leaf, p_clip=p_clip)


def test_small_against_oracle():
    for n in (1, 2, 5, 17, 100, 1000, W + 7, 3 * W + 1):
        check(walk(n, n), use_oracle=True)
        check(walk(n, 100 + n, p_leaf=0.0, p_clip=0.5), use_oracle=True)
    for v in (0, 1, 2, 3, 9):
        check(torch.full((10,), v, dtype=torch.uint8), use_oracle=True)


def test_more_shards_than_elements():
    for n in (1, 3, 7):
        check(walk(n, 3 * n + 1), Gs=(8, 16), use_oracle=True)


@pytest.mark.parametrize("n", [64 * W, 64 * W + 777, 300 * W + 5])
def test_random_walks(n):
    check(walk(n, 1))
    check(walk(n, 2, p_leaf=0.2, p_clip=0.5))
    check(walk(n, 3, p_leaf=0.9, p_clip=1.0))
    check(walk(n, 4, p_leaf=0.5, p_clip=0.0))  # blend opens only: unions cross chunks


def test_configs():
    check(scenegen.config("C1", seed=11)[0], Gs=(2, 4, 8), use_oracle=True)
    check(scenegen.config("C2", seed=11)[0], Gs=(2, 4, 8))
    # bursts of up to 65536 nested opens: deeper than the default capacity
    check(scenegen.compacted_tags(1 << 20, 11), Gs=(2, 4, 8), cap=(1 << 20) + 2)


def test_deep_chains_need_capacity():
    tb = gpu()
    n = 1 << 16
    t = torch.cat([torch.ones(n // 2, dtype=torch.uint8), torch.full((n // 2,), 3, dtype=torch.uint8)])
    t[1::5] = 2  # some blend opens
    b = scenegen.boxes(n, 9, t).float().reshape(n, 4)
    with pytest.raises(tb.TreeBBoxError, match="-6"):
        tb.pair_vshard(t.cuda(), b.cuda(), 2)  # default cap ~ 4 sqrt(n / 2) + 4096 < n / 2
    check(t, Gs=(2, 3, 8), cap=n + 2, use_oracle=True)
    check(scenegen.deep_chain_tags(n, 3), Gs=(2, 5), cap=n + 2)
    check(scenegen.deep_chain_tags(n, 4, leaves_mid=True), Gs=(2, 5), cap=n + 2)


def test_root_pops_in_later_chunks():
    # more closes than opens: later chunks pop the global root
    n = 20 * W
    t = walk(n, 8)
    t[::7] = 3
    check(t, Gs=(2, 4, 7), use_oracle=True)


def test_junk_and_specials():
    n = 9 * W + 3
    t = walk(n, 12)
    g = torch.Generator().manual_seed(3)
    junk = torch.randint(4, 256, (n,), generator=g, dtype=torch.int32).to(torch.uint8)
    sel = torch.rand(n, generator=g) < 0.05
    t[sel] = junk[sel]
    check(t, Gs=(2, 3), use_oracle=True)
