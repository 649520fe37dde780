"""The largest stream of BASELINE.json's configs on ONE device: 2^30 elements
(the 1B-element C5 stream) through the bench step, paren_match_tree_bbox.

Every output is checked over the whole stream on the GPU, with plain torch ops
that restate the definitions (R3-R11), given the
matching structure:

* match / parent: involution, parents precede and are opens, a close's parent
  is its open, the unmatched counts equal the stream's Bic value;
* clips: every leaf and clip open equals its box ∩ the output of its nearest
  clip-open ancestor (INF at the root; blend opens pass the clip through);
* unions: every matched close equals the raw union of its node's children
  (leaves: their clipped boxes; child nodes: their unions, at their closes);
  a matched blend open equals its close; an unmatched close is EMPTY; a blend
  open never closed contains every child's contribution;
* the oracle, independently, on the first 2^24 elements (the outputs that
  prefix determines).
"""
import numpy as np
import pytest
import torch

import oracle
import scenegen

pytestmark = pytest.mark.gpu

INF = float("inf")


def isect(a, b):
    return torch.cat([torch.maximum(a[:, :2], b[:, :2]), torch.minimum(a[:, 2:], b[:, 2:])], 1)


def test_one_billion_elements():
    import paper_2205_11659_b200 as tb
    n = 1 << 30
    torch.cuda.empty_cache()  # blocks cached by earlier tests in this process
    free, _ = torch.cuda.mem_get_info()
    if free < 130 << 30:
        pytest.skip("needs ~130 GB of free device memory")
    tags = scenegen.walk_tags(n, 4, device="cuda")
    # boxes by chunks of the same per-index hash (the whole-stream generator
    # holds ~120 GB of fp64 / int64 temporaries at n = 2^30)
    boxes = torch.empty((n, 4), dtype=torch.float32, device="cuda")
    step = 1 << 27
    for s in range(0, n, step):
        e = min(n, s + step)
        boxes[s:e] = scenegen.boxes(e - s, 4, tags[s:e], offset=s, device="cuda")
    torch.cuda.empty_cache()  # the generators' temporaries; the library allocates its own workspace
    m, p, out = tb.paren_match_tree_bbox(tags, boxes)
    torch.cuda.synchronize()
    tb.release_workspaces()
    torch.cuda.empty_cache()

    # ---- matching structure over the whole stream
    ml = m.long()
    has = ml >= 0
    idx = torch.arange(n, device="cuda", dtype=torch.int64)
    assert torch.equal(ml[ml[has]], idx[has])                      # match is an involution
    del idx
    pl = p.long()
    assert bool((pl < torch.arange(n, device="cuda")).all())       # parents precede
    opens = (tags == 1) | (tags == 2)
    close = tags == 3
    assert bool(opens[pl[pl >= 0]].all())                          # parents are opens
    assert torch.equal(p[close & has], m[close & has])             # a close's parent is its open
    a, b = tb.count_unmatched(tags)
    assert int((close & ~has).sum()) == a                          # R3 closes
    assert int((opens & ~has).sum()) == b                          # R4 opens
    del pl

    # ---- clips: nearest clip-open ancestor (blend opens pass the clip through, R7)
    anc = p.clone()
    for _ in range(64):
        blend_anc = (anc >= 0) & (tags[anc.clamp(min=0).long()] == 2)
        if not bool(blend_anc.any()):
            break
        anc = torch.where(blend_anc, p[anc.clamp(min=0).long()], anc)
    else:
        raise AssertionError("blend chains did not resolve")
    clipped = (tags == 1) | ~(opens | close)                        # clip opens and leaves (R2, R6)
    inf = torch.tensor([[-INF, -INF, INF, INF]], device="cuda")
    for s in range(0, n, step):
        e = min(n, s + step)
        sel = clipped[s:e]
        a_ = anc[s:e][sel].long()
        ctx = torch.where((a_ >= 0)[:, None], out[a_.clamp(min=0)], inf)
        want = isect(boxes[s:e][sel], ctx)
        assert torch.equal(out[s:e][sel].view(torch.int32), want.view(torch.int32)), f"clip mismatch in [{s}, {e})"
    del anc

    # ---- unions: children's contributions reduced into their parent node
    U = [torch.full((n,), INF if c < 2 else -INF, dtype=torch.float32, device="cuda") for c in range(4)]
    for s in range(0, n, step):
        e = min(n, s + step)
        ps = p[s:e].long()
        t = tags[s:e]
        leaf = ~((t == 1) | (t == 2) | (t == 3))
        node = ((t == 1) | (t == 2)) & (m[s:e] >= 0)
        sel = (ps >= 0) & (leaf | node)
        contrib = torch.where(leaf[:, None], out[s:e], out[m[s:e].long().clamp(min=0)])[sel]
        tgt = ps[sel]
        for c in range(4):
            U[c].scatter_reduce_(0, tgt, contrib[:, c].contiguous(), reduce="amin" if c < 2 else "amax",
                                 include_self=True)
    for s in range(0, n, step):
        e = min(n, s + step)
        t = tags[s:e]
        ms = m[s:e].long()
        mc = (t == 3) & (ms >= 0)
        um = torch.stack([U[c][ms[mc]] for c in range(4)], 1)
        assert torch.equal(out[s:e][mc].view(torch.int32), um.view(torch.int32)), f"union mismatch in [{s}, {e})"
        mb = (t == 2) & (ms >= 0)
        assert torch.equal(out[s:e][mb].view(torch.int32), out[ms[mb]].view(torch.int32))
        uc = (t == 3) & (ms < 0)
        assert bool((out[s:e][uc] == torch.tensor([INF, INF, -INF, -INF], device="cuda")).all())
        nb = (t == 2) & (ms < 0)
        o_nb = out[s:e][nb]
        u_nb = torch.stack([U[c][s:e][nb] for c in range(4)], 1)
        assert bool((o_nb[:, :2] <= u_nb[:, :2]).all() & (o_nb[:, 2:] >= u_nb[:, 2:]).all())
    del U

    # ---- the oracle on the prefix the first 2^24 elements determine
    k = 1 << 24
    t_k = tags[:k].cpu().numpy()
    m_ref, p_ref = oracle.paren_match(t_k)
    assert np.array_equal(p[:k].cpu().numpy(), p_ref)
    mk = m[:k].cpu().numpy()
    opk = (t_k == 1) | (t_k == 2)
    done = m_ref >= 0
    assert np.array_equal(mk[done], m_ref[done])                   # partners found inside the prefix
    assert ((mk[opk & ~done] == -1) | (mk[opk & ~done] >= k)).all()   # the others close later or never
    ref = oracle.tree_bbox(t_k, boxes[:k].cpu().numpy())
    got = out[:k].cpu().numpy()
    det = (t_k == 1) | ~np.isin(t_k, [1, 2, 3]) | (t_k == 3) | ((t_k == 2) & done)
    assert np.array_equal(got[det].view(np.uint32), ref[det].view(np.uint32))
