"""The NCCL-backed shard entry points (tb_get_unique_id, tb_comm_init,
paren_match_shard, tree_bbox_shard, tree_bbox_matched_shard,
paren_match_tree_bbox_shard, tb_shard_status) through ShardContext, with a world of one
rank (the GPU box has one GPU; multi-rank exchange logic is covered by the
virtual-shard parity tests and the gloo protocol tests)."""
import os

import numpy as np
import pytest
import torch

import oracle
import scenegen

pytestmark = pytest.mark.gpu


def test_nccl_shard_world1():
    import torch.distributed as dist
    import paper_2205_11659_b200 as tb
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n = 700_001
        t = scenegen.walk_tags(n, 5)
        b = scenegen.boxes(n, 5, t)
        ctx = tb.ShardContext(1, 0, 0, n)
        m = torch.empty(n, dtype=torch.int32, device="cuda")
        p = torch.empty_like(m)
        ctx.paren_match(t.cuda(), m, p)
        out = torch.empty((n, 4), dtype=torch.float32, device="cuda")
        ctx.tree_bbox(t.cuda(), b.cuda(), out)
        torch.cuda.synchronize()
        m_ref, p_ref = oracle.paren_match(t.numpy())
        o_ref = oracle.tree_bbox(t.numpy(), b.numpy())
        assert np.array_equal(m.cpu().numpy(), m_ref) and np.array_equal(p.cpu().numpy(), p_ref)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), o_ref.view(np.uint32))
        out2 = torch.empty_like(out)
        ctx.tree_bbox_matched(t.cuda(), b.cuda(), m, p, out2)
        torch.cuda.synchronize()
        assert np.array_equal(out2.cpu().numpy().view(np.uint32), o_ref.view(np.uint32))
        # the bench's multi-GPU step: the sharded fused pass (two all-gathers, no host sync)
        m3, p3, out3 = torch.full_like(m, -7), torch.full_like(p, -7), torch.full_like(out, 7.0)
        for check in (True, False):
            ctx.paren_match_tree_bbox(t.cuda(), b.cuda(), m3, p3, out3, check=check)
        ctx.status()
        assert np.array_equal(m3.cpu().numpy(), m_ref) and np.array_equal(p3.cpu().numpy(), p_ref)
        assert np.array_equal(out3.cpu().numpy().view(np.uint32), o_ref.view(np.uint32))
        # a capacity too small for this chunk is reported, not silently wrong
        with pytest.raises(tb.TreeBBoxError, match="-6"):
            ctx.paren_match_tree_bbox(t.cuda(), b.cuda(), m3, p3, out3, cap=16)
        ctx.close()
    finally:
        dist.destroy_process_group()
