"""Multi-process (torch.distributed, gloo, CPU) tests of the shard protocols'
host logic: each rank holds one contiguous chunk of a global stream, the
protocol models (tests/shard_model.py, mirroring csrc/shard.cu) exchange
chunk summaries with real all-gathers, and every rank's slice of parent /
match (paren_match) or node_bbox (tree_bbox, bit-exact) must equal the oracle
on the whole stream."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import oracle
    import scenegen
    import shard_model as M
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_per = 6000
        seed = 11 + case
        if case == 0:   # random walk, one global stream generated shard by shard
            off = rank * n_per
            s_before = sum(scenegen.walk_step_sum(n_per, seed, offset=r * n_per) for r in range(rank))
            mine = scenegen.walk_tags(n_per, seed, offset=off, s_before=s_before).numpy()
            full = scenegen.walk_tags(world * n_per, seed).numpy()
        else:           # deep chain spanning all ranks, plus underflowing closes
            full = np.concatenate([scenegen.deep_chain_tags(world * n_per - 500, seed).numpy(),
                                   np.full(500, 3, np.uint8)])
            off = rank * n_per
            mine = full[off:off + n_per]

        def allgather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out

        parent, match = M.protocol(list(mine), off, rank, allgather)
        m_ref, p_ref = oracle.paren_match(full)
        ok = (np.array_equal(np.array(parent), p_ref[off:off + len(mine)]) and
              np.array_equal(np.array(match), m_ref[off:off + len(mine)]))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def _bbox_worker(rank, world, port, case, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import oracle
    import scenegen
    import shard_model as M
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_per = 3000
        seed = 21 + case
        if case == 0:
            full = scenegen.walk_tags(world * n_per, seed, p_leaf=0.4).numpy()
        else:  # deep chain with leaves spanning all ranks, blend opens never closed
            t = scenegen.deep_chain_tags(world * n_per - 300, seed, leaves_mid=True).numpy()
            full = np.concatenate([np.full(300, 2, np.uint8), t])
        boxes = scenegen.boxes(len(full), seed, torch.from_numpy(full)).numpy()
        m_ref, p_ref = oracle.paren_match(full)
        ref = oracle.tree_bbox(full, boxes)
        off = rank * n_per
        sl = slice(off, off + n_per)

        def allgather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out

        out = M.bbox_protocol(list(full[sl]), boxes[sl].tolist(), list(p_ref[sl]), list(m_ref[sl]), off, rank,
                              allgather)
        got = np.array(out, dtype=np.float32)
        q.put((rank, bool(np.array_equal(got.view(np.uint32), ref[sl].view(np.uint32)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", [0, 1])
def test_tree_bbox_shard_protocol_gloo(world, case):
    """The tree_bbox shard protocol (final stacks with chunk-local clips, chunk
    context chain, imported contexts, exported unions, fix-up) over gloo."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bbox_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", [0, 1])
def test_shard_protocol_gloo(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res
