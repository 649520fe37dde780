"""Multi-process (torch.distributed, gloo, CPU) test of the sharded fused
protocol (csrc/fused_shard.cuh) through its model (tests/fused_shard_model.py):
each rank holds one contiguous chunk of a global stream, the two exchanges
are real all-gathers, and every rank's slice of parent / match / node_bbox
(fp32 bit patterns) must equal the oracle on the whole stream."""
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


def _stream(case, n):
    import scenegen
    if case == 0:  # random walk
        return scenegen.walk_tags(n, 31, p_leaf=0.4).numpy()
    if case == 1:  # blend opens only: unions cross every chunk
        return scenegen.walk_tags(n, 32, p_clip=0.0).numpy()
    if case == 2:  # deep chain with leaves spanning all ranks, blend opens never closed
        t = scenegen.deep_chain_tags(n - 300, 33, leaves_mid=True).numpy()
        return np.concatenate([np.full(300, 2, np.uint8), t])
    t = scenegen.walk_tags(n, 34).numpy()  # root pops in later chunks
    t[::5] = 3
    return t


def _worker(rank, world, port, case, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import oracle
    import scenegen
    import fused_shard_model as M
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 2500 * world + 37
        full = _stream(case, n)
        boxes = scenegen.boxes(n, 5, torch.from_numpy(full)).numpy()
        m_ref, p_ref = oracle.paren_match(full)
        ref = oracle.tree_bbox(full, boxes)
        off = [(n * k // world) & ~15 for k in range(world)] + [n]
        lo, hi = off[rank], off[rank + 1]

        def allgather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out

        m, p, o = M.protocol(full[lo:hi], boxes[lo:hi], lo, rank, allgather)
        ok = (np.array_equal(p, p_ref[lo:hi]) and np.array_equal(m, m_ref[lo:hi]) and
              np.array_equal(o.view(np.uint32), ref[lo:hi].view(np.uint32)))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", [0, 1, 2, 3])
def test_fused_shard_protocol_gloo(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res
