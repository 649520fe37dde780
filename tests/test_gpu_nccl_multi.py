"""Multi-GPU parity of the sharded bench step (paren_match_tree_bbox_shard over
NCCL, one process per GPU): every rank's chunk of match / parent / node_bbox
must equal the oracle on the whole stream, bit for bit.

Under pytest this launches itself with torchrun for G = 2, 4, 8 ranks (those
that fit the box's GPUs) and skips on a box with fewer than two GPUs; it can
also be run directly:
    python -m torch.distributed.run --standalone --nproc-per-node G tests/test_gpu_nccl_multi.py
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rank_main():
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    import oracle
    import scenegen
    import paper_2205_11659_b200 as tb

    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    fails = []

    def run(name, t, cap=None):
        n = t.numel()
        b = scenegen.boxes(n, 3, t).float().reshape(n, 4)
        m_ref, p_ref = oracle.paren_match(t.numpy())
        o_ref = oracle.tree_bbox(t.numpy(), b.numpy()).view(np.uint32)
        off = [(n * k // world) & ~15 for k in range(world)] + [n]
        lo, hi = off[rank], off[rank + 1]
        ctx = tb.ShardContext(world, rank, lo, hi - lo, device=dev)
        tt, bb = t[lo:hi].to(dev), b[lo:hi].to(dev)
        m = torch.empty(hi - lo, dtype=torch.int32, device=dev)
        p = torch.empty_like(m)
        o = torch.empty((hi - lo, 4), dtype=torch.float32, device=dev)
        ctx.paren_match_tree_bbox(tt, bb, m, p, o, cap=cap)
        ok = (np.array_equal(m.cpu().numpy(), m_ref[lo:hi]) and np.array_equal(p.cpu().numpy(), p_ref[lo:hi])
              and np.array_equal(o.cpu().numpy().view(np.uint32), o_ref[lo:hi]))
        if cap is None:  # tree_bbox alone and paren_match alone (the same protocol)
            o2 = torch.empty_like(o)
            ctx.tree_bbox(tt, bb, o2)
            m2, p2 = torch.empty_like(m), torch.empty_like(p)
            ctx.paren_match(tt, m2, p2)
            torch.cuda.synchronize()
            ok = ok and np.array_equal(o2.cpu().numpy().view(np.uint32), o_ref[lo:hi])
            ok = ok and np.array_equal(m2.cpu().numpy(), m_ref[lo:hi]) and np.array_equal(p2.cpu().numpy(), p_ref[lo:hi])
        ctx.close()
        if not ok:
            fails.append(f"{name} rank {rank}/{world}")

    run("random walk", scenegen.walk_tags((1 << 20) + 12345, 7))
    run("blend-only walk", scenegen.walk_tags(1 << 19, 8, p_clip=0.0))
    run("root pops", torch.where(torch.arange(1 << 18) % 7 == 0, 3, scenegen.walk_tags(1 << 18, 9)).to(torch.uint8))
    run("deep chain", scenegen.deep_chain_tags(1 << 18, 4), cap=(1 << 18) + 2)
    run("empty ranks", scenegen.walk_tags(16 * world - 13, 6))  # chunk borders at multiples of 16: some empty
    flag = torch.tensor([len(fails)], device=dev)
    dist.all_reduce(flag)
    dist.destroy_process_group()
    if fails:
        print("FAIL", fails, flush=True)
    return 0 if int(flag.item()) == 0 else 1


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 4, 8])
def test_multi_gpu_parity(G):
    if torch.cuda.device_count() < G:
        pytest.skip(f"needs {G} GPUs (this box has {torch.cuda.device_count()})")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "tests"),
                                                      os.environ.get("PYTHONPATH", "")]))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", str(G),
                        os.path.abspath(__file__)], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


if __name__ == "__main__":
    sys.exit(rank_main())
