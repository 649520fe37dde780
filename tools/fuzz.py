"""Randomised sweep of the hot path against the oracle (GPU):

    python tools/fuzz.py [seconds] [seed]

Each case draws a size (1 .. ~400k, often near tile multiples), a tag mix
(leaf / clip / blend / close probabilities, including close-heavy underflow
mixes, deep chains and pure runs) and boxes, then checks bit-exact equality
with the oracle for: paren_match_tree_bbox (the bench step), the virtual-shard
protocol with a random shard count, and the chunked host pipeline with a
random chunk size.  Prints one line per failure and a summary."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_2205_11659_b200 as tb
import scenegen


def draw_tags(rng: np.random.Generator, n: int) -> torch.Tensor:
    kind = rng.integers(0, 6)
    if kind == 0:  # random walk with a random leaf share
        return scenegen.walk_tags(n, int(rng.integers(1 << 30)), p_leaf=float(rng.uniform(0.0, 0.9)),
                                  p_clip=float(rng.uniform(0.0, 1.0)))
    if kind == 1:  # i.i.d. tags (underflow-heavy when closes dominate)
        p = rng.dirichlet(np.ones(4))
        return torch.from_numpy(rng.choice(4, size=n, p=p).astype(np.uint8))
    if kind == 2:  # deep chain, optionally with leaves
        return scenegen.deep_chain_tags(n, int(rng.integers(1 << 30)), leaves_mid=bool(rng.integers(2)))
    if kind == 3:  # runs of one tag
        out = np.empty(n, np.uint8)
        i = 0
        while i < n:
            k = int(rng.integers(1, 3000))
            out[i:i + k] = rng.integers(0, 4)
            i += k
        return torch.from_numpy(out)
    if kind == 4:  # nested blocks: opens then closes, with leaves between
        d = int(rng.integers(1, 5000))
        one = np.concatenate([rng.choice([1, 2], size=d), np.zeros(int(rng.integers(0, 50)), np.uint8),
                              np.full(d, 3, np.uint8)]).astype(np.uint8)
        return torch.from_numpy(np.resize(one, n))
    return scenegen.walk_tags(n, int(rng.integers(1 << 30)))


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    lib = tb.load()
    t_end = time.time() + budget
    cases = fails = 0
    while time.time() < t_end:
        base = int(rng.choice([1, 1024, 4096, 8192, 65536]))
        n = int(max(1, base * int(rng.integers(1, 50)) + int(rng.integers(-3, 4)))) if rng.random() < 0.5 \
            else int(rng.integers(1, 400_000))
        t = draw_tags(rng, n)
        b = scenegen.boxes(n, int(rng.integers(1 << 30)), t)
        m_ref, p_ref = oracle.paren_match(t.numpy())
        ref = oracle.tree_bbox(t.numpy(), b.numpy()).view(np.uint32)
        td, bd = t.cuda(), b.cuda()
        m, p, out = tb.paren_match_tree_bbox(td, bd)
        torch.cuda.synchronize()
        ok = (np.array_equal(m.cpu().numpy(), m_ref) and np.array_equal(p.cpu().numpy(), p_ref)
              and np.array_equal(out.cpu().numpy().view(np.uint32), ref))
        g = min(int(rng.integers(1, 9)), n)
        vs = tb.tree_bbox_vshard(td, bd, g)
        torch.cuda.synchronize()
        ok_v = np.array_equal(vs.cpu().numpy().view(np.uint32), ref)
        shift = int(rng.integers(10, 16))
        old = lib.tb_debug_host_chunk_shift(shift)
        hm = torch.empty(n, dtype=torch.int32).pin_memory()
        hp = torch.empty_like(hm).pin_memory()
        ho = torch.empty((n, 4), dtype=torch.float32).pin_memory()
        tb.paren_match_tree_bbox_host(t.pin_memory(), b.pin_memory(), hm, hp, ho)
        lib.tb_debug_host_chunk_shift(old)
        ok_h = np.array_equal(ho.numpy().view(np.uint32), ref) and np.array_equal(hm.numpy(), m_ref)
        cases += 1
        if not (ok and ok_v and ok_h):
            fails += 1
            print(f"FAIL n={n} fused={ok} vshard(G={g})={ok_v} host(shift={shift})={ok_h}", flush=True)
    print(f"fuzz: {cases} cases, {fails} failures")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
