"""Randomised sweep of the hot path against the oracle (GPU):

    python tools/fuzz.py [seconds] [seed]

Each case draws a size (1 .. ~400k, often near tile multiples), a tag mix
(leaf / clip / blend / close probabilities, including close-heavy underflow
mixes, deep chains and pure runs) and boxes, then checks bit-exact equality
with the oracle for: paren_match_tree_bbox (the bench step), paren_match and
tree_bbox alone, the round-1 virtual-shard box protocol and the sharded fused
pass (random shard counts), the chunked host pipeline (random chunk size), the
fused compaction (random commands inserted and dropped) and tree_fold.  Prints one line per failure and a summary."""
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
        # paren_match alone (fz_match), tree_bbox alone, the sharded fused pass
        m2, p2 = tb.paren_match(td)
        ok_m = np.array_equal(m2.cpu().numpy(), m_ref) and np.array_equal(p2.cpu().numpy(), p_ref)
        ok_t = np.array_equal(tb.tree_bbox(td, bd).cpu().numpy().view(np.uint32), ref)
        gs = int(rng.integers(1, 17))
        ms, ps, os_ = tb.pair_vshard(td, bd, gs, cap=n + 2)
        ok_s = (np.array_equal(ms.cpu().numpy(), m_ref) and np.array_equal(ps.cpu().numpy(), p_ref)
                and np.array_equal(os_.cpu().numpy().view(np.uint32), ref))
        # the fused compaction: commands (bytes 4-15) inserted at random, dropped by the keep map
        k = int(rng.integers(0, 2 * n + 1))
        pos = np.sort(rng.integers(0, n + 1, size=k))
        full = np.insert(t.numpy(), pos, rng.integers(4, 16, size=k).astype(np.uint8))
        fb = np.insert(b.numpy(), pos, rng.normal(size=(k, 4)).astype(np.float32), axis=0)
        tt, ii, mm, pp, oo, kk = tb.paren_match_tree_bbox_scene(torch.from_numpy(full).cuda(),
                                                              torch.from_numpy(np.ascontiguousarray(fb)).cuda())
        ok_c = (kk == n and np.array_equal(mm.cpu().numpy(), m_ref) and np.array_equal(pp.cpu().numpy(), p_ref)
                and np.array_equal(oo.cpu().numpy().view(np.uint32), ref))
        # tree_fold (2x2 matrices mod 2^32 up the tree)
        x = rng.integers(0, 1 << 32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
        f = tb.tree_fold(td, torch.from_numpy(x.view(np.int32)).cuda(), torch.from_numpy(m_ref).cuda())
        ok_f = np.array_equal(f.cpu().numpy().view(np.uint32), oracle.tree_fold(t.numpy(), x))
        cases += 1
        if not (ok and ok_v and ok_h and ok_m and ok_t and ok_s and ok_c and ok_f):
            fails += 1
            print(f"FAIL n={n} fused={ok} vshard(G={g})={ok_v} host(shift={shift})={ok_h} pm={ok_m} tb={ok_t} "
                  f"shard(G={gs})={ok_s} scene={ok_c} fold={ok_f}", flush=True)
    print(f"fuzz: {cases} cases, {fails} failures")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
