"""Dev driver: fused path parity on a corpus + A/B timing against the two-call path.

    python tools/dev/fz_quick.py [check|time|both] [log2n]
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import oracle
import paper_2205_11659_b200 as tb
import scenegen


def cases():
    for n in (1, 2, 15, 16, 17, 2047, 2048, 2049, 4096 + 5, 3 * 2048 + 7, 40 * 2048 + 3, 200_003):
        for seed in range(2):
            yield f"walk n={n} s={seed}", scenegen.walk_tags(n, seed, p_leaf=0.5)
            yield f"walk0 n={n} s={seed}", scenegen.walk_tags(n, 50 + seed, p_leaf=0.0, p_clip=0.5)
    for n in (2048, 2049, 3 * 2048, 40 * 2048 + 3, 300 * 2048 + 9):
        yield f"opens n={n}", torch.full((n,), 1, dtype=torch.uint8)
        yield f"blends n={n}", torch.full((n,), 2, dtype=torch.uint8)
        yield f"closes n={n}", torch.full((n,), 3, dtype=torch.uint8)
        yield f"leaves n={n}", torch.zeros(n, dtype=torch.uint8)
        yield f"chain n={n}", scenegen.deep_chain_tags(n, 1)
        yield f"chainL n={n}", scenegen.deep_chain_tags(n, 2, leaves_mid=True)
        alt = torch.tensor([2, 0, 3], dtype=torch.uint8).repeat(n // 3 + 1)[:n]
        yield f"alt n={n}", alt
    g = torch.Generator().manual_seed(5)
    for n in (1000, 50_000, 300_000):
        t = torch.multinomial(torch.tensor([0.3, 0.15, 0.1, 0.45]), n, replacement=True, generator=g)
        yield f"iid n={n}", t.to(torch.uint8)
    n = 300_000
    opens = torch.where(torch.rand(n // 2, generator=g) < 0.7, 1, 2).to(torch.uint8)
    t = torch.stack([opens, torch.zeros(n // 2, dtype=torch.uint8)], 1).reshape(-1)
    yield "chain+leaves", torch.cat([t, torch.full((n // 2,), 3, dtype=torch.uint8)])
    yield "C4 2^20", scenegen.compacted_tags(1 << 20, 3)


def check():
    fails = 0
    for name, t in cases():
        if os.environ.get("FZ_VERBOSE"):
            print("case", name, flush=True)
        t = t.contiguous()
        n = t.numel()
        b = scenegen.boxes(n, 7, t)
        m_ref, p_ref = oracle.paren_match(t.numpy())
        o_ref = oracle.tree_bbox(t.numpy(), b.numpy()).view(np.uint32)
        m, p, o = tb.paren_match_tree_bbox(t.cuda(), b.cuda())
        o2 = tb.tree_bbox(t.cuda(), b.cuda())
        torch.cuda.synchronize()
        m, p = m.cpu().numpy(), p.cpu().numpy()
        o, o2 = o.cpu().numpy().view(np.uint32), o2.cpu().numpy().view(np.uint32)
        msg = []
        for nm, got, ref in (("parent", p, p_ref), ("match", m, m_ref)):
            if not np.array_equal(got, ref):
                bad = np.nonzero(got != ref)[0]
                msg.append(f"{nm}: {len(bad)} bad, first {bad[:5].tolist()} got {got[bad[:5]].tolist()} "
                           f"want {ref[bad[:5]].tolist()} tags {t.numpy()[bad[:5]].tolist()}")
        for nm, got in (("bbox(pair)", o), ("bbox(tree_bbox)", o2)):
            if not np.array_equal(got, o_ref):
                bad = np.nonzero((got != o_ref).any(1))[0]
                msg.append(f"{nm}: {len(bad)} bad, first {bad[:5].tolist()} tags {t.numpy()[bad[:5]].tolist()}")
        if msg:
            fails += 1
            print(f"FAIL {name}: " + " | ".join(msg), flush=True)
    print(f"check: {fails} failing cases", flush=True)
    return fails


def timing(log2n=27):
    lib = tb.load()
    lib.tb_profile_read.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
    n = 1 << log2n
    dev = torch.device("cuda")
    tags = scenegen.walk_tags(n, 4, device=dev)
    boxes = scenegen.boxes(n, 4, tags, device=dev)
    match = torch.empty(n, dtype=torch.int32, device=dev)
    parent = torch.empty(n, dtype=torch.int32, device=dev)
    out = torch.empty((n, 4), dtype=torch.float32, device=dev)
    res = {}
    for fused in (1, 0):
        lib.tb_debug_use_fused(fused)
        for _ in range(3):
            tb.paren_match_tree_bbox(tags, boxes, match, parent, out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 20
        a.record()
        for _ in range(K):
            tb.paren_match_tree_bbox(tags, boxes, match, parent, out)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / K
        lib.tb_profile_enable(1)
        for _ in range(5):
            tb.paren_match_tree_bbox(tags, boxes, match, parent, out)
        torch.cuda.synchronize()
        lib.tb_profile_enable(0)
        buf = ctypes.create_string_buffer(8192)
        lib.tb_profile_read(buf, 8192)
        per = {k: round(v[1] / v[0], 4) for k, v in json.loads(buf.value.decode()).items()}
        res["fused" if fused else "two-call"] = {"ms": round(ms, 4), "Gelem/s": round(n / ms / 1e6, 2), "kernels": per}
    lib.tb_debug_use_fused(1)
    tr = torch.zeros(16, dtype=torch.int64, device=dev)
    lib.tb_debug_fz_trace(tr.data_ptr())
    tb.paren_match_tree_bbox(tags, boxes, match, parent, out)
    torch.cuda.synchronize()
    lib.tb_debug_fz_trace(None)
    t = tr.cpu().tolist()
    res["fz_ctrl_phases_us"] = {"P0": (t[1] - t[0]) / 1e3, "P1": (t[2] - t[1]) / 1e3, "P2": (t[3] - t[2]) / 1e3,
                                "P3": (t[4] - t[3]) / 1e3, "P3_ansv": (t[9] - t[3]) / 1e3,
                                "P3_unres": (t[10] - t[9]) / 1e3, "P3_jump": (t[4] - t[10]) / 1e3,
                                "P4": (t[5] - t[4]) / 1e3, "P4_runs": (t[8] - t[4]) / 1e3, "P5": (t[7] - t[5]) / 1e3,
                                "rounds": t[6]}
    print(json.dumps(res, indent=1), flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "both"
    rc = 0
    if what in ("check", "both"):
        rc = check()
    if what in ("notma",):
        tb.load().tb_debug_fz_tma(0)
        rc = check()
        tb.load().tb_debug_fz_tma(1)
    if what in ("time", "both"):
        timing(int(sys.argv[2]) if len(sys.argv) > 2 else 27)
    sys.exit(1 if rc else 0)
