"""The two-pass Bic scan's share of the fused step (fz_reduce + fz_ctrl, which
read the tags once more and scan the tile aggregates) at 2^24, 2^27 and 2^30
elements of the C5 walk: per-kernel CUDA-event times over 5 steps.
    python tools/time_scan_share.py"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import scenegen
import paper_2205_11659_b200 as tb

lib = tb.load()
lib.tb_profile_read.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
res = []
for lg in (24, 27, 30):
    n = 1 << lg
    t = scenegen.walk_tags(n, 4, device="cuda")
    b = torch.empty((n, 4), dtype=torch.float32, device="cuda")
    step = 1 << 26
    for s0 in range(0, n, step):
        e = min(n, s0 + step)
        b[s0:e] = scenegen.boxes(e - s0, 4, t[s0:e], offset=s0, device="cuda")
    m = torch.empty(n, dtype=torch.int32, device="cuda")
    p = torch.empty_like(m)
    o = torch.empty_like(b)
    for _ in range(2):
        tb.paren_match_tree_bbox(t, b, m, p, o)
    torch.cuda.synchronize()
    lib.tb_profile_enable(1)
    lib.tb_profile_read(None, 0)
    for _ in range(5):
        tb.paren_match_tree_bbox(t, b, m, p, o)
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16)
    lib.tb_profile_read(buf, len(buf))
    lib.tb_profile_enable(0)
    pk = {k: v[1] / 5 for k, v in json.loads(buf.value.decode() or "{}").items()}
    tot = sum(pk.values())
    scan = pk.get("fz_reduce", 0) + pk.get("fz_ctrl", 0)
    res.append({"log2n": lg, "step_ms": tot, "scan_ms": scan, "scan_share": scan / tot,
                "kernels_ms": {k: round(v, 4) for k, v in pk.items()}})
    del t, b, m, p, o
    tb.release_workspaces()
    torch.cuda.empty_cache()
print(json.dumps(res))
