"""Launch-bound configs (C1: 1000 elements, C2: 2^20 + closing tail): the
bench step (paren_match_tree_bbox) eager vs replayed from a CUDA graph
(torch.cuda.CUDAGraph capture of one call; the library's launches, the
cooperative control kernel included, are stream-ordered and capturable).
CUDA events around K back-to-back steps after warm-up.
    python tools/time_graph.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import scenegen
import paper_2205_11659_b200 as tb


def run(name):
    t = scenegen.config(name)[0].cuda()
    n = t.numel()
    b = scenegen.boxes(n, 1, t.cpu()).float().cuda()
    m = torch.empty(n, dtype=torch.int32, device="cuda")
    p = torch.empty_like(m)
    o = torch.empty_like(b)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(5):
            tb.paren_match_tree_bbox(t, b, m, p, o)
    torch.cuda.synchronize()
    ref = (m.clone(), p.clone(), o.clone())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        tb.paren_match_tree_bbox(t, b, m, p, o)
    torch.cuda.synchronize()
    m.fill_(-9), p.fill_(-9), o.fill_(0)
    g.replay()
    torch.cuda.synchronize()
    same = torch.equal(m, ref[0]) and torch.equal(p, ref[1]) and torch.equal(o.view(torch.int32), ref[2].view(torch.int32))
    K = 200

    def ev(fn):
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(K):
            fn()
        e.record()
        torch.cuda.synchronize()
        return a.elapsed_time(e) / K

    eager = ev(lambda: tb.paren_match_tree_bbox(t, b, m, p, o))
    graph = ev(g.replay)
    return {"config": name, "n": n, "eager_us": eager * 1e3, "graph_us": graph * 1e3,
            "graph_Gelem_s": n / graph / 1e6, "eager_Gelem_s": n / eager / 1e6, "graph_equal": same}


print(json.dumps([run("C1"), run("C2")]))
import ctypes
lib = tb.load()
lib.tb_profile_read.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
for name in ("C1", "C2"):
    t = scenegen.config(name)[0].cuda()
    b = scenegen.boxes(t.numel(), 1, t.cpu()).float().cuda()
    tb.paren_match_tree_bbox(t, b)
    torch.cuda.synchronize()
    lib.tb_profile_enable(1)
    lib.tb_profile_read(None, 0)
    for _ in range(20):
        tb.paren_match_tree_bbox(t, b)
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16)
    lib.tb_profile_read(buf, len(buf))
    lib.tb_profile_enable(0)
    pk = json.loads(buf.value.decode() or "{}")
    print(name, {k: round(v[1] / 20 * 1e3, 1) for k, v in pk.items()}, "us per call")
