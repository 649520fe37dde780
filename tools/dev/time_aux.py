"""Dev: compact_scene (2^27 scene stream) and bin_leaves (C5) per-kernel split."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, scenegen, paper_2205_11659_b200 as tb
lib = tb.load(); lib.tb_profile_read.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
def prof(name, fn, k=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    lib.tb_profile_enable(1); lib.tb_profile_read(None, 0)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(k): fn()
    e.record(); torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16); lib.tb_profile_read(buf, len(buf)); lib.tb_profile_enable(0)
    pk = json.loads(buf.value.decode() or "{}")
    print(name, f"{s.elapsed_time(e) / k:.3f} ms/call", {kk: round(v[1] / k, 4) for kk, v in sorted(pk.items(), key=lambda kv: -kv[1][1])})
n = 1 << 27
t, b = scenegen.scene_stream(n, 3, device="cuda")
prof("compact", lambda: tb.compact_scene(t, b, scenegen.SCENE_KEEP_MAP))
tags, _ = scenegen.config("C5", device="cuda")
node = tb.tree_bbox(tags, scenegen.boxes(tags.numel(), 7, tags, device="cuda"))
for gw, bs in ((16, 256.0), (64, 64.0)):
    prof(f"bins {gw}x{gw}", lambda: tb.bin_leaves(tags, node, gw, gw, bs))
