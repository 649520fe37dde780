"""Fused stream compaction (paren_match_tree_bbox_scene) against the two-step
path (compact_scene, then paren_match_tree_bbox on its output) on the S1 scene
stream, CUDA events after warm-up.
    python tools/time_scene.py [log2n] [p_cmd]"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import scenegen
import paper_2205_11659_b200 as tb

n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 27)
p_cmd = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
s, b = scenegen.scene_stream(n, 4, p_cmd=p_cmd, device="cuda")
keep = bytes([1, 1, 1, 1] + [0] * 252)


def ev(fn, k=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    e.record()
    torch.cuda.synchronize()
    return a.elapsed_time(e) / k


fused = ev(lambda: tb.paren_match_tree_bbox_scene(s, b, keep, sync=False))
t2, b2, _ = tb.compact_scene(s, b, keep)
kept = t2.numel()
comp = ev(lambda: tb.compact_scene(s, b, keep))
t2, b2 = t2.contiguous(), b2.contiguous()
pair = ev(lambda: tb.paren_match_tree_bbox(t2, b2))
lib = tb.load()
lib.tb_profile_read.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
lib.tb_profile_enable(1)
lib.tb_profile_read(None, 0)
for _ in range(5):
    tb.paren_match_tree_bbox_scene(s, b, keep, sync=False)
torch.cuda.synchronize()
buf = ctypes.create_string_buffer(1 << 16)
lib.tb_profile_read(buf, len(buf))
lib.tb_profile_enable(0)
pk = json.loads(buf.value.decode() or "{}")
# algorithmic bytes: the full stream in (tags 1 + boxes 16 per element), kept outputs
# (tags 1 + index 4 + match 4 + parent 4 + node_bbox 16 = 29 per kept element)
byt = 17 * n + 29 * kept
print(json.dumps({"n": n, "p_cmd": p_cmd, "kept": kept, "fused_ms": fused, "two_step_ms": comp + pair,
                  "compact_ms": comp, "pair_ms": pair, "fused_GBs": byt / fused / 1e6,
                  "fused_Gelem_s_full_stream": n / fused / 1e6,
                  "kernels_ms": {kk: v[1] / 5 for kk, v in pk.items()}}))
