"""Timing experiment: fz_main with phases skipped (results are wrong)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, scenegen, paper_2205_11659_b200 as tb
lib = tb.load()
lib.tb_profile_read.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
n = 1 << 27
tags = scenegen.walk_tags(n, 4, device="cuda"); boxes = scenegen.boxes(n, 4, tags, device="cuda")
m = torch.empty(n, dtype=torch.int32, device="cuda"); p = torch.empty_like(m); out = torch.empty_like(boxes)
for mask in [0] + [int(x) for x in sys.argv[1:]]:
    lib.tb_debug_fz_abl(mask)
    for _ in range(3): tb.paren_match_tree_bbox(tags, boxes, m, p, out)
    torch.cuda.synchronize()
    lib.tb_profile_enable(1); lib.tb_profile_read(None, 0)
    for _ in range(10): tb.paren_match_tree_bbox(tags, boxes, m, p, out)
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(8192); lib.tb_profile_read(buf, 8192); lib.tb_profile_enable(0)
    d = json.loads(buf.value.decode())
    print(mask, "fz_main ms", round(d["fz_main"][1] / d["fz_main"][0], 4), flush=True)
lib.tb_debug_fz_abl(0)
