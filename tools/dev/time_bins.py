"""Dev: time bin_leaves on the C5 scene (boxes from tree_bbox)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, scenegen, paper_2205_11659_b200 as tb
tags, _ = scenegen.config("C5", device="cuda")
n = tags.numel()
node = tb.tree_bbox(tags, scenegen.boxes(n, 7, tags, device="cuda"))
for gw, bs in ((16, 256.0), (64, 64.0)):
    tb.bin_leaves(tags, node, gw, gw, bs)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    c, o, it = tb.bin_leaves(tags, node, gw, gw, bs)
    e.record(); e.synchronize()
    print(f"grid {gw}x{gw} bin {bs}: {s.elapsed_time(e):.2f} ms, items {it.numel()}, leaves {(tags == 0).sum().item()}")
