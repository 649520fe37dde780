"""Dev helper: run one config through paren_match / tree_bbox a few times (for ncu)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import scenegen
import paper_2205_11659_b200 as tb
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--op", default="pm")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
tags, _ = scenegen.config(a.config, device="cuda")
n = tags.numel()
if a.op == "pm":
    m = torch.empty(n, dtype=torch.int32, device="cuda"); p = torch.empty_like(m)
    for _ in range(a.reps): tb.paren_match(tags, m, p)
elif a.op == "pair":
    boxes = scenegen.boxes(n, 7, tags, device="cuda"); out = torch.empty_like(boxes)
    m = torch.empty(n, dtype=torch.int32, device="cuda"); p = torch.empty_like(m)
    for _ in range(a.reps): tb.paren_match_tree_bbox(tags, boxes, m, p, out)
else:
    boxes = scenegen.boxes(n, 7, tags, device="cuda"); out = torch.empty_like(boxes)
    for _ in range(a.reps): tb.tree_bbox(tags, boxes, out)
torch.cuda.synchronize()
print("ok", n)
