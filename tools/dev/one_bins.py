import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, scenegen, paper_2205_11659_b200 as tb
tags, _ = scenegen.config("C5", device="cuda")
node = tb.tree_bbox(tags, scenegen.boxes(tags.numel(), 7, tags, device="cuda"))
tb.bin_leaves(tags, node, 16, 16, 256.0); torch.cuda.synchronize(); print("ok")
