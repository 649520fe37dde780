import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, scenegen, paper_2205_11659_b200 as tb
for n in (1, 5000, 100000):
    t = scenegen.walk_tags(n, 0, p_leaf=0.5)
    b = scenegen.boxes(n, 7, t)
    m, p, o = tb.paren_match_tree_bbox(t.cuda(), b.cuda())
    torch.cuda.synchronize()
    print("ok pair", n, flush=True)
    o2 = tb.tree_bbox(t.cuda(), b.cuda())
    torch.cuda.synchronize()
    print("ok tb", n, flush=True)
