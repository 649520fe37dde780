"""Dev: inspect tree_bbox virtual-shard mismatches (prints a few bad elements)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch, oracle, scenegen, paper_2205_11659_b200 as tb
G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
t = scenegen.walk_tags(1_000_003, 7, p_leaf=0.5)
b = scenegen.boxes(t.numel(), 0, t)
n = t.numel()
ref = oracle.tree_bbox(t.numpy(), b.numpy())
m, p = oracle.paren_match(t.numpy())
out = tb.tree_bbox_vshard(t.cuda(), b.cuda(), G).cpu().numpy()
bad = np.nonzero((out.view(np.uint32) != ref.view(np.uint32)).any(1))[0]
splits = [((n * g // G) & ~63) if g else 0 for g in range(G)] + [n]
print("n", n, "splits", splits, "bad", len(bad))
tn = t.numpy(); bn = b.numpy()
# clipped leaf boxes from the oracle output
leafm = ~np.isin(tn, [1, 2, 3])
for i in bad[:8]:
    o = m[i]
    print(f"i={i} tag={tn[i]} match={o} parent={p[i]} got={out[i]} ref={ref[i]}")
    if tn[i] == 3 and o >= 0:
        lo, hi = o, i
    elif tn[i] in (1, 2):
        lo, hi = i, (o if o >= 0 else n)
    else:
        continue
    for a, c in [(lo + 1, hi)]:
        seg = np.arange(a, c)
        lv = seg[leafm[seg]]
        U = np.array([ref[lv, 0].min(), ref[lv, 1].min(), ref[lv, 2].max(), ref[lv, 3].max()]) if len(lv) else None
        # per-chunk partials
        parts = []
        for g in range(G):
            s0, s1 = max(a, splits[g]), min(c, splits[g + 1])
            if s0 < s1:
                sl = np.arange(s0, s1); sl = sl[leafm[sl]]
                if len(sl): parts.append((g, [ref[sl, 0].min(), ref[sl, 1].min(), ref[sl, 2].max(), ref[sl, 3].max()]))
        print("   range", a, c, "U", U, "parts", parts)
