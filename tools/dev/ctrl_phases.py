"""Dev: fz_ctrl phase times (block 0 globaltimer trace) on a bench config: python tools/dev/ctrl_phases.py C2"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, scenegen, paper_2205_11659_b200 as tb
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
tags, _ = scenegen.config(cfg, device="cuda")
n = tags.numel()
boxes = scenegen.boxes(n, 3, tags.cpu()).float().reshape(n, 4).cuda()
m = torch.empty(n, dtype=torch.int32, device="cuda"); p = torch.empty_like(m)
o = torch.empty((n, 4), dtype=torch.float32, device="cuda")
lib = tb.load()
for _ in range(3): tb.paren_match_tree_bbox(tags, boxes, m, p, o)
torch.cuda.synchronize()
res = []
for _ in range(5):
    tr = torch.zeros(16, dtype=torch.int64, device="cuda")
    lib.tb_debug_fz_trace(tr.data_ptr())
    tb.paren_match_tree_bbox(tags, boxes, m, p, o)
    torch.cuda.synchronize()
    lib.tb_debug_fz_trace(None)
    t = tr.cpu().tolist()
    res.append({"P0": (t[1] - t[0]) / 1e3, "P1": (t[2] - t[1]) / 1e3, "P2": (t[3] - t[2]) / 1e3,
                "P3_ansv": (t[9] - t[3]) / 1e3, "P3_unres": (t[10] - t[9]) / 1e3, "P3_jump": (t[4] - t[10]) / 1e3,
                "P4_runs": (t[8] - t[4]) / 1e3, "P4_rounds": (t[5] - t[8]) / 1e3, "P5": (t[7] - t[5]) / 1e3,
                "rounds": t[6], "total": (t[7] - t[0]) / 1e3})
print(cfg, n, json.dumps(res[-1]))
