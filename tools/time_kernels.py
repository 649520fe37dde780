"""Dev timing helper: CUDA-event timing of the C-ABI calls on one GPU."""
import argparse
import json
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import scenegen
import paper_2205_11659_b200 as tb


def time_fn(fn, iters=20, warmup=3, flush=None):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        if flush is not None:
            flush.zero_()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2], ts[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C3,C4,C5")
    ap.add_argument("--bbox", action="store_true")
    ap.add_argument("--transform", action="store_true", help="also time tree_transform (57 B/element)")
    args = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for name in args.configs.split(","):
        tags, info = scenegen.config(name, device="cuda")
        n = tags.numel()
        m = torch.empty(n, dtype=torch.int32, device="cuda")
        p = torch.empty(n, dtype=torch.int32, device="cuda")
        if name.upper() == "J1":  # raw text bytes through the JSON class map
            med, mn = time_fn(lambda: tb.paren_match_bytes(tags, scenegen.JSON_CLASS_MAP, m, p), flush=flush)
        else:
            med, mn = time_fn(lambda: tb.paren_match(tags, m, p), flush=flush)
        row = {"config": name, "n": n, "pm_ms": med, "pm_min_ms": mn,
               "pm_Gelem_s": n / med / 1e6, "pm_GBs": 9 * n / med / 1e6}
        if args.bbox and name.upper() != "J1":
            boxes = scenegen.boxes(n, 7, tags, device="cuda")
            out = torch.empty_like(boxes)
            med, mn = time_fn(lambda: tb.tree_bbox(tags, boxes, out), flush=flush)
            row.update({"tb_ms": med, "tb_Gelem_s": n / med / 1e6, "tb_GBs": 33 * n / med / 1e6})
            med, mn = time_fn(lambda: tb.paren_match_tree_bbox(tags, boxes, m, p, out), flush=flush)
            row.update({"pair_ms": med, "pair_Gelem_s": n / med / 1e6, "pair_GBs": 41 * n / med / 1e6})
        if args.transform and name.upper() != "J1":
            tb.paren_match(tags, m, p)
            loc = torch.zeros((n, 6), dtype=torch.float32, device="cuda")
            loc[:, 0] = 1
            loc[:, 3] = 1
            loc[:, 4:] = torch.rand((n, 2), device="cuda")
            world = torch.empty_like(loc)
            med, mn = time_fn(lambda: tb.tree_transform(tags, loc, m, p, world), flush=flush)
            row.update({"tt_ms": med, "tt_Gelem_s": n / med / 1e6, "tt_GBs": 57 * n / med / 1e6})
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
