"""Drive every C-ABI entry point once on small seeded inputs that still span
many tiles, checking the results of the paths that must agree bit for bit
(tree_bbox vs tree_bbox_matched, virtual shards vs one device, the chunked
host pipeline vs the device call).  Meant to run under compute-sanitizer
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize.py

(compute-sanitizer is disabled on the round-1 GPU pool; the driver itself ran
clean there.)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2205_11659_b200 as tb
import scenegen


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 150_001
    cases = [scenegen.walk_tags(n, 3), scenegen.deep_chain_tags(n // 2, 4, leaves_mid=True),
             torch.full((20_000,), 2, dtype=torch.uint8)]
    for i, t in enumerate(cases):
        tags = t.cuda()
        boxes = scenegen.boxes(t.numel(), 10 + i, t).cuda()
        m, p = tb.paren_match(tags)
        out = tb.tree_bbox_matched(tags, boxes, m, p)
        out2 = tb.tree_bbox(tags, boxes)
        assert torch.equal(out.view(torch.int32), out2.view(torch.int32))
        loc = torch.zeros((t.numel(), 6), device="cuda")
        loc[:, 0] = 1
        loc[:, 3] = 1
        loc[:, 4:] = torch.rand((t.numel(), 2), device="cuda")
        tb.tree_transform(tags, loc, m, p)
        tb.bin_leaves(tags, out, 16, 16, 64.0)
        tb.compact_scene(tags, boxes, scenegen.SCENE_KEEP_MAP)
        vs = tb.tree_bbox_vshard(tags, boxes, 3)
        assert torch.equal(vs.view(torch.int32), out.view(torch.int32))
        mv, pv = tb.paren_match_vshard(tags, 3)
        assert torch.equal(mv, m) and torch.equal(pv, p)
        # chunked host path (small chunks)
        lib = tb.load()
        old = lib.tb_debug_host_chunk_shift(12)
        hb = boxes.cpu().pin_memory()
        hm = torch.empty(t.numel(), dtype=torch.int32).pin_memory()
        hp = torch.empty_like(hm).pin_memory()
        ho = torch.empty_like(hb).pin_memory()
        tb.paren_match_tree_bbox_host(t.pin_memory(), hb, hm, hp, ho)
        lib.tb_debug_host_chunk_shift(old)
        assert torch.equal(ho.view(torch.int32), out.cpu().view(torch.int32))
    text = scenegen.json_text(100_000, 5).cuda()
    tb.paren_match_bytes(text, scenegen.JSON_CLASS_MAP)
    torch.cuda.synchronize()
    print("sanitize driver ok", n)


if __name__ == "__main__":
    main()
