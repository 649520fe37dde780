"""Dev: the sharded bench step (paren_match_tree_bbox_shard, NCCL world of one
rank) against the unsharded fused step on the same stream (CUDA events): the
protocol's own overhead (export / compose / fix-up kernels, two all-gathers)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, torch.distributed as dist
import scenegen, paper_2205_11659_b200 as tb
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 27)
tags = scenegen.walk_tags(n, 4, device="cuda"); boxes = scenegen.boxes(n, 4, tags, device="cuda")
m = torch.empty(n, dtype=torch.int32, device="cuda"); p = torch.empty_like(m); out = torch.empty_like(boxes)
ctx = tb.ShardContext(1, 0, 0, n)
def t(fn, k=10):
    for _ in range(3): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(k): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / k
plain = t(lambda: tb.paren_match_tree_bbox(tags, boxes, m, p, out))
ref = (m.clone(), p.clone(), out.clone())
shard = t(lambda: ctx.paren_match_tree_bbox(tags, boxes, m, p, out, check=False))
ctx.status()
same = torch.equal(m, ref[0]) and torch.equal(p, ref[1]) and torch.equal(out.view(torch.int32), ref[2].view(torch.int32))
print(f"n=2^{n.bit_length()-1} plain {plain:.3f} ms  shard(world 1) {shard:.3f} ms  (+{(shard / plain - 1) * 100:.1f} %)  same={same}")
import ctypes, json
lib = tb.load()
lib.tb_profile_read.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
for name, fn in (("plain", lambda: tb.paren_match_tree_bbox(tags, boxes, m, p, out)),
                 ("shard", lambda: ctx.paren_match_tree_bbox(tags, boxes, m, p, out, check=False))):
    lib.tb_profile_enable(1); lib.tb_profile_read(None, 0)
    for _ in range(5): fn()
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16); lib.tb_profile_read(buf, len(buf)); lib.tb_profile_enable(0)
    pk = json.loads(buf.value.decode() or "{}")
    tot = sum(v[1] for v in pk.values()) / 5
    print(name, f"kernel sum {tot:.3f} ms/step", {k: round(v[1] / 5, 4) for k, v in sorted(pk.items(), key=lambda kv: -kv[1][1])})
ctx.close(); dist.destroy_process_group()
