"""Dev: per-kernel split of tree_transform on C5 (library profile hook)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, scenegen, paper_2205_11659_b200 as tb
tags, _ = scenegen.config(sys.argv[1] if len(sys.argv) > 1 else "C5", device="cuda")
n = tags.numel()
m, p = tb.paren_match(tags)
loc = torch.zeros((n, 6), device="cuda"); loc[:, 0] = 1; loc[:, 3] = 1; loc[:, 4:] = torch.rand((n, 2), device="cuda")
world = torch.empty_like(loc)
lib = tb.load(); lib.tb_profile_read.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
for _ in range(3): tb.tree_transform(tags, loc, m, p, world)
torch.cuda.synchronize()
lib.tb_profile_enable(1); lib.tb_profile_read(None, 0)
for _ in range(5): tb.tree_transform(tags, loc, m, p, world)
torch.cuda.synchronize()
buf = ctypes.create_string_buffer(1 << 16); lib.tb_profile_read(buf, len(buf)); lib.tb_profile_enable(0)
pk = json.loads(buf.value.decode() or "{}")
print({k: round(v[1] / 5, 4) for k, v in sorted(pk.items(), key=lambda kv: -kv[1][1])}, "n", n)
