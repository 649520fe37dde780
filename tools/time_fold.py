"""tree_fold at C5 size (2^27 elements): CUDA-event time per call (after
warm-up), per-kernel times, and the effective bandwidth at its algorithmic
bytes (tags 1 + payload 16 + match 4 + out 16 = 37 B/element).
    python tools/time_fold.py [log2n]"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import scenegen
import paper_2205_11659_b200 as tb

n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 27)
t = scenegen.walk_tags(n, 4, device="cuda")
x = torch.randint(0, 1 << 31, (n, 4), dtype=torch.int32, device="cuda")
m, _ = tb.paren_match(t)
out = torch.empty_like(x)
for _ in range(3):
    tb.tree_fold(t, x, m, out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
k = 10
a.record()
for _ in range(k):
    tb.tree_fold(t, x, m, out)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / k
lib = tb.load()
lib.tb_profile_read.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
lib.tb_profile_enable(1)
lib.tb_profile_read(None, 0)
for _ in range(k):
    tb.tree_fold(t, x, m, out)
torch.cuda.synchronize()
buf = ctypes.create_string_buffer(1 << 16)
lib.tb_profile_read(buf, len(buf))
lib.tb_profile_enable(0)
pk = json.loads(buf.value.decode() or "{}")
print(json.dumps({"n": n, "ms": ms, "Gelem_s": n / ms / 1e6, "GB_s_at_37B": 37 * n / ms / 1e6,
                  "kernels_ms": {kk: v[1] / k for kk, v in pk.items()}}))
