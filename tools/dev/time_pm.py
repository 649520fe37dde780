"""Dev: paren_match alone at 2^27 (C5), per-kernel CUDA-event times."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, scenegen, paper_2205_11659_b200 as tb
n = 1 << 27
t = scenegen.walk_tags(n, 4, device="cuda")
m = torch.empty(n, dtype=torch.int32, device="cuda"); p = torch.empty_like(m)
for _ in range(3): tb.paren_match(t, m, p)
torch.cuda.synchronize()
lib = tb.load(); lib.tb_profile_read.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
lib.tb_profile_enable(1); lib.tb_profile_read(None, 0)
for _ in range(10): tb.paren_match(t, m, p)
torch.cuda.synchronize()
buf = ctypes.create_string_buffer(1 << 16); lib.tb_profile_read(buf, len(buf)); lib.tb_profile_enable(0)
pk = json.loads(buf.value.decode() or "{}")
print({k: round(v[1] / 10, 4) for k, v in pk.items()})
