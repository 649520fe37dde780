"""Dev: paren_match alone, per-kernel CUDA-event times (C5 walk 2^27, or C3 with arg 'C3')."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, scenegen, paper_2205_11659_b200 as tb
cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
t = scenegen.deep_chain_tags(1 << 24, 2, device="cuda") if cfg == "C3" else scenegen.walk_tags(1 << 27, 4, device="cuda")
n = t.numel()
m = torch.empty(n, dtype=torch.int32, device="cuda"); p = torch.empty_like(m)
lib = tb.load(); lib.tb_profile_read.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
for fused in (1, 0):
    lib.tb_debug_use_fused(fused)
    for _ in range(3): tb.paren_match(t, m, p)
    torch.cuda.synchronize()
    lib.tb_profile_enable(1); lib.tb_profile_read(None, 0)
    for _ in range(10): tb.paren_match(t, m, p)
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16); lib.tb_profile_read(buf, len(buf)); lib.tb_profile_enable(0)
    pk = json.loads(buf.value.decode() or "{}")
    print(cfg, "fused" if fused else "round-1", {k: round(v[1] / 10, 4) for k, v in pk.items()})
lib.tb_debug_use_fused(1)
