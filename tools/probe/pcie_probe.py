"""PCIe bound of the e2e step: pinned host <-> device copies of the bench's
per-step bytes (H2D 17 B, D2H 24 B per element at 2^27), each direction alone
and both at once on two streams."""
import json
import torch

n = 1 << 27
hi = torch.empty(17 * n, dtype=torch.uint8).pin_memory()
ho = torch.empty(24 * n, dtype=torch.uint8).pin_memory()
di = torch.empty(17 * n, dtype=torch.uint8, device="cuda")
do = torch.empty(24 * n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def h2d():
    di.copy_(hi, non_blocking=True)


def d2h():
    ho.copy_(do, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        di.copy_(hi, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


r = {"h2d_ms": t(h2d), "d2h_ms": t(d2h), "both_ms": t(both)}
r["h2d_GBs"] = 17 * n / r["h2d_ms"] / 1e6
r["d2h_GBs"] = 24 * n / r["d2h_ms"] / 1e6
r["e2e_bound_Gelem_s"] = n / r["both_ms"] / 1e6
print(json.dumps(r))
