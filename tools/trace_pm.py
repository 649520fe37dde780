"""Dev: per-tile phase timing of the paren_match kernel (globaltimer)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, scenegen, paper_2205_11659_b200 as tb
lib = tb.load()
lib.tb_debug_paren_match_trace.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
names = ["start", "scanned", "w0_begin", "lookback_done", "published", "runs_found", "w1_query_begin", "w1_query_done", "syncC", "inc_ready", "end"]
for cfg in sys.argv[1:] or ["C5"]:
    tags, _ = scenegen.config(cfg, device="cuda")
    n = tags.numel(); nt = (n + 4095) // 4096
    m = torch.empty(n, dtype=torch.int32, device="cuda"); p = torch.empty_like(m)
    tr = torch.zeros(nt * 16, dtype=torch.int64, device="cuda")
    for _ in range(3):
        tr.zero_()
        lib.tb_debug_paren_match_trace(tags.data_ptr(), n, m.data_ptr(), p.data_ptr(), tr.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    t = tr.view(nt, 16).cpu().numpy()[:, :11].astype(np.float64)
    t0 = t[:, 0].min()
    t -= t0
    print(f"== {cfg} n={n} tiles={nt} kernel span {t[:,10].max()/1e3:.1f} us")
    for a, b in [(0,1),(1,2),(2,3),(3,4),(4,5),(6,7),(5,8),(8,9),(9,10),(0,10)]:
        d = (t[:, b] - t[:, a]) / 1e3
        print(f"  {names[a]:>14} -> {names[b]:<14} med {np.median(d):7.2f} p90 {np.percentile(d,90):7.2f} max {d.max():8.2f} us")
    # look-back depth: how far behind the INC frontier
    order = np.argsort(t[:, 0])
    print("  start spacing (us/tile):", np.median(np.diff(t[order, 0])) / 1e3)
