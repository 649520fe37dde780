"""Dev: per-tile phase timing of bb_finish (globaltimer)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, scenegen, paper_2205_11659_b200 as tb
lib = tb.load()
P = ctypes.c_void_p
lib.tb_debug_tree_bbox_trace.argtypes = [P, P, ctypes.c_int64, P, P, P]
names = ["A load+B", "C ptrjump", "D pending", "E walk", "F publish", "G closes", "H copyout", "end"]
for cfg in sys.argv[1:] or ["C5"]:
    tags, _ = scenegen.config(cfg, device="cuda")
    n = tags.numel(); TL = lib.tb_debug_bb_tile(); nt = (n + TL - 1) // TL
    b = scenegen.boxes(n, 7, tags, device="cuda"); out = torch.empty_like(b)
    tr = torch.zeros(nt * 16, dtype=torch.int64, device="cuda")
    for _ in range(2):
        tr.zero_()
        rc = lib.tb_debug_tree_bbox_trace(tags.data_ptr(), b.data_ptr(), n, out.data_ptr(), tr.data_ptr(), torch.cuda.current_stream().cuda_stream); assert rc == 0, (rc, lib.tb_last_error())
    torch.cuda.synchronize()
    t = tr.view(nt, 16).cpu().numpy()[:, :8].astype(np.float64)
    t -= t[:, 0].min()
    print(f"== {cfg} n={n} tiles={nt} span {t[:,7].max()/1e3:.1f} us")
    for a in range(7):
        d = (t[:, a + 1] - t[:, a]) / 1e3
        print(f"  {names[a]:>10} -> {names[a+1]:<10} med {np.median(d):7.2f} p90 {np.percentile(d,90):7.2f} max {d.max():8.2f} us")
    full = tr.view(nt, 16).cpu().numpy().astype(np.float64)
    for a, b, nm in ((4, 8, "F windows+bar"), (8, 9, "F wmid+bar"), (9, 10, "F backward"), (10, 5, "F tile union")):
        if full[:, b].max() > 0:
            d = (full[:, b] - full[:, a]) / 1e3
            print(f"  {nm:>24} med {np.median(d):7.2f} p90 {np.percentile(d,90):7.2f} us")
    d = (t[:, 7] - t[:, 0]) / 1e3
    print(f"  tile total med {np.median(d):.2f} p90 {np.percentile(d,90):.2f}")
