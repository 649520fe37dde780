"""Per-phase stall reasons (sampled) from an ncu source page.
    python tools/ncu_phase_stalls.py rep file A:1-10 B:11-20 ..."""
import csv, subprocess, sys
rep, fname = sys.argv[1], sys.argv[2]
ranges = []
for a in sys.argv[3:]:
    nm, r = a.split(":"); lo, hi = r.split("-"); ranges.append((nm, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
def f(x):
    try: return float(x.replace(",", ""))
    except: return 0.0
cur = "?"; idx = None; acc = {}
reasons = ["stall_barrier", "stall_branch_resolving", "stall_long_sb", "stall_short_sb", "stall_wait", "stall_mio",
           "stall_math", "stall_no_inst", "stall_lg", "stall_selected", "stall_not_selected", "stall_dispatch", "stall_drain", "stall_membar"]
for r in csv.reader(out.splitlines()):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": idx = {n: i for i, n in enumerate(r)}; continue
    if idx and len(r) > 10 and r[2] == "-":
        ln = int(r[0]); key = "helpers:" + cur
        if cur == fname:
            key = "other"
            for nm, lo, hi in ranges:
                if lo <= ln <= hi: key = nm
        d = acc.setdefault(key, {})
        d["instr"] = d.get("instr", 0) + f(r[idx["Instructions Executed"]])
        for rs in reasons:
            if rs in idx: d[rs] = d.get(rs, 0) + f(r[idx[rs]])
tot = sum(sum(v.get(rs, 0) for rs in reasons) for v in acc.values()) or 1
ti = sum(v["instr"] for v in acc.values()) or 1
print(f"{'phase':24} {'instr':>6} {'stall':>6} " + " ".join(f"{rs[6:14]:>8}" for rs in reasons[:9]))
for k, v in sorted(acc.items(), key=lambda x: -sum(x[1].get(rs, 0) for rs in reasons)):
    st = sum(v.get(rs, 0) for rs in reasons)
    print(f"{k:24} {v['instr']/ti*100:5.1f}% {st/tot*100:5.1f}% " + " ".join(f"{v.get(rs,0)/tot*100:7.1f}%" for rs in reasons[:9]))
