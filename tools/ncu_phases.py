"""Per-phase share of executed warp instructions and stall samples of a kernel,
from an ncu source page (needs -lineinfo).  Phases are line ranges of one file:
    python tools/ncu_phases.py rep.ncu-rep fused.cu A:456-480 B:481-497 ...
Lines of other files (inlined helpers) are attributed to 'helpers:<file>'."""
import csv, subprocess, sys
rep, fname = sys.argv[1], sys.argv[2]
ranges = []
for a in sys.argv[3:]:
    nm, r = a.split(":")
    lo, hi = r.split("-")
    ranges.append((nm, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
def f(x):
    try: return float(x.replace(",", ""))
    except: return 0.0
cur = "?"; hdr = None; acc = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr and len(r) >= 8 and r[2] == "-":
        ln = int(r[0]); key = "helpers:" + cur
        if cur == fname:
            key = "other"
            for nm, lo, hi in ranges:
                if lo <= ln <= hi: key = nm
        s, i = acc.get(key, (0.0, 0.0))
        acc[key] = (s + f(r[4]), i + f(r[7]))
ts = sum(v[0] for v in acc.values()) or 1; ti = sum(v[1] for v in acc.values()) or 1
for k, (s, i) in sorted(acc.items(), key=lambda x: -x[1][1]):
    print(f"{k:28} instr {i/ti*100:5.1f}%  stalls {s/ts*100:5.1f}%")
