"""Summarise an ncu source page per CUDA source line (needs -lineinfo):
share of warp-stall samples and of executed warp instructions."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
def f(x):
    try: return float(x.replace(",", ""))
    except: return 0.0
recs = []
fname = "?"
hdr = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr and len(r) >= 8 and r[2] == "-":
        recs.append((fname, r[0], r[1], f(r[4]), f(r[7])))
tot_s = sum(x[3] for x in recs) or 1
tot_i = sum(x[4] for x in recs) or 1
print(f"stall samples={tot_s:.0f} warp-instr={tot_i:.0f}")
for fn, ln, src, s, i in sorted(recs, key=lambda x: -x[3])[:top]:
    print(f"{fn[:14]:14} {ln:>4} {s/tot_s*100:5.1f}%s {i/tot_i*100:5.1f}%i  {src.strip()[:80]}")
