"""Per-source-line table from an ncu report (needs -lineinfo): executed warp
instructions, average active threads, stall samples, excess shared wavefronts.
    python tools/ncu_lines.py rep.ncu-rep [sort=instr|stall|conf] [top]"""
import csv, subprocess, sys
rep = sys.argv[1]
key = sys.argv[2] if len(sys.argv) > 2 else "instr"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
def f(x):
    try: return float(x.replace(",", ""))
    except: return 0.0
cur = "?"; idx = None; recs = []
for r in csv.reader(out.splitlines()):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": idx = {n: i for i, n in enumerate(r)}; continue
    if idx and len(r) > 10 and r[2] == "-":
        col = lambda name: f(r[idx[name]]) if name in idx else 0.0  # absent when the kernel has no such traffic
        recs.append(dict(file=cur, line=r[0], src=r[1].strip(), instr=col("Instructions Executed"),
                         thr=col("Thread Instructions Executed"), stall=col("Warp Stall Sampling (All Samples)"),
                         conf=col("L1 Wavefronts Shared Excessive")))
ti = sum(x["instr"] for x in recs) or 1; ts = sum(x["stall"] for x in recs) or 1; tc = sum(x["conf"] for x in recs) or 1
print(f"warp-instr {ti:.3g}  stall samples {ts:.3g}  excess shared wavefronts {tc:.3g}")
for x in sorted(recs, key=lambda x: -x[key])[:top]:
    act = x["thr"] / x["instr"] if x["instr"] else 0
    print(f"{x['file'][:12]:12} {x['line']:>4} i{x['instr']/ti*100:5.1f}% s{x['stall']/ts*100:5.1f}% c{x['conf']/tc*100:5.1f}% act{act:5.1f}  {x['src'][:70]}")
