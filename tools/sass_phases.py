"""Static SASS instruction count of a kernel per source phase (needs -lineinfo).
    python tools/sass_phases.py file.cubin kernel_substring source.cu"""
import re, sys, collections, subprocess
cub, kname, srcf = sys.argv[1], sys.argv[2], sys.argv[3]
lines = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout.split("\n")
start = [i for i, l in enumerate(lines) if l.startswith("//---") and kname in l][0]
end = next((i for i in range(start + 5, len(lines)) if lines[i].startswith("//---") and ".text." in lines[i]), len(lines))
cur = None; cnt = collections.Counter(); total = 0
for l in lines[start:end]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: cur = (m.group(1).split("/")[-1], int(m.group(2))); continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", l):
        total += 1
        if cur: cnt[cur] += 1
src = open(srcf).read().split("\n")
marks = [(i + 1, l.strip()[8:12]) for i, l in enumerate(src) if "// ---- " in l]
base = srcf.split("/")[-1]
def phase(ln):
    best = "pre"
    for m, l in marks:
        if m <= ln: best = l
    return best
ph = collections.Counter()
for (f, l), c in cnt.items():
    ph[f if f != base else base + ":" + phase(l)] += c
print("total", total, "instructions,", total * 16, "bytes")
for k, c in ph.most_common(): print(f"  {k:32} {c}")
