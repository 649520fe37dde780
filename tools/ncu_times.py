"""Parse an ncu --csv metrics log: per-kernel launch times and DRAM bytes."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
acc = collections.OrderedDict()
for r in rows[1:]:
    key = (r[ix["ID"]], r[ix["Kernel Name"]])
    acc.setdefault(key, {})[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
for (i, k), m in acc.items():
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    rd = m.get("dram__bytes_read.sum", 0) / 1e6
    wr = m.get("dram__bytes_write.sum", 0) / 1e6
    print(f"{i:>4} {k[:40]:40} {t:9.1f} us  read {rd:9.1f} MB  write {wr:9.1f} MB  {(rd+wr)/max(t,1e-9)*1e-3:7.1f} GB/s")
