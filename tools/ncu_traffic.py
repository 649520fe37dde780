"""Per-kernel mean DRAM traffic per launch (dram__bytes_read.sum +
dram__bytes_write.sum) and mean duration from an ncu --csv launch list:

    python tools/ncu_traffic.py launches.csv [traffic.json]

Only our kernels (the library's names) are kept; units are normalised to bytes
and microseconds.  Writes the traffic map bench.py reads (profiles/traffic.json)."""
import collections
import csv
import json
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}
OURS = ("fz_", "sh_", "sc_", "tf_", "pm_", "tile_scan", "bbm_", "tt_", "bin_", "count_k", "scatter_k", "excl_scan", "scan_", "classify_bytes")


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    rows = rows[next(i for i, r in enumerate(rows) if "Kernel Name" in r):]  # skip the program's own output
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ix["Kernel Name"]]
        short = name.split("(")[0].split("<")[0].split("::")[-1].split()[-1]
        if not short.startswith(OURS):
            continue
        v = float(r[ix["Metric Value"]].replace(",", "")) * UNIT.get(r[ix["Metric Unit"]], 1)
        per.setdefault((r[ix["ID"]], short), {})[r[ix["Metric Name"]]] = v
    agg = collections.OrderedDict()
    for (_, k), m in per.items():
        a = agg.setdefault(k, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        a[2] += m.get("gpu__time_duration.sum", 0)
    tot_t = sum(a[2] for a in agg.values()) or 1
    for k, (c, b, t) in agg.items():
        print(f"{k:16} launches {c:3}  {t / c:9.1f} us  {b / c / 1e6:9.1f} MB/launch  share {t / tot_t * 100:5.1f} %")
    if len(sys.argv) > 2:
        json.dump({k: b / c for k, (c, b, t) in agg.items()}, open(sys.argv[2], "w"), indent=1)


if __name__ == "__main__":
    main()
