"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    data[d["Kernel Name"]][d["Metric Name"]].append((float(d["Metric Value"].replace(",", "")), d["Metric Unit"]))
print("| kernel | launches | mean time | DRAM read | DRAM write |\n|---|---|---|---|---|")
for k, m in data.items():
    f = lambda xs: f"{sum(x for x, _ in xs) / len(xs):.1f} {xs[0][1]}" if xs else "-"  # noqa: E731
    print(f"| {k[:90]} | {len(m.get('gpu__time_duration.sum', []))} | {f(m.get('gpu__time_duration.sum', []))} | "
          f"{f(m.get('dram__bytes_read.sum', []))} | {f(m.get('dram__bytes_write.sum', []))} |")
