"""Summarise an ncu --csv launch list: per kernel mean time, DRAM bytes, GB/s."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = defaultdict(lambda: defaultdict(list))
for d in data:
    agg[d["Kernel Name"][:70]][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
tot = 0.0
for k, v in agg.items():
    t = v["gpu__time_duration.sum"]
    rd, wr = v.get("dram__bytes_read.sum", [0]), v.get("dram__bytes_write.sum", [0])
    n = len(t)
    tot += sum(t)
    print(f"{k:70s} n={n:3d} t_us={sum(t)/n/1e3:8.1f} rdMB={sum(rd)/n/1e6:7.1f} wrMB={sum(wr)/n/1e6:7.1f} "
          f"GB/s={(sum(rd)+sum(wr))/max(sum(t),1):6.0f}")
