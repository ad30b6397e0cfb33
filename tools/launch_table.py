"""Per-kernel totals of an ncu launch list with DRAM bytes (gpu_quick.sh output)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize_launches import load  # noqa: E402

rows = load(sys.argv[1])
per = collections.defaultdict(dict)
names = {}
grids = {}
for r in rows:
    try:
        per[int(r["ID"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    except ValueError:
        continue
    names[int(r["ID"])] = r["Kernel Name"].split("(")[0].replace("void ", "")
    grids[int(r["ID"])] = r["Grid Size"]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
tot = 0.0
for i in sorted(per):
    m = per[i]
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    b = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6
    key = names[i] + ("  grid=" + grids[i] if len(sys.argv) > 2 else "")
    a = agg[key]
    a[0] += 1
    a[1] += t
    a[2] += b
    tot += t
print(f"total {tot:.1f} us over {sum(a[0] for a in agg.values())} launches")
for n, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:60s} n={c:4d} {t:9.1f}us avg {t / c:7.2f}us {b / c:7.1f}MB/launch {b / t:5.2f} TB/s")
