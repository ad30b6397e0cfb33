"""Summarize an ncu --csv launch list (gpu__time_duration.sum) by kernel name and grid."""
import collections
import csv
import io
import sys


def load(path):
    text = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(text) if ln.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(text[start:]))))


def main(path, top=30):
    rows = load(path)
    agg = collections.defaultdict(list)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        agg[(name, r["Grid Size"])].append(float(r["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    by_name = collections.defaultdict(float)
    for (n, _), v in agg.items():
        by_name[n] += sum(v)
    print(f"launches={sum(len(v) for v in agg.values())} total={tot/1e3:.1f} us")
    for n, v in sorted(by_name.items(), key=lambda kv: -kv[1]):
        print(f"  {v/1e3:10.1f} us {100*v/tot:5.1f}%  {n}")
    print("by (kernel, grid):")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:top]:
        print(f"  {sum(v)/1e3:9.1f} us n={len(v):4d} avg={sum(v)/len(v)/1e3:8.2f} us  {k[0]} grid={k[1]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
