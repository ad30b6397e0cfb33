"""Per-kernel summary of an ncu --csv launch list with several metrics (duration, DRAM bytes,
tcgen05 pipe utilisation): writes a markdown table and a compact CSV (one row per launch).

  python tools/launch_metrics.py gpurun_out/r02/launches_llama2-7b.csv profiles/r02_launches_llama2-7b
"""
import collections
import csv
import io
import sys

TIME = "gpu__time_duration.sum"
RD, WR = "dram__bytes_read.sum", "dram__bytes_write.sum"
TC = "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed"


def load(path):
    text = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(text) if ln.startswith('"ID"'))
    launches = collections.OrderedDict()
    for r in csv.DictReader(io.StringIO("\n".join(text[start:]))):
        key = int(r["ID"])
        d = launches.setdefault(key, {"kernel": r["Kernel Name"].split("(")[0].replace("void ", ""),
                                      "grid": r["Grid Size"]})
        v = r["Metric Value"].replace(",", "")
        unit = r.get("Metric Unit", "")
        x = float(v) if v not in ("", "n/a") else float("nan")
        scale = {"nsecond": 1e-3, "ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0, "msecond": 1e3, "byte": 1.0, "Kbyte": 1e3,
                 "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        d[r["Metric Name"]] = x * scale
    return list(launches.values())


def main(src, dst):
    rows = load(src)
    with open(dst + ".csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["launch", "kernel", "grid", "us", "dram_MB", "tc_pct"])
        for i, r in enumerate(rows):
            w.writerow([i, r["kernel"], r["grid"], f"{r.get(TIME, 0):.2f}",
                        f"{(r.get(RD, 0) + r.get(WR, 0)) / 1e6:.2f}",
                        f"{r.get(TC, float('nan')):.1f}"])
    agg = collections.defaultdict(list)
    for r in rows:
        agg[(r["kernel"], r["grid"])].append(r)
    total = sum(r.get(TIME, 0) for r in rows)
    out = [f"# {src.split('/')[-1]}: {len(rows)} launches, {total / 1e3:.2f} ms serialized "
           "(ncu, cold cache, --clock-control none)", "",
           "| kernel | grid | n | total us | share | avg us | avg DRAM MB | avg GB/s | avg tc-pipe % |",
           "|---|---|---|---|---|---|---|---|---|"]
    for (k, g), rs in sorted(agg.items(), key=lambda kv: -sum(r.get(TIME, 0) for r in kv[1])):
        t = sum(r.get(TIME, 0) for r in rs)
        mb = sum(r.get(RD, 0) + r.get(WR, 0) for r in rs) / len(rs) / 1e6
        tc = [r[TC] for r in rs if TC in r and r[TC] == r[TC]]
        out.append(f"| `{k}` | {g} | {len(rs)} | {t:.1f} | {100 * t / total:.1f}% | {t / len(rs):.2f} "
                   f"| {mb:.2f} | {mb * len(rs) / t * 1e3:.0f} | "
                   f"{(sum(tc) / len(tc)) if tc else float('nan'):.1f} |")
    open(dst + ".md", "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
