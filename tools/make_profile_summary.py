"""Summarise a round's ncu captures into profiles/ (committed evidence).

usage: python tools/make_profile_summary.py r01 llama2-7b
"""
import collections
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize_launches import load  # noqa: E402

TAG, CFG = sys.argv[1], sys.argv[2]
SRC = f"gpurun_out/{TAG}"
DST = "profiles"
os.makedirs(DST, exist_ok=True)

# per-launch metrics of one full step (cold-cache, serialised by ncu)
rows = load(f"{SRC}/metrics_{CFG}.csv")
per = collections.defaultdict(dict)
names = {}
for r in rows:
    try:
        per[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    except ValueError:
        continue
    names[r["ID"]] = r["Kernel Name"].split("(")[0].replace("void ", "")
ids = sorted(per, key=int)
agg = collections.defaultdict(lambda: collections.defaultdict(float))
for i in ids:
    m = per[i]
    k = names[i]
    a = agg[k]
    a["n"] += 1
    a["us"] += m.get("gpu__time_duration.sum", 0) / 1e3
    a["dram"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    a["tensor_pct_x_us"] += m.get("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 0) * m.get("gpu__time_duration.sum", 0) / 1e3
    a["dram_pct_x_us"] += m.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 0) * m.get("gpu__time_duration.sum", 0) / 1e3
tot_us = sum(a["us"] for a in agg.values())
lines = [f"# {TAG}: ncu per-launch metrics of one {CFG} step ({len(ids)} launches, cold cache, serialised)",
         "", f"total kernel time {tot_us/1e3:.2f} ms", "",
         "| kernel | launches | time (ms) | share | DRAM bytes/launch (MB) | DRAM throughput (time-weighted % of peak) |",
         "|---|---|---|---|---|---|"]
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
    lines.append(f"| {k} | {int(a['n'])} | {a['us']/1e3:.2f} | {100*a['us']/tot_us:.1f}% | "
                 f"{a['dram']/a['n']/1e6:.1f} | {a['dram_pct_x_us']/a['us']:.1f} |")
gemm_keys = [k for k in agg if k.startswith("collm::gemm_lora_kernel") or k.startswith("gemm_lora_kernel")]
g_launch = sum(agg[k]["n"] for k in gemm_keys)
g_dram = sum(agg[k]["dram"] for k in gemm_keys)
traffic = g_dram / max(g_launch, 1)
lines += ["", f"GEMM average DRAM traffic per launch: {traffic/1e6:.1f} MB over {int(g_launch)} launches "
          "(bench.py reports it as roofline.traffic)"]
open(f"{DST}/{TAG}_{CFG}_step_metrics.md", "w").write("\n".join(lines) + "\n")
tf = f"{DST}/gemm_traffic.json"
d = json.load(open(tf)) if os.path.exists(tf) else {}
d[CFG] = traffic
json.dump(d, open(tf, "w"), indent=1)

# launch list (gpu__time_duration only) -> copy + summary
import shutil  # noqa: E402
shutil.copy(f"{SRC}/launches_{CFG}.csv", f"{DST}/{TAG}_launches_{CFG}.csv")
summ = subprocess.run([sys.executable, "tools/summarize_launches.py", f"{SRC}/launches_{CFG}.csv", "20"],
                      capture_output=True, text=True).stdout
open(f"{DST}/{TAG}_launches_{CFG}_summary.txt", "w").write(summ)

# full captures -> details + hotspot text
for f in sorted(os.listdir(SRC)):
    if f.startswith("full_") and f.endswith(".ncu-rep"):
        base = f[:-8]
        det = subprocess.run([sys.executable, "tools/ncu_summary.py", f"{SRC}/{f}"], capture_output=True, text=True).stdout
        raw = subprocess.run(["ncu", "-i", f"{SRC}/{f}", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        import csv, io  # noqa: E401,E402
        rr = list(csv.reader(io.StringIO(raw)))
        keep = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
                "sm__warps_active.avg.pct_of_peak_sustained_active",
                "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed",
                "lts__throughput.avg.pct_of_peak_sustained_elapsed",
                "lts__t_sectors_srcunit_tex.sum", "lts__t_sector_hit_rate.pct",
                "sm__cycles_elapsed.avg.per_second"]
        extra = []
        if len(rr) > 2:
            hdr, units, vals = rr[0], rr[1], rr[2]
            for k in keep:
                if k in hdr:
                    i = hdr.index(k)
                    extra.append(f"    {k:75s} {vals[i]} {units[i]}")
        hot = subprocess.run([sys.executable, "tools/ncu_hotspots.py", f"{SRC}/{f}",
                              "gemm|lora|expand"], capture_output=True, text=True).stdout
        open(f"{DST}/{TAG}_{base}.txt", "w").write(
            det + "\n  raw:\n" + "\n".join(extra) + "\n\n  SASS stall hotspots:\n" + hot)
print(open(f"{DST}/{TAG}_{CFG}_step_metrics.md").read())
