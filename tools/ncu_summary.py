"""Key per-kernel metrics from an ncu report (details page)."""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Grid Size", "Block Size", "L2 Hit Rate",
        "Compute (SM) Throughput", "Waves Per SM", "Dynamic Shared Memory Per Block",
        "No Eligible", "Eligible Warps Per Scheduler", "Issued Warp Per Scheduler"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value",
                                                 "Metric Unit", "ID"))
    cur = None
    for r in rows[1:]:
        if r[mi] not in WANT:
            continue
        if r[ii] != cur:
            cur = r[ii]
            print(f"--- [{cur}] {r[ki][:90]}")
        print(f"    {r[mi]:34s} {r[vi]:>12s} {r[ui]}")


if __name__ == "__main__":
    main(sys.argv[1])
