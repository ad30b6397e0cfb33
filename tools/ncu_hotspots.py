"""Top stalled SASS instructions of one kernel in an ncu report (needs -lineinfo / --import-source)."""
import csv
import io
import subprocess
import sys


def main(rep, regex, skip=0, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{regex}", "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    data = [r for r in rows if len(r) == len(hdr) and r[0] not in ("Address",)]
    si = hdr.index("Warp Stall Sampling (All Samples)")

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    seen = set()
    uniq = []
    for r in data:
        if r[0] in seen:
            continue
        seen.add(r[0])
        uniq.append(r)
    tot = sum(f(r[si]) for r in uniq)
    print(f"samples={tot:.0f} instructions={len(uniq)}")
    order = sorted(range(len(uniq)), key=lambda i: -f(uniq[i][si]))[:top]
    for i in sorted(order):
        r = uniq[i]
        print(f"{f(r[si]):6.0f} {100*f(r[si])/max(tot,1):5.1f}%  [{i:4d}] {r[1][:110]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0)
