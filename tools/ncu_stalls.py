"""Per-reason warp-stall totals from an ncu report's source page.

    python tools/ncu_stalls.py gpurun_out/prof.ncu-rep [top_lines]
"""
import collections
import csv
import io
import subprocess
import sys


def main(path, top=12):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[1]
    cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    iS = h.index("Source")
    tot = collections.Counter()
    lines = []
    for r in rows[2:]:
        if len(r) <= max(cols):
            continue
        per = {h[i]: int(r[i] or 0) for i in cols}
        for k, v in per.items():
            tot[k] += v
        lines.append((sum(per.values()), r[iS].strip(), max(per, key=per.get)))
    s = sum(tot.values()) or 1
    for k, v in tot.most_common(10):
        print(f"{k:26s} {100 * v / s:5.1f}%")
    print("top lines:")
    for n, src, why in sorted(lines, reverse=True)[:int(top)]:
        print(f"{100 * n / s:5.1f}% {why:18s} {src}")


if __name__ == "__main__":
    main(*sys.argv[1:])
