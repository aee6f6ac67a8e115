"""Stall samples and warp instructions per CUDA source line of one kernel in
an ncu report (source page, cuda+sass view).

    python tools/ncu_lines.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys


def main(path, kern, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kern}", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, agg, hdr = None, {}, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "" or len(r) < 6:
            continue
        try:
            samples = float(r[4])
            inst = float(r[7])
        except ValueError:
            continue
        key = (fname, int(r[0]), r[1].strip()[:70])
        a = agg.setdefault(key, [0.0, 0.0])
        a[0] += samples
        a[1] += inst
    tot = sum(v[0] for v in agg.values()) or 1.0
    toti = sum(v[1] for v in agg.values()) or 1.0
    print(f"{tot:.0f} samples, {toti:.3g} warp instructions")
    for (f, ln, src), (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * s / tot:5.1f}% samp {100 * i / toti:5.1f}% inst  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
