"""Per-instruction view of an ncu report (source page, SASS): top stall
lines, shared-memory excess wavefronts and global L1 requests.

    python tools/ncu_sass.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys


def load(path, kern):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kern}", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    recs = []
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        d = dict(zip(h, r))
        for k in h[2:]:
            try:
                d[k] = float(d[k])
            except ValueError:
                pass
        recs.append(d)
    return h, recs


def main(path, kern, top=30):
    h, recs = load(path, kern)
    tot = sum(r["Warp Stall Sampling (All Samples)"] for r in recs)
    stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    print(f"{len(recs)} instructions, {tot:.0f} samples")
    agg = {k: sum(r[k] for r in recs if isinstance(r[k], float)) for k in stalls}
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
        print(f"  {k:24s} {100 * v / tot:5.1f}%")
    for key in ("L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal", "L1 Wavefronts Shared Excessive",
                "L1 Tag Requests Global", "L2 Theoretical Sectors Global",
                "L2 Theoretical Sectors Global Excessive", "Instructions Executed"):
        print(f"  total {key:40s} {sum(r[key] for r in recs if isinstance(r[key], float)):.4g}")
    # opcode mix
    ops = {}
    for r in recs:
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + r["Instructions Executed"]
    ie = sum(ops.values())
    print("  opcode mix (warp instructions):",
          ", ".join(f"{k} {100 * v / ie:.1f}%" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:12]))
    print(f"\ntop {top} by stall samples:")
    for r in sorted(recs, key=lambda r: -r["Warp Stall Sampling (All Samples)"])[:top]:
        s = r["Warp Stall Sampling (All Samples)"]
        st = sorted(((r[k], k[6:]) for k in stalls if isinstance(r[k], float) and r[k] > 0), reverse=True)[:3]
        print(f"  {100 * s / tot:5.2f}% {r['Source'].strip()[:60]:60s} "
              + " ".join(f"{n}:{100 * v / tot:.1f}" for v, n in st))
    print(f"\ntop 15 by excess shared wavefronts:")
    for r in sorted(recs, key=lambda r: -(r["L1 Wavefronts Shared Excessive"] or 0))[:15]:
        if not r["L1 Wavefronts Shared Excessive"]:
            break
        print(f"  {r['L1 Wavefronts Shared Excessive']:.3g} of {r['L1 Wavefronts Shared']:.3g} "
              f"{r['Source'].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
