"""Group an ncu source page (one kernel) by source-line ranges: instruction and stall shares.

    python scripts/ncu_regions.py REPORT KERNEL_REGEX name:lo-hi [name:lo-hi ...]
"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
regions = []
for a in sys.argv[3:]:
    name, rng = a.split(":")
    lo, hi = rng.split("-")
    regions.append((name, int(lo), int(hi)))
sel = ["--launch-skip", kern[5:], "--launch-count", "1"] if kern.startswith("skip:") else ["--kernel-name", f"regex:{kern}"]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + sel,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = None, []
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        try:
            data.append((int(r[0]), float(r[hdr.index("Instructions Executed")] or 0),
                         float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)))
        except ValueError:
            pass
ti = sum(d[1] for d in data) or 1
ts = sum(d[2] for d in data) or 1
acc = {}
for ln, i, st in data:
    name = next((n for n, lo, hi in regions if lo <= ln <= hi), "other")
    a = acc.setdefault(name, [0, 0])
    a[0] += i
    a[1] += st
print(f"total warp instructions {ti:.0f}")
for n, (i, st) in sorted(acc.items(), key=lambda x: -x[1][0]):
    print(f"{n:14s} {100*i/ti:5.1f}% inst {100*st/ts:5.1f}% stall")
