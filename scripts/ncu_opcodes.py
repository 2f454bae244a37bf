"""Aggregate an ncu source page (SASS) by opcode: stall samples, instructions, smem wavefronts."""
import csv, io, re, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
while rows and "Source" not in rows[0]:
    rows = rows[1:]
h = rows[0]
ix = {k: h.index(k) for k in ["Source", "Warp Stall Sampling (All Samples)", "Instructions Executed", "L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive"]}
agg = defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
for r in rows[1:]:
    try:
        s = r[ix["Source"]].strip()
        s = re.sub(r"^@!?U?P\w+\s+", "", s)
        op = s.split()[0] if s else "?"
        a = agg[op]
        for k, j in zip(["Warp Stall Sampling (All Samples)", "Instructions Executed", "L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive"], range(4)):
            v = r[ix[k]]
            a[j] += float(v) if v not in ("", "-") else 0.0
    except (IndexError, ValueError):
        pass
tot = [sum(v[i] for v in agg.values()) or 1 for i in range(4)]
print(f"{'opcode':22s} {'stall%':>7s} {'inst%':>7s} {'smemwf':>12s} {'excess':>12s}")
for op, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:22]:
    print(f"{op:22s} {100*v[0]/tot[0]:7.1f} {100*v[1]/tot[1]:7.1f} {v[2]:12.0f} {v[3]:12.0f}")
print("total instructions", tot[1], "smem wavefronts", tot[2], "excess", tot[3])
