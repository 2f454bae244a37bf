"""Per-opcode totals of one kernel of an ncu report (SASS source page):
stall samples, executed instructions, shared wavefronts (and excess) and
global L1 tag requests.

    python scripts/ncu_ops.py report.ncu-rep k2_pair
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:k"],
                     capture_output=True, text=True).stdout
# the page holds one block per kernel (each starting with a "Kernel Name" line);
# keep the first block whose name contains `kern`
keep, lines = False, []
for line in src.splitlines():
    if line.startswith('"Kernel Name"'):
        if keep:
            break
        keep = kern in line
        continue
    if keep:
        lines.append(line)
rows = list(csv.reader(io.StringIO("\n".join(lines))))
while rows and "Source" not in rows[0]:
    rows = rows[1:]
h = rows[0]
cols = ["Warp Stall Sampling (All Samples)", "Instructions Executed", "L1 Wavefronts Shared",
        "L1 Wavefronts Shared Excessive", "L1 Tag Requests Global"]
ix = {k: h.index(k) for k in cols + ["Source"]}
agg = defaultdict(lambda: [0.0] * len(cols))
seen = set()  # the source page repeats every SASS line (once per view): count each address once
ia = h.index("Address")
for r in rows[1:]:
    if len(r) < len(h) or r[ia] in seen:
        continue
    seen.add(r[ia])
    s = re.sub(r"^@!?U?P\w+\s+", "", r[ix["Source"]].strip())
    op = s.split()[0] if s else "?"
    for j, k in enumerate(cols):
        v = r[ix[k]]
        try:
            agg[op][j] += float(v)
        except ValueError:
            pass
tot = [sum(v[i] for v in agg.values()) or 1 for i in range(len(cols))]
print(f"{'opcode':24s} {'stall%':>7s} {'inst':>12s} {'smem_wf':>12s} {'excess':>11s} {'gl_tags':>11s}")
for op, v in sorted(agg.items(), key=lambda kv: -(kv[1][2] + kv[1][4] + kv[1][0]))[:28]:
    print(f"{op:24s} {100 * v[0] / tot[0]:7.1f} {v[1]:12.0f} {v[2]:12.0f} {v[3]:11.0f} {v[4]:11.0f}")
print("totals: inst", int(tot[1]), "smem wavefronts", int(tot[2]), "excess", int(tot[3]), "global tags", int(tot[4]))
