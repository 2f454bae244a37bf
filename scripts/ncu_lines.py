"""Per-CUDA-line instruction and stall share for one kernel of an ncu report."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
data = []
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        try:
            data.append((float(r[hdr.index("Instructions Executed")] or 0),
                         float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0), r[0], r[1].strip()[:100]))
        except ValueError:
            pass
ti = sum(d[0] for d in data) or 1
ts = sum(d[1] for d in data) or 1
print("total warp instructions", ti)
for d in sorted(data, key=lambda x: -x[0])[:top]:
    print(f"{100*d[0]/ti:5.1f}% inst {100*d[1]/ts:5.1f}% stall  L{d[2]}: {d[3]}")
