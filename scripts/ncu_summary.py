"""Summarise an ncu report: key metrics + top source lines by stall samples."""
import csv
import io
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Compute (SM) Throughput',
        'Achieved Occupancy', 'Theoretical Occupancy', 'Registers Per Thread', 'Dynamic Shared Memory Per Block',
        'L1/TEX Cache Throughput', 'L2 Cache Throughput', 'Executed Ipc Active', 'Issue Slots Busy',
        'Warp Cycles Per Issued Instruction', 'Executed Instructions', 'Grid Size', 'Block Size']


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(io.StringIO(out))
    hdr = next(r)
    for row in r:
        d = dict(zip(hdr, row))
        if d.get('Metric Name') in WANT:
            print(f"{d['Section Name'][:28]:28s} | {d['Metric Name']} = {d['Metric Value']} {d['Metric Unit']}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, units = (rr[0], rr[1]) if len(rr) > 2 else ([], [])
    for vals in rr[2:]:
        kname = dict(zip(h, vals)).get("Kernel Name", "?").split("(")[0]
        print(f"raw [{kname}]")
        for k, u, v in zip(h, units, vals):
            if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum",
                     "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                     "sm__sass_inst_executed_op_shared_ld.sum", "sm__sass_inst_executed_op_shared_st.sum",
                     "sm__sass_inst_executed_op_global_ld.sum", "gpu__time_duration.sum",
                     "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
                     "smsp__issue_active.avg.pct_of_peak_sustained_active"):
                print(f"raw   {k} = {v} {u}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    if not src:
        return
    rows = list(csv.reader(io.StringIO(src)))
    while rows and "Source" not in rows[0]:
        rows = rows[1:]
    if not rows:
        return
    h = rows[0]
    try:
        ci = h.index("Warp Stall Sampling (All Samples)")
    except ValueError:
        print("source columns:", h[:12])
        return
    si = h.index("Source") if "Source" in h else 1
    cw = h.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in h else None
    ce = h.index("L1 Wavefronts Shared Excessive") if "L1 Wavefronts Shared Excessive" in h else None
    data = []
    for row in rows[1:]:
        try:
            extra = ""
            if cw is not None and row[cw] not in ("", "0"):
                extra = f"  [smem wf {row[cw]} excess {row[ce]}]"
            data.append((float(row[ci] or 0), row[si].strip() + extra))
        except (ValueError, IndexError):
            pass
    tot = sum(x for x, _ in data) or 1
    print("top SASS by stall samples:")
    for v, s in sorted(data, reverse=True)[:top]:
        print(f"{100 * v / tot:5.1f}%  {s}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
