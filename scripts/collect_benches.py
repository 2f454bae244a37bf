"""Copy evidence-run bench lines into profiles/<round>_bench_<config>.json, with the
roofline's ncu fields (traffic, LSU / issue fractions) taken from the committed
profiles/ncu_traffic.json -- the capture of the same build, made after the benches ran.

    python scripts/collect_benches.py r01 gpurun_out/ev c4 c5 c3 c2 c1
"""
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
rnd, src, cfgs = sys.argv[1], pathlib.Path(sys.argv[2]), sys.argv[3:]
tj = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
for c in cfgs:
    d = json.loads((src / f"bench_{c}.json").read_text().strip().splitlines()[-1])
    r = d.get("roofline")
    if r:
        k = r["kernel"]
        r["traffic"] = tj.get(c, {}).get(k)
        lsu = tj.get("lsu_issue", {}).get(c, {}).get(k)
        if lsu:
            r["lsu_pipe_frac_ncu"], r["issue_frac_ncu"] = lsu
            r["lsu_floor_ms"] = round(lsu[0] * r["avg_launch_ms"], 4)
            r["frac_at_lsu_floor"] = round(r["achieved"] / lsu[0] / r["peak"], 4)
        else:
            for k in ("lsu_pipe_frac_ncu", "issue_frac_ncu", "lsu_floor_ms", "frac_at_lsu_floor"):
                r.pop(k, None)
    (ROOT / "profiles" / f"{rnd}_bench_{c}.json").write_text(json.dumps(d) + "\n")
    print(c, d["value"], r and (r["kernel"], r["frac"], r["traffic"]))
ref = src / "bench_reference_c4.json"
if ref.exists():
    (ROOT / "profiles" / f"{rnd}_bench_reference_c4.json").write_text(ref.read_text().strip().splitlines()[-1] + "\n")
