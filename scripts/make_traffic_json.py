"""profiles/ncu_traffic.json from the committed ncu summaries (scripts/ncu_summary.py
output, profiles/<round>_ncu_<config>.txt): per kernel of one launch, DRAM bytes
(read + write) and the LSU data-pipe / issue-slot fractions of peak.

    python scripts/make_traffic_json.py r01 c4 c5
"""
import json
import pathlib
import re
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]


def parse(path: pathlib.Path):
    traffic, frac = {}, {}
    cur, k2 = None, 0
    for line in path.read_text().splitlines():
        m = re.match(r"raw \[.*::(k\w+)", line)
        if m:
            cur = m.group(1)
            if cur in ("k1_by32", "k1_by32_pair"):  # k1_by32_pair: the u16 pair-mode K1P
                cur = "k1p_by32"
            if cur == "k2_pair_pipe":  # the pair-mode root band (double-buffered windows)
                cur = "k2_pass_root"
            if cur == "k2_pass":
                k2 += 1
                cur = "k2_pass" if k2 == 1 else "k2_pass_root"
            traffic[cur] = 0
            frac[cur] = [None, None]
            continue
        if cur is None:
            continue
        m = re.match(r"raw\s+dram__bytes_(read|write)\.sum = ([\d.]+) (Gbyte|Mbyte|Kbyte)", line)
        if m:
            traffic[cur] += round(float(m.group(2)) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3}[m.group(3)])
        m = re.match(r"raw\s+l1tex__data_pipe_lsu_wavefronts\.avg\.pct_of_peak_sustained_elapsed = ([\d.]+)", line)
        if m:
            frac[cur][0] = round(float(m.group(1)) / 100, 3)
        m = re.match(r"raw\s+smsp__issue_active\.avg\.pct_of_peak_sustained_active = ([\d.]+)", line)
        if m:
            frac[cur][1] = round(float(m.group(1)) / 100, 3)
    return traffic, frac


def main(rnd, configs):
    out = {"_note": "per launch of each kernel, from one ncu --set full capture (profiles/%s_ncu_<config>.txt): "
                    "dram__bytes_read.sum + dram__bytes_write.sum; lsu_issue = [LSU data-pipe wavefronts, "
                    "issue slots] as fractions of peak" % rnd, "lsu_issue": {}}
    for cfg in configs:
        tr, fr = parse(ROOT / "profiles" / f"{rnd}_ncu_{cfg}.txt")
        if "k2_pass" in tr and "k2_pass_root" not in tr:  # a single band is the root band
            tr["k2_pass_root"] = tr.pop("k2_pass")
            fr["k2_pass_root"] = fr.pop("k2_pass")
        out[cfg] = tr
        out["lsu_issue"][cfg] = {k: v for k, v in fr.items() if None not in v}
    (ROOT / "profiles" / "ncu_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:] or ["c4", "c5"])
