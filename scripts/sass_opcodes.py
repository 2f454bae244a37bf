"""Memory/sync opcode counts of the production kernels in libfht_b200.so (static
SASS, cuobjdump): shows which copy engines each kernel uses (UBLKCP = TMA bulk
copy, UTMALDG/UTMASTG = TMA tensor load/store, LDGSTS = cp.async).

    python scripts/sass_opcodes.py [kernel-substring ...]
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

SO = Path(__file__).resolve().parents[1] / "paper_2411_07351_b200" / "libfht_b200.so"
KEEP = ("UBLKCP", "UTMA", "LDGSTS", "SYNCS", "LDS", "STS", "STG", "LDG", "BAR", "SHFL")
sass = subprocess.run(["cuobjdump", "-sass", str(SO)], capture_output=True, text=True).stdout
want = sys.argv[1:] or ["k2_pair_pipeIiLb1ELb0E", "k1_by32_pairIiE", "k_stage_u8", "k2_passIffLi2ELb0E"]
for f in re.split(r"\n\s*Function : ", sass)[1:]:
    name = f.split("\n", 1)[0].strip()
    if not any(w in name for w in want):
        continue
    ops = collections.Counter(re.findall(r"^\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", f, re.M))
    keep = {k: v for k, v in sorted(ops.items()) if any(x in k for x in KEEP)}
    print(name)
    print("  " + ", ".join(f"{k} {v}" for k, v in keep.items()))
