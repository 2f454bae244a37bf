"""Print the c4 plan (describe JSON) -- slot counts and row capacities of the root band."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2411_07351_b200 import fht  # noqa: E402

plan = fht.Plan(509, 509, "tweaked", in_dtype="u8", acc_dtype="i32", batch=256)
d = plan.describe()
g = d["groups"][0]
print(json.dumps({k: v for k, v in g.items() if k != "plan"}, indent=None))
print(json.dumps(g["plan"])[:3000])
