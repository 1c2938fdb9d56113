"""Print a sweep JSONL (tools/sweep_allreduce.py) as a table of microseconds per launch."""
import json
import sys
from collections import defaultdict

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
t = defaultdict(dict)
for r in rows:
    m = r["mode"].replace("_nvls", "")
    arm = m + ("" if m == "nccl" else ("_os" if r.get("oneshot_max", 0) > 0 else "_2s")) + \
        ("_nvls" if r["mode"].endswith("_nvls") else "")
    t[(r["dtype"], r["bytes"])][arm] = r["ms"] * 1000
arms = sorted({a for v in t.values() for a in v})
print("| dtype | bytes | " + " | ".join(f"{a} us" for a in arms) + " |")
print("|---|---|" + "---|" * len(arms))
for k in sorted(t):
    print(f"| {k[0]} | {k[1]} | " + " | ".join("%.1f" % t[k][a] if a in t[k] else "-" for a in arms) + " |")
