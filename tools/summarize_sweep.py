"""Markdown table of a tools/sweep_allreduce.py JSONL file (C3)."""
import collections
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
by = collections.defaultdict(dict)
for r in rows:
    key = r["mode"] + ("" if r["mode"] != "nccl" else (" (NVLS off)" if r["nvls"] == "0" else " (default)"))
    by[r["bytes"]][key] = r
cols = ["ours", "nccl (default)", "nccl (NVLS off)", "ours_tap", "ours_tap_direct"]
n = rows[0]["n"]
print(f"n = {n} GPUs, {rows[0]['dtype']}; time = median of reps (max over ranks); busBW = 2(n-1)/n*S/t\n")
print("| size | " + " | ".join(f"{c} ms / busBW GB/s" for c in cols) + " | tap GB/s per GPU |")
print("|---|" + "---|" * (len(cols) + 1))
for b in sorted(by):
    cells = []
    for c in cols:
        r = by[b].get(c)
        cells.append(f"{r['ms']:.3f} / {r['busbw_GBps']:.0f}" if r else "-")
    tap = by[b].get("ours_tap_direct") or by[b].get("ours_tap")
    mib = b >> 20
    print(f"| {mib} MiB | " + " | ".join(cells) + f" | {tap['tap_GBps_per_gpu']:.1f} |" if tap else " | - |")
