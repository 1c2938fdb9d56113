"""Summaries of ncu output for profiles/: per-kernel share of a launch list, and selected
metrics of --set full captures.

  python tools/summarize_ncu.py launches <launches.csv>
  python tools/summarize_ncu.py full <report.ncu-rep> [...]
"""
import collections
import csv
import io
import subprocess
import sys

FULL = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "pcie__read_bytes.sum", "pcie__write_bytes.sum",
        "nvlrx__bytes.sum", "nvltx__bytes.sum"]


def launches(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        tot[name] += float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
        cnt[name] += 1
    all_us = sum(tot.values())
    print(f"| kernel | launches | total us | share of device time |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {cnt[k]} | {v:.1f} | {v / all_us:.3f} |")
    print(f"\n{len(rows)} launches, {all_us:.1f} us total (cold-cache, serialised: compare shares).")


def full(paths):
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            print(f"### {p.split('/')[-1]}\n")
            print("| metric | value | unit |\n|---|---|---|")
            for m in FULL:
                if m in hdr:
                    i = hdr.index(m)
                    print(f"| {m} | {r[i]} | {units[i]} |")
            print()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2:])
