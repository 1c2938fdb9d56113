"""Summary of ncu NVLink counters (tools/ncu_nvlink_probe.sh; one process, 2 GPUs, barriers off) per
kernel launch of the last iteration: user bytes received / transmitted over NVLink against
the algorithmic per-rank bytes of the launch ((n-1)/n of the bucket each way for the two-shot
all-reduce: the pulls in, the all-gather pushes out; ZeRO-1: the pulls only, and the AdamW
kernel's parameter pushes 4 (n-1) B per shard element out), protocol overhead, and rates.

  python tools/summarize_nvlink_ncu.py <ncu.csv> [n]
"""
import collections
import csv
import sys

MULT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
        "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}


def main(path, n=2):
    lines = [l for l in open(path) if not l.startswith("==")]
    L = collections.OrderedDict()
    for r in csv.DictReader(lines):
        key = (int(r["ID"]), r["Kernel Name"].split("(")[0].replace("void ", ""), r["Device"])
        L.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * MULT[r["Metric Unit"]]
    items = list(L.items())
    last = items[len(items) // 2:]
    print("| launch | kernel | GPU | µs | NVLink rx user MB | tx user MB | rx / tx raw MB | user rx GB/s | user tx GB/s | DRAM MB |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    tot = collections.Counter()
    for (i, name, dev), m in last:
        t = m["gpu__time_duration.sum"]
        rxu, txu = m["nvlrx__bytes_data_user.sum"], m["nvltx__bytes_data_user.sum"]
        rx, tx = m["nvlrx__bytes.sum"], m["nvltx__bytes.sum"]
        dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        k = name.split("<")[0]
        tot[(k, "t")] += t
        tot[(k, "rxu")] += rxu
        tot[(k, "txu")] += txu
        tot[(k, "rx")] += rx
        tot[(k, "tx")] += tx
        print(f"| {i} | `{name}` | {dev} | {t * 1e6:.1f} | {rxu / 1e6:.2f} | {txu / 1e6:.2f} | {rx / 1e6:.2f} / {tx / 1e6:.2f} | "
              f"{rxu / t / 1e9:.0f} | {txu / t / 1e9:.0f} | {dram / 1e6:.1f} |")
    print()
    for k in sorted({k for k, _ in tot}):
        t = tot[(k, "t")]
        ratio = lambda a, b: f"{a / b:.3f}" if b > 0 else "n/a (no user bytes)"   # noqa: E731
        print(f"- `{k}`: user rx {tot[(k, 'rxu')] / 1e6:.1f} MB, tx {tot[(k, 'txu')] / 1e6:.1f} MB in {t * 1e6:.1f} µs "
              f"summed over its launches (both GPUs); raw/user rx {ratio(tot[(k, 'rx')], tot[(k, 'rxu')])}, "
              f"tx {ratio(tot[(k, 'tx')], tot[(k, 'txu')])}; user rate rx {tot[(k, 'rxu')] / t / 1e9:.0f} GB/s, "
              f"tx {tot[(k, 'txu')] / t / 1e9:.0f} GB/s")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 2)
