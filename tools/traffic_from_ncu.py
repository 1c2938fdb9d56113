"""profiles/traffic.json from an ncu per-launch CSV (tools/ncu_final.sh step 2): the measured
DRAM bytes (read + write) per launch next to the algorithmic bytes of the SAME launches, for
the kernels bench.py reports: the all-reduce (average over one iteration's 17 buckets; n=1,
staged tap: a copy of the bucket into the HBM staging half, 2 S_b), the training AdamW
(28 B/elem) and the shadow AdamW (28 B/elem of the shard).

  python tools/traffic_from_ncu.py gpurun_out/<tag>_dram.csv profiles/traffic.json
Launch order per iteration (virtual rank n=1): gen_grads, 17 x rs_tap_ag, training adamw_wt,
shadow adamw_wt (one launch: no persist in iterations 1, 2 with K=8)."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(path, out):
    from paper_2507_13522_b200 import workloads as W
    numel = W.numels(W.gpt2_small())
    P = sum(numel)                                   # no padding for GPT-2 at n=1
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.DictReader(lines))
    launches = {}
    for r in rows:
        key = (int(r["ID"]), r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if unit in ("Kbyte", "KB"):
            v *= 1e3
        elif unit in ("Mbyte", "MB"):
            v *= 1e6
        elif unit in ("Gbyte", "GB"):
            v *= 1e9
        elif unit == "usecond":
            v *= 1e3
        elif unit == "msecond":
            v *= 1e6
        launches.setdefault(key, {})[r["Metric Name"]] = v
    seq = [(k[1].split("(")[0].replace("void ", ""), m) for k, m in sorted(launches.items())]
    # the last complete iteration: gen, 17 AR, train adamw, shadow adamw
    it = []
    for i in range(len(seq) - 1, -1, -1):
        if "gen_grads" in seq[i][0]:
            it = seq[i:i + 20]
            break
    ar = [m for nm, m in it if "rs_tap_ag" in nm]
    ad = [m for nm, m in it if "adamw_wt" in nm]
    assert len(ar) == 17 and len(ad) == 2, (len(ar), len(ad))
    dram = lambda m: m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]   # noqa: E731
    S = P * 4
    table = json.load(open(out)) if os.path.exists(out) else {}
    table["gpt2_n1_host"] = {
        "rs_tap_ag": {"dram_bytes_per_launch": sum(dram(m) for m in ar) / 17,
                      "algorithmic": 2 * S / 17,
                      "what": "average over one iteration's 17 launches (staged tap at n=1: bucket -> HBM staging)",
                      "source": os.path.basename(path)},
        "adamw_step": {"dram_bytes_per_launch": dram(ad[0]), "algorithmic": 28 * P,
                       "source": os.path.basename(path)},
        "shadow_adamw": {"dram_bytes_per_launch": dram(ad[1]), "algorithmic": 28 * P,
                         "source": os.path.basename(path)},
    }
    json.dump(table, open(out, "w"), indent=1)
    print(json.dumps(table["gpt2_n1_host"], indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
