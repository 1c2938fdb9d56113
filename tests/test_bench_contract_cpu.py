"""The bench JSON line contract, checked on lines bench.py printed on B200 (committed under
profiles/r02/): the base keys, `roofline` (the dominant kernel: bound, achieved, peak, frac,
traffic), `cpu_baseline`, `e2e` with its copy bytes, `clocks`, `gpu_launches`, and the
reference arm's line.  A field renamed or dropped in bench.py shows up here when the next
GPU line is committed; the checker itself runs on the CPU."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R02 = os.path.join(ROOT, "profiles", "r02")

BASE = {"metric": str, "value": float, "unit": str, "n_gpus": int, "steps": int, "warmup": int,
        "ms_per_step": float, "higher_is_better": bool, "scaling": str, "dtype": str, "data": str,
        "config": dict}


def _line(name):
    with open(os.path.join(R02, name)) as f:
        return json.loads([ln for ln in f if ln.startswith("{")][-1])


def _check_base(d):
    for k, t in BASE.items():
        assert k in d, k
        assert isinstance(d[k], (int, float) if t is float else t), (k, d[k])
    assert "vs_baseline" in d and d["vs_baseline"] is None       # no paper number for this metric
    assert d["scaling"] == "weak" and d["higher_is_better"] is True
    assert "workload" in d["config"]
    assert d["warmup"] >= 3
    assert d["value"] > 0 and d["ms_per_step"] > 0


@pytest.mark.parametrize("name,n", [("r02bg_bench_n1_model200.json", 1), ("r02bg_bench_n2_model200.json", 2),
                                    ("r02bh_bench_n4_model200.json", 4)])
def test_bench_line(name, n):
    d = _line(name)
    _check_base(d)
    assert d["n_gpus"] == n
    # value = whole-job rank-iterations per second = n * 1000 / ms_per_step (max over ranks)
    assert abs(d["value"] - n * 1000.0 / d["ms_per_step"]) / d["value"] < 1e-6
    r = d["roofline"]
    for k in ("kernel", "bound", "achieved", "peak", "unit", "frac", "bytes_per_launch", "avg_ms"):
        assert k in r, k
    assert r["bound"] in ("hbm", "nvlink") and r["unit"] == "GB/s"
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert abs(r["achieved"] - r["bytes_per_launch"] / (r["avg_ms"] * 1e-3) / 1e9) / r["achieved"] < 1e-9
    assert 0 < r["frac"] <= 1.05
    if n == 1:
        assert r["kernel"] == "adamw_step" and r["traffic"] is not None
        assert 0.9 < r["traffic"] / r["bytes_per_launch"] <= 1.05     # ncu DRAM bytes vs algorithmic
    else:
        assert r["kernel"] == "rs_tap_ag" and 0.5 < r["lockstep_frac"] <= 1.0
    s = d["step_roofline"]
    assert s["bound"] == "host_link" and 0 < s["frac"] <= 1.05
    e = d["e2e"]
    assert e["unit"] == d["unit"] and e["value"] > 0
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0     # copies inside the timed region
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and c["sm_max_mhz"] > 0
    assert not set(c["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert isinstance(d["gpu_launches"], int) and d["gpu_launches"] > 0
    if n == 1:
        cb = d["cpu_baseline"]
        for k in ("value", "unit", "cores", "kind", "sample"):
            assert k in cb, k
        assert cb["kind"] == "oracle" and cb["cores"] >= 1
    else:
        assert d["cpu_baseline"] is None                      # rank 0 at N=1 only
    assert d["checkpoint_verified"] == {"shadow": True, "host_log": True, "ring": True}
    m = d["model_mode"]
    assert m["timed_iterations"] == 200 and m["ours_ckpt"]["shadow_bit_identical"] is True


def test_reference_arm_line():
    d = _line("r02ba_reference_arm_n1_final.json")
    _check_base(d)
    assert d["impl"] == "reference"
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == d["value"] and cb["cores"] >= 1 and cb["sample"]
    assert d["steps"] == 20 and d["warmup"] == 5                  # the steps it actually ran
