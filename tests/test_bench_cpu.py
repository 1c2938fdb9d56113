"""Host logic of bench.py that needs no GPU: the clock sampler reports only rows read
inside the timed region, and a short region still gets samples because nvidia-smi is
started (and its first row awaited) before the region opens."""
import os
import stat
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _fake_smi(tmp_path, reason="Not Active", startup_s=0.4):
    p = tmp_path / "nvidia-smi"
    p.write_text("#!/bin/bash\n"
                 f"sleep {startup_s}\n"
                 f"while true; do echo \"0, 1965, 1965, {reason}, Not Active, Not Active, Not Active\"; sleep 0.05; done\n")
    p.chmod(p.stat().st_mode | stat.S_IEXEC)
    return str(tmp_path)


def test_short_region_is_sampled(tmp_path, monkeypatch):
    monkeypatch.setenv("PATH", _fake_smi(tmp_path) + os.pathsep + os.environ["PATH"])
    with bench.ClockSampler(0) as c:
        time.sleep(0.2)
    s = c.summary()
    assert s["samples"] >= 2 and s["sm_mhz"] == 1965.0 and s["reasons"] == []


def test_throttle_reason_reported(tmp_path, monkeypatch):
    monkeypatch.setenv("PATH", _fake_smi(tmp_path, reason="Active") + os.pathsep + os.environ["PATH"])
    with bench.ClockSampler(0) as c:
        time.sleep(0.15)
    assert c.summary()["reasons"] == ["hw_slowdown"]


def test_missing_nvidia_smi_is_unsampled(tmp_path, monkeypatch):
    monkeypatch.setenv("PATH", str(tmp_path))
    with bench.ClockSampler(0) as c:
        time.sleep(0.01)
    assert c.summary()["reasons"] == ["unsampled"]


def test_reference_arm_prints_one_contract_line():
    """`bench.py --impl reference` (the CPU oracle arm) prints exactly one JSON line with the
    base contract's keys, the oracle's cpu_baseline and a host-only e2e."""
    import json
    import subprocess
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--cpu-sample-s", "0.2"], capture_output=True, text=True, timeout=300,
                       cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["steps"] == 1 and d["warmup"] == 0            # the steps it actually ran
    cb = d["cpu_baseline"]
    assert cb["steps"] == 1 and cb["cores"] >= 1 and cb["kind"] == "oracle"


def test_oracle_all_core_build_gives_the_same_bits():
    """bench.py times the oracle on every host core with the -fopenmp build of the same
    source: the sampled trajectories must be bit-identical to the single-threaded build."""
    import numpy as np
    from oracle import oracle as O
    rng = np.random.default_rng(5)
    idx = np.sort(rng.choice(1 << 24, 200_000, replace=False)).astype(np.int64)
    used = (rng.random(len(idx)) < 0.95).astype(np.uint8)
    for dtype in (O.F32, O.BF16):
        a = O.run_sample(3, 4, dtype, 10, 5, idx, used, t0=2)
        b = O.run_sample(3, 4, dtype, 10, 5, idx, used, t0=2, omp=True)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x.view(np.uint32), y.view(np.uint32))
    assert O.threads(True) >= 1 and O.threads(False) == 1
