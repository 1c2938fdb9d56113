"""Multi-process GPU tests: one process per GPU over real NVLink peer memory (CUDA IPC),
cross-GPU flag barriers inside the kernels.  Need >= 2 GPUs (skipped otherwise)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def launch(n, mode, name, timeout=300):
    port = 29500 + (os.getpid() % 2000)
    cmd = [sys.executable, "-m", "torch.distributed.run", f"--nproc-per-node={n}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.join(ROOT, "tests", "mp_worker.py"), mode, name]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    return p


def counts():
    return [n for n in (2, 4, 8) if n <= NGPU]


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("mode", ["parity_f32", "parity_bf16", "parity_zero1", "parity_sgd",
                                  "parity_oneshot", "parity_oneshot_bf16", "parity_oneshot_direct",
                                  "parity_nvls", "parity_nvls_bf16", "parity_zero1_oneshot",
                                  "parity_bucket_step", "parity_bucket_step_zero1", "nonfinite",
                                  "restore_soft", "model_parity", "kd_rule"])
def test_multiprocess(mode):
    for n in counts():
        name = f"cmmp{os.getpid()}_{mode}_{n}"
        p = launch(n, mode, name)
        assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
        assert p.stdout.count(f"{mode} ok") == n


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_hard_kill_restore():
    """SIGKILL-equivalent: every rank exits without cleanup after iteration 5; a fresh set of
    processes attaches to the surviving shadow segments, restores and continues bit-exact."""
    n = counts()[0]
    name = f"cmhk{os.getpid()}"
    p = launch(n, "hardkill_phase1", name)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    p = launch(n, "hardkill_phase2", name)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert p.stdout.count("hardkill_phase2 ok") == n


@pytest.mark.skipif(NGPU < 4, reason="needs >= 4 GPUs (8 B params of ZeRO-1 state + shadow per GPU)")
def test_llama8b_full_size_zero1_sampled():
    """BASELINE.json configs[3] (Llama-3-8B-shaped, bf16 grads, fp32 AdamW, host shadow) at
    full size in the bench's launch configuration (ZeRO-1, one process per GPU): sampled
    elements of every rank's state bit-exact vs the oracle after 3 iterations."""
    name = f"cmll{os.getpid()}"
    p = launch(4, "llama_full_zero1", name, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert p.stdout.count("llama_full_zero1 ok") == 4
