"""Multi-GPU parity (needs >= 2 GPUs; skipped otherwise): runs tests/mgpu_parity.py under
torchrun with one rank per GPU and checks rank 0's verdict."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def n_gpus():
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("world", [2, 4])
def test_multi_gpu_parity(world):
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world), os.path.join(ROOT, "tests", "mgpu_parity.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [l for l in res.stdout.splitlines() if l.startswith("MGPU_RESULT ")]
    assert res.returncode == 0 and lines, res.stdout[-3000:] + res.stderr[-3000:]
    out = json.loads(lines[-1][len("MGPU_RESULT "):])
    assert out["world"] == world
    for name, r in out["cases"].items():
        assert r["ok"], (name, r)


@pytest.mark.parametrize("world", [2, 4])
def test_multi_gpu_full_size_c4_bloch(world):
    """C4 (400x400x40, N = 25.6M) at V = 0 on 2 / 4 GPUs against the exact partial-Bloch
    trace (tests/mgpu_bloch.py)."""
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world), os.path.join(ROOT, "tests", "mgpu_bloch.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    lines = [l for l in res.stdout.splitlines() if l.startswith("MGPU_BLOCH ")]
    assert res.returncode == 0 and lines, res.stdout[-3000:] + res.stderr[-3000:]
    out = json.loads(lines[-1][len("MGPU_BLOCH "):])
    assert out["world"] == world and out["ok"], out

