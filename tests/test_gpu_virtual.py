"""The multi-rank path on ONE GPU (§8(e)) through KPM_VIRTUAL_RANKS: P
contexts on cuda:0, one host thread each, joined in an in-process group (kpm_vgroup).  Each
context owns a row block of the global matrix (the row distribution of P:849-854) and runs the
multi-GPU code: edge / interior chunk split, the fused halo exchange (the edge kernels' epilogue
stores boundary rows straight into the neighbours' halo slots -- plain device pointers here
instead of CUDA IPC mappings), the flag-epoch ordering (cuStreamWaitValue32 / WriteValue32), and
the single eta reduction at the end (host all-gather in rank order here instead of
ncclAllReduce).  Checked against the oracle on the global matrix (1e-10 gate), the SELL copy and
halo plan bit for bit against the numpy references, and P-invariance.  Each case runs in a
subprocess (tests/vranks_parity.py) with CUDA_DEVICE_MAX_CONNECTIONS=32 and a hard timeout."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args, timeout=600):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "vranks_parity.py"), *map(str, args)],
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    lines = [l for l in res.stdout.splitlines() if l.startswith("VRANKS_RESULT ")]
    assert res.returncode == 0 and lines, res.stdout[-3000:] + res.stderr[-3000:]
    out = json.loads(lines[-1][len("VRANKS_RESULT "):])
    assert out["ok"], out
    return out


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("R", [32, 8])
def test_virtual_ranks_ti_slabs(P, R):
    out = run("ti", P, R)
    if R == 32:
        assert out["kernel"].startswith("tiled.bc")  # the block-cache feed, one plan per list


@pytest.mark.parametrize("P", [2, 4])
def test_virtual_ranks_uneven_irregular(P):
    run("uneven", P)


def test_virtual_group_rejects_mismatch():
    assert run("mismatch")["rejected"]
