"""Real multi-GPU parity (needs >= 2 visible B200s; skipped otherwise): launches
tests/mgpu_worker.py under torchrun, one process per GPU, for the fused
one-launch-per-layer path and the two-kernel path. Each rank's kernels
exchange tokens with the others over NVLink P2P; rank 0 checks every layer
against the CPU oracle (see the worker's docstring)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("phased,vanilla,migrate", [(False, False, False), (True, False, False),
                                                    (False, True, False), (False, False, True)])
def test_two_gpu_parity(phased, vanilla, migrate):
    n = _gpus()
    if n < 2:
        pytest.skip("needs two GPUs")
    port = "29631" if phased else ("29635" if vanilla else ("29637" if migrate else "29633"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", port,
           os.path.join(HERE, "mgpu_worker.py")] + (["--phased"] if phased else []) + \
        (["--vanilla"] if vanilla else []) + (["--migrate"] if migrate else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " OK " in r.stdout
    if migrate:
        assert "migrated" in r.stdout


@pytest.mark.parametrize("vanilla", [False, True])
def test_four_gpu_parity(vanilla):
    # G=4: 2 experts per GPU at E=8, every layer checked against the oracle
    n = _gpus()
    if n < 4:
        pytest.skip("needs four GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "4",
           "--master-addr", "127.0.0.1", "--master-port", "29645" if vanilla else "29643",
           os.path.join(HERE, "mgpu_worker.py"), "--batch", "32"] + (["--vanilla"] if vanilla else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " OK " in r.stdout


def test_kv_append_replicated():
    """exf_kv_append writing every rank's replica over NVLink (CUDA-IPC peers)."""
    n = _gpus()
    if n < 2:
        pytest.skip("needs two GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29641",
           os.path.join(HERE, "kv_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout
