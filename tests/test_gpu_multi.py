"""Multi-GPU parity (needs >= 2 GPUs; skipped otherwise): P-rank NCCL forward
== 1-GPU forward bit for bit (tools/multi_gpu_check.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def n_gpus():
    """GPUs visible to child processes (torch's count, else nvidia-smi's)."""
    n = 0
    try:
        import torch
        n = torch.cuda.device_count()
    except Exception:
        pass
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=30).stdout
        n = max(n, sum(1 for line in out.splitlines() if line.startswith("GPU ")))
    except Exception:
        pass
    return n


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_partitioned_forward_bit_exact(world, precision):
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world),
           os.path.join(ROOT, "tools", "multi_gpu_check.py"), "--precision", precision]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0
    assert "bit-exact True" in r.stdout


@pytest.mark.parametrize("world", [2, 4])
def test_partitioned_training_step_matches_serial(world):
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + world),
           os.path.join(ROOT, "tools", "multi_gpu_train_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0
    assert "train lockstep True" in r.stdout
