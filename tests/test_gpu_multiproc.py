"""GPU parity tests, real mode: one process per GPU over CUDA-IPC peer memory
(NVLink / NVSwitch). Skipped when the box has fewer than 2 GPUs."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus() -> int:
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("nproc", [2, 4, 8])
def test_real_mode_parity(nproc):
    if _ngpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs, box has {_ngpus()}")
    env = dict(os.environ, PCCL_TIMEOUT_MS="10000")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + nproc}", os.path.join(ROOT, "tests", "mp_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count("OK") >= nproc, out[-4000:]
