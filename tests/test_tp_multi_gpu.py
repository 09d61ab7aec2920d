"""TP > 1 parity on real GPUs: launches tests/mp_tp_check.py under torchrun with
one process per visible GPU (2, 4 or 8) and requires exit code 0."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("T", [2, 4, 8])
def test_tp_parity_multi_gpu(T):
    if torch.cuda.device_count() < T:
        pytest.skip(f"needs {T} GPUs, have {torch.cuda.device_count()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={T}",
           "--master-addr", "127.0.0.1", "--master-port", str(29400 + T), os.path.join(ROOT, "tests", "mp_tp_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]


def test_pipeline_stage_sendrecv_2gpu():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29477", os.path.join(ROOT, "tests", "mp_pp_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]


def test_peer_barrier_timeout_2gpu():
    """A TP peer that never reaches the barrier -> PeerTimeoutError naming it."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29478", os.path.join(ROOT, "tests", "mp_timeout_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    print(r.stdout[-4000:])
    assert r.returncode == 0 and "PeerTimeoutError" in r.stdout, r.stdout[-4000:] + r.stderr[-4000:]


def test_tp2_x_pp2_step_4gpu():
    """BASELINE.json configs[0]: TP=2 x PP=2 pipelined step vs the fp64 oracle (mp_tppp_check.py)."""
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
           "--master-addr", "127.0.0.1", "--master-port", "29479", os.path.join(ROOT, "tests", "mp_tppp_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
