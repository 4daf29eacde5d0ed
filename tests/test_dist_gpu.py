"""Multi-GPU parity: slab-partitioned SpMV / PCG / pipelined CG over NCCL (halo send/recv and
fused-sum allgathers) equal the single-domain oracle.  Runs tests/dist_worker.py
under torchrun with 2 (and 4 when present) ranks; skipped on boxes with fewer GPUs."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.parametrize("mode", ["p2p_fused", "p2p_split", "nccl"])
@pytest.mark.parametrize("nproc", [2, 4])
def test_distributed_parity(nproc, mode):
    """Peer-memory path (default; fused and split pipelined passes) and the NCCL fallback."""
    if _ngpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    env = dict(os.environ)
    env["LDU_P2P"] = "0" if mode == "nccl" else "1"
    env["LDU_PIPE_FUSE"] = "0" if mode == "p2p_split" else "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", "--master-port=29533",
           os.path.join(ROOT, "tests", "dist_worker.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert p.returncode == 0 and "DIST_OK" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]


@pytest.mark.parametrize("nproc", [2, 4])
def test_distributed_amg_parity(nproc):
    """Block-Jacobi AMG-PCG / AMG-PipeCG across ranks (reading Z33) = the oracle's emulation."""
    if _ngpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", "--master-port=29534",
           os.path.join(ROOT, "tests", "dist_amg_worker.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0 and "DIST_AMG_OK" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]


@pytest.mark.parametrize("nproc", [2, 4])
def test_distributed_dic_parity(nproc):
    """Block-Jacobi DIC-PCG / DIC-PipeCG across ranks (readings Z33, Z35) = the oracle's block DIC."""
    if _ngpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", "--master-port=29535",
           os.path.join(ROOT, "tests", "dist_amg_worker.py"), "dic"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0 and "DIST_AMG_OK" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]
