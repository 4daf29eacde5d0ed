"""Multi-rank parity: slab-partitioned SpMV / PCG / pipelined CG (halo exchange + fused-sum
reductions) equal the single-domain oracle.  Runs tests/dist_worker.py
(and dist_amg_worker.py) under torchrun.

* ``*_shared_gpu`` tests: host-bootstrapped communicator (gloo + ldu_comm_init_host, no NCCL);
  ranks share the box's GPUs (all on cuda:0 on a 1-GPU box) and talk through the peer-memory
  mailboxes over CUDA IPC -- the same kernels as the one-rank-per-GPU path.  Never skipped.
* the others: one rank per GPU over NCCL bootstrap; skipped on boxes with fewer GPUs."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _torchrun(nproc, port, script_args, env_extra=None, timeout=900):
    env = dict(os.environ)
    env.update(env_extra or {})
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={port}",
           *script_args]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)


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


# ---- ranks sharing the box's GPU(s): host bootstrap, peer-memory path only ------------------

@pytest.mark.parametrize("mode,nproc", [("p2p_fused", 2), ("p2p_split", 2), ("p2p_fused", 4),
                                        ("p2p_fused", 8)])
def test_distributed_parity_shared_gpu(nproc, mode):
    """SpMV, PCG, PipeCG (fused and split passes), OpenFOAM norm / relTol / minIter and the
    device-counted reductions (1 + 2 it classical, 2 + it pipelined) across nproc ranks."""
    p = _torchrun(nproc, 29541 + nproc, [os.path.join(ROOT, "tests", "dist_worker.py")],
                  {"LDU_DIST_BOOT": "host", "LDU_PIPE_FUSE": "0" if mode == "p2p_split" else "1"})
    assert p.returncode == 0 and "DIST_OK" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]


@pytest.mark.parametrize("bounds,nproc", [("weighted", 2), ("weighted", 3), ("nnz", 3)])
def test_distributed_unequal_slabs_shared_gpu(bounds, nproc):
    """NEXT-3 through the library: Eq 5-8 weighted slabs (work fractions 1 : 2 : .. : nproc)
    and equal-non-zero slabs of every case (incl. the irregular RCM mesh, whose slab boundaries
    are ragged) -- the one-kernel loop's interface-free run and boundary rows on unequal ranks."""
    p = _torchrun(nproc, 29591 + nproc + (10 if bounds == "nnz" else 0),
                  [os.path.join(ROOT, "tests", "dist_worker.py")],
                  {"LDU_DIST_BOOT": "host", "LDU_DIST_BOUNDS": bounds})
    assert p.returncode == 0 and "DIST_OK" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]


@pytest.mark.parametrize("nproc", [2, 4])
def test_distributed_amg_parity_shared_gpu(nproc):
    p = _torchrun(nproc, 29551 + nproc, [os.path.join(ROOT, "tests", "dist_amg_worker.py")],
                  {"LDU_DIST_BOOT": "host"})
    assert p.returncode == 0 and "DIST_AMG_OK" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]


@pytest.mark.parametrize("nproc", [2])
def test_distributed_dic_parity_shared_gpu(nproc):
    p = _torchrun(nproc, 29561 + nproc, [os.path.join(ROOT, "tests", "dist_amg_worker.py"), "dic"],
                  {"LDU_DIST_BOOT": "host"})
    assert p.returncode == 0 and "DIST_AMG_OK" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]


@pytest.mark.parametrize("pdl", ["1"])
def test_distributed_pipecg_stress_shared_gpu(pdl):
    """Regression for the halo-pack race of the fused multi-rank loop (the pack of exchange i+1
    read the State the concurrent control step was advancing): >= 10^4 fused iterations over
    repeated solves on 4 ranks, with and without programmatic dependent launch; every repeat
    must be bitwise identical (the path is deterministic) and match the oracle.  (PDL is the
    default; LDU_PDL=0 passed the same test, profiles/r02_dist.)"""
    p = _torchrun(4, 29571, [os.path.join(ROOT, "tests", "dist_worker.py"), "stress"],
                  {"LDU_DIST_BOOT": "host", "LDU_PDL": pdl}, timeout=1500)
    assert p.returncode == 0 and "DIST_STRESS_OK" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]
