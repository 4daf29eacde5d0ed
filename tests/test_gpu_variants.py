"""Every SpMV-bearing kernel variant of the DIA layout (LDU_VARIANT: 0 generic row gather,
1/2 hoisted loads, 3 plane-marching smem ring, 4 TMA-fed plane march, 5 chunked wavefront, 6 warp-shuffle neighbours, 7 split update + SpMV) against the oracle, on meshes whose far offset
nx*ny >= 4096 so the marching geometry applies (incl. ragged tiles and a partial last tile)."""
import os

import numpy as np
import pytest

import meshgen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

MESHES = {
    "64x64x12": lambda: meshgen.hex_laplacian(64, 64, 12, dirichlet=dict(x0=1.0)),
    "70x61x13_sigma": lambda: meshgen.hex_laplacian(70, 61, 13, conductance_sigma=0.7, seed=9,
                                                    dirichlet=dict(x0=1.0)),
    "130x33x5_ddt": lambda: meshgen.hex_laplacian(130, 33, 5, ddt=0.5, dirichlet=dict(z0=2.0)),
    "96x43x7_sigma": lambda: meshgen.hex_laplacian(96, 43, 7, conductance_sigma=0.4, seed=3,
                                                   dirichlet=dict(y1=1.0)),
}


@pytest.fixture(scope="module")
def ldu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1505_07630_b200 as m
    return m


def _make(ldu, sys, variant):
    """Variants live in the CUDA-graph pass kernels: force them (no persistent kernel)."""
    saved = {k: os.environ.get(k) for k in ("LDU_VARIANT", "LDU_PERSIST")}
    os.environ["LDU_VARIANT"] = str(variant)
    os.environ["LDU_PERSIST"] = "0"
    try:
        return ldu.LduMatrix.from_system(sys)
    finally:
        for k, v in saved.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("mesh", sorted(MESHES))
def test_amul_variants_bitwise(ldu, mesh):
    sys = MESHES[mesh]()
    x = np.random.default_rng(4).uniform(-1, 1, sys.nCells)
    yo = oracle.amul(sys, x)
    ys = []
    for v in (0, 1, 2, 3, 4, 5, 6, 7):
        with _make(ldu, sys, v) as A:
            assert A.info()["layout_name"] == "DIA_SYM"
            y = np.empty(sys.nCells)
            A.amul(x, y)
            ys.append(y)
        assert np.linalg.norm(y - yo) <= 1e-12 * np.linalg.norm(yo)
    for y in ys[1:]:  # same per-row order and arithmetic in every variant
        np.testing.assert_array_equal(y, ys[0])


@pytest.mark.parametrize("solver", ["pcg", "pipecg"])
@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("mesh", sorted(MESHES))
def test_solve_variants(ldu, mesh, variant, solver):
    sys = MESHES[mesh]()
    ofn = oracle.pcg if solver == "pcg" else oracle.pipecg
    ost, ox, oit, ores = ofn(sys, sys.b, tol=1e-10, maxIter=5000)
    with _make(ldu, sys, variant) as A:
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        x = torch.zeros(sys.nCells, dtype=torch.float64, device="cuda")
        st, it, res = fn(torch.from_numpy(sys.b).cuda(), x, tol=1e-10, maxIter=5000)
        # fixed-iteration tracking as in bench.py
        xf = np.zeros(sys.nCells)
        st2, it2, res2 = fn(sys.b, xf, tol=0.0, maxIter=17)
    assert st == ldu.OK and abs(it - oit) <= max(1, round(0.02 * oit))
    assert np.linalg.norm(x.cpu().numpy() - ox) <= 1e-8 * np.linalg.norm(ox)
    _, oxf, _, _ = ofn(sys, sys.b, tol=0.0, maxIter=17)
    assert st2 == ldu.NOT_CONVERGED and it2 == 17
    assert np.linalg.norm(xf - oxf) <= 1e-11 * np.linalg.norm(oxf)


@pytest.mark.parametrize("fuse", [0, 1])
@pytest.mark.parametrize("mesh", sorted(MESHES))
def test_pipelined_fused_and_split(ldu, mesh, fuse):
    """Single rank: pipelined CG with S and U fused (default) and split (LDU_PIPE_FUSE=0)."""
    sys = MESHES[mesh]()
    ost, ox, oit, ores = oracle.pipecg(sys, sys.b, tol=1e-10, maxIter=5000)
    saved = {k: os.environ.get(k) for k in ("LDU_PIPE_FUSE", "LDU_PERSIST")}
    os.environ["LDU_PIPE_FUSE"] = str(fuse)
    os.environ["LDU_PERSIST"] = "0"
    try:
        A = ldu.LduMatrix.from_system(sys)
    finally:
        for k, v in saved.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
    with A:
        assert A.info()["pipeFused"] == fuse
        x = np.zeros(sys.nCells)
        st, it, res = A.pipecg_solve(sys.b, x, tol=1e-10, maxIter=5000)
        xf = np.zeros(sys.nCells)
        A.pipecg_solve(sys.b, xf, tol=0.0, maxIter=23)
    assert st == ldu.OK and abs(it - oit) <= max(1, round(0.02 * oit))
    assert np.linalg.norm(x - ox) <= 1e-8 * np.linalg.norm(ox)
    _, oxf, _, _ = oracle.pipecg(sys, sys.b, tol=0.0, maxIter=23)
    assert np.linalg.norm(xf - oxf) <= 1e-11 * np.linalg.norm(oxf)
