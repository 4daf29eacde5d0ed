"""Parity at the bench geometry (VERDICT r1 "untested configs"): solves to tolerance on meshes
large enough that every streaming pass takes several grid-stride wavefronts and the CUDA-graph
batches exit early on the device `done` flag, against the oracle on the same seeded inputs.

Bars (BASELINE.json north_star): solution rel-L2 <= 1e-8 at tol 1e-10; iteration counts within
+-2 %.  Configs: c3-like 96^3 / 128^3 Poisson (DIA layout) with both criteria (reading Z1) and
x0 = 0 / x0 != 0; c5-like irregular RCM mesh at 80^3 base (SELL-32 layout, > 2 wavefronts); the
c2 icoFoam pressure sequence (warm-started, OpenFOAM norm) on the 512^2 cavity; c2 at its full
1024^2 size solved to its tolerance (PCG) and 60 fixed iterations of both solvers; config 5 at one
GPU's share (184^3 irregular, SELL-32) and config 4 at full size on one GPU (512^3) sampled."""
import numpy as np
import pytest

import meshgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ldu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1505_07630_b200 as m
    torch.cuda.set_device(0)
    return m


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _case(n, x0kind, seed=7630):
    s = meshgen.hex_laplacian(n, n, n, dirichlet=dict(x0=1.0))
    x0 = (np.zeros(s.nCells) if x0kind == "zero"
          else np.random.default_rng(seed).uniform(-1, 1, s.nCells))
    return s, x0


# (size, x0, norm): every combination of criterion and initial guess appears at a multi-wave size
CASES = [(128, "zero", "L2"), (128, "warm", "OpenFOAM"), (96, "warm", "L2"), (96, "zero", "OpenFOAM")]


@pytest.mark.parametrize("solver", ["pcg", "pipecg"])
@pytest.mark.parametrize("n,x0kind,norm", CASES)
def test_poisson_to_tolerance_large(ldu, n, x0kind, norm, solver):
    s, x0 = _case(n, x0kind)
    tol = 1e-10
    onorm = oracle.NORM_L2 if norm == "L2" else oracle.NORM_OPENFOAM
    gnorm = ldu.NORM_L2 if norm == "L2" else ldu.NORM_OPENFOAM
    ofn = oracle.pcg if solver == "pcg" else oracle.pipecg
    ost, ox, oit, ores = ofn(s, s.b, x0=x0, tol=tol, maxIter=20000, norm=onorm)
    assert ost == oracle.OK
    with ldu.LduMatrix.from_system(s) as A:
        assert A.info()["layout_name"] == "DIA_SYM"
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        x = cuda(x0)
        st, it, res = fn(cuda(s.b), x, tol=tol, maxIter=20000, norm=gnorm)
        stats = A.stats()
    assert st == ldu.OK and res < tol
    assert abs(it - oit) <= max(1, round(0.02 * oit)), (it, oit)
    assert rel(x.cpu().numpy(), ox) <= 1e-8
    extra = 1 if norm == "OpenFOAM" else 0  # the xbar reduction (reading Z1)
    assert stats["reductions"] == extra + (1 + 2 * it if solver == "pcg" else 2 + it)


@pytest.mark.parametrize("solver", ["pcg", "pipecg"])
def test_irregular_sell_to_tolerance_large(ldu, solver):
    """c5 recipe (exp(0.5 xi) conductances, dropped and diagonal faces, RCM renumbering) at a
    96^3 base (884,736 cells): SELL-32 over > 2 grid-stride wavefronts of every pass."""
    s = meshgen.irregular_mesh(96, seed=1505)
    ofn = oracle.pcg if solver == "pcg" else oracle.pipecg
    ost, ox, oit, ores = ofn(s, s.b, tol=1e-10, maxIter=20000)
    assert ost == oracle.OK
    with ldu.LduMatrix.from_system(s) as A:
        info = A.info()
        assert info["layout_name"] == "SELL32"
        assert s.nCells > 2 * info["gridBlocks"] * info["blockThreads"]
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        x = torch.zeros(s.nCells, dtype=torch.float64, device="cuda")
        st, it, res = fn(cuda(s.b), x, tol=1e-10, maxIter=20000)
    assert st == ldu.OK
    assert abs(it - oit) <= max(1, round(0.02 * oit)), (it, oit)
    assert rel(x.cpu().numpy(), ox) <= 1e-8


@pytest.mark.parametrize("solver,norm", [("pcg", "OpenFOAM"), ("pipecg", "L2")])
def test_cavity_piso_sequence_512(ldu, solver, norm):
    """Config 2 semantics at 512^2: 3 time steps x 2 correctors, warm start, tol 1e-6.
    Bars (DESIGN.md §4 "c2 sequence"): per-solve iteration counts within +-2 %; the final field
    within 1e-5 of the oracle's (two iterates that both meet a 1e-6 criterion on this
    Neumann operator, kappa ~ 1e5, may differ by up to kappa * tol; the warm-started sequence of
    pipelined solves carries the recurrence/true residual gap forward); the GPU's true residual
    within 10 x tol (L2)."""
    nx = 512
    s = meshgen.cavity_pressure_2d(nx, nx)
    onorm = oracle.NORM_L2 if norm == "L2" else oracle.NORM_OPENFOAM
    gnorm = ldu.NORM_L2 if norm == "L2" else ldu.NORM_OPENFOAM
    ofn = oracle.pcg if solver == "pcg" else oracle.pipecg
    xo = np.zeros(s.nCells)
    its, its_o = [], []
    with ldu.LduMatrix.from_system(s) as A:
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        x = torch.zeros(s.nCells, dtype=torch.float64, device="cuda")
        for t in range(3):
            b = meshgen.cavity_rhs(nx, nx, t)
            for c in range(2):
                st, it, res = fn(cuda(b), x, tol=1e-6, maxIter=100000, norm=gnorm)
                ost, xo, oit, ores = ofn(s, b, x0=xo, tol=1e-6, maxIter=100000, norm=onorm)
                assert st == ldu.OK and ost == oracle.OK
                its.append(it)
                its_o.append(oit)
    for a, b_ in zip(its, its_o):
        assert abs(a - b_) <= max(1, round(0.02 * b_)), (its, its_o)
    xg = x.cpu().numpy()
    assert rel(xg, xo) <= 1e-5
    if norm == "L2":
        r = b - oracle.amul(s, xg)
        assert np.linalg.norm(r) / np.linalg.norm(b) <= 10 * 1e-6


@pytest.mark.parametrize("solver", ["pcg", "pipecg"])
def test_cavity_1024_fixed_iterations(ldu, solver):
    """Config 2 at its full size (1024^2 cavity, OpenFOAM criterion): 60 fixed iterations from a
    warm start, in the launch configuration the library picks there (the persistent cooperative
    kernels: the working set fits in L2), against the oracle's 60 (a full solve takes the oracle
    ~2 min: 5648 iterations)."""
    nx = 1024
    s = meshgen.cavity_pressure_2d(nx, nx)
    b = meshgen.cavity_rhs(nx, nx, 4)
    x0 = np.random.default_rng(9).uniform(-1, 1, s.nCells)
    ofn = oracle.pcg if solver == "pcg" else oracle.pipecg
    ost, ox, oit, ores, ohist = ofn(s, b, x0=x0, tol=0.0, maxIter=60, norm=oracle.NORM_OPENFOAM,
                                    history=True)
    with ldu.LduMatrix.from_system(s) as A:
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        x = cuda(x0)
        st, it, res = fn(cuda(b), x, tol=0.0, maxIter=60, norm=ldu.NORM_OPENFOAM,
                         record_history=True)
        hist = A.history()
    assert st == ldu.NOT_CONVERGED == ost and it == oit == 60
    assert rel(x.cpu().numpy(), ox) <= 1e-10
    np.testing.assert_allclose(hist, ohist, rtol=1e-9)


def test_cavity_1024_to_tolerance():
    """Config 2 at its full size solved to its tolerance: the 1024^2 cavity pressure equation, PCG,
    OpenFOAM criterion, tol 1e-6 from x0 = 0 (5648 iterations; the oracle takes ~80 s), in the
    persistent-kernel configuration the library picks at this size, exiting on the device flag.
    Bars as the 512^2 sequence (DESIGN.md §4 "c2 sequence"): iterations within +-2 %, the field
    within 1e-5 of the oracle's (kappa ~ 4e5 at 1024^2 bounds how far two iterates meeting a 1e-6
    criterion may differ), both final residuals below tol."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1505_07630_b200 as ldu
    torch.cuda.set_device(0)
    nx = 1024
    s = meshgen.cavity_pressure_2d(nx, nx)
    b = meshgen.cavity_rhs(nx, nx, 0)
    ost, ox, oit, ores = oracle.pcg(s, b, x0=np.zeros(s.nCells), tol=1e-6, maxIter=100000,
                                    norm=oracle.NORM_OPENFOAM)
    assert ost == oracle.OK
    with ldu.LduMatrix.from_system(s) as A:
        x = torch.zeros(s.nCells, dtype=torch.float64, device="cuda")
        st, it, res = A.pcg_solve(cuda(b), x, tol=1e-6, maxIter=100000, norm=ldu.NORM_OPENFOAM)
    assert st == ldu.OK and res < 1e-6 and ores < 1e-6
    assert abs(it - oit) <= max(1, round(0.02 * oit)), (it, oit)
    assert rel(x.cpu().numpy(), ox) <= 1e-5


@pytest.mark.parametrize("solver", ["pcg", "pipecg"])
def test_c5_share_184_sampled(ldu, solver):
    """Config 5's recipe at one GPU's share of its 50M cells (184^3 base, 6.2M cells, RCM,
    SELL-32), the mesh and launch configuration of bench.py's c5 leg: SpMV over all rows vs the
    oracle; 30 fixed iterations vs the oracle's 30; then a solve to 1e-10 whose true residual
    (recomputed by the oracle's SpMV) meets the tolerance within the pipelined recurrence gap."""
    s = meshgen.irregular_mesh(184, seed=1505)
    xr = np.random.default_rng(5).uniform(-1, 1, s.nCells)
    ofn = oracle.pcg if solver == "pcg" else oracle.pipecg
    ost, ox, oit, ores = ofn(s, s.b, tol=0.0, maxIter=30)
    with ldu.LduMatrix.from_system(s) as A:
        assert A.info()["layout_name"] == "SELL32"
        y = torch.empty(s.nCells, dtype=torch.float64, device="cuda")
        A.amul(cuda(xr), y)
        assert rel(y.cpu().numpy(), oracle.amul(s, xr)) <= 1e-12
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        x = torch.zeros(s.nCells, dtype=torch.float64, device="cuda")
        st, it, res = fn(cuda(s.b), x, tol=0.0, maxIter=30)
        assert it == oit == 30
        assert rel(x.cpu().numpy(), ox) <= 1e-10
        assert abs(res - ores) <= 1e-8 * ores
        x.zero_()
        st, it, res = fn(cuda(s.b), x, tol=1e-10, maxIter=100000)
    assert st == ldu.OK and res < 1e-10
    xg = x.cpu().numpy()
    true = np.linalg.norm(s.b - oracle.amul(s, xg)) / np.linalg.norm(s.b)
    assert true < 1e-9, true


def test_c4_512_cube_sampled(ldu):
    """Config 4 at its full size on one GPU (512^3, 134M cells: the N = 1 point of the 1/2/4/8
    scaling run): SpMV over all rows vs the oracle, and 5 fixed pipelined iterations vs the
    oracle's 5 (the oracle needs ~1 min for them at this size)."""
    n = 512
    s = meshgen.hex_laplacian(n, n, n)
    b = meshgen.rhs_hot_face(n, n, n)
    xr = np.random.default_rng(3).uniform(-1, 1, s.nCells)
    yo = oracle.amul(s, xr)
    ost, ox, oit, ores = oracle.pipecg(s, b, tol=0.0, maxIter=5)
    with ldu.LduMatrix.from_system(s) as A:
        y = torch.empty(s.nCells, dtype=torch.float64, device="cuda")
        A.amul(cuda(xr), y)
        assert rel(y.cpu().numpy(), yo) <= 1e-12
        del y
        x = torch.zeros(s.nCells, dtype=torch.float64, device="cuda")
        st, it, res = A.pipecg_solve(cuda(b), x, tol=0.0, maxIter=5)
    assert it == oit == 5
    assert rel(x.cpu().numpy(), ox) <= 1e-10
    assert abs(res - ores) <= 1e-8 * ores
