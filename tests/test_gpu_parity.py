"""Parity of the CUDA path (through the C ABI) with the CPU oracle, element by element on the same
seeded inputs.  Bars (BASELINE.json north_star): SpMV rel-L2 <= 1e-12; solution rel-L2 <= 1e-8
at tol 1e-10; iteration counts within +-2%."""
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
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


SPMV_CASES = {
    "hex16_dia": lambda: meshgen.hex_laplacian(16, 16, 16),
    "hex_ragged_dia": lambda: meshgen.hex_laplacian(13, 7, 5, conductance_sigma=0.7, seed=5),
    "hex_ghost": lambda: meshgen.hex_laplacian(9, 8, 7, bc="ghost"),
    "single_cell": lambda: meshgen.hex_laplacian(1, 1, 1),
    "line_dia1": lambda: meshgen.hex_laplacian(37, 1, 1),
    "cavity_dia2": lambda: meshgen.cavity_pressure_2d(45, 33),
    "random_sell": lambda: meshgen.random_ldu(64, seed=1),
    "random_nonsym_sell": lambda: meshgen.random_ldu(61, seed=2, symmetric=False),
    "random_shuffled_sell": lambda: meshgen.random_ldu(50, seed=3, sort_faces=False),
    "irregular_sell": lambda: meshgen.irregular_mesh(12, seed=4),
    "irregular_norcm_sell": lambda: meshgen.irregular_mesh(9, seed=6, rcm=False),
}


@pytest.mark.parametrize("case", sorted(SPMV_CASES))
def test_amul_parity(ldu, case):
    sys = SPMV_CASES[case]()
    x = np.random.default_rng(11).uniform(-1, 1, sys.nCells)
    yo = oracle.amul(sys, x)
    with ldu.LduMatrix.from_system(sys) as A:
        info = A.info()
        if case.endswith("_dia") or case.endswith("dia1") or case.endswith("dia2") or case == "hex_ghost":
            assert info["layout_name"] == "DIA_SYM", info
        if case.endswith("_sell"):
            assert info["layout_name"] == "SELL32", info
        y = torch.empty(sys.nCells, dtype=torch.float64, device="cuda")
        A.amul(cuda(x), y)
        assert rel(y.cpu().numpy(), yo) <= 1e-12
        # host pointers through the same C ABI
        yh = np.empty(sys.nCells)
        A.amul(x, yh)
        np.testing.assert_array_equal(yh, y.cpu().numpy())


def test_amul_row_sums_exact(ldu):
    """A 1 = 2 x #walls exactly (integers) -- holds in any summation order."""
    nx, ny, nz = 20, 9, 11
    sys = meshgen.hex_laplacian(nx, ny, nz)
    with ldu.LduMatrix.from_system(sys) as A:
        y = np.empty(sys.nCells)
        A.amul(np.ones(sys.nCells), y)
    np.testing.assert_array_equal(y, oracle.amul(sys, np.ones(sys.nCells)))


SOLVE_CASES = {
    "c1_hot": lambda: (meshgen.hex_laplacian(16, 16, 16), meshgen.rhs_hot_face(16, 16, 16)),
    "c1_manufactured": lambda: (lambda s: (s, oracle.amul(s, np.random.default_rng(7630).uniform(-1, 1, s.nCells))))(meshgen.hex_laplacian(16, 16, 16)),
    "ragged_sigma": lambda: (lambda s: (s, meshgen.rhs_random(s.nCells, 3)))(meshgen.hex_laplacian(21, 10, 7, conductance_sigma=1.0, seed=8)),
    "cavity": lambda: (lambda s: (s, meshgen.cavity_rhs(40, 30, 0)))(meshgen.cavity_pressure_2d(40, 30)),
    "random_sell": lambda: (lambda s: (s, s.b))(meshgen.random_ldu(64, seed=21)),
    "irregular_sell": lambda: (lambda s: (s, s.b))(meshgen.irregular_mesh(14, seed=5)),
}


@pytest.mark.parametrize("persist", ["0", "1"])
@pytest.mark.parametrize("solver", ["pcg", "pipecg"])
@pytest.mark.parametrize("case", sorted(SOLVE_CASES))
def test_solve_parity(ldu, case, solver, persist, monkeypatch):
    """persist=1: the persistent cooperative kernels; 0: CUDA-graph batches of pass kernels."""
    monkeypatch.setenv("LDU_PERSIST", persist)
    sys, b = SOLVE_CASES[case]()
    tol = 1e-10
    ofn = oracle.pcg if solver == "pcg" else oracle.pipecg
    ost, ox, oit, ores, ohist = ofn(sys, b, tol=tol, maxIter=20000, history=True)
    assert ost == oracle.OK
    with ldu.LduMatrix.from_system(sys) as A:
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        xt = torch.zeros(sys.nCells, dtype=torch.float64, device="cuda")
        st, it, res = fn(cuda(b), xt, tol=tol, maxIter=20000, record_history=True)
        hist = A.history()
        stats = A.stats()
    assert st == ldu.OK and res < tol
    assert abs(it - oit) <= max(1, round(0.02 * oit)), (it, oit)
    assert rel(xt.cpu().numpy(), ox) <= 1e-8
    # residual histories overlay while the residual is well above rounding
    m = min(len(hist), len(ohist))
    assert len(hist) == it + 1
    keep = ohist[:m] > 1e-6
    np.testing.assert_allclose(hist[:m][keep], ohist[:m][keep], rtol=1e-5)
    assert stats["iterations"] == it and stats["kernels"] > 0 and stats["allreduces"] == 0
    # device-counted grid-wide reductions (reading Z4): the r0 reduction plus 2 per
    # classical iteration; pipelined: r0, (gamma_0, delta_0, rr_0), then ONE per iteration
    assert stats["reductions"] == (1 + 2 * it if solver == "pcg" else 2 + it), stats


@pytest.mark.parametrize("persist", ["0", "1"])
@pytest.mark.parametrize("solver", ["pcg", "pipecg"])
def test_fixed_iterations_track_oracle(ldu, solver, persist, monkeypatch):
    monkeypatch.setenv("LDU_PERSIST", persist)
    """tol = 0 runs exactly maxIter iterations; iterate after k steps matches the oracle's."""
    sys = meshgen.hex_laplacian(24, 20, 18)
    b = meshgen.rhs_hot_face(24, 20, 18)
    ofn = oracle.pcg if solver == "pcg" else oracle.pipecg
    for k in (1, 2, 7, 40):
        ost, ox, oit, ores = ofn(sys, b, tol=0.0, maxIter=k)
        with ldu.LduMatrix.from_system(sys) as A:
            fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
            x = np.zeros(sys.nCells)
            st, it, res = fn(b, x, tol=0.0, maxIter=k, batch=4)
        assert st == ldu.NOT_CONVERGED == ost and it == k == oit
        assert rel(x, ox) <= 1e-11
        assert abs(res - ores) <= 1e-9 * ores


@pytest.mark.parametrize("persist", ["0", "1"])
@pytest.mark.parametrize("solver", ["pcg", "pipecg"])
def test_edge_cases(ldu, solver, persist, monkeypatch):
    monkeypatch.setenv("LDU_PERSIST", persist)
    sys = meshgen.hex_laplacian(6, 5, 4)
    with ldu.LduMatrix.from_system(sys) as A:
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        # b = 0 => x = 0, nIter 0
        x = np.ones(sys.nCells)
        assert fn(np.zeros(sys.nCells), x) == (ldu.OK, 0, 0.0) and not np.any(x)
        # exact initial guess => 0 iterations, x unchanged
        xs = np.random.default_rng(1).uniform(-1, 1, sys.nCells)
        b = oracle.amul(sys, xs)
        x = xs.copy()
        st, it, res = fn(b, x, tol=1e-10)
        assert st == ldu.OK and it == 0 and np.array_equal(x, xs)
        # maxIter = 0
        x = np.zeros(sys.nCells)
        st, it, res = fn(b, x, tol=1e-10, maxIter=0)
        assert st == ldu.NOT_CONVERGED and it == 0 and not np.any(x)
        # bad arguments
        with pytest.raises(ldu.LduError):
            fn(b, x, tol=-1.0)
        with pytest.raises(ldu.LduError):
            fn(b, x, maxIter=-1)
    # identity -> 1 iteration, x = b
    I = meshgen.LduSystem(5, np.zeros(0, np.int32), np.zeros(0, np.int32), np.ones(5), np.zeros(0))
    with ldu.LduMatrix.from_system(I) as A:
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        b = np.array([3.0, -1.0, 2.0, 0.5, 7.0])
        x = np.zeros(5)
        st, it, res = fn(b, x, tol=1e-12)
        assert st == ldu.OK and it == 1 and np.array_equal(x, b)
    # indefinite 2x2 -> breakdown at iteration 1, x = (1, 0) (oracle test_breakdown_indefinite)
    B = meshgen.LduSystem(2, np.array([0], np.int32), np.array([1], np.int32), np.array([1.0, 1.0]),
                          np.array([2.0]))
    with ldu.LduMatrix.from_system(B) as A:
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        x = np.zeros(2)
        st, it, res = fn(np.array([1.0, 0.0]), x, tol=1e-12, maxIter=10)
        assert st == ldu.BREAKDOWN and it == 1
        np.testing.assert_allclose(x, [1.0, 0.0], atol=1e-15)


def test_setup_validation(ldu):
    l = np.array([0, 1], np.int32)
    u = np.array([1, 2], np.int32)
    d = np.ones(3)
    up = -0.1 * np.ones(2)
    for bad, msg in (((l, np.array([1, 3], np.int32), d, up), "outside"),
                     ((l, np.array([1, 1], np.int32), d, up), "lowerAddr == upperAddr"),
                     ((l, u, np.array([1.0, 0.0, 1.0]), up), "diag"),
                     ((l, u, d, np.array([np.nan, 1.0])), "non-finite")):
        with pytest.raises(ldu.LduError) as ei:
            ldu.LduMatrix(3, *bad)
        assert ei.value.status == ldu.ERR_INVALID_ARG and msg in str(ei.value)


@pytest.mark.parametrize("persist", ["0", "1"])
def test_determinism_bitwise(ldu, persist, monkeypatch):
    monkeypatch.setenv("LDU_PERSIST", persist)
    sys = meshgen.hex_laplacian(30, 30, 30, conductance_sigma=0.5, seed=2)
    b = meshgen.rhs_random(sys.nCells, 5)
    xs = []
    with ldu.LduMatrix.from_system(sys) as A:
        for solver in ("pcg", "pcg", "pipecg", "pipecg"):
            fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
            x = np.zeros(sys.nCells)
            fn(b, x, tol=1e-9)
            xs.append(x)
    assert np.array_equal(xs[0], xs[1]) and np.array_equal(xs[2], xs[3])


@pytest.mark.parametrize("solver", ["pcg", "pipecg"])
def test_openfoam_norm_parity(ldu, solver):
    sys = meshgen.cavity_pressure_2d(64, 48)
    b = meshgen.cavity_rhs(64, 48, 3)
    x0 = np.random.default_rng(2).uniform(-1, 1, sys.nCells)
    ofn = oracle.pcg if solver == "pcg" else oracle.pipecg
    ost, ox, oit, ores = ofn(sys, b, x0=x0, tol=1e-6, maxIter=5000, norm=oracle.NORM_OPENFOAM)
    with ldu.LduMatrix.from_system(sys) as A:
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        x = x0.copy()
        st, it, res = fn(b, x, tol=1e-6, maxIter=5000, norm=ldu.NORM_OPENFOAM)
    assert st == ldu.OK == ost
    assert abs(it - oit) <= max(1, round(0.02 * oit))
    assert rel(x, ox) <= 1e-6


@pytest.mark.parametrize("solver", ["pcg", "pipecg"])
def test_bench_config_256cube_sampled(ldu, solver):
    """BASELINE config 3 at full size (256^3, 16.8M cells) in the launch configuration bench.py
    times: SpMV over all rows vs the oracle; 30 fixed iterations vs the oracle's 30."""
    n = 256
    sys = meshgen.hex_laplacian(n, n, n)
    b = meshgen.rhs_hot_face(n, n, n)
    x = np.random.default_rng(3).uniform(-1, 1, sys.nCells)
    with ldu.LduMatrix.from_system(sys) as A:
        y = torch.empty(sys.nCells, dtype=torch.float64, device="cuda")
        A.amul(cuda(x), y)
        assert rel(y.cpu().numpy(), oracle.amul(sys, x)) <= 1e-12
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        xt = torch.zeros(sys.nCells, dtype=torch.float64, device="cuda")
        st, it, res = fn(cuda(b), xt, tol=0.0, maxIter=30)
    ofn = oracle.pcg if solver == "pcg" else oracle.pipecg
    ost, ox, oit, ores = ofn(sys, b, tol=0.0, maxIter=30)
    assert it == oit == 30
    assert rel(xt.cpu().numpy(), ox) <= 1e-10
    assert abs(res - ores) <= 1e-8 * ores


def test_stream_triad(ldu):
    g = ldu.stream_triad(0, 1 << 27, 3)
    assert 3000 < g < 9000, g


@pytest.mark.parametrize("norm", ["L2", "OpenFOAM"])
@pytest.mark.parametrize("solver", ["pcg", "pipecg"])
def test_cavity_piso_sequence_parity(ldu, solver, norm):
    """Config 2 semantics: warm-started sequence of pressure solves (6 steps x 2 correctors,
    tol 1e-6) on the 2-D cavity matrix; per-solve iteration counts and the final field match
    the oracle's sequence (pipelined CG's true-vs-recurrence residual gap included)."""
    nx = 128
    sys = meshgen.cavity_pressure_2d(nx, nx)
    onorm = oracle.NORM_L2 if norm == "L2" else oracle.NORM_OPENFOAM
    gnorm = ldu.NORM_L2 if norm == "L2" else ldu.NORM_OPENFOAM
    ofn = oracle.pcg if solver == "pcg" else oracle.pipecg
    xo = np.zeros(sys.nCells)
    its_o = []
    with ldu.LduMatrix.from_system(sys) as A:
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        x = np.zeros(sys.nCells)
        its = []
        for t in range(6):
            b = meshgen.cavity_rhs(nx, nx, t)
            for c in range(2):
                st, it, res = fn(b, x, tol=1e-6, maxIter=100000, norm=gnorm)
                ost, xo, oit, ores = ofn(sys, b, x0=xo, tol=1e-6, maxIter=100000, norm=onorm)
                assert st == ldu.OK and ost == oracle.OK
                its.append(it)
                its_o.append(oit)
    for a, b_ in zip(its, its_o):
        assert abs(a - b_) <= max(1, round(0.02 * b_)), (its, its_o)
    assert rel(x, xo) <= 1e-6


@pytest.mark.parametrize("solver", ["pcg", "pipecg"])
def test_reltol_miniter_parity(ldu, solver):
    """OpenFOAM relTol / minIter (reading Z26) through the C ABI vs the oracle."""
    sys = meshgen.cavity_pressure_2d(48, 40)
    b = meshgen.cavity_rhs(48, 40, 2)
    ofn = oracle.pcg if solver == "pcg" else oracle.pipecg
    with ldu.LduMatrix.from_system(sys) as A:
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        for kw in (dict(tol=1e-14, relTol=0.05), dict(tol=1e-14, relTol=0.5),
                   dict(tol=1e300, minIter=9), dict(tol=1e-6, relTol=0.05, minIter=3),
                   dict(tol=1e300, minIter=50, maxIter=20)):
            kw = dict(kw)
            maxIter = kw.pop("maxIter", 5000)
            ost, ox, oit, ores = ofn(sys, b, maxIter=maxIter, norm=oracle.NORM_OPENFOAM, **kw)
            x = np.zeros(sys.nCells)
            st, it, res = fn(b, x, maxIter=maxIter, norm=ldu.NORM_OPENFOAM, **kw)
            assert st == ost and it == oit, (kw, st, ost, it, oit)
            assert rel(x, ox) <= 1e-10


# ---- residual replacement in pipelined CG (NEXT-4) ------------------------------------------------
def test_pipecg_replacement_parity(ldu):
    """replaceEvery = 25 on the device = the oracle's pipelined CG with the same replacement
    (counts, solution, residual history across two replacements) -- fixed and to tolerance."""
    s = meshgen.hex_laplacian(24, 24, 24, conductance_sigma=0.3, seed=4, dirichlet=dict(x0=1.0))
    ost, ox, oit, ores, ohist = oracle.pipecg(s, s.b, tol=1e-10, maxIter=2000, history=True,
                                              replace_every=25)
    with ldu.LduMatrix.from_system(s) as A:
        x = torch.zeros(s.nCells, dtype=torch.float64, device="cuda")
        st, it, res = A.pipecg_solve(cuda(s.b), x, tol=1e-10, maxIter=2000, record_history=True,
                                     replaceEvery=25)
        hist = A.history()
        assert st == ldu.OK and ost == oracle.OK and abs(it - oit) <= 1, (it, oit)
        assert rel(x.cpu().numpy(), ox) <= 1e-8
        np.testing.assert_allclose(hist[:60], ohist[:60], rtol=1e-8)
        fst, fox, foit, fores, fohist = oracle.pipecg(s, s.b, tol=0.0, maxIter=60, history=True,
                                                      replace_every=25)
        x = torch.zeros(s.nCells, dtype=torch.float64, device="cuda")
        st, it, res = A.pipecg_solve(cuda(s.b), x, tol=0.0, maxIter=60, record_history=True,
                                     replaceEvery=25)
        assert st == fst == ldu.NOT_CONVERGED and it == foit == 60
        np.testing.assert_allclose(A.history(), fohist, rtol=1e-8)
        assert rel(x.cpu().numpy(), fox) <= 1e-9
        with pytest.raises(ldu.LduError) as e:
            A.pcg_solve(cuda(s.b), x, tol=1e-8, maxIter=10, replaceEvery=5)
        assert e.value.status == ldu.ERR_INVALID_ARG


def test_pipecg_replacement_restores_attainable_accuracy(ldu):
    """On the device, as in the oracle pin: plain GV pipelined CG at 64^3 stalls (true residual
    above tol 1e-12) and breaks down at tol 1e-14; with replacement every 50 iterations the TRUE
    residual (library SpMV) meets the tolerance in the classical iteration count."""
    s = meshgen.hex_laplacian(64, 64, 64, dirichlet=dict(x0=1.0))
    with ldu.LduMatrix.from_system(s) as A:
        b = cuda(s.b)

        def true_res(x):
            y = torch.empty_like(x)
            A.amul(x, y)
            return (torch.linalg.norm(b - y) / torch.linalg.norm(b)).item()
        x = torch.zeros_like(b)
        st, it, res = A.pipecg_solve(b, x, tol=1e-12, maxIter=3000)
        assert st == ldu.OK and true_res(x) > 2e-12
        x = torch.zeros_like(b)
        st, it, res = A.pipecg_solve(b, x, tol=1e-12, maxIter=3000, replaceEvery=50)
        assert st == ldu.OK and true_res(x) < 1e-12
        x = torch.zeros_like(b)
        st0, _, _ = A.pipecg_solve(b, x, tol=1e-14, maxIter=3000)
        assert st0 == ldu.BREAKDOWN
        x = torch.zeros_like(b)
        _, it_cg, _ = A.pcg_solve(b, x, tol=1e-14, maxIter=3000)
        x = torch.zeros_like(b)
        st, it, res = A.pipecg_solve(b, x, tol=1e-14, maxIter=3000, replaceEvery=50)
        assert st == ldu.OK and abs(it - it_cg) <= 2 and true_res(x) < 1.1e-14
