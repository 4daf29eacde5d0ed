"""Pins for oracle.pcg / oracle.pipecg against things other than the
oracle: the worked examples S:332-333, LAPACK Cholesky, exact-arithmetic termination, closed-form
eigen RHS, manufactured solutions (algebraic and continuum O(h^2)), A-norm monotonicity,
iterate-wise equivalence of pipelined and classical CG, Table 2's 128^3/64^3 ratio."""
import numpy as np
import pytest

import meshgen
import oracle
from conftest import load_spec_examples, load_table2
from test_oracle_spmv import ghost_eigpair


def _ex_sys(ex):
    return meshgen.LduSystem(ex["n"], ex["l"], ex["u"], ex["diag"], ex["upper"])


@pytest.mark.parametrize("solver", ["pcg", "pipecg_j", "pipecg_l"])
def test_spec_2x2(solver):
    ex = load_spec_examples()["cg_2x2"]
    f = _solver(solver)
    st, x, it, res = f(_ex_sys(ex), ex["vec"], tol=1e-14, maxIter=10)
    exp = np.array([float(v) for v in ex["expected"]["x"].split(",")])
    assert st == oracle.OK
    np.testing.assert_allclose(x, exp, rtol=0, atol=1e-15)
    np.testing.assert_allclose(x, [1 / 11, 7 / 11], rtol=0, atol=1e-15)
    assert it <= 2  # n = 2: exact termination


@pytest.mark.parametrize("solver", ["pcg", "pipecg_j", "pipecg_l"])
def test_spec_identity(solver):
    ex = load_spec_examples()["cg_identity"]
    st, x, it, res = _solver(solver)(_ex_sys(ex), ex["vec"], tol=1e-12, maxIter=10)
    assert st == oracle.OK
    assert it == int(ex["expected"]["iters"])
    np.testing.assert_array_equal(x, np.array([float(v) for v in ex["expected"]["x"].split(",")]))


def _solver(name):
    if name == "pcg":
        return oracle.pcg
    if name == "pipecg_j":
        return lambda *a, **k: oracle.pipecg(*a, mode=oracle.JACOBI, **k)
    return lambda *a, **k: oracle.pipecg(*a, mode=oracle.LITERAL, **k)


def _kappa_jacobi(A):
    d = np.sqrt(np.diag(A))
    ev = np.linalg.eigvalsh(A / d[:, None] / d[None, :])
    return ev[-1] / ev[0]


CHOL_CASES = [
    ("hex_hot", lambda: meshgen.hex_laplacian(8, 7, 6, dirichlet=dict(x0=1.0))),
    ("hex_sigma", lambda: meshgen.hex_laplacian(6, 6, 6, conductance_sigma=1.0, seed=9)),
    ("cavity", lambda: meshgen.cavity_pressure_2d(12, 9)),
    ("random", lambda: meshgen.random_ldu(64, seed=21)),
    ("random_shuffled", lambda: meshgen.random_ldu(48, seed=22, sort_faces=False)),
]


@pytest.mark.parametrize("solver", ["pcg", "pipecg_j", "pipecg_l"])
@pytest.mark.parametrize("case", range(len(CHOL_CASES)))
def test_against_cholesky(solver, case):
    name, mk = CHOL_CASES[case]
    sys = mk()
    A = sys.dense()
    b = sys.b if np.any(sys.b) else meshgen.rhs_random(sys.nCells, seed=case)
    L = np.linalg.cholesky(A)
    xc = np.linalg.solve(L.T, np.linalg.solve(L, b))
    tol = 1e-10
    st, x, it, res = _solver(solver)(sys, b, tol=tol, maxIter=5000)
    assert st == oracle.OK and res < tol
    kappa = np.linalg.cond(A)
    assert np.linalg.norm(x - xc) / np.linalg.norm(xc) <= kappa * tol * 1.01
    # true residual agrees with the recurrence residual
    rt = np.linalg.norm(b - A @ x) / np.linalg.norm(b)
    assert rt < 10 * tol


@pytest.mark.parametrize("seed", range(6))
def test_termination_in_n_steps(seed):
    """Exact-arithmetic property: CG terminates in <= n iterations (n <= 32, well conditioned)."""
    n = 24 + seed
    sys = meshgen.random_ldu(n, seed=100 + seed, density=0.3, margin=2.0)
    st, x, it, res = oracle.pcg(sys, sys.b, tol=1e-12, maxIter=200)
    assert st == oracle.OK and it <= n


@pytest.mark.parametrize("m", [1, 3, 5])
@pytest.mark.parametrize("solver", ["pcg", "pipecg_j", "pipecg_l"])
def test_eigen_rhs_exact_iterations(m, solver):
    """Ghost-h (constant diag 6, so Jacobi is a scaling): b = sum of m eigenvectors with distinct
    eigenvalues => exactly m iterations and x = sum v_i / lambda_i (closed form)."""
    nx, ny, nz = 6, 5, 7
    sys = meshgen.hex_laplacian(nx, ny, nz, bc="ghost")
    ks = [(1, 1, 1), (2, 1, 3), (3, 4, 2), (5, 2, 6), (6, 5, 7)][:m]
    b = np.zeros(sys.nCells)
    xe = np.zeros(sys.nCells)
    for k in ks:
        v, lam = ghost_eigpair(nx, ny, nz, *k)
        b += v
        xe += v / lam
    st, x, it, res = _solver(solver)(sys, b, tol=1e-10, maxIter=100)
    assert st == oracle.OK and it == m
    assert np.linalg.norm(x - xe) <= 1e-10 * np.linalg.norm(xe)


def test_anorm_error_monotone():
    """the A-norm error of CG iterates decreases monotonically."""
    sys = meshgen.random_ldu(60, seed=5, density=0.1, margin=0.05)
    A = sys.dense()
    xs = np.linalg.solve(A, sys.b)
    errs = []
    for k in range(0, 40):
        st, x, it, res = oracle.pcg(sys, sys.b, tol=0.0, maxIter=k)
        e = x - xs
        errs.append(e @ A @ e)
    errs = np.array(errs)
    assert np.all(np.diff(errs) <= 1e-12 * errs[0])
    assert errs[-1] < 1e-6 * errs[0]


def test_manufactured_ghost_closed_form_kappa():
    """x* ~ U(-1,1) (seed 7630), b = A x* (numpy dense): ||x - x*|| / ||x*|| <= kappa tol with
    kappa = lambda_max / lambda_min in closed form for ghost-h."""
    n = 12
    sys = meshgen.hex_laplacian(n, n, n, bc="ghost")
    xs = np.random.default_rng(7630).uniform(-1, 1, sys.nCells)
    b = sys.dense() @ xs
    lmin = 3 * 2 * (1 - np.cos(np.pi / (n + 1)))
    lmax = 3 * 2 * (1 - np.cos(np.pi * n / (n + 1)))
    tol = 1e-10
    for solver in ("pcg", "pipecg_j"):
        st, x, it, res = _solver(solver)(sys, b, tol=tol, maxIter=5000)
        assert st == oracle.OK
        assert np.linalg.norm(x - xs) / np.linalg.norm(xs) <= (lmax / lmin) * tol


def test_continuum_manufactured_second_order():
    """T = sin(pi x) sin(pi y) sin(pi z) on the unit cube, T = 0 on the walls, f = 3 pi^2 T.
    With h = 1/n, the h=1 FV system reads A T = h^2 f.  Max error must fall ~4x per refinement
    (O(h^2)); this pins the generator's half-cell Dirichlet convention (reading Z11)."""
    errs = []
    for n in (8, 16, 32):
        sys = meshgen.hex_laplacian(n, n, n)
        c = np.arange(sys.nCells)
        xc = ((c % n) + 0.5) / n
        yc = (((c // n) % n) + 0.5) / n
        zc = ((c // (n * n)) + 0.5) / n
        T = np.sin(np.pi * xc) * np.sin(np.pi * yc) * np.sin(np.pi * zc)
        b = (1.0 / n) ** 2 * 3 * np.pi ** 2 * T
        st, x, it, res = oracle.pcg(sys, b, tol=1e-12, maxIter=10000)
        assert st == oracle.OK
        errs.append(np.abs(x - T).max())
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.5 < r1 < 4.5 and 3.7 < r2 < 4.3, errs


@pytest.mark.parametrize("seed", range(10))
def test_pipelined_iteratewise_equals_classical(seed):
    """on SPD n <= 32, kappa < 1e4, pipelined iterates match classical ones within 1e-6
    at equal iteration counts (equivalent in exact arithmetic)."""
    n = 16 + seed
    sys = meshgen.random_ldu(n, seed=300 + seed, density=0.3, margin=0.2)
    assert np.linalg.cond(sys.dense()) < 1e4
    for k in range(1, min(n, 12)):
        _, xc, itc, _ = oracle.pcg(sys, sys.b, tol=0.0, maxIter=k)
        for mode in (oracle.JACOBI, oracle.LITERAL):
            _, xp, itp, _ = oracle.pipecg(sys, sys.b, tol=0.0, maxIter=k, mode=mode)
            assert itc == itp == k
            assert np.linalg.norm(xp - xc) <= 1e-6 * np.linalg.norm(xc)


@pytest.mark.parametrize("rhs", ["hot", "manufactured"])
def test_pipelined_equal_counts_16cube(rhs):
    """Config 1 (16^3, tol 1e-10): pipelined (both forms) and classical stop at the same
    iteration; solutions agree far below tolerance; residual histories overlay."""
    sys = meshgen.hex_laplacian(16, 16, 16)
    if rhs == "hot":
        b = meshgen.rhs_hot_face(16, 16, 16)
    else:
        b = sys.dense() @ np.random.default_rng(7630).uniform(-1, 1, sys.nCells)
    st, xc, itc, rc, hc = oracle.pcg(sys, b, tol=1e-10, maxIter=1000, history=True)
    st2, xj, itj, rj, hj = oracle.pipecg(sys, b, tol=1e-10, maxIter=1000, history=True)
    st3, xl, itl, rl, hl = oracle.pipecg(sys, b, tol=1e-10, maxIter=1000, mode=oracle.LITERAL,
                                         history=True)
    assert st == st2 == st3 == oracle.OK
    assert itc == itj == itl
    assert np.linalg.norm(xj - xc) <= 1e-10 * np.linalg.norm(xc)
    assert np.linalg.norm(xl - xj) <= 1e-11 * np.linalg.norm(xc)
    np.testing.assert_allclose(hj, hc, rtol=1e-4)


@pytest.mark.parametrize("solver", ["pcg", "pipecg_j", "pipecg_l"])
def test_breakdown_indefinite(solver):
    """A = [[1,2],[2,1]] (positive diagonal, indefinite), b = (1,0): p.Ap = -12 at k = 1
    (hand computation) -> BREAKDOWN naming iteration 1; x is the last valid iterate (1, 0)."""
    sys = meshgen.LduSystem(2, np.array([0], np.int32), np.array([1], np.int32),
                            np.array([1.0, 1.0]), np.array([2.0]))
    st, x, it, res = _solver(solver)(sys, np.array([1.0, 0.0]), tol=1e-12, maxIter=10)
    assert st == oracle.BREAKDOWN and it == 1
    np.testing.assert_allclose(x, [1.0, 0.0], atol=1e-15)


@pytest.mark.parametrize("solver", ["pcg", "pipecg_j", "pipecg_l"])
def test_zero_rhs_and_exact_guess(solver):
    sys = meshgen.hex_laplacian(5, 4, 3)
    st, x, it, res = _solver(solver)(sys, np.zeros(sys.nCells), x0=np.ones(sys.nCells))
    assert st == oracle.OK and it == 0 and res == 0.0 and not np.any(x)
    xs = np.random.default_rng(1).uniform(-1, 1, sys.nCells)
    st, x, it, res = _solver(solver)(sys, sys.dense() @ xs, x0=xs, tol=1e-10)
    assert st == oracle.OK and it == 0


@pytest.mark.parametrize("solver", ["pcg", "pipecg_j"])
def test_not_converged_returns_last_iterate(solver):
    sys = meshgen.hex_laplacian(8, 8, 8)
    b = meshgen.rhs_hot_face(8, 8, 8)
    st, x, it, res = _solver(solver)(sys, b, tol=1e-10, maxIter=5)
    assert st == oracle.NOT_CONVERGED and it == 5 and res > 1e-10
    r = b - sys.dense() @ x
    assert abs(np.linalg.norm(r) / np.linalg.norm(b) - res) < 1e-8


def test_openfoam_norm_factor():
    """Reading Z1 option: with x0 = 0, normFactor = sum|b| + 1e-20, so res0 = 1 (to 1e-15) and
    the final residual equals sum|b - A x| / sum|b| recomputed with numpy."""
    sys = meshgen.hex_laplacian(6, 5, 4)
    b = meshgen.rhs_random(sys.nCells, seed=4)
    st, x, it, res, h = oracle.pcg(sys, b, tol=1e-6, norm=oracle.NORM_OPENFOAM, history=True)
    assert st == oracle.OK
    assert abs(h[0] - 1.0) < 1e-14
    r = b - sys.dense() @ x
    assert abs(np.abs(r).sum() / np.abs(b).sum() - res) < 1e-8 * max(res, 1e-12) + 1e-12


@pytest.mark.parametrize("solver", ["pcg", "pipecg_j", "pipecg_l"])
def test_openfoam_norm_factor_warm_start_golden(solver):
    """Reading Z1 OpenFOAM normFactor with x0 != 0 against the hand-computed 3-cell example of
    tests/golden/spec_examples.txt (of_norm_3cell): res0 = 7/11 exactly as printed there; both
    xbar*sumA terms, the mean (not the sum) of x0 and the sign of r0 all enter it."""
    ex = load_spec_examples()["of_norm_3cell"]
    sys = meshgen.LduSystem(nCells=ex["n"], lowerAddr=ex["l"], upperAddr=ex["u"],
                            diag=ex["diag"], upper=ex["upper"])
    x0 = np.array([float(v) for v in ex["expected"]["x0"].split(",")])
    res0 = float(ex["expected"]["res0"])
    nf = float(ex["expected"]["normFactor"])
    kw = dict(tol=1e-12, maxIter=50, norm=oracle.NORM_OPENFOAM, history=True)
    if solver == "pcg":
        st, x, it, res, h = oracle.pcg(sys, ex["vec"], x0=x0, **kw)
    else:
        mode = oracle.JACOBI if solver == "pipecg_j" else oracle.LITERAL
        st, x, it, res, h = oracle.pipecg(sys, ex["vec"], x0=x0, mode=mode, **kw)
    assert st == oracle.OK
    assert abs(h[0] - res0) <= 1e-15
    # the final criterion is sum|b - A x| / normFactor, normFactor fixed at the x0 value (11)
    r = ex["vec"] - sys.dense() @ x
    assert abs(np.abs(r).sum() / nf - res) <= 1e-10
    assert it <= 3  # n = 3: exact termination in <= n steps


@pytest.mark.slow
def test_table2_iteration_ratio():
    """Table 2: absolute counts are unpinned (RHS/criterion unknown), but the
    128^3/64^3 ratio is ~2 for every row (1.89-2.01); Jacobi-PCG on the FV Dirichlet cube with a
    hot-face RHS at rel-L2 1e-8 must land in [1.8, 2.1]."""
    rows = load_table2()
    paper = [b / a for a, b, _ in rows.values()]
    assert all(1.8 < r < 2.1 for r in paper)
    its = []
    for n in (64, 128):
        sys = meshgen.hex_laplacian(n, n, n)
        st, x, it, res = oracle.pcg(sys, meshgen.rhs_hot_face(n, n, n), tol=1e-8, maxIter=5000)
        assert st == oracle.OK
        its.append(it)
    assert 1.8 <= its[1] / its[0] <= 2.1, its


@pytest.mark.parametrize("solver", ["pcg", "pipecg_j"])
def test_reltol_and_miniter(solver):
    """OpenFOAM relTol / minIter (reading Z26): the solve stops at the FIRST iteration i >= minIter
    whose criterion value is below tol or below relTol * res0 -- checked against the residual
    history of an unstopped run (tol = 0), and minIter forces iterations past convergence."""
    sys = meshgen.cavity_pressure_2d(24, 20)
    b = meshgen.cavity_rhs(24, 20, 1)
    f = _solver(solver)
    _, _, _, _, h = f(sys, b, tol=0.0, maxIter=200, history=True)
    for relTol in (0.5, 0.05, 1e-3):
        first = int(np.argmax(h < relTol * h[0]))
        st, x, it, res = f(sys, b, tol=1e-14, maxIter=200, relTol=relTol)
        assert st == oracle.OK and it == first and res == h[first]
    # minIter: a huge tol passes at iteration 0 unless minIter forces more iterations
    st, x, it, res = f(sys, b, tol=1e300, maxIter=200)
    assert st == oracle.OK and it == 0
    st, x, it, res = f(sys, b, tol=1e300, maxIter=200, minIter=7)
    _, x7, it7, _ = f(sys, b, tol=0.0, maxIter=7)
    assert st == oracle.OK and it == 7 and np.array_equal(x, x7)


# ---- residual replacement in pipelined CG (NEXT-4) ------------------------------------------------
def _true_res(s, b, x):
    return np.linalg.norm(b - oracle.amul(s, x)) / np.linalg.norm(b)


def test_pipecg_replacement_identical_until_first_replacement():
    s = meshgen.hex_laplacian(20, 20, 20, dirichlet=dict(x0=1.0))
    _, _, _, _, h0 = oracle.pipecg(s, s.b, tol=0.0, maxIter=40, history=True)
    _, _, _, _, h1 = oracle.pipecg(s, s.b, tol=0.0, maxIter=40, history=True, replace_every=25)
    np.testing.assert_array_equal(h0[:25], h1[:25])  # residuals 0..24: the first replacement follows update 24
    assert np.allclose(h0[25:], h1[25:], rtol=1e-6)   # equal in exact arithmetic


def test_pipecg_replacement_restores_attainable_accuracy():
    """Plain Ghysels-Vanroose CG drifts: at 64^3 its true residual stalls above tol and at
    tol 1e-14 the recurrences break down; with the residual recomputed every 50 iterations the
    TRUE residual meets the tolerance in classical CG's iteration count (the methods coincide in
    exact arithmetic)."""
    s = meshgen.hex_laplacian(64, 64, 64, dirichlet=dict(x0=1.0))
    b = s.b
    st, x, it, res = oracle.pipecg(s, b, tol=1e-12, maxIter=3000)
    assert st == oracle.OK and _true_res(s, b, x) > 2e-12            # recurrence says < 1e-12
    st, x, it, res = oracle.pipecg(s, b, tol=1e-12, maxIter=3000, replace_every=50)
    assert st == oracle.OK and _true_res(s, b, x) < 1e-12
    _, _, it_cg, _ = oracle.pcg(s, b, tol=1e-14, maxIter=3000)
    st0, _, _, _ = oracle.pipecg(s, b, tol=1e-14, maxIter=3000)
    assert st0 == oracle.BREAKDOWN
    st, x, it, res = oracle.pipecg(s, b, tol=1e-14, maxIter=3000, replace_every=50)
    assert st == oracle.OK and abs(it - it_cg) <= 2 and _true_res(s, b, x) < 1.1e-14
