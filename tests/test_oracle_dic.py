"""Pins of the oracle's DIC preconditioner (readings Z35, Z36).

The oracle follows OpenFOAM's DICPreconditioner face loops (oracle/ldu_oracle.c).  These checks
hold it against what the mathematics fixes, not against a retyped copy of the loops:
  - the defining property of DIC: M = (D + L) D^-1 (D + L^T) has diag(M) = diag(A) (assembled
    densely here from the oracle's rD alone); on a triangle-free cell graph (hex meshes) DIC is
    IC(0), so M also equals A on A's whole off-diagonal pattern (reading Z35);
  - on a tridiagonal matrix there is no fill, so DIC is the exact Cholesky factorisation: D is
    the squared diagonal of numpy's Cholesky factor and DIC-PCG converges in one iteration;
  - the preconditioner apply solves M w = r (dense check);
  - DIC-PCG solutions against a dense direct solve, fewer iterations than Jacobi-PCG;
  - unsorted / swapped / duplicated faces give the same operator (reading Z36);
  - the block form equals DIC of block-diag(A) (reading Z33 applied to DIC).
"""
import numpy as np
import pytest

import meshgen
import oracle
from oracle import amg


def dense(sys):
    return amg.csr_of_ldu(sys).toarray()


def dic_M(A, rD):
    D = np.diag(1.0 / rD)
    L = np.tril(A, -1)
    return (D + L) @ np.diag(rD) @ (D + L.T)


def systems():
    yield "hex5x4x3", meshgen.hex_laplacian(5, 4, 3)
    yield "hex_cavity2d", meshgen.cavity_pressure_2d(9, 7)
    yield "irregular6", meshgen.irregular_mesh(6, seed=3)
    yield "random40", meshgen.random_ldu(40, seed=7, density=0.2)
    yield "random40_unsorted", meshgen.random_ldu(40, seed=8, density=0.2, sort_faces=False)


@pytest.mark.parametrize("name,sys", list(systems()), ids=lambda v: v if isinstance(v, str) else "")
def test_dic_matches_A_on_pattern(name, sys):
    A = dense(sys)
    st, rD, _ = oracle.dic(sys)
    assert st == oracle.OK
    assert np.all(rD > 0)
    M = dic_M(A, rD)
    scale = np.abs(A).max()
    assert np.max(np.abs(np.diag(M) - np.diag(A))) <= 1e-13 * scale
    G = (A != 0) & ~np.eye(A.shape[0], dtype=bool)
    Gi = G.astype(np.int64)
    triangle_free = not np.any((Gi @ Gi)[G])
    assert triangle_free == name.startswith("hex")
    if triangle_free:  # IC(0): every entry of A's pattern reproduced
        pat = G | np.eye(A.shape[0], dtype=bool)
        assert np.max(np.abs((M - A)[pat])) <= 1e-13 * scale
    # fill-in outside the pattern (M != A) unless the graph is a forest
    assert np.max(np.abs(M - A)) > 1e-6 * scale


@pytest.mark.parametrize("name,sys", list(systems()), ids=lambda v: v if isinstance(v, str) else "")
def test_dic_apply_solves_M(name, sys):
    A = dense(sys)
    r = meshgen.rhs_random(sys.nCells, seed=11)
    st, rD, w = oracle.dic(sys, r)
    assert st == oracle.OK
    M = dic_M(A, rD)
    assert np.linalg.norm(M @ w - r) <= 1e-13 * np.linalg.norm(r) * np.linalg.cond(M)


def test_dic_tridiagonal_is_cholesky():
    sys = meshgen.hex_laplacian(17, 1, 1)  # 1-D chain: tridiagonal, no fill
    A = dense(sys)
    st, rD, _ = oracle.dic(sys)
    Lc = np.linalg.cholesky(A)
    np.testing.assert_allclose(1.0 / rD, np.diag(Lc) ** 2, rtol=1e-14)
    b = meshgen.rhs_random(sys.nCells, seed=5)
    for pipelined in (False, True):
        st, x, it, res = oracle.dic_pcg(sys, b, tol=1e-12, maxIter=50, pipelined=pipelined)
        assert st == oracle.OK and it == 1, (pipelined, st, it, res)
        np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-12, atol=1e-14)


def test_dic_duplicate_and_swapped_faces():
    sys = meshgen.hex_laplacian(4, 3, 3)
    rng = np.random.default_rng(2)
    nf = sys.lowerAddr.shape[0]
    perm = rng.permutation(nf)
    l, u, a = sys.lowerAddr[perm].copy(), sys.upperAddr[perm].copy(), sys.upper[perm].copy()
    sw = rng.random(nf) < 0.5
    l[sw], u[sw] = u[sw], l[sw].copy()
    # split every third face into two halves (duplicates are summed, reading Z36)
    dup = np.arange(0, nf, 3)
    l2 = np.concatenate([l, l[dup]]).astype(np.int32)
    u2 = np.concatenate([u, u[dup]]).astype(np.int32)
    a2 = np.concatenate([a, a[dup] * 0.5])
    a2[dup] *= 0.5
    s2 = meshgen.LduSystem(sys.nCells, l2, u2, sys.diag.copy(), a2, None, sys.b)
    np.testing.assert_allclose(dense(s2), dense(sys), rtol=1e-15, atol=1e-15)
    _, rD1, _ = oracle.dic(sys)
    _, rD2, _ = oracle.dic(s2)
    np.testing.assert_allclose(rD2, rD1, rtol=1e-14)


@pytest.mark.parametrize("n", [8, 12])
def test_dic_pcg_solution_and_iterations(n):
    sys = meshgen.hex_laplacian(n, n, n)
    b = meshgen.rhs_hot_face(n, n, n)
    xd = np.linalg.solve(dense(sys), b)
    st, x, it, res = oracle.dic_pcg(sys, b, tol=1e-12, maxIter=2000)
    assert st == oracle.OK
    assert np.linalg.norm(x - xd) <= 1e-9 * np.linalg.norm(xd)
    _, _, itj, _ = oracle.pcg(sys, b, tol=1e-12, maxIter=2000)
    assert it < itj, (it, itj)
    # pipelined DIC-CG: same iterates in exact arithmetic -> residual histories agree early on
    st2, x2, it2, _, h2 = oracle.dic_pcg(sys, b, tol=1e-12, maxIter=2000, pipelined=True,
                                         history=True)
    _, _, _, _, h1 = oracle.dic_pcg(sys, b, tol=1e-12, maxIter=2000, history=True)
    assert st2 == oracle.OK and abs(it2 - it) <= max(1, it // 50)
    np.testing.assert_allclose(h2[:10], h1[:10], rtol=1e-7)
    assert np.linalg.norm(x2 - xd) <= 1e-9 * np.linalg.norm(xd)


def test_dic_block_form_is_dic_of_block_diagonal():
    sys = meshgen.irregular_mesh(6, seed=4)
    n = sys.nCells
    bounds = np.array([0, n // 3, (2 * n) // 3, n], dtype=np.int32)
    A = dense(sys)
    Ab = np.zeros_like(A)
    for g in range(3):
        s, e = bounds[g], bounds[g + 1]
        Ab[s:e, s:e] = A[s:e, s:e]
    st, rD, _ = oracle.dic(sys, bounds=bounds)
    M = dic_M(Ab, rD)
    assert np.max(np.abs(np.diag(M) - np.diag(A))) <= 1e-13 * np.abs(A).max()
    # block-diagonal preconditioner: no coupling between blocks
    assert np.all(M[: bounds[1], bounds[1]:] == 0)
    b = meshgen.rhs_random(n, seed=9)
    st, x, it, _ = oracle.dic_pcg(sys, b, tol=1e-11, maxIter=500, bounds=bounds)
    assert st == oracle.OK
    xd = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xd) <= 1e-8 * np.linalg.norm(xd)


def test_dic_zero_rhs_and_nonpositive_pivot():
    sys = meshgen.hex_laplacian(4, 4, 4)
    st, x, it, res = oracle.dic_pcg(sys, np.zeros(sys.nCells), tol=1e-10, maxIter=10)
    assert st == oracle.OK and it == 0 and not x.any()
    bad = meshgen.LduSystem(2, np.array([0], np.int32), np.array([1], np.int32),
                            np.array([1.0, 1.0]), np.array([-2.0]), None, np.ones(2))
    st, _, _ = oracle.dic(bad)
    assert st == oracle.BREAKDOWN


@pytest.mark.parametrize("p", [2, 3])
def test_dic_block_form_equals_per_rank_local_factors(p):
    """The multi-rank reading (Z33 applied to DIC): the block form over the slab bounds is the DIC
    of each rank's LOCAL matrix, as meshgen.slab_partition hands it to ldu_setup."""
    g = meshgen.hex_laplacian(7, 6, 9, conductance_sigma=0.4, seed=2)
    parts = meshgen.slab_partition(g, p)
    bounds = meshgen.slab_bounds(g.nCells, p)
    r = meshgen.rhs_random(g.nCells, seed=3)
    _, rD, w = oracle.dic(g, r, bounds=bounds)
    for k, part in enumerate(parts):
        lo, hi = int(bounds[k]), int(bounds[k + 1])
        _, rDk, wk = oracle.dic(part, r[lo:hi])
        np.testing.assert_allclose(rD[lo:hi], rDk, rtol=1e-14)
        np.testing.assert_allclose(w[lo:hi], wk, rtol=1e-12, atol=1e-14)
