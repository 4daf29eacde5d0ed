"""Input generators (structure the paper and SPEC fix) and the slab decomposition
(reconstruction invariants S:198-204, message counts S:359-361), checked with the oracle's
serial halo emulation and with dense numpy algebra."""
import numpy as np
import pytest

import meshgen
import oracle


def test_single_cell_examples():
    """1x1x1, unit spacing, zero Dirichlet -> A = [6] (ghost-h); the FV half-cell
    convention doubles the wall coefficient -> [12]."""
    g = meshgen.hex_laplacian(1, 1, 1, bc="ghost")
    assert g.nFaces == 0 and g.diag.tolist() == [6.0] and not np.any(g.b)
    f = meshgen.hex_laplacian(1, 1, 1)
    assert f.diag.tolist() == [12.0]


def test_2cube_ghost():
    """2x2x2 -> every diagonal 6, every row exactly 3 off-diagonals of -1."""
    s = meshgen.hex_laplacian(2, 2, 2, bc="ghost")
    A = s.dense()
    assert np.all(np.diag(A) == 6.0)
    off = A - np.diag(np.diag(A))
    assert np.all((off != 0).sum(1) == 3) and set(np.unique(off)) == {-1.0, 0.0}


@pytest.mark.parametrize("nx,ny,nz", [(4, 4, 4), (5, 3, 2), (16, 16, 16), (1, 7, 3)])
def test_hex_structure(nx, ny, nz):
    s = meshgen.hex_laplacian(nx, ny, nz)
    N = nx * ny * nz
    assert s.nFaces == (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1)
    # upper-triangular order: sorted by owner then neighbour, l < u
    assert np.all(s.lowerAddr < s.upperAddr)
    key = s.lowerAddr.astype(np.int64) * N + s.upperAddr
    assert np.all(np.diff(key) > 0)
    # row nnz = 7 - #boundary faces, symmetric, weakly diagonally dominant (strict on walls)
    deg = np.bincount(s.lowerAddr, minlength=N) + np.bincount(s.upperAddr, minlength=N)
    c = np.arange(N)
    i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
    walls = (i == 0).astype(int) + (i == nx - 1) + (j == 0) + (j == ny - 1) + (k == 0) + (k == nz - 1)
    assert np.all(deg + 1 == 7 - walls)
    offsum = np.bincount(s.lowerAddr, weights=-s.upper, minlength=N) + \
        np.bincount(s.upperAddr, weights=-s.upper, minlength=N)
    np.testing.assert_array_equal(s.diag - offsum, 2.0 * walls)


def test_cavity_matrix():
    """Config 2: symmetric, SPD after setReference (Cholesky succeeds), zero-mean sources."""
    s = meshgen.cavity_pressure_2d(10, 8)
    A = s.dense()
    assert np.array_equal(A, A.T)
    np.linalg.cholesky(A)
    for t in range(3):
        f = meshgen.cavity_rhs(10, 8, t)
        assert abs(f.sum()) < 1e-12


def test_irregular_mesh():
    s = meshgen.irregular_mesh(10, seed=3)
    N = s.nCells
    deg = np.bincount(s.lowerAddr, minlength=N) + np.bincount(s.upperAddr, minlength=N)
    assert deg.min() >= 2 and deg.max() <= 10
    assert np.all(s.lowerAddr < s.upperAddr)
    key = s.lowerAddr.astype(np.int64) * N + s.upperAddr
    assert np.all(np.diff(key) > 0)
    np.linalg.cholesky(s.dense())


DIST_CASES = [
    ("hex8", lambda: meshgen.hex_laplacian(8, 8, 8, dirichlet=dict(x0=1.0))),
    ("hex_sigma", lambda: meshgen.hex_laplacian(6, 5, 8, conductance_sigma=1.0, seed=2)),
    ("random", lambda: meshgen.random_ldu(64, seed=8)),
    ("random_nonsym", lambda: meshgen.random_ldu(50, seed=9, symmetric=False)),
    ("irregular", lambda: meshgen.irregular_mesh(8, seed=4)),
]


@pytest.mark.parametrize("p", [1, 2, 4, 8])
@pytest.mark.parametrize("case", range(len(DIST_CASES)))
def test_distributed_spmv_reconstruction(case, p):
    """S:201 / S:587: slab-partitioned SpMV (local LDU + interfaces + halo) equals the global
    SpMV to 1e-12; per-call message count = 2 x adjacent slab pairs."""
    sys = DIST_CASES[case][1]()
    parts = meshgen.slab_partition(sys, p)
    x = np.random.default_rng(case).uniform(-1, 1, sys.nCells)
    bounds = meshgen.slab_bounds(sys.nCells, p)
    xs = [x[bounds[g]:bounds[g + 1]] for g in range(p)]
    y = np.concatenate(oracle.dist_amul(parts, xs))
    ref = sys.dense() @ x
    assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref)
    pairs = {(g, itf.neighbRank) for g, part in enumerate(parts) for itf in part.interfaces}
    adjacent = {tuple(sorted(pr)) for pr in pairs}
    assert len(pairs) == 2 * len(adjacent)
    if p == 1:
        assert not parts[0].interfaces
    # interface pairing is consistent: equal lengths both ways
    for g, part in enumerate(parts):
        for itf in part.interfaces:
            back = [t for t in parts[itf.neighbRank].interfaces if t.neighbRank == g]
            assert len(back) == 1 and len(back[0].faceCells) == len(itf.faceCells)


def test_two_cell_chain():
    """S:202-203 / S:360: a 2-cell chain split in 2 -> each local block is [diag] with one
    coupling entry; one message each way; result matches the global SpMV."""
    s = meshgen.LduSystem(2, np.array([0], np.int32), np.array([1], np.int32),
                          np.array([2.0, 3.0]), np.array([-1.0]))
    parts = meshgen.slab_partition(s, 2)
    for part in parts:
        assert part.nCells == 1 and part.nFaces == 0 and len(part.interfaces) == 1
        assert part.interfaces[0].coeffs.tolist() == [1.0]
    ys = oracle.dist_amul(parts, [np.array([1.0]), np.array([2.0])])
    np.testing.assert_array_equal(np.concatenate(ys), [0.0, 5.0])


def test_reconstruction_dense():
    """Reassembling every part's local block plus its interface couplings reproduces A exactly."""
    sys = meshgen.random_ldu(40, seed=12, symmetric=False)
    p = 3
    parts = meshgen.slab_partition(sys, p)
    bounds = meshgen.slab_bounds(sys.nCells, p)
    A = np.zeros((sys.nCells, sys.nCells))
    for g, part in enumerate(parts):
        lo = bounds[g]
        A[lo:lo + part.nCells, lo:lo + part.nCells] += part.dense()
        for itf in part.interfaces:
            h = itf.neighbRank
            back = [t for t in parts[h].interfaces if t.neighbRank == g][0]
            A[lo + itf.faceCells, bounds[h] + back.faceCells] += -itf.coeffs
    np.testing.assert_array_equal(A, sys.dense())


@pytest.mark.parametrize("p", [1, 2, 4])
def test_direct_slab_equals_partition(p):
    kw = dict(dirichlet=dict(x0=1.0, z1=0.5))
    a = meshgen.slab_partition(meshgen.hex_laplacian(5, 4, 8, **kw), p)
    b = [meshgen.hex_laplacian_slab(5, 4, 8, p, g, **kw) for g in range(p)]
    for x, y in zip(a, b):
        for f in ("lowerAddr", "upperAddr", "diag", "upper", "b"):
            np.testing.assert_array_equal(getattr(x, f), getattr(y, f))
        assert len(x.interfaces) == len(y.interfaces)
        for i, j in zip(x.interfaces, y.interfaces):
            assert i.neighbRank == j.neighbRank
            np.testing.assert_array_equal(i.faceCells, j.faceCells)
            np.testing.assert_array_equal(i.coeffs, j.coeffs)
