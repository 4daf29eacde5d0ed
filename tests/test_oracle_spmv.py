"""Pins for oracle.amul (SpMV) against things other than itself:
worked examples, a dense numpy mat-vec of the plain matrix definition, the symmetry
identity, exact row sums, closed-form eigenpairs of the ghost-h Laplacian."""
import numpy as np
import pytest

import meshgen
import oracle
from conftest import load_spec_examples


def _sys_from_example(ex):
    return meshgen.LduSystem(ex["n"], ex["l"], ex["u"], ex["diag"], ex["upper"])


@pytest.mark.parametrize("name", ["spmv_identity", "spmv_1d_laplacian"])
def test_spec_examples(name):
    ex = load_spec_examples()[name]
    y = oracle.amul(_sys_from_example(ex), ex["vec"])
    np.testing.assert_array_equal(y, np.array([float(v) for v in ex["expected"]["y"].split(",")]))


def _dense_from_definition(sys):
    """A[c,c] = diag; A[l,u] = upper; A[u,l] = lower, built entry by entry."""
    n = sys.nCells
    A = np.zeros((n, n))
    lo = sys.upper if sys.lower is None else sys.lower
    for c in range(n):
        A[c, c] += sys.diag[c]
    for f in range(sys.nFaces):
        A[sys.lowerAddr[f], sys.upperAddr[f]] += sys.upper[f]
        A[sys.upperAddr[f], sys.lowerAddr[f]] += lo[f]
    return A


SMALL = [
    meshgen.hex_laplacian(4, 3, 5),
    meshgen.hex_laplacian(4, 3, 5, bc="ghost"),
    meshgen.hex_laplacian(1, 1, 1),
    meshgen.hex_laplacian(2, 2, 2, conductance_sigma=0.5, seed=3),
    meshgen.hex_laplacian(5, 1, 1, ddt=0.25),
    meshgen.cavity_pressure_2d(6, 5),
    meshgen.random_ldu(64, seed=1),
    meshgen.random_ldu(40, seed=2, symmetric=False),
    meshgen.random_ldu(33, seed=3, sort_faces=False),
    meshgen.random_ldu(17, seed=4, symmetric=False, sort_faces=False, density=0.4),
]


@pytest.mark.parametrize("k", range(len(SMALL)))
def test_dense_matvec(k):
    sys = SMALL[k]
    x = np.random.default_rng(100 + k).uniform(-1, 1, sys.nCells)
    ref = _dense_from_definition(sys) @ x
    y = oracle.amul(sys, x)
    assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("k", [0, 1, 3, 5, 6, 8])
def test_symmetry_identity(k):
    sys = SMALL[k]
    rng = np.random.default_rng(7 + k)
    x, z = rng.uniform(-1, 1, (2, sys.nCells))
    a = x @ oracle.amul(sys, z)
    b = z @ oracle.amul(sys, x)
    assert abs(a - b) <= 1e-10 * max(abs(a), 1.0)


@pytest.mark.parametrize("nx,ny,nz", [(4, 3, 5), (7, 7, 7), (1, 1, 6)])
def test_row_sums_exact(nx, ny, nz):
    """A * 1 = 0 on interior rows, 2 * (#Dirichlet walls) on wall rows (FV, reading Z11): exact."""
    sys = meshgen.hex_laplacian(nx, ny, nz)
    y = oracle.amul(sys, np.ones(sys.nCells))
    c = np.arange(sys.nCells)
    i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
    walls = (i == 0).astype(int) + (i == nx - 1) + (j == 0) + (j == ny - 1) + (k == 0) + (k == nz - 1)
    np.testing.assert_array_equal(y, 2.0 * walls)


def ghost_eigpair(nx, ny, nz, kx, ky, kz):
    """Ghost-h 7-point Laplacian (diag 6, off -1) is a Kronecker sum of 1-D tridiag(-1, 2, -1)
    chains: v = prod_d sin(pi k_d (i_d+1)/(n_d+1)), lambda = sum_d 2 (1 - cos(pi k_d/(n_d+1)))."""
    c = np.arange(nx * ny * nz)
    i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
    v = (np.sin(np.pi * kx * (i + 1) / (nx + 1)) * np.sin(np.pi * ky * (j + 1) / (ny + 1))
         * np.sin(np.pi * kz * (k + 1) / (nz + 1)))
    lam = sum(2.0 * (1 - np.cos(np.pi * kk / (n + 1))) for kk, n in ((kx, nx), (ky, ny), (kz, nz)))
    return v, lam


@pytest.mark.parametrize("k", [(1, 1, 1), (2, 3, 1), (5, 4, 6), (6, 5, 7)])
def test_ghost_eigenvectors(k):
    nx, ny, nz = 6, 5, 7
    sys = meshgen.hex_laplacian(nx, ny, nz, bc="ghost")
    v, lam = ghost_eigpair(nx, ny, nz, *k)
    y = oracle.amul(sys, v)
    assert np.abs(y - lam * v).max() <= 1e-13 * 12


def test_face_loop_equals_row_order_bitwise():
    """Summing diag first, then the row's entries in ascending column order, reproduces the
    face loop bit for bit for upper-triangular-ordered faces (SURVEY App. B check 1); this is
    the order the GPU row-gathered layout uses."""
    sys = meshgen.hex_laplacian(5, 4, 3, conductance_sigma=1.0, seed=11)
    x = np.random.default_rng(5).uniform(-1, 1, sys.nCells)
    y = oracle.amul(sys, x)
    rows = [[] for _ in range(sys.nCells)]
    for f in range(sys.nFaces):
        rows[sys.upperAddr[f]].append((int(sys.lowerAddr[f]), sys.upper[f]))
        rows[sys.lowerAddr[f]].append((int(sys.upperAddr[f]), sys.upper[f]))
    y2 = np.empty(sys.nCells)
    for c in range(sys.nCells):
        s = sys.diag[c] * x[c]
        for col, a in sorted(rows[c]):
            s = s + a * x[col]
        y2[c] = s
    np.testing.assert_array_equal(y, y2)
