"""Heterogeneous decomposition, Eq 5-8.  Pins: SPEC acceptance criterion 6
worked values, exact sum over random fraction vectors (Eq 7), weighted slabs reproduce
the global SpMV, nnz balancing on an irregular mesh."""
import numpy as np
import pytest

import meshgen
import oracle


def test_eq5_to_eq8_worked_values():
    # SPEC acceptance 6: measure_speed(100,300,0.7)=1000; relative_speeds(2,6)=(0.25,0.75);
    # rebalance_cells(1000,(0.25,0.75))=(250,750)
    assert meshgen.speed(100, 300, 0.7) == pytest.approx(1000.0, rel=1e-15)
    np.testing.assert_array_equal(meshgen.relative_speeds([2, 6]), [0.25, 0.75])
    np.testing.assert_array_equal(meshgen.rebalance(1000, [0.25, 0.75]), [250, 750])


def test_rebalance_sums_to_N():
    rng = np.random.default_rng(0)
    for _ in range(1000):
        p = rng.integers(1, 12)
        r = rng.random(p)
        r /= r.sum()
        N = int(rng.integers(p, 10 ** 6))
        n = meshgen.rebalance(N, r)
        assert n.sum() == N and np.all(n >= 0)
        assert np.all(np.abs(n - N * r) < 1.0 + 1e-9)


def test_speed_factors_4_to_1():
    """Two devices with speed factors (4, 1) on a 1M-cell slab (P:174 setting): Eq 8 assigns
    80% / 20% of the cells."""
    s = [meshgen.speed(500_000, 1_500_000, 1.0 / 4), meshgen.speed(500_000, 1_500_000, 1.0)]
    n = meshgen.rebalance(1_000_000, meshgen.relative_speeds(s))
    np.testing.assert_array_equal(n, [800_000, 200_000])


@pytest.mark.parametrize("fr", [[0.7, 0.3], [0.1, 0.2, 0.3, 0.4]])
def test_weighted_slabs_reconstruct_spmv(fr):
    sys = meshgen.hex_laplacian(7, 6, 10, conductance_sigma=0.5, seed=1)
    bounds = meshgen.slab_bounds_weighted(sys.nCells, fr)
    parts = meshgen.slab_partition(sys, len(fr), bounds=bounds)
    assert [q.nCells for q in parts] == list(meshgen.rebalance(sys.nCells, fr))
    x = np.random.default_rng(3).uniform(-1, 1, sys.nCells)
    y = np.concatenate(oracle.dist_amul(parts, [x[bounds[g]:bounds[g + 1]] for g in range(len(fr))]))
    ref = oracle.amul(sys, x)
    assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref)


def test_nnz_balanced_bounds():
    sys = meshgen.irregular_mesh(12, seed=2)
    p = 4
    b = meshgen.nnz_balanced_bounds(sys, p)
    N = sys.nCells
    w = 1 + np.bincount(sys.lowerAddr, minlength=N) + np.bincount(sys.upperAddr, minlength=N)
    loads = np.array([w[b[g]:b[g + 1]].sum() for g in range(p)])
    assert b[0] == 0 and b[-1] == N and np.all(np.diff(b) > 0)
    assert loads.max() - loads.min() <= 2 * w.max()
