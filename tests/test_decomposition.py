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


# ---- functional performance model (FuPerMod, the paper's reference for Eq 5; NEXT-3) -----------
def test_fpm_single_point_is_eq5_to_eq8():
    """One measurement per device (a = 0): the FPM partition is exactly Eq 5-8."""
    ns = [250_000, 250_000, 250_000, 250_000]
    Ts = [0.004, 0.001, 0.002, 0.0013]
    models = [meshgen.fit_time_model([n], [T]) for n, T in zip(ns, Ts)]
    assert all(a == 0.0 for a, _ in models)
    fp = meshgen.fpm_partition(1_000_000, models)
    eq8 = meshgen.rebalance(1_000_000, meshgen.relative_speeds(
        [meshgen.speed(n, 0, T) for n, T in zip(ns, Ts)]))
    np.testing.assert_array_equal(fp, eq8)


def test_fpm_equalises_affine_devices_where_eq8_overshoots():
    """Devices with a fixed per-iteration cost (T_i(n) = a_i + b_i n): Eq 5-8 from one
    measurement leaves the times unequal (the one-shot re-decomposition over-corrects, as
    measured in r01); the model fitted from two measurements equalises them up to rounding."""
    a = np.array([20e-6, 15e-6, 15e-6, 15e-6])
    b = np.array([25e-12, 14e-12, 14e-12, 14e-12])
    T = lambda n: a + b * n  # noqa: E731
    N = 4_096_000
    n0 = meshgen.slab_bounds(N, 4)
    n0 = np.diff(n0)
    eq8 = meshgen.rebalance(N, meshgen.relative_speeds(n0 / T(n0)))
    t8 = T(eq8)
    models = [meshgen.fit_time_model([n0[i], eq8[i]], [T(n0)[i], t8[i]]) for i in range(4)]
    for (ai, bi), at, bt in zip(models, a, b):
        assert abs(ai - at) <= 1e-12 and abs(bi - bt) <= 1e-18
    fp = meshgen.fpm_partition(N, models)
    tf = T(fp)
    assert fp.sum() == N
    assert tf.max() / tf.min() < 1 + 1e-5          # equal up to the rounding of cells
    assert t8.max() / t8.min() > 1.05              # Eq 8 alone: several % apart
    assert tf.max() < t8.max()                     # so the step time improves


def test_fpm_min_cells_clamp():
    models = [(1.0, 1e-6), (0.0, 1e-6), (0.0, 1e-6)]  # device 0: a fixed cost above the balance
    n = meshgen.fpm_partition(1000, models, min_cells=5)
    assert n.sum() == 1000 and n[0] == 5 and abs(int(n[1]) - int(n[2])) <= 1
