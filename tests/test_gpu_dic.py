"""Parity of the device DIC preconditioner and DIC-CG / DIC-PipeCG (readings
Z35-Z36) with the oracle (oracle.dic / oracle.dic_pcg), through the C ABI.

  * factor 1/D                      ~ oracle.dic rD                    (rel 1e-12 per cell);
  * level count on a lexicographic hex mesh = nx + ny + nz - 2 (the i+j+k wavefronts);
  * z = M^-1 r                      ~ oracle.dic w                     (rel-L2 1e-12);
  * solves: iteration counts within +-2% (+-1), solution rel-L2 <= 1e-8 at tol 1e-10.
"""
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


CASES = {
    "hex16": lambda: meshgen.hex_laplacian(16, 16, 16),
    "hex_ragged": lambda: meshgen.hex_laplacian(23, 17, 11, conductance_sigma=0.5, seed=3),
    "chain": lambda: meshgen.hex_laplacian(300, 1, 1),
    "cavity": lambda: meshgen.cavity_pressure_2d(96, 80),
    "irregular": lambda: meshgen.irregular_mesh(14, seed=4),
    "random_unsorted": lambda: meshgen.random_ldu(400, seed=5, density=0.02, sort_faces=False),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_dic_factor_and_apply(ldu, case):
    sys_ = CASES[case]()
    n = sys_.nCells
    st, rD_o, _ = oracle.dic(sys_)
    assert st == oracle.OK
    r = meshgen.rhs_random(n, seed=21)
    _, _, w_o = oracle.dic(sys_, r)
    with ldu.LduMatrix.from_system(sys_) as A:
        info = A.dic_setup()
        assert info["nLevels"] >= 1 and info["widestLevel"] >= 1
        rD = A.dic_rD(np.empty(n))
        np.testing.assert_allclose(rD, rD_o, rtol=1e-12)
        zt = torch.empty(n, dtype=torch.float64, device="cuda")
        A.dic_apply(cuda(r), zt)
        assert rel(zt.cpu().numpy(), w_o) <= 1e-12
        zh = A.dic_apply(r, np.empty(n))  # host pointers
        assert rel(zh, w_o) <= 1e-12
        if case == "hex_ragged":
            assert info["nLevels"] == 23 + 17 + 11 - 2
        if case == "chain":
            assert info["nLevels"] == 300 and info["widestLevel"] == 1


def star_chain(hubs):
    """40-cell chain plus extra faces {k -> hub}: hub rows with len(ks)+1 lower entries."""
    n = 40
    l = list(range(n - 1))
    u = list(range(1, n))
    for hub, ks in hubs.items():
        l += ks
        u += [hub] * len(ks)
    l, u = np.array(l, np.int32), np.array(u, np.int32)
    a = -np.linspace(0.5, 1.5, l.shape[0])
    diag = np.bincount(l, np.abs(a), n) + np.bincount(u, np.abs(a), n) + 1.0
    return meshgen.LduSystem(n, l, u, diag, a, None, np.ones(n))


@pytest.mark.parametrize("hubs,wlo", [({30: [1, 2, 3, 4]}, 6),            # width 5 -> kernel 6
                                      ({39: [0, 5, 10, 15, 20, 25]}, 8),  # width 7 -> kernel 8
                                      ({39: list(range(0, 32, 4))}, 0)])  # width 9 -> CSR rows
def test_dic_ell_widths(ldu, hubs, wlo):
    sys_ = star_chain(hubs)
    r = meshgen.rhs_random(sys_.nCells, seed=4)
    _, rD_o, w_o = oracle.dic(sys_, r)
    with ldu.LduMatrix.from_system(sys_) as A:
        info = A.dic_setup()
        assert info["ellWidthLower"] == wlo, info
        np.testing.assert_allclose(A.dic_rD(np.empty(sys_.nCells)), rD_o, rtol=1e-12)
        assert rel(A.dic_apply(r, np.empty(sys_.nCells)), w_o) <= 1e-12
        x = np.zeros(sys_.nCells)
        st, it, _ = A.dic_pcg_solve(sys_.b, x, tol=1e-10, maxIter=200)
        ost, ox, oit, _ = oracle.dic_pcg(sys_, sys_.b, tol=1e-10, maxIter=200)
        assert st == ldu.OK and abs(it - oit) <= 1 and rel(x, ox) <= 1e-8


@pytest.mark.parametrize("case", ["hex16", "hex_ragged", "cavity", "irregular"])
@pytest.mark.parametrize("pipelined", [False, True])
def test_dic_solve_parity(ldu, case, pipelined):
    sys_ = CASES[case]()
    n = sys_.nCells
    b = meshgen.rhs_random(n, seed=8)
    ost, ox, oit, ores = oracle.dic_pcg(sys_, b, tol=1e-10, maxIter=5000, pipelined=pipelined)
    assert ost == oracle.OK
    with ldu.LduMatrix.from_system(sys_) as A:
        A.dic_setup()
        fn = A.dic_pipecg_solve if pipelined else A.dic_pcg_solve
        xt = torch.zeros(n, dtype=torch.float64, device="cuda")
        st, it, res = fn(cuda(b), xt, tol=1e-10, maxIter=5000)
        assert st == ldu.OK, (st, it, res)
        assert abs(it - oit) <= max(1, int(0.02 * oit)), (it, oit)
        assert rel(xt.cpu().numpy(), ox) <= 1e-8
        # host buffers, warm start from the solution: converges at once
        x = xt.cpu().numpy()
        st2, it2, _ = fn(b, x, tol=1e-10, maxIter=5000)
        assert st2 == ldu.OK and it2 <= 1


def test_dic_openfoam_criterion_history(ldu):
    sys_ = meshgen.cavity_pressure_2d(64, 64)
    b = meshgen.cavity_rhs(64, 64, 3)
    ost, ox, oit, ores, oh = oracle.dic_pcg(sys_, b, tol=1e-6, relTol=0.05, maxIter=1000,
                                            norm=oracle.NORM_OPENFOAM, history=True)
    with ldu.LduMatrix.from_system(sys_) as A:
        A.dic_setup()
        x = np.zeros(sys_.nCells)
        st, it, res = A.dic_pcg_solve(b, x, tol=1e-6, relTol=0.05, maxIter=1000,
                                      norm=ldu.NORM_OPENFOAM, record_history=True)
        assert st == ost and abs(it - oit) <= 1
        h = A.history()
        m = min(len(h), len(oh))
        np.testing.assert_allclose(h[:m], oh[:m], rtol=1e-8)


def test_dic_fewer_iterations_than_jacobi(ldu):
    sys_ = meshgen.hex_laplacian(32, 32, 32)
    b = meshgen.rhs_hot_face(32, 32, 32)
    with ldu.LduMatrix.from_system(sys_) as A:
        x = np.zeros(sys_.nCells)
        _, itj, _ = A.pcg_solve(b, x, tol=1e-10, maxIter=5000)
        A.dic_setup()
        x = np.zeros(sys_.nCells)
        st, itd, _ = A.dic_pcg_solve(b, x, tol=1e-10, maxIter=5000)
        assert st == ldu.OK and itd < 0.75 * itj, (itd, itj)


def test_dic_errors(ldu):
    sys_ = meshgen.hex_laplacian(6, 5, 4)
    b = np.ones(sys_.nCells)
    with ldu.LduMatrix.from_system(sys_) as A:
        with pytest.raises(ldu.LduError) as e:
            A.dic_pcg_solve(b, np.zeros(sys_.nCells))
        assert e.value.status == ldu.ERR_STATE
        A.amg_setup()
        with pytest.raises(ldu.LduError):
            A.dic_apply(b, np.zeros(sys_.nCells))
        A.dic_setup()  # replaces the hierarchy
        with pytest.raises(ldu.LduError):
            A.amg_info()
        with pytest.raises(ldu.LduError):
            A.amg_pcg_solve(b, np.zeros(sys_.nCells))
    ns = meshgen.random_ldu(50, seed=2, symmetric=False)
    with ldu.LduMatrix.from_system(ns) as A:
        with pytest.raises(ldu.LduError) as e:
            A.dic_setup()
        assert e.value.status == ldu.ERR_INVALID_ARG
