"""Aggregation-AMG preconditioner for the oracle (NEXT-2) -- TEST INFRASTRUCTURE ONLY.

The paper preconditions both CG solvers with CUSP's aggregation AMG (Table 2):
"a V-cycle of an aggregation-based AMG with weighted Jacobi iterations with omega = 4/3 as a
smoother", aggregates from "the parallel aggregation method based on a distance-2
maximal-independent-set".  Readings Z27-Z33 fix the rest:

* Z27  smoothed aggregation: P = (I - w D^-1 A) T, T the piecewise-constant aggregate indicator,
       w = (4/3) / rho, rho = 1.05 x the largest Ritz value of 20 Lanczos steps on
       D^-1/2 A D^-1/2 from the fixed start vector v0_i = mix32(i) / 2^32 - 1/2 (``spectral_radius``;
       CUSP scales the smoother by an estimate of rho(D^-1 A) too; the Gershgorin bound, 2.05 on
       the coarse levels where rho ~ 1.3, damps them too much: 27 / 41 iterations at 64^3 / 128^3
       vs 22 / 28).
* Z28  smoother: one pre- and one post-sweep of x += w D^-1 (f - A x) from x = 0, same w.
* Z29  all couplings strong (no strength threshold).
* Z30  MIS-2 = greedy distance-2 MIS in key order (``oracle_mis2_aggregate`` in ldu_oracle.c).
* Z31  coarsening stops at n <= ``coarsest`` (default 64), when a level does not shrink, or at
       ``max_levels``; the coarsest system is solved exactly (Cholesky factor from numpy).
* Z32  V-cycle as ``vcycle`` in ldu_oracle.c; Galerkin A_{l+1} = P^T A_l P (scipy product).
* Z33  multi-rank: block-Jacobi -- each rank's hierarchy is built from its local matrix only.

Library primitives used as steps (allowed for the oracle): scipy.sparse products for T, P and
P^T A P, numpy's Cholesky for the coarsest factor.  The integer aggregation and every V-cycle /
Krylov operation run in the plain C of ldu_oracle.c.  Pinned by tests/test_oracle_amg.py.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import NORM_L2, _arrays, _load, _p

KEY_INDEX, KEY_HASH = 0, 1


def csr_of_ldu(sys) -> sp.csr_matrix:
    """The full matrix A of an LDU system (A[c,c] = diag, A[l,u] = upper,
    A[u,l] = lower), CSR with ascending columns per row, the diagonal stored."""
    n = sys.nCells
    l = np.asarray(sys.lowerAddr, dtype=np.int64)
    u = np.asarray(sys.upperAddr, dtype=np.int64)
    lo = sys.upper if sys.lower is None else sys.lower
    rows = np.concatenate([np.arange(n), l, u])
    cols = np.concatenate([np.arange(n), u, l])
    vals = np.concatenate([sys.diag, sys.upper, lo]).astype(np.float64)
    A = sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    return A


def _lib():
    lib = _load()
    if not getattr(lib, "_amg_ready", False):
        P, I = ctypes.c_void_p, ctypes.c_int
        D = ctypes.c_double
        lib.oracle_mis2_aggregate.argtypes = [I, P, P, I, P]
        lib.oracle_mis2_aggregate.restype = I
        lib.oracle_amg_vcycle.argtypes = [P, P, P]
        lib.oracle_amg_vcycle.restype = None
        lib.oracle_amg_pcg.argtypes = [I, I, P, P, P, P, P, P, P, D, I, I, P, P, P, D, I, P, I]
        lib.oracle_amg_pcg.restype = I
        lib.oracle_amg_block_vcycle.argtypes = [I, I, P, P, P, P]
        lib.oracle_amg_block_vcycle.restype = I
        lib.oracle_amg_block_pcg.argtypes = [I, I, P, P, P, P, P, P, P, D, I, I, P, P, P, D, I, I,
                                             P, P, I]
        lib.oracle_amg_block_pcg.restype = I
        lib._amg_ready = True
    return lib


def mis2_aggregate(A: sp.csr_matrix, key_mode: int = KEY_HASH):
    """Distance-2 MIS aggregation of A's graph (reading Z30).  Returns (agg[n], nAgg)."""
    A = A.tocsr()
    A.sort_indices()
    n = A.shape[0]
    ptr = np.ascontiguousarray(A.indptr, dtype=np.int32)
    col = np.ascontiguousarray(A.indices, dtype=np.int32)
    agg = np.empty(n, dtype=np.int32)
    na = _lib().oracle_mis2_aggregate(n, _p(ptr), _p(col), key_mode, _p(agg))
    if na < 0:
        raise ValueError("mis2_aggregate: bad arguments")
    return agg, na


LANCZOS_STEPS, RHO_SAFETY = 20, 1.05


def mix32(i) -> np.ndarray:
    """The "lowbias32" integer mixer (shared definition with ldu_oracle.c's amg_key, reading Z30)."""
    m = np.uint64(0xFFFFFFFF)
    h = np.asarray(i, dtype=np.uint64) & m
    h ^= h >> np.uint64(16)
    h = (h * np.uint64(0x7FEB352D)) & m
    h ^= h >> np.uint64(15)
    h = (h * np.uint64(0x846CA68B)) & m
    h ^= h >> np.uint64(16)
    return h


def lanczos_ritz_max(A: sp.csr_matrix, steps: int = LANCZOS_STEPS) -> float:
    """Largest Ritz value of ``steps`` plain Lanczos steps on M = D^-1/2 A D^-1/2 (same spectrum
    as D^-1 A) from v0_i = mix32(i)/2^32 - 1/2, normalised (reading Z27).  Stops early on an
    invariant subspace (beta = 0) or after n steps."""
    n = A.shape[0]
    s = 1.0 / np.sqrt(A.diagonal())
    v = mix32(np.arange(n)).astype(np.float64) / 2.0**32 - 0.5
    v /= np.linalg.norm(v)
    v_prev = np.zeros(n)
    beta = 0.0
    alphas, betas = [], []
    for j in range(min(steps, n)):
        w = s * (A @ (s * v)) - beta * v_prev
        a = float(w @ v)
        w -= a * v
        alphas.append(a)
        beta = float(np.linalg.norm(w))
        if beta == 0.0 or j == min(steps, n) - 1:
            break
        betas.append(beta)
        v_prev, v = v, w / beta
    return float(sla.eigvalsh_tridiagonal(np.array(alphas), np.array(betas)).max())


def spectral_radius(A: sp.csr_matrix) -> float:
    """rho = RHO_SAFETY x lanczos_ritz_max(A) (reading Z27)."""
    return RHO_SAFETY * lanczos_ritz_max(A)


def jacobi_weight(A: sp.csr_matrix) -> float:
    """w = (4/3) / rho(D^-1 A) (readings Z27, Z28; "weighted Jacobi ... omega = 4/3")."""
    return (4.0 / 3.0) / spectral_radius(A)


@dataclass
class Level:
    A: sp.csr_matrix
    agg: np.ndarray
    nAgg: int
    omega: float
    P: sp.csr_matrix
    R: sp.csr_matrix


@dataclass
class Hierarchy:
    levels: List[Level]
    Ac: sp.csr_matrix                 # coarsest matrix
    Lc: np.ndarray                    # its lower Cholesky factor (empty if factor=False)
    _keep: list = field(default_factory=list, repr=False)

    @property
    def sizes(self):
        return [lv.A.shape[0] for lv in self.levels] + [self.Ac.shape[0]]

    def operator_complexity(self) -> float:
        nnz = [lv.A.nnz for lv in self.levels] + [self.Ac.nnz]
        return sum(nnz) / nnz[0]


def prolongator(A: sp.csr_matrix, agg: np.ndarray, nAgg: int, w: float,
                smooth: bool = True) -> sp.csr_matrix:
    """P = (I - w D^-1 A) T (smoothed aggregation, reading Z27) or P = T; T[i, agg[i]] = 1."""
    n = A.shape[0]
    T = sp.csr_matrix((np.ones(n), (np.arange(n), agg)), shape=(n, nAgg))
    if smooth:
        P = (T - sp.diags(w / A.diagonal()) @ (A @ T)).tocsr()
    else:
        P = T
    P.sort_indices()
    return P


def galerkin(A: sp.csr_matrix, P: sp.csr_matrix):
    """R = P^T and the Galerkin coarse matrix A_c = R A P (reading Z32)."""
    R = P.T.tocsr()
    R.sort_indices()
    Ac = (R @ A @ P).tocsr()
    Ac.sort_indices()
    return R, Ac


def build_hierarchy(A, coarsest: int = 64, max_levels: int = 25, key_mode: int = KEY_HASH,
                    smooth: bool = True, max_dense: int = 8192, factor: bool = True) -> Hierarchy:
    """Smoothed-aggregation hierarchy (readings Z27-Z32).  ``A`` is an LDU system or a CSR."""
    if not sp.issparse(A):
        A = csr_of_ldu(A)
    A = A.tocsr()
    A.sort_indices()
    levels: List[Level] = []
    while A.shape[0] > coarsest and len(levels) < max_levels:
        n = A.shape[0]
        agg, na = mis2_aggregate(A, key_mode)
        if na >= n:                                   # no coarsening possible (Z31)
            break
        w = jacobi_weight(A)
        P = prolongator(A, agg, na, w, smooth)
        R, Ac = galerkin(A, P)
        levels.append(Level(A, agg, na, w, P, R))
        A = Ac
    if A.shape[0] > max_dense:
        raise ValueError(f"coarsest level too large for the dense solve ({A.shape[0]})")
    Lc = np.linalg.cholesky(A.toarray()) if factor else np.zeros((0, 0))
    return Hierarchy(levels, A, np.ascontiguousarray(Lc))


class _Flat(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int), ("nc", ctypes.c_int), ("n", ctypes.c_void_p)] + \
        [(k, ctypes.c_void_p) for k in ("Aptr", "Acol", "Aval", "Pptr", "Pcol", "Pval",
                                        "Rptr", "Rcol", "Rval", "nR", "rD", "omega", "Lc")]


def _flatten(H: Hierarchy) -> _Flat:
    keep = []

    def arr(a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        keep.append(a)
        return a

    def ptrs(lst):
        a = (ctypes.c_void_p * max(1, len(lst)))(*[x.ctypes.data for x in lst])
        keep.append(a)
        return ctypes.cast(a, ctypes.c_void_p)

    L = len(H.levels)
    f = _Flat()
    f.L = L
    f.nc = H.Ac.shape[0]
    f.n = arr([lv.A.shape[0] for lv in H.levels] or [0], np.int32).ctypes.data
    f.nR = arr([lv.R.shape[0] for lv in H.levels] or [0], np.int32).ctypes.data
    for name, get in (("A", lambda lv: lv.A), ("P", lambda lv: lv.P), ("R", lambda lv: lv.R)):
        mats = [get(lv) for lv in H.levels]
        setattr(f, name + "ptr", ptrs([arr(m.indptr, np.int32) for m in mats]))
        setattr(f, name + "col", ptrs([arr(m.indices, np.int32) for m in mats]))
        setattr(f, name + "val", ptrs([arr(m.data, np.float64) for m in mats]))
    f.rD = ptrs([arr(1.0 / lv.A.diagonal(), np.float64) for lv in H.levels])
    f.omega = arr([lv.omega for lv in H.levels] or [0.0], np.float64).ctypes.data
    f.Lc = arr(H.Lc, np.float64).ctypes.data
    H._keep = keep
    return f


def vcycle(H: Hierarchy, r: np.ndarray) -> np.ndarray:
    """z = B r: one V-cycle (reading Z32)."""
    f = _flatten(H)
    r = np.ascontiguousarray(r, dtype=np.float64)
    z = np.empty_like(r)
    _lib().oracle_amg_vcycle(ctypes.byref(f), _p(r), _p(z))
    return z


def amg_solve(sys, b: np.ndarray, H: Optional[Hierarchy] = None, x0: Optional[np.ndarray] = None,
              tol: float = 1e-8, maxIter: int = 1000, norm: int = NORM_L2, history: bool = False,
              relTol: float = 0.0, minIter: int = 0, pipelined: bool = False, **build_kw):
    """AMG-preconditioned CG (``pipelined=False``, SURVEY §8(c) c2 with z = B r) or pipelined CG
    (c3 literal form, u = B r, m = B w).  Returns (status, x, nIter, finalRes[, hist])."""
    if H is None:
        H = build_hierarchy(sys, **build_kw)
    f = _flatten(H)
    l, u, d, lo, up = _arrays(sys)
    bb = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(sys.nCells) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    it, res = ctypes.c_int(0), ctypes.c_double(0.0)
    hist = np.full(maxIter + 1, np.nan) if history else None
    st = _lib().oracle_amg_pcg(sys.nCells, l.shape[0], _p(l), _p(u), _p(d), _p(lo), _p(up),
                               _p(bb), _p(x), tol, maxIter, norm, ctypes.byref(it),
                               ctypes.byref(res), _p(hist), relTol, minIter, ctypes.byref(f),
                               1 if pipelined else 0)
    if st < 0:
        raise ValueError("oracle_amg_pcg: bad arguments")
    if history:
        return st, x, it.value, res.value, hist[: it.value + 1]
    return st, x, it.value, res.value


# ---- block-Jacobi AMG across ranks (reading Z33) -------------------------------------------
def block_hierarchies(parts, **build_kw) -> List[Hierarchy]:
    """One hierarchy per rank, each from the rank's LOCAL matrix (its own faces only; the
    interface couplings are dropped) -- ``parts`` as from meshgen.slab_partition."""
    return [build_hierarchy(csr_of_ldu(p), **build_kw) for p in parts]


def _blocks(Hs, bounds):
    flats = [_flatten(H) for H in Hs]
    arr = (ctypes.c_void_p * len(flats))(*[ctypes.addressof(f) for f in flats])
    start = np.ascontiguousarray(bounds, dtype=np.int32)
    return flats, arr, start


def block_vcycle(Hs, bounds, r: np.ndarray) -> np.ndarray:
    """z = B r, B = blockdiag(B_0 .. B_{p-1}) over the row ranges ``bounds``."""
    flats, arr, start = _blocks(Hs, bounds)
    r = np.ascontiguousarray(r, dtype=np.float64)
    z = np.empty_like(r)
    st = _lib().oracle_amg_block_vcycle(r.shape[0], len(Hs), _p(start),
                                        ctypes.cast(arr, ctypes.c_void_p), _p(r), _p(z))
    if st < 0:
        raise ValueError("oracle_amg_block_vcycle: bad arguments")
    return z


def amg_block_solve(sys, b: np.ndarray, bounds, Hs, x0: Optional[np.ndarray] = None,
                    tol: float = 1e-8, maxIter: int = 1000, norm: int = NORM_L2,
                    history: bool = False, relTol: float = 0.0, minIter: int = 0,
                    pipelined: bool = False):
    """Block-Jacobi AMG-CG / AMG-PipeCG on the GLOBAL system ``sys`` with one local hierarchy per
    row range (the distributed solve of reading Z33, emulated serially)."""
    flats, arr, start = _blocks(Hs, bounds)
    l, u, d, lo, up = _arrays(sys)
    bb = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(sys.nCells) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    it, res = ctypes.c_int(0), ctypes.c_double(0.0)
    hist = np.full(maxIter + 1, np.nan) if history else None
    st = _lib().oracle_amg_block_pcg(sys.nCells, l.shape[0], _p(l), _p(u), _p(d), _p(lo), _p(up),
                                     _p(bb), _p(x), tol, maxIter, norm, ctypes.byref(it),
                                     ctypes.byref(res), _p(hist), relTol, minIter, len(Hs),
                                     _p(start), ctypes.cast(arr, ctypes.c_void_p),
                                     1 if pipelined else 0)
    if st < 0:
        raise ValueError("oracle_amg_block_pcg: bad arguments")
    if history:
        return st, x, it.value, res.value, hist[: it.value + 1]
    return st, x, it.value, res.value

