"""CPU oracle for the hot path of arXiv 1505.07630 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  It wraps ``ldu_oracle.c`` (plain fp64 C,
``-O2 -ffp-contract=off``, single thread) through ctypes and shares no code with the CUDA library
``paper_1505_07630_b200``.  See ``ldu_oracle.c`` for the passage each function follows and the
pins that hold it; DESIGN.md lists the readings Z1..Z33 of the paper it relies on.
``dic`` / ``dic_pcg`` add OpenFOAM's DIC preconditioner (NEXT-1; readings Z35-Z36).
``oracle.amg`` adds the aggregation-AMG preconditioner of P:236 (NEXT-2; readings Z27-Z33).

Parity status: every function here is pinned by ``tests/test_oracle_*.py`` (no "parity unpinned"
functions), except that Table 2's absolute iteration counts are unpinned (RHS and stopping
criterion unknown) -- only their 128^3/64^3 ratio is a pin.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ldu_oracle.c")
_LIB = os.path.join(_HERE, "libldu_oracle.so")

OK, NOT_CONVERGED, BREAKDOWN = 0, 1, 2
NORM_L2, NORM_OPENFOAM = 0, 1
LITERAL, JACOBI = 0, 1

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc, no FMA contraction, no fast-math, no OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int
        D = ctypes.c_double
        lib.oracle_amul.argtypes = [I, I, P, P, P, P, P, P, P]
        lib.oracle_amul.restype = None
        lib.oracle_iface.argtypes = [I, P, P, P, P]
        lib.oracle_iface.restype = None
        lib.oracle_pcg.argtypes = [I, I, P, P, P, P, P, P, P, D, I, I, P, P, P, D, I]
        lib.oracle_pcg.restype = I
        lib.oracle_pipecg.argtypes = [I, I, P, P, P, P, P, P, P, D, I, I, I, P, P, P, D, I]
        lib.oracle_pipecg.restype = I
        lib.oracle_pipecg_rr.argtypes = [I, I, P, P, P, P, P, P, P, D, I, I, I, P, P, P, D, I, I]
        lib.oracle_pipecg_rr.restype = I
        lib.oracle_dic.argtypes = [I, I, P, P, P, P, I, P, P, P, P]
        lib.oracle_dic.restype = I
        lib.oracle_dic_pcg.argtypes = [I, I, P, P, P, P, P, P, D, I, I, P, P, P, D, I, I, P, I]
        lib.oracle_dic_pcg.restype = I
        _lib = lib
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _arrays(sys):
    l = np.ascontiguousarray(sys.lowerAddr, dtype=np.int32)
    u = np.ascontiguousarray(sys.upperAddr, dtype=np.int32)
    d = np.ascontiguousarray(sys.diag, dtype=np.float64)
    up = np.ascontiguousarray(sys.upper, dtype=np.float64)
    lo = None if sys.lower is None else np.ascontiguousarray(sys.lower, dtype=np.float64)
    return l, u, d, lo, up


def amul(sys, x: np.ndarray) -> np.ndarray:
    """y = A x over internal faces (interfaces excluded), OpenFOAM face loop."""
    lib = _load()
    l, u, d, lo, up = _arrays(sys)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(sys.nCells, dtype=np.float64)
    lib.oracle_amul(sys.nCells, l.shape[0], _p(l), _p(u), _p(d), _p(lo), _p(up), _p(x), _p(y))
    return y


def iface_update(y: np.ndarray, faceCells: np.ndarray, coeffs: np.ndarray, xnbr: np.ndarray):
    lib = _load()
    fc = np.ascontiguousarray(faceCells, dtype=np.int32)
    cf = np.ascontiguousarray(coeffs, dtype=np.float64)
    xn = np.ascontiguousarray(xnbr, dtype=np.float64)
    lib.oracle_iface(fc.shape[0], _p(fc), _p(cf), _p(xn), _p(y))


def halo_values(parts: Sequence, xs: Sequence[np.ndarray], g: int, k: int) -> np.ndarray:
    """Serial emulation of the halo exchange: the values rank g receives on its k-th
    interface are the neighbour's x at the neighbour's faceCells of the interface back to g, in
    the shared face order (reading Z22).  Multiple interfaces to the same neighbour pair in order."""
    me = parts[g].interfaces[k]
    h = me.neighbRank
    mine = [i for i, itf in enumerate(parts[g].interfaces) if itf.neighbRank == h].index(k)
    back = [itf for itf in parts[h].interfaces if itf.neighbRank == g][mine]
    return xs[h][back.faceCells]


def dist_amul(parts: Sequence, xs: Sequence[np.ndarray]) -> List[np.ndarray]:
    """Distributed SpMV emulated serially over all slabs: local face loop, then interface updates
    in interface order, face order (readings Z10, Z23)."""
    ys = []
    for g, part in enumerate(parts):
        y = amul(part, xs[g])
        for k, itf in enumerate(part.interfaces):
            iface_update(y, itf.faceCells, itf.coeffs, halo_values(parts, xs, g, k))
        ys.append(y)
    return ys


def pcg(sys, b: np.ndarray, x0: Optional[np.ndarray] = None, tol: float = 1e-10,
        maxIter: int = 10000, norm: int = NORM_L2, history: bool = False, relTol: float = 0.0,
        minIter: int = 0):
    """Jacobi-PCG.  Returns (status, x, nIter, finalRes[, hist])."""
    lib = _load()
    l, u, d, lo, up = _arrays(sys)
    bb = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(sys.nCells) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    it = ctypes.c_int(0)
    res = ctypes.c_double(0.0)
    hist = np.full(maxIter + 1, np.nan) if history else None
    st = lib.oracle_pcg(sys.nCells, l.shape[0], _p(l), _p(u), _p(d), _p(lo), _p(up), _p(bb),
                        _p(x), tol, maxIter, norm, ctypes.byref(it), ctypes.byref(res), _p(hist),
                        relTol, minIter)
    if history:
        return st, x, it.value, res.value, hist[: it.value + 1]
    return st, x, it.value, res.value


def pipecg(sys, b: np.ndarray, x0: Optional[np.ndarray] = None, tol: float = 1e-10,
           maxIter: int = 10000, norm: int = NORM_L2, mode: int = JACOBI, history: bool = False,
           relTol: float = 0.0, minIter: int = 0, replace_every: int = 0):
    """Ghysels-Vanroose pipelined CG (mode LITERAL or JACOBI), optionally with residual
    replacement every ``replace_every`` iterations (NEXT-4).  Returns like ``pcg``."""
    lib = _load()
    l, u, d, lo, up = _arrays(sys)
    bb = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(sys.nCells) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    it = ctypes.c_int(0)
    res = ctypes.c_double(0.0)
    hist = np.full(maxIter + 1, np.nan) if history else None
    if replace_every:
        st = lib.oracle_pipecg_rr(sys.nCells, l.shape[0], _p(l), _p(u), _p(d), _p(lo), _p(up),
                                  _p(bb), _p(x), tol, maxIter, norm, mode, ctypes.byref(it),
                                  ctypes.byref(res), _p(hist), relTol, minIter, int(replace_every))
    else:
        st = lib.oracle_pipecg(sys.nCells, l.shape[0], _p(l), _p(u), _p(d), _p(lo), _p(up),
                               _p(bb), _p(x), tol, maxIter, norm, mode, ctypes.byref(it),
                               ctypes.byref(res), _p(hist), relTol, minIter)
    if history:
        return st, x, it.value, res.value, hist[: it.value + 1]
    return st, x, it.value, res.value


# ---- DIC preconditioner (readings Z35, Z36) ----------------------------
def _blocks_arg(sys, bounds):
    if bounds is None:
        return 1, None
    st = np.ascontiguousarray(bounds, dtype=np.int32)
    return st.shape[0] - 1, st


def dic(sys, r: Optional[np.ndarray] = None, bounds: Optional[Sequence[int]] = None):
    """OpenFOAM DIC: returns (status, rD, w) with rD the reciprocal D of
    M = (D + L) D^-1 (D + L^T) and w = M^-1 r (None without r).  ``bounds`` = contiguous row
    blocks (block-Jacobi DIC across ranks: faces joining two blocks dropped)."""
    assert sys.lower is None or np.array_equal(sys.lower, sys.upper), "DIC needs a symmetric matrix"
    lib = _load()
    l, u, d, _, up = _arrays(sys)
    nb, st = _blocks_arg(sys, bounds)
    rD = np.empty(sys.nCells)
    rr = None if r is None else np.ascontiguousarray(r, dtype=np.float64)
    w = None if r is None else np.empty(sys.nCells)
    status = lib.oracle_dic(sys.nCells, l.shape[0], _p(l), _p(u), _p(d), _p(up), nb, _p(st),
                            _p(rD), _p(rr), _p(w))
    if status < 0:
        raise ValueError("oracle_dic: bad arguments")
    return status, rD, w


def dic_pcg(sys, b: np.ndarray, x0: Optional[np.ndarray] = None, tol: float = 1e-10,
            maxIter: int = 10000, norm: int = NORM_L2, history: bool = False,
            relTol: float = 0.0, minIter: int = 0, pipelined: bool = False,
            bounds: Optional[Sequence[int]] = None):
    """DIC-preconditioned CG (c2 with z = M^-1 r) or pipelined CG (c3 literal form).
    Returns (status, x, nIter, finalRes[, hist])."""
    assert sys.lower is None or np.array_equal(sys.lower, sys.upper), "DIC needs a symmetric matrix"
    lib = _load()
    l, u, d, _, up = _arrays(sys)
    nb, st = _blocks_arg(sys, bounds)
    bb = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(sys.nCells) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    it = ctypes.c_int(0)
    res = ctypes.c_double(0.0)
    hist = np.full(maxIter + 1, np.nan) if history else None
    status = lib.oracle_dic_pcg(sys.nCells, l.shape[0], _p(l), _p(u), _p(d), _p(up), _p(bb),
                                _p(x), tol, maxIter, norm, ctypes.byref(it), ctypes.byref(res),
                                _p(hist), relTol, minIter, nb, _p(st), 1 if pipelined else 0)
    if status < 0:
        raise ValueError("oracle_dic_pcg: bad arguments")
    if history:
        return status, x, it.value, res.value, hist[: it.value + 1]
    return status, x, it.value, res.value
