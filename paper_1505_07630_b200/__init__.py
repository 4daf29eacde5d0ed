"""B200-native hot path of arXiv 1505.07630 (OpenFOAM LDU SpMV, Jacobi-PCG, pipelined CG).

Thin ctypes binding over the C ABI in ``include/ldu.h`` (``libldu_b200.so``): argument
marshalling only -- every step of the solve runs in the library's CUDA kernels.  There is no CPU
fallback: importing this package without the built library raises ImportError, and every call
that fails in the library raises :class:`LduError`.

Arrays may be numpy arrays (host) or torch tensors (CUDA on the handle's device, or CPU); they
must be contiguous, float64 for values and int32 for indices.  Names follow the paper / OpenFOAM
(lowerAddr, upperAddr, diag, upper, lower, interfaces, pcg_solve, pipecg_solve).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libldu_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build` "
                      "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)

# status codes (ldu_status)
OK, NOT_CONVERGED, BREAKDOWN = 0, 1, 2
ERR_INVALID_ARG, ERR_CUDA, ERR_NCCL, ERR_OOM, ERR_STATE = -1, -2, -3, -4, -5
NORM_L2, NORM_OPENFOAM = 0, 1
LAYOUT_DIA_SYM, LAYOUT_SELL32 = 1, 2
STATUS_NAMES = {0: "OK", 1: "NOT_CONVERGED", 2: "BREAKDOWN", -1: "ERR_INVALID_ARG",
                -2: "ERR_CUDA", -3: "ERR_NCCL", -4: "ERR_OOM", -5: "ERR_STATE"}


class LduError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class _Interface(ctypes.Structure):
    _fields_ = [("neighbRank", ctypes.c_int), ("nFaces", ctypes.c_int),
                ("faceCells", ctypes.c_void_p), ("coeffs", ctypes.c_void_p)]


class _Interfaces(ctypes.Structure):
    _fields_ = [("nInterfaces", ctypes.c_int), ("list", ctypes.POINTER(_Interface)),
                ("comm", ctypes.c_void_p)]


class SolveOpts(ctypes.Structure):
    _fields_ = [("norm", ctypes.c_int), ("recordHistory", ctypes.c_int), ("batch", ctypes.c_int),
                ("profile", ctypes.c_int), ("minIter", ctypes.c_int), ("replaceEvery", ctypes.c_int),
                ("relTol", ctypes.c_double), ("reserved2", ctypes.c_double * 2)]


class SolveStats(ctypes.Structure):
    _fields_ = [("solveMs", ctypes.c_double), ("iterMs", ctypes.c_double),
                ("kernels", ctypes.c_longlong), ("allreduces", ctypes.c_longlong),
                ("haloBytes", ctypes.c_longlong), ("h2dBytes", ctypes.c_longlong),
                ("d2hBytes", ctypes.c_longlong), ("iterations", ctypes.c_int),
                ("reductions", ctypes.c_int), ("passMs", ctypes.c_double * 2),
                ("passLaunches", ctypes.c_longlong * 2)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["passMs"] = list(self.passMs)
        d["passLaunches"] = list(self.passLaunches)
        return d


class Info(ctypes.Structure):
    _fields_ = [("layout", ctypes.c_int), ("nDiagonals", ctypes.c_int),
                ("offsets", ctypes.c_int * 8), ("storedEntries", ctypes.c_longlong),
                ("matrixBytes", ctypes.c_longlong), ("nCells", ctypes.c_int),
                ("nFaces", ctypes.c_int), ("nInterfaceFaces", ctypes.c_int),
                ("nRanks", ctypes.c_int), ("rank", ctypes.c_int), ("gridBlocks", ctypes.c_int),
                ("blockThreads", ctypes.c_int), ("variant", ctypes.c_int),
                ("pipeFused", ctypes.c_int)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["offsets"] = list(self.offsets)[: self.nDiagonals]
        d["layout_name"] = {1: "DIA_SYM", 2: "SELL32"}.get(self.layout, "?")
        return d


AMG_MAX_LEVELS = 25


class AmgOpts(ctypes.Structure):
    _fields_ = [("coarsest", ctypes.c_int), ("maxLevels", ctypes.c_int),
                ("keyIndexOrder", ctypes.c_int), ("unsmoothed", ctypes.c_int),
                ("lanczosSteps", ctypes.c_int), ("reserved", ctypes.c_int * 3)]


class AmgInfo(ctypes.Structure):
    _fields_ = [("nLevels", ctypes.c_int), ("coarsestN", ctypes.c_int),
                ("n", ctypes.c_int * (AMG_MAX_LEVELS + 1)),
                ("nnzA", ctypes.c_longlong * (AMG_MAX_LEVELS + 1)),
                ("nnzP", ctypes.c_longlong * AMG_MAX_LEVELS),
                ("omega", ctypes.c_double * AMG_MAX_LEVELS),
                ("operatorComplexity", ctypes.c_double), ("setupMs", ctypes.c_double),
                ("deviceBytes", ctypes.c_longlong)]

    def as_dict(self):
        L = self.nLevels
        return {"nLevels": L, "coarsestN": self.coarsestN, "n": list(self.n)[: L + 1],
                "nnzA": list(self.nnzA)[: L + 1], "nnzP": list(self.nnzP)[:L],
                "omega": list(self.omega)[:L], "operatorComplexity": self.operatorComplexity,
                "setupMs": self.setupMs, "deviceBytes": self.deviceBytes}


class DicInfo(ctypes.Structure):
    """ldu_dic_info (include/ldu.h)."""
    _fields_ = [("nLevels", ctypes.c_int), ("widestLevel", ctypes.c_int),
                ("lowerEntries", ctypes.c_longlong), ("setupMs", ctypes.c_double),
                ("ellWidthLower", ctypes.c_int), ("ellWidthUpper", ctypes.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_S = ctypes.c_int  # ldu_status

# exported symbols: name -> (restype, argtypes); tests check this matches include/ldu.h
SIGNATURES = {
    "ldu_abi_version": (_I, []),
    "ldu_last_error": (ctypes.c_char_p, []),
    "ldu_get_unique_id": (_S, [_P]),
    "ldu_comm_init": (_S, [_I, _I, _P, _I, ctypes.POINTER(_P)]),
    "ldu_comm_init_host": (_S, [_I, _I, _I, _P, _P, ctypes.POINTER(_P)]),
    "ldu_comm_destroy": (_S, [_P]),
    "ldu_setup": (_S, [_I, _I, _P, _P, _P, _P, _P, ctypes.POINTER(_Interfaces), ctypes.POINTER(_P)]),
    "ldu_set_stream": (_S, [_P, _P]),
    "ldu_amul": (_S, [_P, _P, _P]),
    "pcg_solve": (_S, [_P, _P, _P, _D, _I, ctypes.POINTER(_I), ctypes.POINTER(_D)]),
    "pipecg_solve": (_S, [_P, _P, _P, _D, _I, ctypes.POINTER(_I), ctypes.POINTER(_D)]),
    "pcg_solve_ex": (_S, [_P, _P, _P, _D, _I, ctypes.POINTER(SolveOpts), ctypes.POINTER(_I),
                          ctypes.POINTER(_D)]),
    "pipecg_solve_ex": (_S, [_P, _P, _P, _D, _I, ctypes.POINTER(SolveOpts), ctypes.POINTER(_I),
                             ctypes.POINTER(_D)]),
    "ldu_get_residual_history": (_S, [_P, _P, _I, ctypes.POINTER(_I)]),
    "ldu_get_solve_stats": (_S, [_P, ctypes.POINTER(SolveStats)]),
    "ldu_get_info": (_S, [_P, ctypes.POINTER(Info)]),
    "ldu_stream_triad": (_S, [_I, ctypes.c_longlong, _I, ctypes.POINTER(_D)]),
    "ldu_amg_setup": (_S, [_P, ctypes.POINTER(AmgOpts)]),
    "ldu_amg_get_info": (_S, [_P, ctypes.POINTER(AmgInfo)]),
    "ldu_amg_get_matrix": (_S, [_P, _I, _I, _P, _P, _P]),
    "ldu_amg_get_aggregates": (_S, [_P, _I, _P]),
    "ldu_amg_vcycle": (_S, [_P, _P, _P]),
    "amg_pcg_solve": (_S, [_P, _P, _P, _D, _I, ctypes.POINTER(SolveOpts), ctypes.POINTER(_I),
                           ctypes.POINTER(_D)]),
    "amg_pipecg_solve": (_S, [_P, _P, _P, _D, _I, ctypes.POINTER(SolveOpts), ctypes.POINTER(_I),
                              ctypes.POINTER(_D)]),
    "ldu_dic_setup": (_S, [_P]),
    "ldu_dic_get": (_S, [_P, _P, ctypes.POINTER(DicInfo)]),
    "ldu_dic_apply": (_S, [_P, _P, _P]),
    "dic_pcg_solve": (_S, [_P, _P, _P, _D, _I, ctypes.POINTER(SolveOpts), ctypes.POINTER(_I),
                           ctypes.POINTER(_D)]),
    "dic_pipecg_solve": (_S, [_P, _P, _P, _D, _I, ctypes.POINTER(SolveOpts), ctypes.POINTER(_I),
                              ctypes.POINTER(_D)]),
    "ldu_destroy": (_S, [_P]),
}
for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def last_error() -> str:
    return _lib.ldu_last_error().decode()


def _check(status: int) -> int:
    if status < 0:
        raise LduError(status, last_error())
    return status


def _ptr(a, dtype: str):
    """Raw pointer of a contiguous numpy array or torch tensor of the given dtype."""
    if a is None:
        return None
    mod = type(a).__module__
    if mod.startswith("torch"):
        import torch
        want = {"f64": torch.float64, "i32": torch.int32}[dtype]
        if a.dtype != want or not a.is_contiguous():
            raise TypeError(f"expected a contiguous {want} tensor")
        return a.data_ptr()
    import numpy as np
    want = {"f64": np.float64, "i32": np.int32}[dtype]
    if not isinstance(a, np.ndarray) or a.dtype != want or not a.flags["C_CONTIGUOUS"]:
        raise TypeError(f"expected a C-contiguous numpy {want.__name__} array")
    return a.ctypes.data


def _len(a) -> int:
    return int(a.shape[0])


_HostAllgather = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_ulonglong)


class Comm:
    """One rank's communicator.  ``Comm(rank, n, uid, device)``: two NCCL communicators
    (ldu_comm_init).  ``Comm.host(rank, n, device, group)``: no NCCL -- every exchange runs over
    the peer-memory mailboxes and the one-time setup exchange goes through torch.distributed on
    ``group`` (gloo), so several ranks may share one GPU (ldu_comm_init_host)."""

    def __init__(self, rank: int, nranks: int, unique_id: Optional[bytes], device: int,
                 _host_group=None):
        h = _P()
        self._cb = None
        if unique_id is None:
            import torch
            import torch.distributed as dist
            group = _host_group

            def _allgather(ctx, send, recv, nbytes):  # plumbing: bytes in, bytes out
                try:
                    src = torch.frombuffer(bytearray(ctypes.string_at(send, nbytes)),
                                           dtype=torch.uint8)
                    outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(nranks)]
                    dist.all_gather(outs, src, group=group)
                    allb = b"".join(bytes(o.numpy().tobytes()) for o in outs)
                    ctypes.memmove(recv, allb, len(allb))
                    return 0
                except Exception:  # noqa: BLE001 -- reported as a failed setup by the library
                    return 1

            self._cb = _HostAllgather(_allgather)
            _check(_lib.ldu_comm_init_host(rank, nranks, device, ctypes.cast(self._cb, _P), None,
                                           ctypes.byref(h)))
        else:
            if len(unique_id) != 128:
                raise ValueError("unique id must be 128 bytes")
            self._id = ctypes.create_string_buffer(unique_id, 128)
            _check(_lib.ldu_comm_init(rank, nranks, self._id, device, ctypes.byref(h)))
        self.handle = h
        self.rank, self.nranks, self.device = rank, nranks, device

    @classmethod
    def host(cls, rank: int, nranks: int, device: int, group=None) -> "Comm":
        """Peer-memory-only communicator bootstrapped over torch.distributed (gloo) ``group``."""
        return cls(rank, nranks, None, device, _host_group=group)

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(_lib.ldu_get_unique_id(buf))
        return buf.raw

    def close(self):
        if self.handle:
            _check(_lib.ldu_comm_destroy(self.handle))
            self.handle = None


class LduMatrix:
    """A device-resident OpenFOAM lduMatrix (``ldu_setup``) and its solvers."""

    def __init__(self, nCells: int, lowerAddr, upperAddr, diag, upper, lower=None,
                 interfaces: Optional[Sequence] = None, comm: Optional[Comm] = None):
        keep = []
        ifs_p = None
        if interfaces or comm is not None:
            arr = (_Interface * max(1, len(interfaces or [])))()
            for k, itf in enumerate(interfaces or []):
                fc, cf = itf.faceCells, itf.coeffs
                keep += [fc, cf]
                arr[k] = _Interface(int(itf.neighbRank), _len(fc), _ptr(fc, "i32"), _ptr(cf, "f64"))
            self._ifs = _Interfaces(len(interfaces or []), arr,
                                    comm.handle if comm is not None else None)
            keep.append(arr)
            ifs_p = ctypes.byref(self._ifs)
        h = _P()
        nf = _len(lowerAddr)
        st = _lib.ldu_setup(int(nCells), nf, _ptr(lowerAddr, "i32"), _ptr(upperAddr, "i32"),
                            _ptr(diag, "f64"), _ptr(lower, "f64"), _ptr(upper, "f64"), ifs_p,
                            ctypes.byref(h))
        _check(st)
        self.handle = h
        self.nCells = int(nCells)
        self.comm = comm

    @classmethod
    def from_system(cls, sys, comm: Optional[Comm] = None):
        """Build from a ``meshgen.LduSystem``-like object (duck-typed)."""
        return cls(sys.nCells, sys.lowerAddr, sys.upperAddr, sys.diag, sys.upper, sys.lower,
                   getattr(sys, "interfaces", None), comm)

    # -- operations ----------------------------------------------------------------------------
    def set_stream(self, stream_ptr: Optional[int]):
        _check(_lib.ldu_set_stream(self.handle, stream_ptr))

    def amul(self, x, y):
        """y = A x (incl. interfaces; collective across ranks)."""
        _check(_lib.ldu_amul(self.handle, _ptr(x, "f64"), _ptr(y, "f64")))
        return y

    def _solve(self, fn, b, x, tol, maxIter, norm, record_history, batch, profile=False,
               relTol=0.0, minIter=0, replaceEvery=0):
        it = _I(0)
        res = _D(0.0)
        opts = SolveOpts(norm, 1 if record_history else 0, batch, 1 if profile else 0,
                         int(minIter), int(replaceEvery), float(relTol))
        st = fn(self.handle, _ptr(b, "f64"), _ptr(x, "f64"), float(tol), int(maxIter),
                ctypes.byref(opts), ctypes.byref(it), ctypes.byref(res))
        if st < 0:
            raise LduError(st, last_error())
        return st, it.value, res.value

    def pcg_solve(self, b, x, tol: float = 1e-10, maxIter: int = 10000, norm: int = NORM_L2,
                  record_history: bool = False, batch: int = 0, profile: bool = False,
                  relTol: float = 0.0, minIter: int = 0, replaceEvery: int = 0):
        """Jacobi-PCG; x is in/out.  Returns (status, nIter, finalRes).  (replaceEvery is passed
        through to the C ABI, which rejects it: residual replacement is pipelined-only.)"""
        return self._solve(_lib.pcg_solve_ex, b, x, tol, maxIter, norm, record_history, batch,
                           profile, relTol, minIter, replaceEvery)

    def pipecg_solve(self, b, x, tol: float = 1e-10, maxIter: int = 10000, norm: int = NORM_L2,
                     record_history: bool = False, batch: int = 0, profile: bool = False,
                     relTol: float = 0.0, minIter: int = 0, replaceEvery: int = 0):
        """Ghysels-Vanroose pipelined CG; x is in/out; replaceEvery > 0 recomputes the recurrence
        vectors every replaceEvery iterations (NEXT-4).  Returns (status, nIter, finalRes)."""
        return self._solve(_lib.pipecg_solve_ex, b, x, tol, maxIter, norm, record_history, batch,
                           profile, relTol, minIter, replaceEvery)

    # -- aggregation-AMG preconditioner (NEXT-2) --------------------------------------
    def amg_setup(self, coarsest: int = 0, maxLevels: int = 0, keyIndexOrder: bool = False,
                  unsmoothed: bool = False, lanczosSteps: int = 0) -> dict:
        """Build the smoothed-aggregation hierarchy on the device; returns amg_info()."""
        o = AmgOpts(int(coarsest), int(maxLevels), 1 if keyIndexOrder else 0,
                    1 if unsmoothed else 0, int(lanczosSteps))
        _check(_lib.ldu_amg_setup(self.handle, ctypes.byref(o)))
        return self.amg_info()

    def amg_info(self) -> dict:
        i = AmgInfo()
        _check(_lib.ldu_amg_get_info(self.handle, ctypes.byref(i)))
        return i.as_dict()

    def amg_matrix(self, level: int, which: str = "A"):
        """(indptr, indices, data) numpy arrays of A_level / P_level / R_level (host copies)."""
        import numpy as np
        info = self.amg_info()
        w = {"A": 0, "P": 1, "R": 2}[which]
        if w == 0:
            rows, nnz = info["n"][level], info["nnzA"][level]
        else:
            rows = info["n"][level] if w == 1 else info["n"][level + 1]
            nnz = info["nnzP"][level]
        ptr = np.empty(rows + 1, dtype=np.int32)
        col = np.empty(max(1, nnz), dtype=np.int32)
        val = np.empty(max(1, nnz), dtype=np.float64)
        _check(_lib.ldu_amg_get_matrix(self.handle, int(level), w, ptr.ctypes.data,
                                       col.ctypes.data, val.ctypes.data))
        return ptr, col[:nnz], val[:nnz]

    def amg_aggregates(self, level: int):
        import numpy as np
        agg = np.empty(self.amg_info()["n"][level], dtype=np.int32)
        _check(_lib.ldu_amg_get_aggregates(self.handle, int(level), agg.ctypes.data))
        return agg

    def amg_vcycle(self, r, z):
        """z = B r (one V-cycle)."""
        _check(_lib.ldu_amg_vcycle(self.handle, _ptr(r, "f64"), _ptr(z, "f64")))
        return z

    def amg_pcg_solve(self, b, x, tol: float = 1e-10, maxIter: int = 10000, norm: int = NORM_L2,
                      record_history: bool = False, batch: int = 0, profile: bool = False,
                      relTol: float = 0.0, minIter: int = 0):
        """AMG-preconditioned CG; x is in/out.  Returns (status, nIter, finalRes)."""
        return self._solve(_lib.amg_pcg_solve, b, x, tol, maxIter, norm, record_history, batch,
                           profile, relTol, minIter)

    def amg_pipecg_solve(self, b, x, tol: float = 1e-10, maxIter: int = 10000,
                         norm: int = NORM_L2, record_history: bool = False, batch: int = 0,
                         profile: bool = False, relTol: float = 0.0, minIter: int = 0):
        """AMG-preconditioned pipelined CG (literal GV form); x is in/out."""
        return self._solve(_lib.amg_pipecg_solve, b, x, tol, maxIter, norm, record_history,
                           batch, profile, relTol, minIter)

    # -- DIC preconditioner (NEXT-1; OpenFOAM's default for p) --------------------------------
    def dic_setup(self) -> dict:
        """Level analysis + factor on the device; returns dic_info()."""
        _check(_lib.ldu_dic_setup(self.handle))
        return self.dic_info()

    def dic_info(self) -> dict:
        i = DicInfo()
        _check(_lib.ldu_dic_get(self.handle, None, ctypes.byref(i)))
        return i.as_dict()

    def dic_rD(self, out):
        """out[c] = 1 / D_c of the factor (host or device array)."""
        _check(_lib.ldu_dic_get(self.handle, _ptr(out, "f64"), None))
        return out

    def dic_apply(self, r, z):
        """z = M^-1 r (forward + backward level-scheduled sweeps)."""
        _check(_lib.ldu_dic_apply(self.handle, _ptr(r, "f64"), _ptr(z, "f64")))
        return z

    def dic_pcg_solve(self, b, x, tol: float = 1e-10, maxIter: int = 10000, norm: int = NORM_L2,
                      record_history: bool = False, batch: int = 0, profile: bool = False,
                      relTol: float = 0.0, minIter: int = 0):
        """DIC-preconditioned CG; x is in/out.  Returns (status, nIter, finalRes)."""
        return self._solve(_lib.dic_pcg_solve, b, x, tol, maxIter, norm, record_history, batch,
                           profile, relTol, minIter)

    def dic_pipecg_solve(self, b, x, tol: float = 1e-10, maxIter: int = 10000,
                         norm: int = NORM_L2, record_history: bool = False, batch: int = 0,
                         profile: bool = False, relTol: float = 0.0, minIter: int = 0):
        """DIC-preconditioned pipelined CG (literal GV form); x is in/out."""
        return self._solve(_lib.dic_pipecg_solve, b, x, tol, maxIter, norm, record_history,
                           batch, profile, relTol, minIter)

    def history(self):
        import numpy as np
        n = _I(0)
        cap = 1 << 20
        buf = np.empty(cap, dtype=np.float64)
        _check(_lib.ldu_get_residual_history(self.handle, buf.ctypes.data, cap, ctypes.byref(n)))
        return buf[: n.value].copy()

    def stats(self) -> dict:
        s = SolveStats()
        _check(_lib.ldu_get_solve_stats(self.handle, ctypes.byref(s)))
        return s.as_dict()

    def info(self) -> dict:
        i = Info()
        _check(_lib.ldu_get_info(self.handle, ctypes.byref(i)))
        return i.as_dict()

    def close(self):
        if getattr(self, "handle", None):
            _check(_lib.ldu_destroy(self.handle))
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def stream_triad(device: int = 0, n: int = 1 << 28, reps: int = 5) -> float:
    """fp64 STREAM triad bandwidth in GB/s."""
    g = _D(0.0)
    _check(_lib.ldu_stream_triad(device, n, reps, ctypes.byref(g)))
    return g.value


def abi_version() -> int:
    return _lib.ldu_abi_version()
