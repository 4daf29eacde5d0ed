"""Seeded synthetic LDU systems and the contiguous-slab decomposition.

This module is shared by the tests, ``bench.py`` and ``__graft_entry__.smoke`` to feed the SAME
inputs to the CPU oracle (``oracle/``) and to the CUDA library (``paper_1505_07630_b200``).
It holds none of the method's arithmetic: no SpMV, no dot products, no Krylov recurrences.  It
only builds matrices in OpenFOAM ``lduMatrix`` form (diag / upper / lower over
lowerAddr = owner, upperAddr = neighbour face addressing) and right-hand
sides, and splits them into per-rank slabs with processor interfaces.

Workload recipes (SURVEY.md §8(d) "Concrete synthetic inputs"):

* ``hex_laplacian``  - laplacianFoam-style 7-point FV Laplacian on an nx*ny*nz hex box with
  Dirichlet walls ("heat equation with Dirichlet boundary condition ... cubic
  geometry"; Eq 3 at PAPER.md:69-71 read as dT/dt - div(D grad T) = 0, reading Z12).  Boundary
  convention ``"fv"`` (default, reading Z11): interior face coefficient -D, a Dirichlet face adds
  2D to diag and 2D*T_b to b (half-cell distance).  ``"ghost"``: a Dirichlet face adds D (every
  diag = 6).  Optional transient term V/dt added to diag (laplacianFoam's
  time-implicit Helmholtz form).
* ``cavity_pressure_2d`` - icoFoam lid-driven-cavity pressure matrix (config 2):
  one cell thick, 5-point, zeroGradient walls, OpenFOAM ``setReference(0, 0)``.
* ``random_ldu``     - small random irregular LDU matrices (n <= 64) for the oracle pins.
* ``irregular_mesh`` - config 5: perturbed, partially-dropped, diagonally-augmented hex graph,
  randomly permuted then RCM-renumbered, faces re-sorted upper-triangular.
* ``slab_partition`` - contiguous cell slabs (decomposePar analogue).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

I32 = np.int32
F64 = np.float64


@dataclass
class Interface:
    """One processor interface (PAPER.md:79 halo layer; OpenFOAM processor patch).

    ``faceCells[i]`` is the local cell next to patch face i; ``coeffs[i]`` is OpenFOAM's
    interfaceBouCoeffs (the NEGATED off-diagonal), so the interface update is
    ``y[faceCells[i]] -= coeffs[i] * x_neighbour[i]`` (reading Z10).  Faces are listed in
    increasing global face index on both sides (reading Z22), so entry i on this rank pairs with
    entry i of the neighbour's interface back to this rank.
    """

    neighbRank: int
    faceCells: np.ndarray  # int32 [nFaces]
    coeffs: np.ndarray  # float64 [nFaces]


@dataclass
class LduSystem:
    """An OpenFOAM-style lduMatrix plus right-hand side (SURVEY.md §8(b) ``ldu_setup`` inputs)."""

    nCells: int
    lowerAddr: np.ndarray  # int32 [nFaces] owner  l[f]
    upperAddr: np.ndarray  # int32 [nFaces] neighbour u[f]
    diag: np.ndarray  # float64 [nCells]
    upper: np.ndarray  # float64 [nFaces]  A[l[f], u[f]]
    lower: Optional[np.ndarray] = None  # float64 [nFaces] A[u[f], l[f]]; None => symmetric
    b: Optional[np.ndarray] = None  # float64 [nCells]
    interfaces: List[Interface] = field(default_factory=list)
    meta: dict = field(default_factory=dict)

    @property
    def nFaces(self) -> int:
        return int(self.lowerAddr.shape[0])

    def dense(self) -> np.ndarray:
        """Dense matrix (internal faces only) - a test helper for tiny systems."""
        n = self.nCells
        A = np.zeros((n, n), dtype=F64)
        A[np.arange(n), np.arange(n)] = self.diag
        lo = self.upper if self.lower is None else self.lower
        np.add.at(A, (self.lowerAddr, self.upperAddr), self.upper)
        np.add.at(A, (self.upperAddr, self.lowerAddr), lo)
        return A


# --------------------------------------------------------------------------------------------
# structured hex box (configs 1, 3, 4)
# --------------------------------------------------------------------------------------------

def _hex_faces(nx: int, ny: int, nz: int):
    """Internal faces of an nx*ny*nz lexicographic (x fastest) hex mesh in OpenFOAM
    upper-triangular order: sorted by owner, then by neighbour (owner c -> c+1, c+nx, c+nx*ny)."""
    N = nx * ny * nz
    c = np.arange(N, dtype=np.int64)
    i = c % nx
    j = (c // nx) % ny
    k = c // (nx * ny)
    valid = np.stack([i < nx - 1, j < ny - 1, k < nz - 1], axis=1)
    nbr = c[:, None] + np.array([1, nx, nx * ny], dtype=np.int64)[None, :]
    owner = np.broadcast_to(c[:, None], nbr.shape)
    l = owner[valid].astype(I32)
    u = nbr[valid].astype(I32)
    axis = np.broadcast_to(np.arange(3)[None, :], nbr.shape)[valid]
    return l, u, axis, (i, j, k)


def hex_laplacian(nx: int, ny: int, nz: int, *, bc: str = "fv", D: float = 1.0,
                  ddt: float = 0.0, conductance_sigma: float = 0.0, seed: int = 7630,
                  dirichlet: Optional[dict] = None) -> LduSystem:
    """7-point FV Laplacian (h = 1) with Dirichlet walls.  See the module docstring.

    ``dirichlet`` maps wall names ('x0','x1','y0','y1','z0','z1') to wall values (default 0);
    the wall terms go into ``b``.  ``conductance_sigma > 0`` multiplies every internal face
    coefficient by exp(sigma*xi), xi ~ N(0,1) (config 5 recipe).
    """
    if bc not in ("fv", "ghost"):
        raise ValueError("bc must be 'fv' or 'ghost'")
    if min(nx, ny, nz) < 1:
        raise ValueError("mesh dimensions must be >= 1")
    N = nx * ny * nz
    l, u, _, (i, j, k) = _hex_faces(nx, ny, nz)
    g = np.full(l.shape[0], D, dtype=F64)
    if conductance_sigma > 0:
        rng = np.random.default_rng(seed)
        g = g * np.exp(conductance_sigma * rng.standard_normal(l.shape[0]))
    upper = -g
    diag = np.bincount(l, weights=g, minlength=N) + np.bincount(u, weights=g, minlength=N)
    wall = 2.0 * D if bc == "fv" else D
    b = np.zeros(N, dtype=F64)
    vals = dict(x0=0.0, x1=0.0, y0=0.0, y1=0.0, z0=0.0, z1=0.0)
    if dirichlet:
        for key in dirichlet:
            if key not in vals:
                raise ValueError(f"unknown wall {key}")
        vals.update(dirichlet)
    for name, mask in (("x0", i == 0), ("x1", i == nx - 1), ("y0", j == 0), ("y1", j == ny - 1),
                       ("z0", k == 0), ("z1", k == nz - 1)):
        diag = diag + wall * mask
        if vals[name] != 0.0:
            b = b + wall * vals[name] * mask
    if ddt:
        diag = diag + ddt
    return LduSystem(N, l, u, diag.astype(F64), upper.astype(F64), None, b,
                     meta=dict(kind="hex", nx=nx, ny=ny, nz=nz, bc=bc, D=D, ddt=ddt))


def rhs_hot_face(nx: int, ny: int, nz: int, bc: str = "fv", D: float = 1.0) -> np.ndarray:
    """Hot-face RHS: T_b = 1 on the x = 0 wall, 0 elsewhere."""
    wall = 2.0 * D if bc == "fv" else D
    N = nx * ny * nz
    i = np.arange(N) % nx
    return (wall * (i == 0)).astype(F64)


def rhs_random(n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    return np.random.default_rng(seed).uniform(lo, hi, n).astype(F64)


# --------------------------------------------------------------------------------------------
# config 2: icoFoam cavity pressure equation (2-D, one cell thick)
# --------------------------------------------------------------------------------------------

def cavity_pressure_2d(nx: int, ny: int) -> LduSystem:
    """Pressure Laplacian of the 2-D lid-driven cavity: off-diagonal -1, zeroGradient walls
    (no wall term), empty front/back, then OpenFOAM ``setReference(0, 0)``:
    diag[0] += diag[0] (reading Z21) so the matrix is SPD."""
    l, u, _, _ = _hex_faces(nx, ny, 1)
    N = nx * ny
    g = np.ones(l.shape[0], dtype=F64)
    diag = np.bincount(l, weights=g, minlength=N) + np.bincount(u, weights=g, minlength=N)
    diag[0] += diag[0]
    return LduSystem(N, l, u, diag.astype(F64), -g, None, np.zeros(N),
                     meta=dict(kind="cavity2d", nx=nx, ny=ny))


def cavity_rhs(nx: int, ny: int, t: int) -> np.ndarray:
    """Zero-mean smoothed random source for PISO step t (seed 1505 + t)."""
    rng = np.random.default_rng(1505 + t)
    f = rng.standard_normal((ny, nx))
    for _ in range(4):  # cheap separable box smoothing, periodic
        f = (np.roll(f, 1, 0) + f + np.roll(f, -1, 0)) / 3.0
        f = (np.roll(f, 1, 1) + f + np.roll(f, -1, 1)) / 3.0
    f = f.ravel()
    f -= f.mean()
    return f.astype(F64)


# --------------------------------------------------------------------------------------------
# random irregular LDU (oracle pins, n <= 64)
# --------------------------------------------------------------------------------------------

def random_ldu(n: int, seed: int, density: float = 0.15, symmetric: bool = True,
               margin: float = 0.5, sort_faces: bool = True) -> LduSystem:
    """Random sparse LDU: unique pairs (l < u), negative off-diagonals, diag = row |off| sum +
    margin (strictly diagonally dominant, so SPD when symmetric).  ``sort_faces=False`` shuffles
    the face order (OpenFOAM does not require it; reading Z10)."""
    rng = np.random.default_rng(seed)
    iu = np.triu_indices(n, 1)
    keep = rng.random(iu[0].shape[0]) < density
    l = iu[0][keep].astype(I32)
    u = iu[1][keep].astype(I32)
    if not sort_faces:
        perm = rng.permutation(l.shape[0])
        l, u = l[perm], u[perm]
    upper = -rng.uniform(0.1, 1.0, l.shape[0])
    lower = None if symmetric else -rng.uniform(0.1, 1.0, l.shape[0])
    lo = upper if lower is None else lower
    off = np.bincount(l, weights=np.abs(upper), minlength=n) + \
        np.bincount(u, weights=np.abs(lo), minlength=n)
    diag = off + margin + rng.uniform(0.0, 1.0, n)
    return LduSystem(n, l, u, diag.astype(F64), upper.astype(F64),
                     None if lower is None else lower.astype(F64),
                     rng.uniform(-1, 1, n).astype(F64), meta=dict(kind="random", seed=seed))


# --------------------------------------------------------------------------------------------
# config 5: unstructured-like mesh
# --------------------------------------------------------------------------------------------

def irregular_mesh(n: int, seed: int = 1505, rcm: bool = True) -> LduSystem:
    """Config-5 recipe: base n^3 hex, conductance exp(0.5 xi); drop 5% of internal
    faces keeping >= 2 faces per cell; add a diagonal face to (i+1, j+1, k) for 10% of cells;
    diag = sum|off| + FV Dirichlet walls + V/dt (0.01); random permutation then (optionally)
    reverse Cuthill-McKee renumbering; faces re-sorted upper-triangular."""
    rng = np.random.default_rng(seed)
    nx = ny = nz = n
    N = n ** 3
    l, u, _, (i, j, k) = _hex_faces(nx, ny, nz)
    # drop 5% keeping >= 2 faces per cell
    drop = rng.random(l.shape[0]) < 0.05
    deg = np.bincount(l, minlength=N) + np.bincount(u, minlength=N)
    cand = np.nonzero(drop)[0]
    keepmask = np.ones(l.shape[0], dtype=bool)
    for f in cand:  # sequential so the >= 2 rule is exact; ~5% of F
        a, c2 = l[f], u[f]
        if deg[a] > 2 and deg[c2] > 2:
            keepmask[f] = False
            deg[a] -= 1
            deg[c2] -= 1
    l, u = l[keepmask], u[keepmask]
    # diagonal faces to (i+1, j+1, k)
    c = np.arange(N)
    ok = (i < nx - 1) & (j < ny - 1) & (rng.random(N) < 0.10)
    dl = c[ok].astype(I32)
    du = (c[ok] + 1 + nx).astype(I32)
    l = np.concatenate([l, dl])
    u = np.concatenate([u, du])
    g = np.exp(0.5 * rng.standard_normal(l.shape[0]))
    diag = np.bincount(l, weights=g, minlength=N) + np.bincount(u, weights=g, minlength=N)
    nwall = (i == 0).astype(int) + (i == nx - 1) + (j == 0) + (j == ny - 1) + (k == 0) + (k == nz - 1)
    diag = diag + 2.0 * nwall + 0.01
    # renumber: random permutation, then RCM
    perm = rng.permutation(N)  # new index of old cell c is perm[c]
    l, u = perm[l], perm[u]
    diag_p = np.empty_like(diag)
    diag_p[perm] = diag
    diag = diag_p
    if rcm:
        import scipy.sparse as sp
        from scipy.sparse.csgraph import reverse_cuthill_mckee
        G = sp.coo_matrix((np.ones(l.shape[0]), (l, u)), shape=(N, N)).tocsr()
        G = G + G.T
        order = reverse_cuthill_mckee(G.tocsr(), symmetric_mode=True)  # order[new] = old
        inv = np.empty(N, dtype=np.int64)
        inv[order] = np.arange(N)
        l, u = inv[l], inv[u]
        diag = diag[order]
    lo = np.minimum(l, u)
    hi = np.maximum(l, u)
    srt = np.lexsort((hi, lo))
    l = lo[srt].astype(I32)
    u = hi[srt].astype(I32)
    g = g[srt]
    b = np.random.default_rng(seed + 1).uniform(0, 1, N)
    return LduSystem(N, l, u, diag.astype(F64), (-g).astype(F64), None, b.astype(F64),
                     meta=dict(kind="irregular", n=n, seed=seed, rcm=rcm))


# --------------------------------------------------------------------------------------------
# contiguous-slab decomposition
# --------------------------------------------------------------------------------------------

def slab_bounds(nCells: int, p: int) -> np.ndarray:
    """Rank g owns cells [floor(g N / p), floor((g+1) N / p))."""
    return np.array([(g * nCells) // p for g in range(p + 1)], dtype=np.int64)


def slab_partition(sys: LduSystem, p: int, bounds: Optional[np.ndarray] = None) -> List[LduSystem]:
    """Split a global LDU system into p contiguous-cell slabs.

    Local faces keep both ends local, in the original relative order.  Each cut face becomes an
    interface face on both ranks; on the owner side coeff = -upper[f] (at faceCell l[f]-lo), on
    the neighbour side coeff = -lower[f] (at faceCell u[f]-lo); interfaces are grouped by
    neighbour rank and list faces in increasing global face index (reading Z22).
    """
    if p < 1:
        raise ValueError("p >= 1")
    if bounds is None:
        bounds = slab_bounds(sys.nCells, p)
    l = sys.lowerAddr.astype(np.int64)
    u = sys.upperAddr.astype(np.int64)
    rl = np.searchsorted(bounds, l, side="right") - 1
    ru = np.searchsorted(bounds, u, side="right") - 1
    lower = sys.upper if sys.lower is None else sys.lower
    out = []
    for g in range(p):
        lo_, hi_ = int(bounds[g]), int(bounds[g + 1])
        loc = (rl == g) & (ru == g)
        ll = (l[loc] - lo_).astype(I32)
        uu = (u[loc] - lo_).astype(I32)
        up = sys.upper[loc].copy()
        lw = None if sys.lower is None else sys.lower[loc].copy()
        ifs = []
        nbrs = sorted(set(ru[(rl == g) & (ru != g)].tolist()) | set(rl[(ru == g) & (rl != g)].tolist()))
        for h in nbrs:
            a = (rl == g) & (ru == h)   # this rank owns l[f]
            bm = (ru == g) & (rl == h)  # this rank owns u[f]
            fids = np.nonzero(a | bm)[0]  # increasing global face index
            fc = np.where(a[fids], l[fids] - lo_, u[fids] - lo_).astype(I32)
            cf = np.where(a[fids], -sys.upper[fids], -lower[fids]).astype(F64)
            ifs.append(Interface(int(h), fc, cf))
        b = None if sys.b is None else sys.b[lo_:hi_].copy()
        out.append(LduSystem(hi_ - lo_, ll, uu, sys.diag[lo_:hi_].copy(), up, lw, b, ifs,
                             meta=dict(sys.meta, rank=g, nranks=p, cell_lo=lo_, cell_hi=hi_)))
    return out


def hex_laplacian_slab(nx: int, ny: int, nz: int, p: int, g: int, **kw) -> LduSystem:
    """Rank g's z-slab of ``hex_laplacian(nx, ny, nz)`` built directly (no global arrays), for
    meshes too large to build whole on one host (config 4, 512^3).  Identical to
    ``slab_partition(hex_laplacian(...), p)[g]`` when the slab bounds fall on whole z-planes,
    which they do when p divides nz; the test suite checks the equality."""
    if nz % p:
        raise ValueError("p must divide nz for direct slab generation")
    if kw.get("conductance_sigma", 0.0):
        raise ValueError("direct slab generation supports uniform conductance only")
    D = kw.get("D", 1.0)
    bc = kw.get("bc", "fv")
    nzl = nz // p
    z0 = g * nzl
    # local slab as its own box, then fix the diag of the cut planes
    loc = hex_laplacian(nx, ny, nzl, bc=bc, D=D, ddt=kw.get("ddt", 0.0),
                        dirichlet=kw.get("dirichlet"))
    plane = nx * ny
    wall = 2.0 * D if bc == "fv" else D
    ifs = []
    if g > 0:  # bottom plane was given a z0 wall; it is a cut instead (neighbour face coeff -D)
        loc.diag[:plane] += -wall + D
        if loc.b is not None:
            zval = (kw.get("dirichlet") or {}).get("z0", 0.0)
            loc.b[:plane] -= wall * zval
        ifs.append(Interface(g - 1, np.arange(plane, dtype=I32), np.full(plane, D, dtype=F64)))
    if g < p - 1:
        loc.diag[-plane:] += -wall + D
        if loc.b is not None:
            zval = (kw.get("dirichlet") or {}).get("z1", 0.0)
            loc.b[-plane:] -= wall * zval
        ifs.append(Interface(g + 1, np.arange(plane * (nzl - 1), plane * nzl, dtype=I32),
                             np.full(plane, D, dtype=F64)))
    loc.interfaces = ifs
    loc.meta.update(kind="hex", nx=nx, ny=ny, nz=nz, rank=g, nranks=p, cell_lo=z0 * plane,
                    cell_hi=(z0 + nzl) * plane)
    return loc


# --------------------------------------------------------------------------------------------
# heterogeneous decomposition (Eq 5-8)
# --------------------------------------------------------------------------------------------

def speed(n_i: int, o_i: int, T: float) -> float:
    """Eq 5: s_i(n_i) = (n_i + 2 o_i) / T(n_i) -- non-zeros of the local matrix
    (n_i rows, o_i upper-triangle off-diagonals) per second of one CG iteration."""
    if T <= 0:
        raise ValueError("T must be > 0")
    return (n_i + 2 * o_i) / T


def relative_speeds(s) -> np.ndarray:
    """Eq 6, index collision read as r_i = s_i / sum_j s_j (reading Z14)."""
    s = np.asarray(s, dtype=F64)
    if s.size == 0 or np.any(s <= 0):
        raise ValueError("speeds must be positive")
    return s / s.sum()


def rebalance(N: int, r) -> np.ndarray:
    """Eq 7-8: n_i,new = N r_i, rounded by largest remainder so that
    sum_i n_i,new = N exactly (Eq 7)."""
    r = np.asarray(r, dtype=F64)
    if r.size == 0 or np.any(r < 0) or abs(r.sum() - 1.0) > 1e-9:
        raise ValueError("fractions must be >= 0 and sum to 1")
    raw = N * r
    n = np.floor(raw).astype(np.int64)
    rem = int(N - n.sum())
    order = np.argsort(-(raw - n), kind="stable")  # ties: lowest index first
    n[order[:rem]] += 1
    return n


def fit_time_model(ns, Ts):
    """Functional performance model of one device (the paper builds Eq 5's speeds with the
    FuPerMod functional performance models, "combines the performance model [fupermode]"):
    T(n) = a + b n, least squares over the measured (cells, seconds per iteration) points.  One
    point gives a = 0 -- the constant-speed model Eq 5 assumes.  Returns (a, b)."""
    ns = np.asarray(ns, dtype=F64)
    Ts = np.asarray(Ts, dtype=F64)
    if ns.size == 0 or ns.size != Ts.size or np.any(ns <= 0) or np.any(Ts <= 0):
        raise ValueError("need matching positive sizes and times")
    if ns.size == 1 or np.ptp(ns) == 0:
        return 0.0, float(Ts.mean() / ns.mean())
    b, a = np.polyfit(ns, Ts, 1)
    if b <= 0:  # not a usable model (noise): fall back to the mean speed
        return 0.0, float(np.sum(Ts) / np.sum(ns))
    return float(a), float(b)


def fpm_partition(N: int, models, min_cells: int = 1) -> np.ndarray:
    """Cells per device with equal predicted iteration times under T_i(n) = a_i + b_i n:
    a_i + b_i n_i = T* for every i and sum_i n_i = N (Eq 7), i.e.
    T* = (N + sum_i a_i / b_i) / sum_i 1 / b_i,  n_i = (T* - a_i) / b_i,
    rounded by the largest remainder (as ``rebalance``); a device whose share would fall below
    ``min_cells`` gets min_cells and the rest is re-solved.  With a_i = 0 this is Eq 5-8."""
    a = np.array([m[0] for m in models], dtype=F64)
    b = np.array([m[1] for m in models], dtype=F64)
    if a.size == 0 or np.any(b <= 0) or N < min_cells * a.size:
        raise ValueError("bad models or too few cells")
    fixed = np.zeros(a.size, dtype=bool)
    n = np.zeros(a.size, dtype=F64)
    for _ in range(a.size):
        free = ~fixed
        rest = N - min_cells * fixed.sum()
        Tstar = (rest + np.sum(a[free] / b[free])) / np.sum(1.0 / b[free])
        n[free] = (Tstar - a[free]) / b[free]
        n[fixed] = min_cells
        low = free & (n < min_cells)
        if not low.any():
            break
        fixed |= low
    return rebalance(N, n / n.sum())


def slab_bounds_weighted(nCells: int, fractions) -> np.ndarray:
    """Contiguous slabs whose sizes follow Eq 8 for the given work fractions (the weights the
    paper hands to MeTiS/SCOTCH)."""
    n = rebalance(nCells, fractions)
    return np.concatenate([[0], np.cumsum(n)]).astype(np.int64)


def nnz_balanced_bounds(sys: LduSystem, p: int) -> np.ndarray:
    """Slab bounds with (nearly) equal local non-zeros n_i + 2 o_i instead of equal cells -- the
    static estimate of Eq 5 for identical devices on irregular meshes (config 5)."""
    N = sys.nCells
    w = np.ones(N) + np.bincount(sys.lowerAddr, minlength=N) + np.bincount(sys.upperAddr, minlength=N)
    cw = np.concatenate([[0.0], np.cumsum(w)])
    targets = cw[-1] * np.arange(1, p) / p
    cuts = np.searchsorted(cw, targets, side="left")
    return np.concatenate([[0], cuts, [N]]).astype(np.int64)
