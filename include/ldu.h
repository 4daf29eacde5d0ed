/*
 * ldu.h -- C ABI of the B200-native hot path of arXiv 1505.07630 (AlOnazi, Keyes, Lastovetsky,
 * Rychkov, "Design and Optimization of OpenFOAM-based CFD Applications for Hybrid and
 * Heterogeneous HPC Platforms", ParCFD 2014): the conjugate-gradient pressure/Poisson solve.
 *
 * Library: paper_1505_07630_b200/libldu_b200.so (hand-written CUDA for sm_100a + NCCL).
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n (reference text read at survey
 * time); readings "Zn" are listed in DESIGN.md.
 *
 * Conventions for every entry point:
 *   - returns ldu_status and never throws; on error ldu_last_error() gives a message
 *     (thread-local, valid until the next call on the same thread);
 *   - a handle is bound to the CUDA device that was current at ldu_setup (or the comm's device)
 *     and is NOT thread-safe: one handle per rank/device;
 *   - all vectors are fp64 (double), all indices int32 (OpenFOAM "label");
 *   - "host or device" pointer arguments are classified with cudaPointerGetAttributes; device
 *     pointers must live on the handle's device (e.g. torch CUDA tensors); host pointers may be
 *     pageable or pinned (pinned is faster);
 *   - across ranks (comm != NULL) ldu_amul and the solves are COLLECTIVE: every rank calls them
 *     in the same order with the same tol / maxIter / options.
 */
#ifndef LDU_B200_H
#define LDU_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define LDU_ABI_VERSION 2

typedef enum {
  LDU_OK = 0,                /* converged: finalRes < tol (or r == 0 exactly; reading Z2)         */
  LDU_NOT_CONVERGED = 1,     /* maxIter reached; x = last iterate; *finalRes >= tol (non-fatal)   */
  LDU_BREAKDOWN = 2,         /* (p,Ap) <= 0, delta - beta*gamma/alpha_old <= 0 or non-finite
                                (reading Z19); x = last valid iterate, *nIter names the iteration */
  LDU_ERR_INVALID_ARG = -1,  /* null pointer, nCells <= 0, nFaces < 0, index outside
                                [0, nCells), lowerAddr == upperAddr, diag <= 0 or non-finite,
                                maxIter < 0, tol < 0 or NaN, unknown option value            */
  LDU_ERR_CUDA = -2,         /* a CUDA runtime error (message in ldu_last_error)                 */
  LDU_ERR_NCCL = -3,         /* an NCCL error                                                    */
  LDU_ERR_OOM = -4,          /* device allocation failed                                         */
  LDU_ERR_STATE = -5         /* call not valid in the current state (e.g. history not recorded) */
} ldu_status;

typedef struct ldu_handle_s *ldu_handle; /* device layout, work vectors, graphs, streams       */
typedef struct ldu_comm_s *ldu_comm;     /* two NCCL communicators + their streams; NULL = 1 rank */

/* One processor interface ("halo-layer approach ... duplicates the cells next to a
 * processor boundary"; OpenFOAM processor patch).  faceCells[i] is the local cell next to patch
 * face i; coeffs[i] is OpenFOAM's interfaceBouCoeffs, i.e. the NEGATED off-diagonal, so the
 * interface contribution to y = A x is  y[faceCells[i]] -= coeffs[i] * x_neighbour[i]  (reading
 * Z10), where x_neighbour[i] is the neighbour rank's x at ITS faceCells[i] of the interface back
 * to this rank (both sides list shared faces in the same order, reading Z22).  Several
 * interfaces may name the same neighbour rank: they pair up in list order.  Host or device
 * pointers; copied by ldu_setup. */
typedef struct {
  int neighbRank;
  int nFaces;
  const int *faceCells;   /* [nFaces] */
  const double *coeffs;   /* [nFaces] */
} ldu_interface;

typedef struct {
  int nInterfaces;
  const ldu_interface *list; /* [nInterfaces] (host memory) */
  ldu_comm comm;             /* required when nInterfaces > 0 or when nRanks > 1 */
} ldu_interfaces;

/* ---- multi-GPU plumbing (P:95 one process per device) ---------------------- */

/* Writes a 128-byte NCCL unique id into id128 (call on rank 0, broadcast the bytes with
 * torch.distributed).  Errors: LDU_ERR_INVALID_ARG (NULL), LDU_ERR_NCCL. */
ldu_status ldu_get_unique_id(void *id128);

/* Creates the rank's communicators (one for reductions, one for halo exchange) on cudaDevice.
 * Collective over nRanks processes.  Errors: INVALID_ARG, CUDA, NCCL. */
ldu_status ldu_comm_init(int rank, int nRanks, const void *id128, int cudaDevice, ldu_comm *out);

/* Host bootstrap of a communicator without NCCL: every exchange inside the library (halo values
 * and the fused reductions) then runs over the peer-memory mailboxes only, and the
 * one-time setup exchange (CUDA IPC handles + interface tables) and setup barriers go through
 * the caller's host all-gather `fn`:
 *     fn(ctx, send, recv, bytes) gathers `bytes` bytes from every rank into recv[nRanks * bytes]
 *     in rank order (host memory) and returns 0 on success.
 * (e.g. torch.distributed over gloo: plumbing only, never called inside a solve.)  Unlike NCCL
 * this allows several ranks on ONE device (processes sharing a GPU through CUDA IPC), which is
 * how the multi-rank path is parity-tested on a single-GPU box.  The function pointer and ctx
 * must stay valid until ldu_comm_destroy.  Errors: INVALID_ARG, CUDA. */
typedef int (*ldu_host_allgather_fn)(void *ctx, const void *send, void *recv, unsigned long long bytes);
ldu_status ldu_comm_init_host(int rank, int nRanks, int cudaDevice, ldu_host_allgather_fn fn,
                              void *ctx, ldu_comm *out);
ldu_status ldu_comm_destroy(ldu_comm comm);

/* ---- setup ------------------------------------------------------------- */

/* Builds the device layout of an OpenFOAM lduMatrix (P:206 names lduMatrix; semantics in
 * SURVEY App. A): A[c][c] = diag[c], A[l[f]][u[f]] = upper[f], A[u[f]][l[f]] = lower[f]
 * (lower == NULL => symmetric, lower := upper).  Local owned rows only ("the local matrix
 * row dimension is number of cells within the subdomain"); couplings to other ranks come through
 * `interfaces`.  Faces need not be sorted (reading Z10); duplicate faces are allowed (summed).
 *
 *   nCells   > 0, nFaces >= 0 (int32; 2*nFaces < 2^31)
 *   lowerAddr, upperAddr [nFaces] int32 in [0, nCells), lowerAddr[f] != upperAddr[f]
 *   diag [nCells] > 0 and finite (Jacobi preconditioner M = diag(A), reading Z9)
 *   lower [nFaces] or NULL, upper [nFaces]
 *   interfaces: NULL for a single-rank matrix.
 * All arrays may be host or device pointers and are copied: the caller may free them on return.
 * With a multi-rank comm, ldu_setup is COLLECTIVE: it maps every rank's communication mailbox
 * (CUDA IPC over NVLink) and pairs the interfaces with the neighbours' (an interface without a
 * matching one of equal face count on its neighbour is LDU_ERR_INVALID_ARG).
 * The one-time conversion runs on the device; it chooses a row-gathered, cell-ordered layout
 * (DESIGN.md "Data layout"): symmetric banded matrices get a symmetric diagonal (DIA) layout
 * storing each face coefficient once; others a SELL-32 layout.  Both are deterministic: SpMV
 * sums diag first, then the row's entries in ascending column order, with no atomics.
 * Errors: INVALID_ARG (message names the first offending index), CUDA, OOM. */
ldu_status ldu_setup(int nCells, int nFaces, const int *lowerAddr, const int *upperAddr,
                     const double *diag, const double *lower, const double *upper,
                     const ldu_interfaces *interfaces, ldu_handle *out);

/* The caller's stream for all subsequent calls on h (e.g. torch.cuda.current_stream().cuda_stream):
 * every call orders its device work after the work already enqueued on that stream (device
 * inputs written there are safe to read) and that stream's later work after the call's.  NULL
 * (the default) = the legacy default stream, CUDA stream 0.  The library computes on its own
 * streams; the solves still return only after completion. */
ldu_status ldu_set_stream(ldu_handle h, void *cudaStream);

/* y = A x including processor interfaces ("point-to-point communication during the
 * matrix-vector multiplication"; SURVEY §8(a) a2+a3).  x, y: [nCells] host or device, must not
 * alias.  Collective when the handle has interfaces/comm.  Errors: INVALID_ARG, CUDA, NCCL. */
ldu_status ldu_amul(ldu_handle h, const double *x, double *y);

/* ---- solvers ----------------------------------------------------------------------------- */

/* Jacobi-preconditioned classical CG (Eq 4): per iteration one
 * SpMV with halo exchange and TWO global reductions ((p,q), then {(r,z),(r,r)} fused; reading
 * Z4).  b: [nCells] host or device (not modified); x: [nCells] host or device, IN/OUT (initial
 * guess in, solution out; reading Z8).  tol >= 0 applies to the criterion of the options (default
 * ||r||_2/||b||_2, reading Z1); tol = 0 runs exactly maxIter iterations (fixed-iteration
 * benchmarking).  Outputs: *nIter = number of x-updates (0 if the initial residual passes),
 * *finalRes = criterion value of the last recurrence residual.  If ||b||_2 == 0: x = 0,
 * nIter = 0, finalRes = 0.  Returns LDU_OK / LDU_NOT_CONVERGED / LDU_BREAKDOWN or an error. */
ldu_status pcg_solve(ldu_handle h, const double *b, double *x, double tol, int maxIter,
                     int *nIter, double *finalRes);

/* Ghysels-Vanroose pipelined CG with M = diag(A) ("only one collective communication per
 * loop body ... overlapped by the sparse matrix-vector multiplication"; SURVEY
 * §8(c) c3 Jacobi-specialised form): ONE fused reduction of (gamma, delta, ||r||^2) per
 * iteration.  Across ranks (peer-memory path) each iteration is ONE kernel: the SpMV with its
 * interface term, the recurrences, the next halo and the rank's share of the reduction written
 * into the peers' memory over NVLink (LL words), the control step in its last block.  Same
 * arguments and semantics as pcg_solve; the convergence test uses r_i at the top of iteration i
 * (reading Z3). */
ldu_status pipecg_solve(ldu_handle h, const double *b, double *x, double tol, int maxIter,
                        int *nIter, double *finalRes);

#define LDU_NORM_L2 0        /* ||r||_2 / ||b||_2 (default, reading Z1)                          */
#define LDU_NORM_OPENFOAM 1  /* sum|r| / (sum|A x0 - xbar sumA| + sum|b - xbar sumA| + 1e-20)    */

typedef struct {
  int norm;          /* LDU_NORM_L2 or LDU_NORM_OPENFOAM                                        */
  int recordHistory; /* 1: keep the criterion value of every iteration (ldu_get_residual_history) */
  int batch;         /* iterations per CUDA-graph launch; 0 = library default                   */
  int profile;       /* 1: bracket each pass kernel with CUDA events inside the graph and report
                        per-pass device time in ldu_solve_stats.passMs (one host sync per batch) */
  int minIter;       /* OpenFOAM minIter: the stopping test cannot pass before minIter x-updates
                        (maxIter still ends the solve, NOT_CONVERGED; reading Z26)            */
  int replaceEvery;  /* pipelined CG only (NEXT-4): > 0 recomputes r = b - A x, w = A M r, s = A p,
                        z = A M s from their definitions after every replaceEvery-th iteration
                        (residual replacement, attainable accuracy); 0 = off.  Single rank, and
                        across ranks on the peer-memory path (not with the NCCL fallback).   */
  double relTol;     /* OpenFOAM relTol: also converged when res < relTol * res0 (0 = off, Z26)  */
  double reserved2[2]; /* must be zero                                                          */
} ldu_solve_opts;

ldu_status pcg_solve_ex(ldu_handle h, const double *b, double *x, double tol, int maxIter,
                        const ldu_solve_opts *opts, int *nIter, double *finalRes);
ldu_status pipecg_solve_ex(ldu_handle h, const double *b, double *x, double tol, int maxIter,
                           const ldu_solve_opts *opts, int *nIter, double *finalRes);

/* Residual history of the last solve with recordHistory = 1: hostOut[0..*n-1] = criterion at
 * iterations 0..nIter (res0 first).  *n = min(cap, nIter + 1).  LDU_ERR_STATE if not recorded. */
ldu_status ldu_get_residual_history(ldu_handle h, double *hostOut, int cap, int *n);

typedef struct {
  double solveMs;        /* device time of the last solve (CUDA events, whole call)            */
  double iterMs;         /* device time of its iteration loop only (excludes r0 and finalize)  */
  long long kernels;     /* kernel launches of this library in the last call (graph nodes incl.) */
  long long allreduces;  /* cross-rank reductions completed in the last solve (per rank; 0 on one
                            rank): counted ON THE DEVICE by the control step that consumes each
                            gathered set of sums (reading Z4 / P:97: 2 per classical iteration,
                            1 per pipelined iteration, plus the r0 reductions)                  */
  long long haloBytes;   /* halo bytes sent by this rank in the last call                      */
  long long h2dBytes;    /* host->device bytes copied for b/x in the last call                 */
  long long d2hBytes;    /* device->host bytes copied for x in the last call                   */
  int iterations;        /* nIter of the last solve                                            */
  int reductions;        /* global (grid-wide, and cross-rank when multi-rank) reductions whose
                            sums were consumed by a control step in the last solve, counted on
                            the device; single rank included                                     */
  double passMs[2];      /* profile = 1: summed device time of pass 0 (classical A / pipelined S)
                            and pass 1 (classical B / pipelined U) over all iterations           */
  long long passLaunches[2]; /* number of timed launches of each pass                          */
} ldu_solve_stats;

ldu_status ldu_get_solve_stats(ldu_handle h, ldu_solve_stats *out);

#define LDU_LAYOUT_DIA_SYM 1  /* symmetric diagonal layout: offsets d_k, coefficient U_k[c] of
                                 face (c, c + d_k); each face stored once                      */
#define LDU_LAYOUT_SELL32 2   /* SELL-32: 32-row slices, per-slice width, lane-interleaved pairs */

typedef struct {
  int layout;            /* LDU_LAYOUT_*                                                        */
  int nDiagonals;        /* DIA: number of offsets                                              */
  int offsets[8];        /* DIA: ascending offsets                                              */
  long long storedEntries; /* off-diagonal entries stored (incl. padding)                       */
  long long matrixBytes;   /* device bytes of the matrix layout (incl. diag and 1/diag)         */
  int nCells, nFaces, nInterfaceFaces, nRanks, rank;
  int gridBlocks, blockThreads;
  int variant;           /* SpMV-pass kernel variant in use (env LDU_VARIANT)          */
  int pipeFused;         /* 1: single-rank pipelined CG runs S and U as one fused pass            */
} ldu_info;

ldu_status ldu_get_info(ldu_handle h, ldu_info *out);

/* fp64 STREAM triad a = b + s*c over n elements ("our implementation of the STREAM
 * benchmark"), repeated `reps` times on the handle's device; *gbps = best 24*n bytes / time.
 * Roofline denominator cross-check.  Uses its own scratch allocation. */
ldu_status ldu_stream_triad(int device, long long n, int reps, double *gbps);

/* ---- aggregation-AMG preconditioner ------------------------------------
 * "a V-cycle of an aggregation-based AMG with weighted Jacobi iterations with omega = 4/3
 * as a smoother ... the parallel aggregation method based on a distance-2
 * maximal-independent-set"; Table 2 runs it inside CG ("GPU AMG-CG") and pipelined
 * CG ("GPU AMG-PipeCG").  Readings Z27-Z34:
 *   - aggregates: greedy distance-2 MIS in the priority order of keyMode (Z30), all couplings
 *     strong (Z29); a DIA-layout coefficient that is exactly 0 is not a coupling (Z34);
 *   - prolongator: smoothed aggregation P = (I - w D^-1 A) T, w = (4/3) / (1.05 x the largest
 *     Ritz value of 20 Lanczos steps on D^-1/2 A D^-1/2) (Z27); R = P^T; A_c = P^T A P (Z32);
 *   - smoother: one pre- and one post-sweep of w-Jacobi from x = 0 (Z28);
 *   - coarsening while n > coarsest, the level shrinks and fewer than maxLevels levels exist; the
 *     coarsest system is solved exactly through its dense inverse (Z31; at most 8192 rows);
 *   - multi-rank handles: the hierarchy is built from the rank's local matrix (interfaces
 *     dropped), i.e. a block-Jacobi preconditioner across ranks; the Krylov operator keeps the
 *     interfaces (Z33).  ldu_amg_setup is then local (not collective); the solves are collective.
 * The matrix must be symmetric (lower == NULL or lower == upper); diag > 0.                     */
typedef struct {
  int coarsest;        /* stop coarsening at n <= coarsest; 0 = 64 (reading Z31)                 */
  int maxLevels;       /* at most this many coarsening steps; 0 = 25                             */
  int keyIndexOrder;   /* MIS-2 priority: 0 = hashed key (mix32(i) << 32 | i, default), 1 = index */
  int unsmoothed;      /* 0 = smoothed aggregation (default), 1 = piecewise-constant P = T       */
  int lanczosSteps;    /* Lanczos steps of the rho(D^-1 A) estimate; 0 = 20                      */
  int reserved[3];     /* must be zero                                                           */
} ldu_amg_opts;

#define LDU_AMG_MAX_LEVELS 25

typedef struct {
  int nLevels;                                  /* L = number of coarsening steps (0: direct)   */
  int coarsestN;                                /* rows of the coarsest matrix A_L              */
  int n[LDU_AMG_MAX_LEVELS + 1];                /* rows of A_0 .. A_L                            */
  long long nnzA[LDU_AMG_MAX_LEVELS + 1];       /* stored entries of A_0 .. A_L (diag included) */
  long long nnzP[LDU_AMG_MAX_LEVELS];           /* stored entries of P_0 .. P_{L-1} (= of R_l)  */
  double omega[LDU_AMG_MAX_LEVELS];             /* Jacobi weights w_0 .. w_{L-1}                 */
  double operatorComplexity;                    /* sum_l nnz(A_l) / nnz(A_0)                     */
  double setupMs;                               /* device time of ldu_amg_setup                  */
  long long deviceBytes;                        /* device memory held by the hierarchy           */
} ldu_amg_info;

/* Builds the hierarchy on the device for handle h (replacing any previous one).  opts NULL =>
 * defaults.  Errors: INVALID_ARG (bad option, non-symmetric matrix, coarsest level > 8192 rows),
 * STATE (a non-positive pivot in the coarsest inverse), CUDA, OOM. */
ldu_status ldu_amg_setup(ldu_handle h, const ldu_amg_opts *opts);
ldu_status ldu_amg_get_info(ldu_handle h, ldu_amg_info *out);

/* Host copies of level `level` of the hierarchy (for verification).  which = 0: A_level
 * (level in [0, L]); 1: P_level; 2: R_level (level in [0, L)).  ptr [rows + 1], col / val [nnz]
 * (sizes from ldu_amg_get_info; R_l has n[l+1] rows and nnzP[l] entries); any of them may be NULL.
 * ldu_amg_get_aggregates: agg [n[level]] (level in [0, L)).  STATE if no hierarchy. */
ldu_status ldu_amg_get_matrix(ldu_handle h, int level, int which, int *ptr, int *col, double *val);
ldu_status ldu_amg_get_aggregates(ldu_handle h, int level, int *agg);

/* z = B r: one V-cycle of the hierarchy (reading Z32).  r, z: [nCells] host or device. */
ldu_status ldu_amg_vcycle(ldu_handle h, const double *r, double *z);

/* AMG-preconditioned classical CG (SURVEY §8(c) c2 with z = B r; 3 global reductions per
 * iteration: (z, r), (p, Ap), crit(r)) and pipelined CG (c3 literal Ghysels-Vanroose form with
 * u = B r, m = B w; ONE fused reduction per iteration, overlapped across ranks with the V-cycle
 * and the SpMV of the next iteration).  Same arguments, options and semantics as
 * pcg_solve_ex; collective on multi-rank handles; STATE if ldu_amg_setup has not been called. */
ldu_status amg_pcg_solve(ldu_handle h, const double *b, double *x, double tol, int maxIter,
                         const ldu_solve_opts *opts, int *nIter, double *finalRes);
ldu_status amg_pipecg_solve(ldu_handle h, const double *b, double *x, double tol, int maxIter,
                            const ldu_solve_opts *opts, int *nIter, double *finalRes);

/* ---- DIC preconditioner ------------------------------------------------
 * OpenFOAM's default preconditioner for the pressure solve (DICPreconditioner [ext]; NEXT-1 "Optional
 * DIC preconditioner (OpenFOAM's default for p)"), readings Z35-Z36:
 *   M = (D + L) D^-1 (D + L^T), L = strictly-lower part of the local matrix,
 *   D_c = A_cc - sum_{l < c} A_cl^2 / D_l  (so diag(M) = diag(A); IC(0) on hex meshes);
 *   z = M^-1 r by a forward and a backward triangular sweep.
 * The sweeps are level-scheduled on the device (a cell's level = 1 + the largest level of its
 * lower neighbours; one launch per level and sweep: 3n-2 levels on an n^3 lexicographic hex mesh),
 * so results equal the sequential face loops up to the summation order within a row.  Multi-rank
 * handles: the factor of the rank's local matrix (interfaces dropped), i.e. block-Jacobi DIC, as
 * OpenFOAM does on processor boundaries; ldu_dic_setup is then local, the solves collective.
 * Symmetric matrices only.  A setup replaces any AMG hierarchy on the handle and vice versa.
 * Errors: INVALID_ARG (non-symmetric matrix), STATE (a pivot D_c <= 0; or, for the calls below,
 * no DIC factor), CUDA, OOM. */
typedef struct {
  int nLevels;              /* number of level-scheduling levels                                  */
  int widestLevel;          /* cells in the widest level                                          */
  long long lowerEntries;   /* stored strictly-lower couplings (non-zero)                         */
  double setupMs;           /* device + host time of ldu_dic_setup                                */
  int ellWidthLower;        /* padded ELL width of the forward-sweep rows (0 = CSR rows used)     */
  int ellWidthUpper;        /* padded ELL width of the backward-sweep rows (0 = CSR rows used)    */
} ldu_dic_info;

ldu_status ldu_dic_setup(ldu_handle h);
/* rD: [nCells] host or device or NULL, receives 1 / D_c; info may be NULL. */
ldu_status ldu_dic_get(ldu_handle h, double *rD, ldu_dic_info *info);
/* z = M^-1 r.  r, z: [nCells] host or device, must not alias. */
ldu_status ldu_dic_apply(ldu_handle h, const double *r, double *z);
/* DIC-preconditioned classical CG (c2 with z = M^-1 r) and pipelined CG (c3 literal GV form with
 * u = M^-1 r, m = M^-1 w; one fused reduction per iteration).  Same arguments, options and
 * semantics as amg_pcg_solve / amg_pipecg_solve (replaceEvery unsupported). */
ldu_status dic_pcg_solve(ldu_handle h, const double *b, double *x, double tol, int maxIter,
                         const ldu_solve_opts *opts, int *nIter, double *finalRes);
ldu_status dic_pipecg_solve(ldu_handle h, const double *b, double *x, double tol, int maxIter,
                            const ldu_solve_opts *opts, int *nIter, double *finalRes);

ldu_status ldu_destroy(ldu_handle h);
const char *ldu_last_error(void);
int ldu_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LDU_B200_H */
