// ldu_amg.cuh -- aggregation-AMG preconditioner of libldu_b200 (NEXT-2; Table 2).
//
// The paper preconditions CG and pipelined CG with "a V-cycle of an aggregation-based AMG with
// weighted Jacobi iterations with omega = 4/3 as a smoother", the aggregates coming from "the
// parallel aggregation method based on a distance-2 maximal-independent-set".  Readings
// Z27-Z34 fix the rest.  Everything is built and applied on the device:
//   setup (ldu_amg_setup.cu): level-0 CSR from the handle's layout, MIS-2 aggregation by parallel
//     local-minimum rounds, Lanczos estimate of rho(D^-1 A), smoothed prolongator
//     P = (I - w D^-1 A) T, R = P^T and the Galerkin product A_c = P^T (A P) by sort-based
//     sparse products (expand -> CUB radix sort -> fixed-order segment sums), coarsest level
//     inverted densely (Gauss-Jordan);
//   solve (ldu_amg_solve.cuh, included by ldu_solve.cu): V-cycle kernels (level 0 in the handle's
//     DIA / SELL layout, coarser levels CSR with a sub-warp per row), AMG-PCG and AMG-PipeCG.
#pragma once

#include <vector>

#include "ldu_impl.cuh"

namespace ldu {

// CSR matrix in device memory, ascending columns per row, diagonal stored.
struct CsrMat {
  int nrows = 0, ncols = 0;
  long long nnz = 0;
  int* ptr = nullptr;     // [nrows + 1]
  int* col = nullptr;     // [nnz]
  double* val = nullptr;  // [nnz]
  int group = 1;          // lanes per row of the CSR-vector SpMV (power of two <= 32)
  // optional SELL-32 copy for the V-cycle (coarse A_l with near-uniform rows): 32-row slices,
  // lane-interleaved (col, val) pairs, padding = (a column of the row, 0.0): no break test
  bool useSell = false;
  long long* slicePtr = nullptr;  // [nslices + 1] in pair rows
  int* npairs = nullptr;          // [nslices]
  int2* scol = nullptr;
  double2* sval = nullptr;
  long long sellSlots = 0;        // pair slots x 32
  void release() {
    for (void* p : {(void*)ptr, (void*)col, (void*)val, (void*)slicePtr, (void*)npairs,
                    (void*)scol, (void*)sval})
      dfree(p);
    ptr = nullptr;
    col = nullptr;
    val = nullptr;
    slicePtr = nullptr;
    npairs = nullptr;
    scol = nullptr;
    sval = nullptr;
    nnz = 0;
    sellSlots = 0;
    useSell = false;
  }
};

// Device view of a CsrMat.
struct CsrView {
  int n;
  const int* __restrict__ ptr;
  const int* __restrict__ col;
  const double* __restrict__ val;
};

inline CsrView view(const CsrMat& m) { return CsrView{m.nrows, m.ptr, m.col, m.val}; }
inline SellView sell_view(const CsrMat& m) {
  return SellView{m.nrows, m.slicePtr, m.npairs, m.scol, m.sval};
}

// One level l < L of the hierarchy: A_l (n x n), aggregates, P_l (n x nc), R_l = P_l^T.
struct AmgLevel {
  int n = 0, nc = 0;
  CsrMat A;                  // A_l (level 0: CSR copy of the handle's matrix; setup / export)
  double* diag = nullptr;    // level 0: the handle's arrays (not owned)
  double* rD = nullptr;
  double omega = 0.0;        // Jacobi weight (4/3) / rho (reading Z27)
  int* agg = nullptr;        // [n] aggregate of each row
  CsrMat P, R;
  double* r = nullptr;       // V-cycle work: residual after the pre-sweep
  double* x = nullptr;       //               iterate after the prolongation
  double* f = nullptr;       // right-hand side (level >= 1)
  double* z = nullptr;       // V-cycle result (level >= 1)
  bool ownsDiag = false;
};

enum { PREC_AMG = 0, PREC_DIC = 1 };

// DIC factor (reading Z35): cells in level order (a cell's level = 1 + the
// largest level of its lower neighbours, so every cell of a level depends only on earlier levels
// in the forward sweep and on later levels in the backward sweep), with each cell's strictly-lower
// and strictly-upper couplings stored row by row in that order.
// ELL width of the DIC sweep rows: the widths k_dic_ell is instantiated for (1-4, 6, 8); rows
// wider than 8 keep CSR (returns 0).  Shared by the setup and the launch dispatch.
inline int dic_ell_width(int W) {
  if (W <= 0 || W > 8) return 0;
  return W <= 4 ? W : (W <= 6 ? 6 : 8);
}

struct DicFactor {
  int nLev = 0;
  std::vector<int> levPtr;       // host [nLev + 1] positions in perm
  int* perm = nullptr;           // [n] cell at level-order position k
  int *loPtr = nullptr, *loCol = nullptr;   // [n + 1], [nnzL]
  double* loVal = nullptr;
  int *upPtr = nullptr, *upCol = nullptr;   // [n + 1], [nnzU]
  double* upVal = nullptr;
  double* rD = nullptr;          // [n] reciprocal D of M = (D + L) D^-1 (D + L^T), by cell
  // level order is padded so that each level starts on a warp boundary (perm = -1 in the gaps):
  // no warp ever holds two levels, so the sync-free sweeps never wait inside a warp
  int nPad = 0;                  // padded positions
  unsigned* flag = nullptr;      // [n] per-cell epoch tag of the sync-free sweeps
  unsigned* ctl = nullptr;       // [3] epoch, forward ticket, backward ticket
  // ELL copy of the same rows (width = the largest row, padded with column -1), [w][nPad]
  // position-major so one level's rows are contiguous; used when the width is <= 8
  int wLo = 0, wUp = 0;
  int* dLevPtr = nullptr;        // device copy of levPtr (runs of narrow levels in one block)
  int *eLoCol = nullptr, *eUpCol = nullptr;
  double *eLoVal = nullptr, *eUpVal = nullptr;
  long long nnzL = 0;
  int maxLevel = 0;              // cells in the widest level
};

struct AmgHierarchy {
  int kind = PREC_AMG;       // PREC_AMG: the hierarchy below; PREC_DIC: `dic` (L = 0, no levels)
  DicFactor dic;
  ldu_amg_opts opts{};
  std::vector<AmgLevel> lv;  // levels 0 .. L-1
  int L = 0;
  int nc = 0;                // coarsest size (level L)
  CsrMat Ac;                 // coarsest matrix (export; level L == 0 => copy of A_0)
  double* Ainv = nullptr;    // [nc * nc] row-major inverse of the coarsest matrix (reading Z31)
  double* fL = nullptr;      // coarsest right-hand side / result (level L >= 1)
  double* zL = nullptr;
  double setupMs = 0.0;
  // AMG Krylov work vectors (lazily allocated by the solves)
  double *u = nullptr, *m = nullptr, *zk = nullptr, *qk = nullptr;
  // occupancy-sized grids of the level-0 kernels (set by the first V-cycle / solve)
  int gPre = 0, gPost = 0, gPassA = 0, gPipe = 0;
  // iteration-batch graphs: [pipelined + 2 * profile]
  cudaGraphExec_t graph[4] = {nullptr, nullptr, nullptr, nullptr};
  int graphBatch[4] = {0, 0, 0, 0};
  long long graphKernels[4] = {0, 0, 0, 0};
};

void amg_setup(ldu_handle h, const ldu_amg_opts* opts);
void dic_setup(ldu_handle h);
void dic_export(ldu_handle h, double* rD, ldu_dic_info* info);
void amg_release(ldu_handle h);
void amg_info(ldu_handle h, ldu_amg_info* out);
void amg_export(ldu_handle h, int level, int which, int* ptr, int* col, double* val);
void amg_export_agg(ldu_handle h, int level, int* agg);
// ldu_solve.cu
void amg_vcycle(ldu_handle h, const double* r, double* z, int kind);
ldu_status amg_solve(ldu_handle h, int kind, bool pipelined, const double* b, double* x, double tol,
                     int maxIter, const ldu_solve_opts* opts, int* nIter, double* finalRes);

// Priority key of node i in the MIS-2 rounds (reading Z30): keyMode 0 = index, 1 = the
// "lowbias32" mixer in the high word and the index in the low word (unique).
__host__ __device__ __forceinline__ unsigned amg_mix32(unsigned h) {
  h ^= h >> 16;
  h *= 0x7feb352du;
  h ^= h >> 15;
  h *= 0x846ca68bu;
  h ^= h >> 16;
  return h;
}
__host__ __device__ __forceinline__ unsigned long long amg_key(int i, int hashed) {
  return hashed ? (((unsigned long long)amg_mix32((unsigned)i) << 32) | (unsigned)i)
                : (unsigned long long)(unsigned)i;
}

}  // namespace ldu
