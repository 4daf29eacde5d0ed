// ldu_impl.cuh -- internal declarations of libldu_b200 (not part of the C ABI).
//
// Device-side matrix views, the solver state machine shared by the CG / pipelined-CG drivers,
// the deterministic block/grid reduction helpers, and the handle / comm structs.
// Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, readings Zn in DESIGN.md.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ldu.h"

namespace ldu {

constexpr int kMaxDiag = 8;      // DIA: max number of distinct symmetric offsets
constexpr int kBlock = 256;      // threads per block of every streaming pass
constexpr int kMaxVals = 4;      // values per fused reduction

// ---------------------------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------------------------
struct Error : std::runtime_error {
  ldu_status status;
  Error(ldu_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

void check_cuda(cudaError_t e, const char* what, const char* file, int line);
void check_nccl(ncclResult_t e, const char* what, const char* file, int line);
#define CUDA_CHECK(x) ::ldu::check_cuda((x), #x, __FILE__, __LINE__)
#define NCCL_CHECK(x) ::ldu::check_nccl((x), #x, __FILE__, __LINE__)

inline void fail_arg(const std::string& m) { throw Error(LDU_ERR_INVALID_ARG, m); }

// ---------------------------------------------------------------------------------------------
// matrix views (row-gathered, cell-ordered layouts)
// ---------------------------------------------------------------------------------------------

// Symmetric diagonal layout: U[k][c] = A[c][c + off[k]] = A[c + off[k]][c] (0 where no face).
// Row c reads U[k][c - off[k]] (lower side) and U[k][c] (upper side): each face coefficient is
// stored once; no column indices.
template <int ND>
struct DiaView {
  int n;
  int off[ND];
  const double* __restrict__ U[ND];
};

// SELL-32: slice s = rows [32 s, 32 s + 32); npairs[s] pair-rows; entry pair jj of row c lives at
// index (slicePtr[s] + jj) * 32 + (c & 31) of col / val (int2 / double2 -> 128-bit loads of
// fp64 coefficients).  Entries of a row are in ascending column order; padding has col = -1.
struct SellView {
  int n;
  const long long* __restrict__ slicePtr;
  const int* __restrict__ npairs;
  const int2* __restrict__ col;
  const double2* __restrict__ val;
};

// ---------------------------------------------------------------------------------------------
// solver state machine (device resident; one writer thread per control step)
// ---------------------------------------------------------------------------------------------
struct State {
  // per-solve inputs
  double tol;
  double relTol;     // OpenFOAM relTol (0 = off)
  double res0;       // criterion value of r0
  int minIter;       // OpenFOAM minIter
  int maxIter;
  int norm;          // LDU_NORM_*
  int record;        // record history
  int histCap;
  double* hist;      // device [histCap]
  // criterion
  double scale;      // ||b||_2 or OpenFOAM normFactor
  double xbar;       // OpenFOAM norm: mean of x0
  // classical CG
  double rho;        // rho_k = (r_k, z_k)
  double alpha;      // alpha_k (after control A) -- also the pending x update
  double beta;       // beta_k
  // pipelined CG
  double gamma_old, alpha_old;
  double pa, pb;     // alpha_i, beta_i of the current pipelined iteration
  double res;        // last criterion value
  int k;             // current iteration index
  int iter;          // x-updates done (reported nIter)
  int done;          // 1 => every pass exits at entry
  int status;        // ldu_status
  int xpending;      // classical: alpha * p_k not yet added to x
  int zero_x;        // ||b|| == 0 => x := 0
  int nRed;          // reductions consumed by a control step this solve (device counter)
};

// ---------------------------------------------------------------------------------------------
// handle / comm
// ---------------------------------------------------------------------------------------------
struct P2PDesc;  // ldu_p2p.cuh

struct DevInterface {
  int neighbRank;
  int nFaces;
  int offset;        // into the packed send / recv buffers
};

}  // namespace ldu

struct ldu_comm_s {
  int rank = 0, nRanks = 1, device = 0;
  ncclComm_t red = nullptr;   // reductions (allgather of fused partial sums)
  ncclComm_t halo = nullptr;  // halo send / recv
  // host bootstrap (ldu_comm_init_host): no NCCL; setup exchanges through the caller's host
  // all-gather, every in-solve exchange over the peer-memory mailboxes
  ldu_host_allgather_fn hostAllgather = nullptr;
  void* hostCtx = nullptr;
  bool nccl() const { return red != nullptr; }
};

namespace ldu {
struct AmgHierarchy;  // ldu_amg.cuh
}

struct ldu_handle_s {
  int device = 0;
  int n = 0, nf = 0;
  bool symmetric = true;              // lower == NULL or bitwise equal to upper
  ldu::AmgHierarchy* amg = nullptr;   // aggregation-AMG hierarchy (ldu_amg_setup)
  cudaStream_t own_stream = nullptr, stream = nullptr;
  cudaStream_t red_stream = nullptr, halo_stream = nullptr;
  int layout = 0;
  // DIA
  int nd = 0;
  int off[ldu::kMaxDiag] = {0};
  double* U = nullptr;  // [nd][n]
  // SELL
  long long* slicePtr = nullptr;
  int* npairs = nullptr;
  int2* col = nullptr;
  double2* val = nullptr;
  long long nPairSlots = 0;
  long long storedEntries = 0;
  // diagonal
  double* diag = nullptr;
  double* rD = nullptr;
  // work vectors (lazily allocated)
  double *x = nullptr, *r = nullptr, *p0 = nullptr, *p1 = nullptr, *q = nullptr;
  double *w = nullptr, *w2 = nullptr, *nv = nullptr, *z = nullptr, *s = nullptr;
  double *bbuf = nullptr, *ybuf = nullptr;
  // reductions
  double* partials = nullptr;  // [kMaxVals][maxParts]
  int maxParts = 0;
  unsigned* ticket = nullptr;
  double* sums = nullptr;      // [kMaxVals] local sums (send buffer of the allgather)
  double* gsums = nullptr;     // [nRanks][kMaxVals]
  ldu::State* st = nullptr;
  ldu::State* st_host = nullptr;  // pinned
  int grid = 0, block = ldu::kBlock;  // streaming passes
  int gridA = 0;                      // SpMV-bearing passes
  int gridSU = 0, suMinB = 0;         // single-rank fused pipelined pass (LDU_SU_MINB)
  int variant = 0;                    // DIA kernel variant (LDU_VARIANT)
  bool marchOk = false;               // plane-marching geometry applies
  bool marchStrict = false;           // ... with the performance geometry (one wave, lockstep)
  int mT = 0, mH = 0, mTiles = 0, mPlanes = 0, mChunk = 0;
  bool tmaOk = false, tmaStrict = false;  // TMA plane march (variant 4)
  int tT = 0, tTiles = 0, tChunk = 0, tGrid = 0, tL = 1;
  int chunkK = 2048;                  // variant 5: rows per chunk
  bool fusePipe = true;               // single rank: pipelined S+U fused (LDU_PIPE_FUSE)
  bool persist = false;               // single rank: persistent cooperative kernels
  bool pdl = false;                   // programmatic dependent launch in the multi-rank loop (LDU_PDL=1)
  int gridP = 0;                      // co-resident grid of the persistent kernels
  double* ppartials = nullptr;        // [2][kMaxVals][gridP]
  // history
  double* hist = nullptr;
  int histCap = 0;
  int histN = -1;
  // graphs
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    int batch = 0;
    long long kernels = 0;  // kernels per captured batch
  };
  Graph graphs[2][2];       // [pipelined][profile]
  Graph graphRR[2];         // pipelined with residual replacement, [profile]
  std::vector<cudaEvent_t> prof_ev;  // profile mode: 4 events per iteration of a batch
  std::vector<cudaEvent_t> trace;    // LDU_TRACE debug events
  // interfaces
  ldu_comm comm = nullptr;
  int nRanks = 1, rank = 0;
  std::vector<ldu::DevInterface> ifaces;
  int nIfFaces = 0;
  int* ifFaceCells = nullptr;   // [nIfFaces] packed
  double* ifCoeffs = nullptr;   // [nIfFaces]
  double* sendbuf = nullptr;    // [nIfFaces]
  double* recvbuf = nullptr;    // [nIfFaces]
  int nIfCells = 0;             // unique interface cells
  int* ifCell = nullptr;        // [nIfCells]
  int* ifCellPtr = nullptr;     // [nIfCells+1] into ifFaceIdx
  int* ifFaceIdx = nullptr;     // [nIfFaces] packed face index, interface order then face order
  // timing / stats
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_red = nullptr, ev_halo = nullptr, ev_pack = nullptr;
  ldu_solve_stats stats = {};
  long long matrixBytes = 0;
  // NVLink peer-memory communication (multi-rank; ldu_p2p.cuh)
  bool p2pOn = false;
  char* mailbox = nullptr;               // this rank's mailbox (peers write into it)
  std::vector<char*> peerMailbox;        // IPC-mapped mailboxes of the other ranks
  ldu::P2PDesc* p2pDesc = nullptr;       // device descriptor
  int* ifFaceIf = nullptr;               // [nIfFaces] interface index of each packed face
  // multi-rank fused pipelined pass (k_pipe_SU_mr): rows are visited in the rotated order
  // c = (mrGapStart + t) mod n so the largest interface-free run of rows (t < mrGapLen) comes
  // first and the rows that need the halo come last; mrTailIf[t - mrGapLen] = interface-cell
  // index of position t (or -1)
  int mrGapStart = 0, mrGapLen = 0;
  int* mrTailIf = nullptr;
  int4* mrTailMeta = nullptr;            // [n - mrGapLen]: {fi, kk, remote face, coeff index} (p2p)
  int gridSUmr = 0, mrPre = 4;           // grid / pre-phase rows per thread (LDU_MR_PRE: 0, 4, 8)
  bool mrFuse = true;                    // one kernel per iteration (LDU_MR_FUSE=0: pack + fix-up)
  bool mrFold = true;                    // ... with the control step in its last block (LDU_MR_FOLD)
  bool cgLL = true;                      // classical multi-rank: LL reductions (LDU_CG_LL)
  unsigned long long* tbuf = nullptr;    // LDU_TRACE device timestamps
};

namespace ldu {
struct P2PDesc;
void p2p_setup(ldu_handle h);
void host_allgather(ldu_comm cm, const void* send, void* recv, size_t bytes);
void p2p_release(ldu_handle h);
// setup (ldu_setup.cu)
void build_layout(ldu_handle h, const int* l, const int* u, const double* diag,
                  const double* lower, const double* upper, const ldu_interfaces* ifs);
// solves (ldu_solve.cu)
ldu_status solve(ldu_handle h, bool pipelined, const double* b, double* x, double tol,
                 int maxIter, const ldu_solve_opts* opts, int* nIter, double* finalRes);
void amul(ldu_handle h, const double* x, double* y);
void release_work(ldu_handle h);
void configure(ldu_handle h);
double stream_triad(int device, long long n, int reps);
// memory helpers
bool is_device_ptr(const void* p);
// Device allocations go through dmalloc / dfree, which record each block's size.  While an
// AllocHook is installed (the AMG setup's block cache, ldu_amg_setup.cu) dmalloc first asks it for
// a cached block (ownership passes to the caller) and dfree hands freed blocks to it instead of
// cudaFree -- a re-setup then reuses the previous hierarchy's memory in stream order.
struct AllocHook {
  virtual void* take(size_t bytes) = 0;          // a cached block of >= bytes, or nullptr
  virtual bool give(void* p, size_t bytes) = 0;  // keep a freed block (true) or not
  virtual ~AllocHook() {}
};
AllocHook*& alloc_hook();  // thread-local (ldu_setup.cu)
void alloc_register(void* p, size_t bytes);
size_t alloc_unregister(void* p);  // the block's size, 0 if unknown
size_t alloc_size(void* p);
void* dmalloc_raw(size_t bytes);  // cudaMalloc + register (trims the pool and retries once)
inline void dfree_raw(void* p) {
  if (!p) return;
  alloc_unregister(p);
  cudaFree(p);
}
template <class T>
T* dmalloc(size_t count) {
  if (count == 0) count = 1;
  if (AllocHook* hk = alloc_hook())
    if (void* q = hk->take(count * sizeof(T))) return static_cast<T*>(q);
  return static_cast<T*>(dmalloc_raw(count * sizeof(T)));
}
inline void dfree(void* p) {
  if (!p) return;
  if (AllocHook* hk = alloc_hook()) {
    const size_t b = alloc_size(p);
    if (b && hk->give(p, b)) return;
  }
  dfree_raw(p);
}
}  // namespace ldu
