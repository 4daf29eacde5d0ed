// ldu_solve.cu -- the hot path: SpMV, Jacobi-PCG and pipelined CG drivers.
//
// Classical Jacobi-PCG, two fused HBM passes per iteration:
//   pass A_k : x += alpha_{k-1} p_{k-1};  p_k = rD.r + beta_k p_{k-1} (recomputed at every
//              neighbour, never re-read);  q = A p_k;  partial (p_k, q)        -> control A (alpha)
//   pass B_k : r -= alpha_k q;  partials (r, rD.r), crit(r)                    -> control B (beta, test)
//   p is ping-pong buffered (pass A gathers p_{k-1} while writing p_k).
// Pipelined CG (Ghysels-Vanroose, Jacobi form: u = rD.r, m = rD.w,
// q = rD.s are never stored):
//   pass S_i : n = A (rD.w)                      (overlaps the single allgather of the partials)
//   control  : alpha_i, beta_i, convergence test on r_i
//   pass U_i : z = n + b z; s = w + b s; p = rD.r + b p; x += a p; r -= a s; w -= a z;
//              partials (r, rD.r), (w, rD.r), crit(r)  -> one fused reduction
// Scalars never leave the device; iterations run as CUDA-graph batches whose kernels exit at
// entry once the device `done` flag is set; the host reads the state once per batch.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <utility>
#include <cstdlib>
#include <vector>

#include "ldu_dia.cuh"
#include "ldu_march.cuh"
#include "ldu_tma.cuh"
#include "ldu_persist.cuh"
#include "ldu_kernels.cuh"

namespace ldu {

namespace {

// ---------------------------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------------------------
#define GRID_STRIDE(c, n) \
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < (n); c += gridDim.x * blockDim.x)

// y = A x over internal faces (diag first, ascending columns).
template <class Fmt>
__global__ void __launch_bounds__(kBlock) k_amul(Fmt A, const double* __restrict__ diag,
                                                 const double* __restrict__ x,
                                                 double* __restrict__ y) {
  GRID_STRIDE(c, A.n) {
    y[c] = row_apply(A, c, __ldg(diag + c) * __ldg(x + c), [&](int j) { return __ldg(x + j); });
  }
}

// Interface update (reading Z10, Z23): y[cell] -= sum_f coeff[f] * recv[f] for every
// interface cell, contributions in interface order then face order.
__global__ void k_iface_apply(int nIfCells, const int* __restrict__ cell,
                              const int* __restrict__ ptr, const int* __restrict__ fidx,
                              const double* __restrict__ coeff, const double* __restrict__ recv,
                              double* __restrict__ y, const State* st) {
  if (st && st->done) return;
  GRID_STRIDE(i, nIfCells) {
    double corr = 0.0;
    for (int t = ptr[i]; t < ptr[i + 1]; ++t) corr = fma(coeff[fidx[t]], recv[fidx[t]], corr);
    y[cell[i]] -= corr;
  }
}

// Interface update of q = A p_k in pass A, plus the (p, q) correction partial.
__global__ void __launch_bounds__(kBlock) k_iface_cg(int nIfCells, const int* __restrict__ cell,
                                                     const int* __restrict__ ptr,
                                                     const int* __restrict__ fidx,
                                                     const double* __restrict__ coeff,
                                                     const double* __restrict__ recv,
                                                     double* __restrict__ q, const double* p0,
                                                     const double* p1, State* st, Red rd) {
  if (st->done) return;
  const double* __restrict__ pnew = (st->k & 1) ? p1 : p0;
  double v[1] = {0.0};
  GRID_STRIDE(i, nIfCells) {
    double corr = 0.0;
    for (int t = ptr[i]; t < ptr[i + 1]; ++t) corr = fma(coeff[fidx[t]], recv[fidx[t]], corr);
    const int c = cell[i];
    q[c] -= corr;
    v[0] -= pnew[c] * corr;
  }
  finish_reduction<1>(v, rd, st);
}

enum Pack : int { PACK_PLAIN = 0, PACK_SCALED = 1, PACK_CG_P = 2, PACK_SCALED_W = 3, PACK_SCALED_LL = 4,
                  PACK_SCALED_LL_W = 5, PACK_CG_P_LL = 6 };

// Halo send buffer: the SpMV operand at the interface cells.
__global__ void k_pack(int nIfFaces, const int* __restrict__ fc, int mode,
                       const double* __restrict__ a, const double* __restrict__ rD,
                       const double* p0, const double* p1, const State* st,
                       double* __restrict__ send) {
  if (st && st->done) return;
  double beta = 0.0;
  const double* pold = nullptr;
  if (mode == PACK_CG_P) {
    beta = st->beta;
    pold = (st->k & 1) ? p0 : p1;
  }
  GRID_STRIDE(i, nIfFaces) {
    const int c = fc[i];
    double v = a[c];
    if (mode == PACK_SCALED) v = rD[c] * v;
    else if (mode == PACK_CG_P) v = fma(beta, pold[c], rD[c] * v);
    send[i] = v;
  }
}

__global__ void k_fill(int n, double v, double* __restrict__ y) {
  GRID_STRIDE(c, n) y[c] = v;
}

// OpenFOAM norm, step 1: partials [sum x0, cell count] -> xbar (reading Z1)
__global__ void __launch_bounds__(kBlock) k_sum_x(int n, const double* __restrict__ x, State* st,
                                                  Red rd) {
  double v[2] = {0.0, 0.0};
  GRID_STRIDE(c, n) {
    v[0] += x[c];
    v[1] += 1.0;
  }
  finish_reduction<2>(v, rd, st);
}

// r = b - Ax (Ax precomputed incl. interfaces).  Partials:
//   L2:       [sum b^2, (r, rD.r), sum r^2]
//   OpenFOAM: [sum |Ax - xbar sumA| + |b - xbar sumA|, (r, rD.r), sum |r|]
__global__ void __launch_bounds__(kBlock) k_resid(int n, const double* __restrict__ b,
                                                  const double* __restrict__ Ax,
                                                  const double* __restrict__ sumA,
                                                  const double* __restrict__ rD,
                                                  double* __restrict__ r, State* st, Red rd) {
  const bool l2 = st->norm == LDU_NORM_L2;
  const double xbar = st->xbar;
  double v[3] = {0.0, 0.0, 0.0};
  GRID_STRIDE(c, n) {
    const double bc = b[c], ax = Ax[c];
    const double rc = bc - ax;
    r[c] = rc;
    if (l2) {
      v[0] += bc * bc;
      v[2] += rc * rc;
    } else {
      const double sa = xbar * sumA[c];
      v[0] += fabs(ax - sa) + fabs(bc - sa);
      v[2] += fabs(rc);
    }
    v[1] += rc * (rD[c] * rc);
  }
  finish_reduction<3>(v, rd, st);
}

// classical pass A_k (see file header)
template <class Fmt>
__global__ void __launch_bounds__(kBlock) k_cg_passA(Fmt A, const double* __restrict__ rD,
                                                     const double* __restrict__ r, double* p0,
                                                     double* p1, double* __restrict__ q,
                                                     double* __restrict__ x, State* st, Red rd) {
  if (st->done) return;
  const int k = st->k;
  const double beta = st->beta, alpha = st->alpha;
  const double* __restrict__ pold = (k & 1) ? p0 : p1;
  double* __restrict__ pnew = (k & 1) ? p1 : p0;
  double v[1] = {0.0};
  GRID_STRIDE(c, A.n) {
    auto op = [&](int j) { return fma(beta, __ldg(pold + j), __ldg(rD + j) * __ldg(r + j)); };
    const double po = __ldg(pold + c);
    const double pc = fma(beta, po, __ldg(rD + c) * __ldg(r + c));
    const double qc = row_apply(A, c, pc / __ldg(rD + c), op);
    pnew[c] = pc;
    q[c] = qc;
    x[c] = fma(alpha, po, x[c]);
    v[0] = fma(pc, qc, v[0]);
  }
  finish_reduction<1>(v, rd, st);
}

// classical pass A_k, chunked wavefront: block b walks chunks b, b + G, ... of K consecutive rows,
// 256 rows at a time, so the +-nx gathers of a tile were loaded by the same block one tile
// earlier (L1 hits) while whole chunks still advance as a wavefront (+-nx*ny gathers in L2).
template <class Fmt>
__global__ void __launch_bounds__(kBlock) k_cg_passA_chunk(Fmt A, const double* __restrict__ rD,
                                                           const double* __restrict__ r, double* p0,
                                                           double* p1, double* __restrict__ q,
                                                           double* __restrict__ x, State* st, Red rd,
                                                           int K) {
  if (st->done) return;
  const int k = st->k;
  const double beta = st->beta, alpha = st->alpha;
  const double* __restrict__ pold = (k & 1) ? p0 : p1;
  double* __restrict__ pnew = (k & 1) ? p1 : p0;
  double v[1] = {0.0};
  const int nchunks = (A.n + K - 1) / K;
  for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int end = min(A.n, (ch + 1) * K);
    for (int c = ch * K + threadIdx.x; c < end; c += kBlock) {
      auto op = [&](int j) { return fma(beta, __ldg(pold + j), __ldg(rD + j) * __ldg(r + j)); };
      const double po = __ldg(pold + c);
      const double pc = fma(beta, po, __ldg(rD + c) * __ldg(r + c));
      const double qc = row_apply(A, c, pc / __ldg(rD + c), op);
      pnew[c] = pc;
      q[c] = qc;
      x[c] = fma(alpha, po, x[c]);
      v[0] = fma(pc, qc, v[0]);
    }
  }
  finish_reduction<1>(v, rd, st);
}

// out = A (rD.in), chunked wavefront (see k_cg_passA_chunk)
template <class Fmt>
__global__ void __launch_bounds__(kBlock) k_spmv_scaled_chunk(Fmt A, const double* __restrict__ rD,
                                                              const double* __restrict__ in,
                                                              double* __restrict__ out,
                                                              const State* st, int K) {
  if (st->done) return;
  const int nchunks = (A.n + K - 1) / K;
  for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int end = min(A.n, (ch + 1) * K);
    for (int c = ch * K + threadIdx.x; c < end; c += kBlock)
      out[c] = row_apply(A, c, __ldg(in + c), [&](int j) { return __ldg(rD + j) * __ldg(in + j); });
  }
}

// classical pass A_k split in two (variant 7): A1 streams p_k = rD.r + beta p_{k-1} and
// x += alpha_{k-1} p_{k-1} (48N bytes); A2 is a plain SpMV q = A p_k gathering one array, with
// partial (p_k, q) (48N bytes, diag term p / rD).  96N instead of the fused 80N, but no operand
// recomputation at the neighbours.
__global__ void __launch_bounds__(kBlock) k_cg_passA1(int n, const double* __restrict__ rD,
                                                      const double* __restrict__ r, double* p0,
                                                      double* p1, double* __restrict__ x,
                                                      const State* st) {
  if (st->done) return;
  const int k = st->k;
  const double beta = st->beta, alpha = st->alpha;
  const double* __restrict__ pold = (k & 1) ? p0 : p1;
  double* __restrict__ pnew = (k & 1) ? p1 : p0;
  GRID_STRIDE(c, n) {
    const double po = pold[c];
    pnew[c] = fma(beta, po, rD[c] * r[c]);
    x[c] = fma(alpha, po, x[c]);
  }
}

template <class Fmt>
__global__ void __launch_bounds__(kBlock, 8) k_cg_passA2(Fmt A, const double* __restrict__ rD,
                                                      const double* p0, const double* p1,
                                                      double* __restrict__ q, State* st, Red rd) {
  if (st->done) return;
  const double* __restrict__ p = (st->k & 1) ? p1 : p0;
  double v[1] = {0.0};
  GRID_STRIDE(c, A.n) {
    const double pc = __ldg(p + c);
    const double qc = row_apply(A, c, pc / __ldg(rD + c), [&](int j) { return __ldg(p + j); });
    q[c] = qc;
    v[0] = fma(pc, qc, v[0]);
  }
  finish_reduction<1>(v, rd, st);
}

// classical pass A_k, DIA layout with off[0] == 1: the operand p_k at c-1 / c+1 is the
// neighbouring lane's own value (warp shuffle), as is the coefficient U_0[c-1]; only the lanes at
// the warp edges load them.  Saves 7 of the ~28 loads per row of the row gather (variant 6).
template <int ND>
__global__ void __launch_bounds__(kBlock) k_cg_passA_shfl(DiaView<ND> A,
                                                          const double* __restrict__ rD,
                                                          const double* __restrict__ r, double* p0,
                                                          double* p1, double* __restrict__ q,
                                                          double* __restrict__ x, State* st,
                                                          Red rd) {
  if (st->done) return;
  const int k = st->k;
  const double beta = st->beta, alpha = st->alpha;
  const double* __restrict__ pold = (k & 1) ? p0 : p1;
  double* __restrict__ pnew = (k & 1) ? p1 : p0;
  const int lane = threadIdx.x & 31;
  const int n = A.n;
  auto op = [&](int j) { return fma(beta, __ldg(pold + j), __ldg(rD + j) * __ldg(r + j)); };
  double v[1] = {0.0};
  // whole warps iterate together (shuffles need all lanes); rows >= n are masked
  for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    const int c = base + threadIdx.x;
    const bool in = c < n;
    const int cc = in ? c : n - 1;
    const double po = __ldg(pold + cc);
    const double rdc = __ldg(rD + cc);
    const double pc = fma(beta, po, rdc * __ldg(r + cc));
    const double u0 = __ldg(A.U[0] + cc);
    double pm = __shfl_up_sync(0xffffffffu, pc, 1);
    double pp = __shfl_down_sync(0xffffffffu, pc, 1);
    double um = __shfl_up_sync(0xffffffffu, u0, 1);
    if (lane == 0) {
      pm = cc >= 1 ? op(cc - 1) : 0.0;
      um = cc >= 1 ? __ldg(A.U[0] + cc - 1) : 0.0;
    }
    if (lane == 31 || c == n - 1) pp = cc + 1 < n ? op(cc + 1) : 0.0;
    if (cc < 1) um = 0.0;
    double s = pc / rdc;
    // ascending columns: far lower offsets, c-1, c+1, far upper offsets
#pragma unroll
    for (int kk = ND - 1; kk >= 1; --kk) {
      const int j = cc - A.off[kk];
      if (j >= 0) s = fma(__ldg(A.U[kk] + j), op(j), s);
    }
    s = fma(um, pm, s);
    s = fma(u0, pp, s);
#pragma unroll
    for (int kk = 1; kk < ND; ++kk) {
      const int j = cc + A.off[kk];
      if (j < n) s = fma(__ldg(A.U[kk] + cc), op(j), s);
    }
    if (in) {
      pnew[c] = pc;
      q[c] = s;
      x[c] = fma(alpha, po, x[c]);
      v[0] = fma(pc, s, v[0]);
    }
  }
  finish_reduction<1>(v, rd, st);
}

// classical pass A_k, DIA layout, all loads of ROWS rows hoisted (ldu_dia.cuh)
template <int ND, int ROWS>
__global__ void __launch_bounds__(kBlock) k_cg_passA_dia(DiaView<ND> A,
                                                         const double* __restrict__ rD,
                                                         const double* __restrict__ r, double* p0,
                                                         double* p1, double* __restrict__ q,
                                                         double* __restrict__ x, State* st, Red rd) {
  if (st->done) return;
  const int k = st->k;
  const double beta = st->beta, alpha = st->alpha;
  const double* __restrict__ pold = (k & 1) ? p0 : p1;
  double* __restrict__ pnew = (k & 1) ? p1 : p0;
  const OpCgP op{rD, r, pold, beta};
  double v[1] = {0.0};
  DIA_TILE_LOOP(base, A.n, ROWS) {
    DiaRow<ND, OpCgP> row[ROWS];
    double xc[ROWS];
#pragma unroll
    for (int u = 0; u < ROWS; ++u) {
      const int c = (int)min(base + u * blockDim.x + threadIdx.x, (long long)A.n - 1);
      row[u].load(A, op, c);
      xc[u] = x[c];
    }
#pragma unroll
    for (int u = 0; u < ROWS; ++u) {
      const long long c = base + u * blockDim.x + threadIdx.x;
      if (c < A.n) {
        const double pc = op.eval(row[u].own);
        const double qc = row[u].apply(op, pc / row[u].own[0]);
        pnew[c] = pc;
        q[c] = qc;
        x[c] = fma(alpha, row[u].own[2], xc[u]);
        v[0] = fma(pc, qc, v[0]);
      }
    }
  }
  finish_reduction<1>(v, rd, st);
}

// classical pass B_k
template <bool LL = false>  // LL: multi-rank, the reduction and control B in the last block
__global__ void __launch_bounds__(kBlock) k_cg_passB(int n, const double* __restrict__ rD,
                                                     const double* __restrict__ q,
                                                     double* __restrict__ r, State* st, Red rd) {
  if (st->done) return;
  const double alpha = st->alpha;
  const bool l2 = st->norm == LDU_NORM_L2;
  double v[2] = {0.0, 0.0};
  GRID_STRIDE(c, n) {
    const double rc = fma(-alpha, q[c], r[c]);
    r[c] = rc;
    v[0] = fma(rc, rD[c] * rc, v[0]);
    v[1] += l2 ? rc * rc : fabs(rc);
  }
  if (LL) finish_reduction_ll<2>(v, rd, st);
  else finish_reduction<2>(v, rd, st);
}

// classical exit: x += alpha_k p_k if pending
__global__ void k_cg_final(int n, const double* p0, const double* p1, double* __restrict__ x,
                           const State* st) {
  if (st->zero_x) {  // ||b|| = 0 => x = 0 (reading Z1), decided on the device
    GRID_STRIDE(c, n) x[c] = 0.0;
    return;
  }
  if (!st->xpending) return;
  const double alpha = st->alpha;
  const double* __restrict__ p = (st->k & 1) ? p1 : p0;
  GRID_STRIDE(c, n) x[c] = fma(alpha, p[c], x[c]);
}

// out = A (rD.in) over internal faces; diag term diag*rD*in taken as in exactly.
template <class Fmt>
__global__ void __launch_bounds__(kBlock) k_spmv_scaled(Fmt A, const double* __restrict__ rD,
                                                        const double* __restrict__ in,
                                                        double* __restrict__ out,
                                                        const State* st) {
  if (st->done) return;
  GRID_STRIDE(c, A.n) {
    out[c] = row_apply(A, c, __ldg(in + c), [&](int j) { return __ldg(rD + j) * __ldg(in + j); });
  }
}

// pipelined: partials [gamma = (r, rD.r), delta = (w, rD.r), crit(r)] over final r, w
__global__ void __launch_bounds__(kBlock) k_pipe_dots(int n, const double* __restrict__ rD,
                                                      const double* __restrict__ r,
                                                      const double* __restrict__ w, State* st,
                                                      Red rd) {
  if (st->done) return;
  const bool l2 = st->norm == LDU_NORM_L2;
  double v[3] = {0.0, 0.0, 0.0};
  GRID_STRIDE(c, n) {
    const double rc = r[c], u = rD[c] * rc;
    v[0] = fma(rc, u, v[0]);
    v[1] = fma(w[c], u, v[1]);
    v[2] += l2 ? rc * rc : fabs(rc);
  }
  finish_reduction<3>(v, rd, st);
}

// pipelined pass U_i (see file header)
__global__ void __launch_bounds__(kBlock) k_pipe_U(int n, const double* __restrict__ rD,
                                                   const double* __restrict__ nv,
                                                   double* __restrict__ z, double* __restrict__ s,
                                                   double* __restrict__ p, double* __restrict__ x,
                                                   double* __restrict__ r, double* __restrict__ w,
                                                   State* st, Red rd) {
  if (st->done) return;
  const double a = st->pa, b = st->pb;
  const bool l2 = st->norm == LDU_NORM_L2;
  double v[3] = {0.0, 0.0, 0.0};
  GRID_STRIDE(c, n) {
    const double rdc = rD[c], rc0 = r[c], wc0 = w[c];
    const double zc = fma(b, z[c], nv[c]);
    const double sc = fma(b, s[c], wc0);
    const double pc = fma(b, p[c], rdc * rc0);
    z[c] = zc;
    s[c] = sc;
    p[c] = pc;
    x[c] = fma(a, pc, x[c]);
    const double rc = fma(-a, sc, rc0);
    const double wc = fma(-a, zc, wc0);
    r[c] = rc;
    w[c] = wc;
    const double u = rdc * rc;
    v[0] = fma(rc, u, v[0]);
    v[1] = fma(wc, u, v[1]);
    v[2] += l2 ? rc * rc : fabs(rc);
  }
  finish_reduction<3>(v, rd, st);
}

// pipelined, single rank: passes S_i and U_i fused.  With one rank there is no global reduction
// to hide behind the SpMV, so n_i = A (rD.w_i) is consumed row by row and never stored (saves the
// 16N bytes of writing and re-reading n).  w is ping-pong buffered: neighbours gather w_i while
// the pass writes w_{i+1}.
// MINB = 6 resident blocks per SM caps the registers at 40 (the unconstrained allocation, 48-84,
// leaves 3-5 blocks): 343 vs 381-418 us per launch at 256^3, 0.96 of the measured copy bandwidth
template <class Fmt, int MINB = 6>
__global__ void __launch_bounds__(kBlock, MINB) k_pipe_SU(Fmt A, const double* __restrict__ rD,
                                                    double* w0, double* w1,
                                                    double* __restrict__ z, double* __restrict__ s,
                                                    double* __restrict__ p, double* __restrict__ x,
                                                    double* __restrict__ r, State* st, Red rd) {
  pdl_wait();  // launched programmatically after the control step (no-op otherwise)
  if (st->done) return;
  if (threadIdx.x == 0) tstamp(rd.p2p, st->k, 2, 1);
  const double a = st->pa, b = st->pb;
  const bool l2 = st->norm == LDU_NORM_L2;
  const double* __restrict__ w = (st->k & 1) ? w1 : w0;
  double* __restrict__ wn = (st->k & 1) ? w0 : w1;
  double v[3] = {0.0, 0.0, 0.0};
  GRID_STRIDE(c, A.n) {
    const double wc0 = __ldg(w + c);
    const double nc = row_apply(A, c, wc0, [&](int j) { return __ldg(rD + j) * __ldg(w + j); });
    const double rdc = __ldg(rD + c), rc0 = r[c];
    const double zc = fma(b, z[c], nc);
    const double sc = fma(b, s[c], wc0);
    const double pc = fma(b, p[c], rdc * rc0);
    z[c] = zc;
    s[c] = sc;
    p[c] = pc;
    x[c] = fma(a, pc, x[c]);
    const double rc = fma(-a, sc, rc0);
    const double wc = fma(-a, zc, wc0);
    r[c] = rc;
    wn[c] = wc;
    const double u = rdc * rc;
    v[0] = fma(rc, u, v[0]);
    v[1] = fma(wc, u, v[1]);
    v[2] += l2 ? rc * rc : fabs(rc);
  }
  pdl_trigger();  // the fix-up may launch now; it waits for this grid before reading
  if (threadIdx.x == 0) tstamp(rd.p2p, st->k, 3, 2);
  finish_reduction<3>(v, rd, st);
}

// ---- NVLink peer-memory halo and reductions (ldu_p2p.cuh) ----------------------------------

// Halo send fused with the pack: the operand at every interface face is stored straight into the
// neighbour's mailbox over NVLink; the last block raises the neighbours' flags.
// gateK / gateDone (NULL = ungated, k = 0): the iteration index that selects the ping-pong half
// and the done flag that skips the send.  The fused pipelined loop passes the fix-up's snapshot
// (P2PDesc::snapK / snapDone), never the live State the concurrent control step is updating.
__global__ void __launch_bounds__(kBlock) k_pack_p2p(int nIfFaces, const int* __restrict__ fc,
                                                     const int* __restrict__ faceIf, int mode,
                                                     const double* a,
                                                     const double* __restrict__ rD,
                                                     const double* p0, const double* p1,
                                                     const State* st, const int* gateK,
                                                     const int* gateDone, P2PDesc* d,
                                                     unsigned* ticket) {
  if (gateDone && *gateDone) return;
  const int k = gateK ? *gateK : 0;
  double beta = 0.0;
  const double* pold = nullptr;
  if (mode == PACK_CG_P || mode == PACK_CG_P_LL) {  // classical: forked / joined between two control steps
    beta = st->beta;
    pold = (k & 1) ? p0 : p1;
  }
  const unsigned long long seq = d->seqHaloSend + 1;
  const int par = (int)(seq & 1);
  if (mode == PACK_SCALED_W || mode == PACK_SCALED_LL_W) a = (k & 1) ? p0 : p1;  // w_{i+1}
  const bool ll = mode == PACK_SCALED_LL || mode == PACK_SCALED_LL_W || mode == PACK_CG_P_LL;
  GRID_STRIDE(i, nIfFaces) {
    const int c = fc[i];
    double v = a[c];
    if (mode == PACK_CG_P || mode == PACK_CG_P_LL) v = fma(beta, pold[c], rD[c] * v);
    else if (mode != PACK_PLAIN) v = rD[c] * v;  // rD w
    const int kk = faceIf[i];
    if (ll) {  // LL words (one-kernel loop, classical CG with cgLL): no flag release
      uint64_t* dst = mb_haloll(d->base[d->ifNeighbor[kk]], par, d->ifRemoteTotal[kk]);
      ll_store(dst + 2 * (size_t)(d->ifRemoteOff[kk] + (i - d->ifLocalOff[kk])), v, (uint32_t)seq);
    } else {
      double* dst = mb_recv(d->base[d->ifNeighbor[kk]], par, d->ifRemoteTotal[kk]);
      dst[d->ifRemoteOff[kk] + (i - d->ifLocalOff[kk])] = v;
    }
  }
  // one cumulative system-scope fence per block (after the barrier) orders the whole block's
  // remote stores before its ticket; the last block then releases the flags
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    if (ll) __threadfence();  // LL words carry their own sequence numbers: no system fence
    else __threadfence_system();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    if (!ll) p2p_release_halo(d, seq);
    d->seqHaloSend = seq;
    *ticket = 0u;
  }
}

// Wait for this exchange's halo (flags of all my interfaces), then read my mailbox.
__device__ __forceinline__ const double* p2p_wait_halo(P2PDesc* d, int nIfFaces) {
  const unsigned long long seq = d->seqHalo + 1;
  const int par = (int)(seq & 1);
  char* me = d->base[d->rank];
  if ((int)threadIdx.x < d->nIf) spin_until_geq(mb_haloflag(me, par, threadIdx.x), seq);
  __syncthreads();
  return mb_recv(me, par, nIfFaces);
}

__global__ void k_iface_apply_p2p(int nIfCells, const int* __restrict__ cell,
                                  const int* __restrict__ ptr, const int* __restrict__ fidx,
                                  const double* __restrict__ coeff, double* __restrict__ y,
                                  const State* st, P2PDesc* d, int nIfFaces) {
  if (st && st->done) return;
  const double* recv = p2p_wait_halo(d, nIfFaces);
  GRID_STRIDE(i, nIfCells) {
    double corr = 0.0;
    for (int t = ptr[i]; t < ptr[i + 1]; ++t) corr = fma(coeff[fidx[t]], __ldcv(recv + fidx[t]), corr);
    y[cell[i]] -= corr;
  }
}

__global__ void __launch_bounds__(kBlock) k_iface_cg_p2p(int nIfCells, const int* __restrict__ cell,
                                                         const int* __restrict__ ptr,
                                                         const int* __restrict__ fidx,
                                                         const double* __restrict__ coeff,
                                                         double* __restrict__ q, const double* p0,
                                                         const double* p1, State* st, Red rd,
                                                         P2PDesc* d, int nIfFaces) {
  if (st->done) return;
  const double* __restrict__ pnew = (st->k & 1) ? p1 : p0;
  double v[1] = {0.0};
  if (rd.llctl) {  // the halo came as LL words (PACK_CG_P_LL): each value carries its sequence number
    const unsigned long long seq = d->seqHalo + 1;
    const uint64_t* recv = mb_haloll(d->base[d->rank], (int)(seq & 1), nIfFaces);
    GRID_STRIDE(i, nIfCells) {
      double corr = 0.0;
      for (int t = ptr[i]; t < ptr[i + 1]; ++t)
        corr = fma(coeff[fidx[t]], ll_load(recv + 2 * (size_t)fidx[t], (uint32_t)seq), corr);
      const int c = cell[i];
      q[c] -= corr;
      v[0] -= pnew[c] * corr;
    }
    finish_reduction_ll<1>(v, rd, st);
    return;
  }
  const double* recv = p2p_wait_halo(d, nIfFaces);
  GRID_STRIDE(i, nIfCells) {
    double corr = 0.0;
    for (int t = ptr[i]; t < ptr[i + 1]; ++t) corr = fma(coeff[fidx[t]], __ldcv(recv + fidx[t]), corr);
    const int c = cell[i];
    q[c] -= corr;
    v[0] -= pnew[c] * corr;
  }
  finish_reduction<1>(v, rd, st);
}

// Multi-rank fused pipelined pass, fix-up of the interface rows once the halo has arrived:
// k_pipe_SU used the internal part of n at every row; n is linear in the interface term
// dn = -sum coeff * recv, so z += dn, w_{i+1} -= alpha dn and the delta partial gains
// -alpha dn (rD r_{i+1}) -- exact algebra, rows touched only here.
__global__ void __launch_bounds__(kBlock) k_pipe_fixup_p2p(int nIfCells, const int* __restrict__ cell,
                                                           const int* __restrict__ ptr,
                                                           const int* __restrict__ fidx,
                                                           const double* __restrict__ coeff,
                                                           const double* __restrict__ rD,
                                                           const double* __restrict__ r,
                                                           double* __restrict__ z, double* w0,
                                                           double* w1, State* st, Red rd,
                                                           P2PDesc* d, int nIfFaces) {
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // snapshot for the pack of the next exchange
    d->snapK = st->k;
    d->snapDone = st->done;
  }
  if (st->done) return;
  if (threadIdx.x == 0) tstamp(d, st->k, 4, 1);
  const double* recv = p2p_wait_halo(d, nIfFaces);
  if (threadIdx.x == 0) tstamp(d, st->k, 5, 2);
  const double a = st->pa;
  double* __restrict__ wn = (st->k & 1) ? w0 : w1;
  double v[3] = {0.0, 0.0, 0.0};
  GRID_STRIDE(i, nIfCells) {
    double corr = 0.0;
    for (int t = ptr[i]; t < ptr[i + 1]; ++t) corr = fma(coeff[fidx[t]], __ldcv(recv + fidx[t]), corr);
    const int c = cell[i];
    const double dn = -corr;
    z[c] += dn;
    wn[c] = fma(-a, dn, wn[c]);
    v[1] = fma(-a * dn, rD[c] * r[c], v[1]);
  }
  if (threadIdx.x == 0) tstamp(d, st->k, 6, 2);
  finish_reduction<3>(v, rd, st);  // last block publishes the iteration's single reduction
  if (threadIdx.x == 0) tstamp(d, st->k, 7, 2);
}

// ---- multi-rank pipelined CG, ONE kernel per iteration -------------------------------------
// ("only one collective communication per loop body ... overlapped by the sparse
// matrix-vector multiplication kernel"; "single reduction followed by matrix-vector
// multiplication".)  Iteration i = control step k_ctl_ll (gathers the single reduction of i-1
// from this rank's mailbox, alpha_i / beta_i) + k_pipe_SU_mr over all rows:
//   * pre-phase, BEFORE griddepcontrol.wait: launched programmatically while the control step
//     runs, every thread computes the internal SpMV n = A (rD w_i) of its first R rows
//     (interface-free rows) into shared memory;
//   * rows are visited in the rotated order c = (gapStart + t) mod n: the interface-free rows
//     (t < gapLen) stream first, the rows next to a processor boundary come last, where the
//     halo of exchange i (rD w_i at the neighbours' interface cells, written by the neighbours'
//     pass i-1) has long arrived, so n_c includes the interface term exactly;
//   * at interface cells the halo of exchange i+1 (rD w_{i+1}) is stored straight into the
//     neighbours' mailboxes over NVLink;
//   * the last block sums the partials in fixed order and stores (gamma, delta, rr) into every
//     rank's mailbox, leaving the iteration index for the next pre-phase (snapK).
// Halo values and sums travel as LL words (32-bit payload + 32-bit sequence number per 8-byte
// word, NCCL's LL protocol): readers spin until the words carry the expected sequence number,
// so the loop has no memory fence and no flag.  No pack, fix-up or halo stream: one HBM pass
// and one kernel boundary per iteration.  MINB = 5 (48 registers): at 6 the accumulators spill
// inside the streaming loop.
struct MrTail {
  int gapStart, gapLen;
  const int4* __restrict__ meta;    // [n - gapLen] single-face boundary rows: {fi, kk, remote, 1};
                                    // no interface: {.., .., .., 0}; several faces: {ic, .., .., 2}
  const int* __restrict__ cellPtr;  // [nIfCells + 1] into faceIdx
  const int* __restrict__ faceIdx;  // packed face index (interface order, then face order)
  const double* __restrict__ coeff; // [nIfFaces] interfaceBouCoeffs
  const int* __restrict__ faceIf;   // [nIfFaces] interface of each packed face
  int nIfFaces;
};

// one row of the GV recurrences (shared by the bulk and the boundary loops of k_pipe_SU_mr)
struct PipeRow {
  double a, b;
  bool l2;
  __device__ __forceinline__ double apply(int c, double wc0, double nc, const double* __restrict__ rD,
                                          double* __restrict__ z, double* __restrict__ s,
                                          double* __restrict__ p, double* __restrict__ x,
                                          double* __restrict__ r, double* __restrict__ wn,
                                          double (&v)[3], double& rdc) const {
    rdc = __ldg(rD + c);
    const double rc0 = r[c];
    const double zc = fma(b, z[c], nc);
    const double sc = fma(b, s[c], wc0);
    const double pc = fma(b, p[c], rdc * rc0);
    z[c] = zc;
    s[c] = sc;
    p[c] = pc;
    x[c] = fma(a, pc, x[c]);
    const double rc = fma(-a, sc, rc0);
    const double wc = fma(-a, zc, wc0);
    r[c] = rc;
    wn[c] = wc;
    const double u = rdc * rc;
    v[0] = fma(rc, u, v[0]);
    v[1] = fma(wc, u, v[1]);
    v[2] += l2 ? rc * rc : fabs(rc);
    return wc;
  }
};

// Boundary row (position t >= gapLen): interface term from the halo of exchange i (LL words,
// sequence number flagIn), the recurrences, and the halo of exchange i+1 (rD w_{i+1}) as LL
// words straight into the neighbours' mailboxes over NVLink (no fence, no flag).
template <class Fmt>
__device__ __forceinline__ void mr_boundary_row(const Fmt& A, int c, int4 m, const double* __restrict__ rD,
                                                const double* __restrict__ w, double* __restrict__ wn,
                                                double* __restrict__ z, double* __restrict__ s,
                                                double* __restrict__ p, double* __restrict__ x,
                                                double* __restrict__ r, const PipeRow& P,
                                                const MrTail& T, const P2PDesc* d,
                                                const uint64_t* recv, uint32_t flagIn,
                                                uint64_t* const* dstBase, uint32_t flagOut,
                                                double (&v)[3]) {
  const double wc0 = __ldg(w + c);
  double nc = row_apply(A, c, wc0, [&](int q) { return __ldg(rD + q) * __ldg(w + q); });
  // interface term of n = A (rD w): y[c] -= coeff * (rD w)_neighbour (Z10, Z23)
  if (m.w == 1) {  // one face (z-slabs): metadata precomputed, two dependent loads
    nc -= __ldg(T.coeff + m.x) * ll_load(recv + 2 * (size_t)m.x, flagIn);
  } else if (m.w == 2) {
    const int ic = m.x;
    double corr = 0.0;
    for (int f = __ldg(T.cellPtr + ic); f < __ldg(T.cellPtr + ic + 1); ++f) {
      const int fi = __ldg(T.faceIdx + f);
      corr = fma(__ldg(T.coeff + fi), ll_load(recv + 2 * (size_t)fi, flagIn), corr);
    }
    nc -= corr;
  }
  double rdc;
  const double wc = P.apply(c, wc0, nc, rD, z, s, p, x, r, wn, v, rdc);
  const double hv = rdc * wc;  // halo of exchange i+1 straight into the neighbours' mailboxes
  if (m.w == 1) {
    ll_store(dstBase[m.y] + 2 * (size_t)m.z, hv, flagOut);
  } else if (m.w == 2) {
    const int ic = m.x;
    for (int f = __ldg(T.cellPtr + ic); f < __ldg(T.cellPtr + ic + 1); ++f) {
      const int fi = __ldg(T.faceIdx + f);
      const int kk = __ldg(T.faceIf + fi);
      ll_store(dstBase[kk] + 2 * (size_t)(d->ifRemoteOff[kk] + (fi - d->ifLocalOff[kk])), hv, flagOut);
    }
  }
}

// Boundary-row metadata of the one-kernel loop (built once after the peer tables are known).
__global__ void k_build_tail_meta(int L, const int* __restrict__ tailIf, const int* __restrict__ cellPtr,
                                  const int* __restrict__ faceIdx, const int* __restrict__ faceIf,
                                  const P2PDesc* d, int4* __restrict__ meta) {
  GRID_STRIDE(j, L) {
    const int ic = tailIf[j];
    int4 m = make_int4(0, 0, 0, 0);
    if (ic >= 0) {
      if (cellPtr[ic + 1] - cellPtr[ic] == 1) {
        const int fi = faceIdx[cellPtr[ic]];
        const int kk = faceIf[fi];
        m = make_int4(fi, kk, d->ifRemoteOff[kk] + (fi - d->ifLocalOff[kk]), 1);
      } else {
        m = make_int4(ic, 0, 0, 2);
      }
    }
    meta[j] = m;
  }
}

// FOLD = true (default loop): no separate control kernel.  The pass launches the next pass
// programmatically as soon as it starts (that pass's blocks take the SMs this one frees and wait
// in griddepcontrol.wait), and its last block, after publishing the sums, gathers every rank's
// sums from its own mailbox and runs the control step of the next iteration itself.
template <class Fmt, int R, int MINB = 5, bool FOLD = false>
__global__ void __launch_bounds__(kBlock, MINB) k_pipe_SU_mr(Fmt A, const double* __restrict__ rD,
                                                       double* w0, double* w1,
                                                       double* __restrict__ z,
                                                       double* __restrict__ s,
                                                       double* __restrict__ p,
                                                       double* __restrict__ x,
                                                       double* __restrict__ r, State* st, Red rd,
                                                       MrTail T, P2PDesc* d) {
  __shared__ double preN[R > 0 ? R : 1][kBlock], preW[R > 0 ? R : 1][kBlock];
  const int n = A.n;
  const int stride = gridDim.x * kBlock;
  const int base0 = blockIdx.x * kBlock;
  const int tid = threadIdx.x;
  const int gap = T.gapLen;
  // ---- pre-phase (may run while the control step of this iteration is still waiting) ----
  const int kpre = d->snapK + 1;  // left by the previous pass (or the init): this iteration
  if (R > 0) {
    const double* __restrict__ w = (kpre & 1) ? w1 : w0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int t = base0 + j * stride + tid;
      if (t < gap) {
        int c = T.gapStart + t;
        if (c >= n) c -= n;
        const double wc = __ldg(w + c);
        preW[j][tid] = wc;
        preN[j][tid] = row_apply(A, c, wc, [&](int q) { return __ldg(rD + q) * __ldg(w + q); });
      }
    }
  }
  pdl_wait();  // the control step has finished: alpha_i, beta_i, done
  if (st->done) return;
  if (FOLD) pdl_trigger();
  const int k = st->k;
  if (tid == 0) tstamp(d, k, 2, 1);
  const PipeRow P{st->pa, st->pb, st->norm == LDU_NORM_L2};
  const double* __restrict__ w = (k & 1) ? w1 : w0;
  double* __restrict__ wn = (k & 1) ? w0 : w1;
  double v[3] = {0.0, 0.0, 0.0};
  const unsigned long long seqIn = d->seqHalo + 1, seqOut = d->seqHaloSend + 1;
  auto boundary = [&]() {  // positions t >= gap, at most one block-row per block
  {
    int bb = base0;  // first block-row of this block that reaches past the gap
    if (bb + kBlock <= gap) bb += ((gap - bb - kBlock) / stride + 1) * stride;
    if (bb < n) {
      if (tid == 0) tstamp(d, k, 4, 1);
      __shared__ uint64_t* dstBase[kP2PMaxIf];  // exchange i+1's LL slots on each neighbour
      if (tid < d->nIf)
        dstBase[tid] = mb_haloll(d->base[d->ifNeighbor[tid]], (int)(seqOut & 1), d->ifRemoteTotal[tid]);
      __syncthreads();
      const uint64_t* recv = mb_haloll(d->base[d->rank], (int)(seqIn & 1), T.nIfFaces);
      for (int t = bb + tid; t < n; t += stride) {
        if (t < gap) continue;
        int c = T.gapStart + t;
        if (c >= n) c -= n;
        mr_boundary_row(A, c, __ldg(T.meta + (t - gap)), rD, w, wn, z, s, p, x, r, P, T, d, recv,
                        (uint32_t)seqIn, dstBase, (uint32_t)seqOut, v);
      }
      if (tid == 0) tstamp(d, k, 6, 2);
    }
  }
  };
  // ---- bulk: interface-free rows (positions t < gap) ----
  {
    int j = 0;
    if (R > 0 && k == kpre) {
#pragma unroll
      for (; j < R; ++j) {
        const int t = base0 + j * stride + tid;
        if (t < gap) {
          int c = T.gapStart + t;
          if (c >= n) c -= n;
          double rdc;
          P.apply(c, preW[j][tid], preN[j][tid], rD, z, s, p, x, r, wn, v, rdc);
        }
      }
    }
    for (int t = base0 + j * stride + tid; t < gap; t += stride) {
      const int c = T.gapStart + t;  // the gap never wraps (ldu_setup)
      const double wc0 = __ldg(w + c);
      const double nc = row_apply(A, c, wc0, [&](int q) { return __ldg(rD + q) * __ldg(w + q); });
      double rdc;
      P.apply(c, wc0, nc, rD, z, s, p, x, r, wn, v, rdc);
    }
  }
  if (tid == 0) tstamp(d, k, 3, 2);
  // ---- boundary rows last: the halo of exchange i has long arrived (measured: the order makes
  // no difference, profiles/r02_multi) ----
  boundary();
  if (tid == 0) tstamp(d, k, 7, 2);
  __shared__ double sm[3][32];
  __shared__ bool last;
  block_reduce<3>(v, sm);
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < 3; ++q) rd.partials[q * rd.ld + blockIdx.x] = v[q];
    __threadfence();
    last = atomicAdd(rd.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  if (tid == 0) tstamp(d, k, 12, 0);
  sum_partials<3>(rd.partials, rd.ld, gridDim.x, rd.sums, rd.ticket);
  // the iteration's single reduction, as LL words, to every rank (lane q -> rank q)
  const unsigned long long sq = d->seqRed + 1;
  __syncthreads();
  if (tid < d->nRanks) {
    uint64_t* dst = mb_redll(d->base[tid], (int)(sq & 1), d->rank);
    const double* sums = rd.sums;
#pragma unroll
    for (int m = 0; m < 3; ++m) ll_store(dst + 2 * m, __ldcg(sums + m), (uint32_t)sq);
  }
  if (tid == 0) {
    d->seqHaloSend = seqOut;
    d->snapK = k;
    tstamp(d, k, 13, 0);
  }
  if (FOLD) {  // the control step of iteration k + 1, in this block
    __shared__ double part[kP2PMaxRanks][3];
    char* me = d->base[d->rank];
    for (int q = tid; q < d->nRanks; q += blockDim.x) {
      const uint64_t* src = mb_redll(me, (int)(sq & 1), q);
#pragma unroll
      for (int m = 0; m < 3; ++m) part[q][m] = ll_load(src + 2 * m, (uint32_t)sq);
    }
    __syncthreads();
    if (tid == 0) {
      double sums[kMaxVals] = {0.0, 0.0, 0.0, 0.0};
      for (int q = 0; q < d->nRanks; ++q)
        for (int m = 0; m < 3; ++m) sums[m] += part[q][m];
      d->seqRed = sq;
      if (d->nIf > 0) d->seqHalo += 1;  // exchange k, read by this pass (every block is done)
      run_ctl(CTL_PIPE_NEXT, st, sums);
      if (d->nIf > 0 && st->done) d->seqHalo += 1;  // exchange k + 1, sent here, never read
      tstamp(d, k + 1, 0, 0);
      tstamp(d, k + 1, 1, 0);
    }
  }
}

// Control step of the one-kernel loop: gather iteration i-1's sums from the LL slots of this
// rank's mailbox (lane q polls rank q), sum them in rank order, run CTL_PIPE_NEXT.  The first
// trip (k = -1) gathers the init's reduction, published with the flag protocol.
// flagFirst = 1: this trip gathers a reduction published with the flag protocol (the first
// trip after a residual replacement).
__global__ void k_ctl_ll(State* st, P2PDesc* d, int flagFirst) {
  pdl_wait();
  pdl_trigger();  // the pass may launch now and run its pre-phase while we wait
  if (st->done) return;
  __shared__ double part[kP2PMaxRanks][3];
  const int lane = threadIdx.x;
  const unsigned long long sq = d->seqRed + 1;
  const bool ll = st->k >= 0 && !flagFirst;
  if (ll) {
    char* me = d->base[d->rank];
    for (int q = lane; q < d->nRanks; q += blockDim.x) {
      const uint64_t* src = mb_redll(me, (int)(sq & 1), q);
#pragma unroll
      for (int m = 0; m < 3; ++m) part[q][m] = ll_load(src + 2 * m, (uint32_t)sq);
    }
  }
  __syncthreads();
  if (lane != 0) return;
  tstamp(d, st->k + 1, 0, 0);
  double sums[kMaxVals] = {0.0, 0.0, 0.0, 0.0};
  if (ll) {
    for (int q = 0; q < d->nRanks; ++q)
      for (int m = 0; m < 3; ++m) sums[m] += part[q][m];
    d->seqRed = sq;
  } else {
    p2p_gather_sums<kMaxVals>(d, sums);
  }
  tstamp(d, st->k + 1, 1, 0);
  // exchange i-1, consumed by pass i-1 (after a replacement the drain retired it already)
  if (d->nIf > 0 && st->k >= 0 && !flagFirst) d->seqHalo += 1;
  run_ctl(CTL_PIPE_NEXT, st, sums);
  if (d->nIf > 0 && st->done) d->seqHalo += 1;    // exchange i, sent by pass i-1, never read
}

// Residual replacement in the one-kernel loop (NEXT-4): the sums of the pass just before the
// replacement are superseded -- drain them (every rank published them), retire that pass's
// consumed exchange and its unread outgoing one.
__global__ void k_ctl_ll_drain(State* st, P2PDesc* d) {
  if (st->done) return;
  const unsigned long long sq = d->seqRed + 1;
  char* me = d->base[d->rank];
  for (int q = threadIdx.x; q < d->nRanks; q += blockDim.x) {
    const uint64_t* src = mb_redll(me, (int)(sq & 1), q);
    for (int m = 0; m < 3; ++m) (void)ll_load(src + 2 * m, (uint32_t)sq);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    d->seqRed = sq;
    if (d->nIf > 0) d->seqHalo += 2;
  }
}

// y = rD . x (residual replacement operands)
__global__ void k_scale_rD(int n, const double* __restrict__ rD, const double* __restrict__ x,
                           double* __restrict__ y) {
  GRID_STRIDE(c, n) y[c] = rD[c] * x[c];
}

// The fused multi-rank loop starts at k = -1 (its first control step evaluates i = 0).
__global__ void k_mr_init(P2PDesc* d, const State* st) {
  if (threadIdx.x == 0 && blockIdx.x == 0) d->snapK = st->k;
}

// advanceHalo: 0 no halo exchange, 1 this step follows the consumption of one exchange,
// 2 (fused pipelined) the previous iteration consumed one -- none before the first trip (k = -1)
__global__ void k_ctl_p2p(int ctl, State* st, P2PDesc* d, int advanceHalo) {
  pdl_wait();
  pdl_trigger();  // let the fused pass launch and park in pdl_wait while we spin
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (st->done) return;
  tstamp(d, st->k + 1, 0, 0);
  double s[kMaxVals];
  p2p_gather_sums<kMaxVals>(d, s);
  tstamp(d, st->k + 1, 1, 0);
  if (advanceHalo == 1 || (advanceHalo == 2 && st->k >= 0)) d->seqHalo += 1;
  run_ctl(ctl, st, s);
  // fused pipelined: the exchange already sent for this iteration (by the previous fix-up or the
  // init) will never be consumed once the solve ends here -- retire its sequence number so the
  // next solve cannot mistake its flag for a fresh one
  if (advanceHalo == 2 && st->done) d->seqHalo += 1;
}

// An ungated halo exchange (ldu_amul's, or amul_dev inside a solve) has been consumed by
// k_iface_apply_p2p: retire its sequence number (one thread, after every block read the flags).
__global__ void k_p2p_halo_consumed(P2PDesc* d) {
  if (threadIdx.x == 0 && blockIdx.x == 0) d->seqHalo += 1;
}

// multi-rank control: sum the allgathered per-rank sums in rank order, then run the step.
__global__ void k_ctl(int ctl, State* st, const double* __restrict__ gsums, int nRanks, int nv) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (st->done && ctl != CTL_XBAR) return;
  double s[kMaxVals] = {0.0, 0.0, 0.0, 0.0};
  for (int r = 0; r < nRanks; ++r)
    for (int k = 0; k < nv; ++k) s[k] += gsums[r * kMaxVals + k];
  run_ctl(ctl, st, s);
}

__global__ void k_triad(long long n, double* __restrict__ a, const double* __restrict__ b,
                        const double* __restrict__ c, double sc) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n / 2; i += stride) {
    double2 bb = reinterpret_cast<const double2*>(b)[i];
    double2 cc = reinterpret_cast<const double2*>(c)[i];
    reinterpret_cast<double2*>(a)[i] = make_double2(fma(sc, cc.x, bb.x), fma(sc, cc.y, bb.y));
  }
}

// ---------------------------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------------------------
// Launch with programmatic stream serialisation (PDL) when enabled (LDU_PDL, default on).
template <class... KArgs, class... Args>
void launch_pdl(bool pdl, void (*kernel)(KArgs...), int grid, int block, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}
template <class F>
void with_format(ldu_handle h, F&& f) {
  if (h->layout == LDU_LAYOUT_SELL32) {
    SellView v{h->n, h->slicePtr, h->npairs, h->col, h->val};
    f(v);
    return;
  }
  auto dia = [&](auto tag) {
    constexpr int ND = decltype(tag)::value;
    DiaView<ND> v;
    v.n = h->n;
    for (int k = 0; k < ND; ++k) {
      v.off[k] = h->off[k];
      v.U[k] = h->U + (size_t)k * h->n;
    }
    f(v);
  };
  switch (h->nd) {
    case 1: dia(std::integral_constant<int, 1>()); break;
    case 2: dia(std::integral_constant<int, 2>()); break;
    case 3: dia(std::integral_constant<int, 3>()); break;
    case 4: dia(std::integral_constant<int, 4>()); break;
    case 5: dia(std::integral_constant<int, 5>()); break;
    case 6: dia(std::integral_constant<int, 6>()); break;
    case 7: dia(std::integral_constant<int, 7>()); break;
    case 8: dia(std::integral_constant<int, 8>()); break;
    default: throw Error(LDU_ERR_STATE, "bad DIA offset count");
  }
}

template <class F>
void with_dia(ldu_handle h, F&& f) {
  auto dia = [&](auto tag) {
    constexpr int ND = decltype(tag)::value;
    DiaView<ND> v;
    v.n = h->n;
    for (int k = 0; k < ND; ++k) {
      v.off[k] = h->off[k];
      v.U[k] = h->U + (size_t)k * h->n;
    }
    f(v);
  };
  switch (h->nd) {
    case 1: dia(std::integral_constant<int, 1>()); break;
    case 2: dia(std::integral_constant<int, 2>()); break;
    case 3: dia(std::integral_constant<int, 3>()); break;
    case 4: dia(std::integral_constant<int, 4>()); break;
    case 5: dia(std::integral_constant<int, 5>()); break;
    case 6: dia(std::integral_constant<int, 6>()); break;
    case 7: dia(std::integral_constant<int, 7>()); break;
    case 8: dia(std::integral_constant<int, 8>()); break;
    default: throw Error(LDU_ERR_STATE, "bad DIA offset count");
  }
}

bool use_dia_kernels(ldu_handle h) {
  return h->layout == LDU_LAYOUT_DIA_SYM && (h->variant == 1 || h->variant == 2);
}
bool use_march(ldu_handle h) { return h->layout == LDU_LAYOUT_DIA_SYM && h->variant == 3 && h->marchOk; }
bool use_tma(ldu_handle h) { return h->layout == LDU_LAYOUT_DIA_SYM && h->variant == 4 && h->tmaOk; }

template <int ND, int MODE>
size_t tma_smem(ldu_handle h) {
  return sizeof(double) * (size_t)(h->tL == 1 ? tma_smem_doubles<ND, MODE, 1>(h->tT, h->mH)
                                              : tma_smem_doubles<ND, MODE, 2>(h->tT, h->mH));
}

template <int ND, int MODE>
void launch_tma(ldu_handle h, const MarchArgs<ND, MODE>& a, const Red& rd, cudaStream_t s) {
  if (h->tL == 1)
    k_tma_march<ND, MODE, 1><<<h->tGrid, kTmaThreads, tma_smem<ND, MODE>(h), s>>>(a, h->st, rd);
  else
    k_tma_march<ND, MODE, 2><<<h->tGrid, kTmaThreads, tma_smem<ND, MODE>(h), s>>>(a, h->st, rd);
}

template <int ND, int MODE>
MarchArgs<ND, MODE> tma_args(ldu_handle h, const DiaView<ND>& A) {
  MarchArgs<ND, MODE> a{};
  a.A = A;
  a.g = MarchGeom{h->tT, h->mH, h->tTiles, h->mPlanes, h->tChunk};
  return a;
}

template <int ND, int MODE>
MarchArgs<ND, MODE> march_args(ldu_handle h, const DiaView<ND>& A) {
  MarchArgs<ND, MODE> a{};
  a.A = A;
  a.g = MarchGeom{h->mT, h->mH, h->mTiles, h->mPlanes, h->mChunk};
  return a;
}

size_t march_smem(ldu_handle h) { return sizeof(double) * 3 * (size_t)(h->mT + 2 * h->mH); }

// y = A x over internal faces
void launch_amul(ldu_handle h, const double* x, double* y, cudaStream_t s) {
  if (use_tma(h)) {
    with_dia(h, [&](auto A) {
      constexpr int ND = sizeof(A.off) / sizeof(int);
      if constexpr (ND >= 2) {
        auto a = tma_args<ND, MARCH_AMUL>(h, A);
        a.in0 = x;
        a.diag = h->diag;
        a.out = y;
        launch_tma<ND, MARCH_AMUL>(h, a, Red{}, s);
      }
    });
  } else if (use_march(h)) {
    with_dia(h, [&](auto A) {
      constexpr int ND = sizeof(A.off) / sizeof(int);
      if constexpr (ND >= 2) {
        auto a = march_args<ND, MARCH_AMUL>(h, A);
        a.in0 = x;
        a.diag = h->diag;
        a.out = y;
        k_march<ND, MARCH_AMUL><<<h->gridA, kBlock, march_smem(h), s>>>(a, h->st, Red{});
      }
    });
  } else if (use_dia_kernels(h)) {
    with_dia(h, [&](auto A) {
      constexpr int ND = sizeof(A.off) / sizeof(int);
      if (h->variant == 2) k_amul_dia<ND, 2><<<h->gridA, kBlock, 0, s>>>(A, h->diag, x, y);
      else k_amul_dia<ND, 1><<<h->gridA, kBlock, 0, s>>>(A, h->diag, x, y);
    });
  } else {
    with_format(h, [&](auto A) { k_amul<<<h->gridA, kBlock, 0, s>>>(A, h->diag, x, y); });
  }
}

// out = A (rD.in) over internal faces
void launch_spmv_scaled(ldu_handle h, const double* in, double* out, cudaStream_t s) {
  if (h->variant == 5) {
    with_format(h, [&](auto A) {
      k_spmv_scaled_chunk<<<h->gridA, kBlock, 0, s>>>(A, h->rD, in, out, h->st, h->chunkK);
    });
  } else if (use_tma(h)) {
    with_dia(h, [&](auto A) {
      constexpr int ND = sizeof(A.off) / sizeof(int);
      if constexpr (ND >= 2) {
        auto a = tma_args<ND, MARCH_S>(h, A);
        a.in0 = h->rD;
        a.in1 = in;
        a.out = out;
        launch_tma<ND, MARCH_S>(h, a, Red{}, s);
      }
    });
  } else if (use_march(h)) {
    with_dia(h, [&](auto A) {
      constexpr int ND = sizeof(A.off) / sizeof(int);
      if constexpr (ND >= 2) {
        auto a = march_args<ND, MARCH_S>(h, A);
        a.in0 = h->rD;
        a.in1 = in;
        a.out = out;
        k_march<ND, MARCH_S><<<h->gridA, kBlock, march_smem(h), s>>>(a, h->st, Red{});
      }
    });
  } else if (use_dia_kernels(h)) {
    with_dia(h, [&](auto A) {
      constexpr int ND = sizeof(A.off) / sizeof(int);
      if (h->variant == 2) k_spmv_scaled_dia<ND, 2><<<h->gridA, kBlock, 0, s>>>(A, h->rD, in, out, h->st);
      else k_spmv_scaled_dia<ND, 1><<<h->gridA, kBlock, 0, s>>>(A, h->rD, in, out, h->st);
    });
  } else {
    with_format(h, [&](auto A) { k_spmv_scaled<<<h->gridA, kBlock, 0, s>>>(A, h->rD, in, out, h->st); });
  }
}

void launch_passA(ldu_handle h, const Red& ra, cudaStream_t s) {
  if (h->variant == 7) {
    k_cg_passA1<<<h->grid, kBlock, 0, s>>>(h->n, h->rD, h->r, h->p0, h->p1, h->x, h->st);
    with_format(h, [&](auto A) {
      k_cg_passA2<<<h->gridA, kBlock, 0, s>>>(A, h->rD, h->p0, h->p1, h->q, h->st, ra);
    });
  } else if (h->variant == 6 && h->layout == LDU_LAYOUT_DIA_SYM && h->off[0] == 1) {
    with_dia(h, [&](auto A) {
      constexpr int ND = sizeof(A.off) / sizeof(int);
      k_cg_passA_shfl<ND><<<h->gridA, kBlock, 0, s>>>(A, h->rD, h->r, h->p0, h->p1, h->q, h->x,
                                                      h->st, ra);
    });
  } else if (h->variant == 5) {
    with_format(h, [&](auto A) {
      k_cg_passA_chunk<<<h->gridA, kBlock, 0, s>>>(A, h->rD, h->r, h->p0, h->p1, h->q, h->x, h->st, ra,
                                                   h->chunkK);
    });
  } else if (use_tma(h)) {
    with_dia(h, [&](auto A) {
      constexpr int ND = sizeof(A.off) / sizeof(int);
      if constexpr (ND >= 2) {
        auto a = tma_args<ND, MARCH_A>(h, A);
        a.in0 = h->rD;
        a.in1 = h->r;
        a.p0 = h->p0;
        a.p1 = h->p1;
        a.out = h->q;
        a.x = h->x;
        launch_tma<ND, MARCH_A>(h, a, ra, s);
      }
    });
  } else if (use_march(h)) {
    with_dia(h, [&](auto A) {
      constexpr int ND = sizeof(A.off) / sizeof(int);
      if constexpr (ND >= 2) {
        auto a = march_args<ND, MARCH_A>(h, A);
        a.in0 = h->rD;
        a.in1 = h->r;
        a.p0 = h->p0;
        a.p1 = h->p1;
        a.out = h->q;
        a.x = h->x;
        k_march<ND, MARCH_A><<<h->gridA, kBlock, march_smem(h), s>>>(a, h->st, ra);
      }
    });
  } else if (use_dia_kernels(h)) {
    with_dia(h, [&](auto A) {
      constexpr int ND = sizeof(A.off) / sizeof(int);
      if (h->variant == 2)
        k_cg_passA_dia<ND, 2><<<h->gridA, kBlock, 0, s>>>(A, h->rD, h->r, h->p0, h->p1, h->q, h->x, h->st, ra);
      else
        k_cg_passA_dia<ND, 1><<<h->gridA, kBlock, 0, s>>>(A, h->rD, h->r, h->p0, h->p1, h->q, h->x, h->st, ra);
    });
  } else {
    with_format(h, [&](auto A) {
      k_cg_passA<<<h->gridA, kBlock, 0, s>>>(A, h->rD, h->r, h->p0, h->p1, h->q, h->x, h->st, ra);
    });
  }
}

int small_grid(long long n) {
  long long b = (n + kBlock - 1) / kBlock;
  return (int)std::max(1LL, std::min(b, 4096LL));
}

struct Launch {
  ldu_handle h;
  long long kernels = 0;
  cudaStream_t s;
};

Red red_of(ldu_handle h, int ctl, bool single, int grid = 0) {
  Red r;
  r.partials = h->partials;
  r.ld = h->maxParts;
  r.ticket = h->ticket;
  r.sums = single ? h->gsums : h->sums;  // single rank: the local sums are the global sums
  r.ctl = single ? ctl : CTL_NONE;
  r.slot_base = 0;
  r.total = grid ? grid : h->grid;
  r.store_only = 0;
  r.p2p = nullptr;
  r.llctl = 0;
  r.llHalo = 0;
  return r;
}

// loop-pass reduction: over peer memory when enabled (multi-rank), else as red_of
Red red_loop(ldu_handle h, int ctl, bool single, int grid = 0) {
  Red r = red_of(h, ctl, single, grid);
  if (!single && h->p2pOn) r.p2p = h->p2pDesc;
  return r;
}

// fork the NVLink halo send onto the halo stream (it overlaps the next bulk pass) / join it
enum Gate : int { GATE_NONE = 0, GATE_LIVE = 1, GATE_SNAP = 2 };
void p2p_pack(ldu_handle h, int mode, const double* a, cudaStream_t s, int gate);
void p2p_pack_async(ldu_handle h, int mode, const double* a, cudaStream_t s, int gate) {
  CUDA_CHECK(cudaEventRecord(h->ev_pack, s));
  CUDA_CHECK(cudaStreamWaitEvent(h->halo_stream, h->ev_pack, 0));
  p2p_pack(h, mode, a, h->halo_stream, gate);
  CUDA_CHECK(cudaEventRecord(h->ev_halo, h->halo_stream));
}
void p2p_join(ldu_handle h, cudaStream_t s) { CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_halo, 0)); }

// gate: GATE_SNAP (fused loop, PACK_SCALED_W) reads the fix-up's snapshot; GATE_LIVE (the
// classical loop and the first exchange of the fused loop) reads the live State, which nothing
// modifies concurrently there; GATE_NONE (amul_dev) always sends -- its consumer always reads.
void p2p_pack(ldu_handle h, int mode, const double* a, cudaStream_t s, int gate) {
  const bool wpair = mode == PACK_SCALED_W || mode == PACK_SCALED_LL_W;
  const double* q0 = wpair ? h->w : h->p0;
  const double* q1 = wpair ? h->w2 : h->p1;
  const int *gk = nullptr, *gd = nullptr;
  if (gate == GATE_SNAP) {
    gk = &h->p2pDesc->snapK;
    gd = &h->p2pDesc->snapDone;
  } else if (gate == GATE_LIVE) {
    gk = &h->st->k;
    gd = &h->st->done;
  }
  k_pack_p2p<<<small_grid(h->nIfFaces), kBlock, 0, s>>>(
      h->nIfFaces, h->ifFaceCells, h->ifFaceIf, mode, a, h->rD, q0, q1, h->st, gk, gd,
      h->p2pDesc, h->ticket + 1);
}

bool multi(ldu_handle h) { return h->comm && h->comm->nRanks > 1; }

// cross-rank reduction of the local sums + the control step (multi-rank only).  Peer-memory
// path: the reducing kernel (launched with red_loop) has published its sums from its last
// block; k_ctl_p2p gathers them in rank order.  NCCL path: allgather on the reduction stream.
void allgather_ctl(ldu_handle h, int ctl, int nv, cudaStream_t s, long long& kernels) {
  if (h->p2pOn) {
    k_ctl_p2p<<<1, 32, 0, s>>>(ctl, h->st, h->p2pDesc, 0);
    ++kernels;
    return;
  }
  ldu_comm cm = h->comm;
  CUDA_CHECK(cudaEventRecord(h->ev_fork, s));
  CUDA_CHECK(cudaStreamWaitEvent(h->red_stream, h->ev_fork, 0));
  NCCL_CHECK(ncclAllGather(h->sums, h->gsums, kMaxVals, ncclDouble, cm->red, h->red_stream));
  CUDA_CHECK(cudaEventRecord(h->ev_red, h->red_stream));
  CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_red, 0));
  k_ctl<<<1, 32, 0, s>>>(ctl, h->st, h->gsums, cm->nRanks, nv);
  ++kernels;
}

// halo exchange of the packed send buffer on the halo stream; returns after enqueueing.
void halo_exchange(ldu_handle h, cudaStream_t s) {
  CUDA_CHECK(cudaEventRecord(h->ev_pack, s));
  CUDA_CHECK(cudaStreamWaitEvent(h->halo_stream, h->ev_pack, 0));
  NCCL_CHECK(ncclGroupStart());
  for (const DevInterface& it : h->ifaces) {
    if (!it.nFaces) continue;
    NCCL_CHECK(ncclSend(h->sendbuf + it.offset, it.nFaces, ncclDouble, it.neighbRank,
                        h->comm->halo, h->halo_stream));
    NCCL_CHECK(ncclRecv(h->recvbuf + it.offset, it.nFaces, ncclDouble, it.neighbRank,
                        h->comm->halo, h->halo_stream));
  }
  NCCL_CHECK(ncclGroupEnd());
  CUDA_CHECK(cudaEventRecord(h->ev_halo, h->halo_stream));
  h->stats.haloBytes += 8LL * h->nIfFaces;
}

void wait_halo(ldu_handle h, cudaStream_t s) { CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_halo, 0)); }

// y = A x including interfaces, all on stream s (x, y device, internal or user)
void amul_dev(ldu_handle h, const double* x, double* y, cudaStream_t s, long long& kernels) {
  const bool haveIf = h->nIfFaces > 0;
  if (haveIf && h->p2pOn) {  // ungated exchange over the peer mailboxes (both sides always run)
    p2p_pack_async(h, PACK_PLAIN, x, s, GATE_NONE);
    launch_amul(h, x, y, s);
    p2p_join(h, s);
    k_iface_apply_p2p<<<small_grid(h->nIfCells), kBlock, 0, s>>>(
        h->nIfCells, h->ifCell, h->ifCellPtr, h->ifFaceIdx, h->ifCoeffs, y, nullptr, h->p2pDesc,
        h->nIfFaces);
    k_p2p_halo_consumed<<<1, 32, 0, s>>>(h->p2pDesc);
    kernels += 4;
    h->stats.haloBytes += 8LL * h->nIfFaces;
    return;
  }
  if (haveIf) {
    k_pack<<<small_grid(h->nIfFaces), kBlock, 0, s>>>(h->nIfFaces, h->ifFaceCells, PACK_PLAIN, x,
                                                      nullptr, nullptr, nullptr, nullptr, h->sendbuf);
    ++kernels;
    halo_exchange(h, s);
  }
  launch_amul(h, x, y, s);
  ++kernels;
  if (haveIf) {
    wait_halo(h, s);
    k_iface_apply<<<small_grid(h->nIfCells), kBlock, 0, s>>>(
        h->nIfCells, h->ifCell, h->ifCellPtr, h->ifFaceIdx, h->ifCoeffs, h->recvbuf, y, nullptr);
    ++kernels;
  }
}

void ensure_vec(double*& p, int n) {
  if (!p) p = dmalloc<double>(n);
}

void ensure_work(ldu_handle h, bool pipelined) {
  const int n = h->n;
  ensure_vec(h->x, n);
  ensure_vec(h->r, n);
  ensure_vec(h->ybuf, n);
  if (!pipelined) {
    ensure_vec(h->p0, n);
    ensure_vec(h->p1, n);
    ensure_vec(h->q, n);
  } else {
    ensure_vec(h->w, n);
    ensure_vec(h->nv, n);
    if (h->fusePipe && (!multi(h) || h->p2pOn)) ensure_vec(h->w2, n);
    ensure_vec(h->z, n);
    ensure_vec(h->s, n);
    ensure_vec(h->p0, n);
  }
}

// One batch of `batch` iterations, enqueued on s (captured into a graph by the caller).
// LDU_TRACE=1 (debug): 5 external event nodes per iteration of the fused multi-rank pipelined
// loop; the per-segment device times are printed to stderr after each solve.
void trace_mark(ldu_handle h, int it, int k, cudaStream_t s) {
  if (!h->trace.empty())
    CUDA_CHECK(cudaEventRecordWithFlags(h->trace[5 * it + k], s, cudaEventRecordExternal));
}

void prof_mark(ldu_handle h, bool profile, int idx, cudaStream_t s) {
  // external event nodes: recorded by the graph on every launch (plain records inside a capture
  // only express dependencies)
  if (profile) CUDA_CHECK(cudaEventRecordWithFlags(h->prof_ev[idx], s, cudaEventRecordExternal));
}

long long enqueue_cg_iters(ldu_handle h, int batch, cudaStream_t s, bool profile) {
  long long kernels = 0;
  const bool mr = multi(h);
  const bool haveIf = h->nIfFaces > 0;
  if (mr && h->p2pOn) {  // halo and both reductions over NVLink peer memory, no NCCL kernels
    for (int it = 0; it < batch; ++it) {
      if (haveIf) {
        p2p_pack_async(h, h->cgLL ? PACK_CG_P_LL : PACK_CG_P, h->r, s, GATE_LIVE);
        ++kernels;
      }
      // the reduction protocol must be the same on every rank: with LL, every rank (also one
      // without interfaces) finishes (p, q) in the fix-up kernel, which then has no cells
      const bool fix = haveIf || h->cgLL;
      Red ra = red_loop(h, CTL_CG_A, false, h->gridA);
      if (fix) ra.store_only = 1;
      prof_mark(h, profile, 4 * it + 0, s);
      launch_passA(h, ra, s);
      prof_mark(h, profile, 4 * it + 1, s);
      ++kernels;
      if (fix) {
        if (haveIf) p2p_join(h, s);
        Red ri = red_loop(h, CTL_CG_A, false);
        const int ig = std::max(1, std::min(small_grid(h->nIfCells), h->maxParts - h->gridA));
        ri.slot_base = h->gridA;
        ri.total = h->gridA + ig;
        if (h->cgLL) {  // (p, q) as LL words; control A in the fix-up's last block
          ri.llctl = CTL_CG_A;
          ri.llHalo = haveIf ? 1 : 0;
        }
        k_iface_cg_p2p<<<ig, kBlock, 0, s>>>(h->nIfCells, h->ifCell, h->ifCellPtr, h->ifFaceIdx,
                                             h->ifCoeffs, h->q, h->p0, h->p1, h->st, ri,
                                             h->p2pDesc, h->nIfFaces);
        ++kernels;
      }
      if (!h->cgLL) {
        k_ctl_p2p<<<1, 32, 0, s>>>(CTL_CG_A, h->st, h->p2pDesc, haveIf ? 1 : 0);
        ++kernels;
      }
      prof_mark(h, profile, 4 * it + 2, s);
      Red rb = red_loop(h, CTL_CG_B, false);
      if (h->cgLL) {
        rb.llctl = CTL_CG_B;
        k_cg_passB<true><<<h->grid, kBlock, 0, s>>>(h->n, h->rD, h->q, h->r, h->st, rb);
      } else {
        k_cg_passB<false><<<h->grid, kBlock, 0, s>>>(h->n, h->rD, h->q, h->r, h->st, rb);
      }
      prof_mark(h, profile, 4 * it + 3, s);
      ++kernels;
      if (!h->cgLL) {
        k_ctl_p2p<<<1, 32, 0, s>>>(CTL_CG_B, h->st, h->p2pDesc, 0);
        ++kernels;
      }
    }
    return kernels;
  }
  for (int it = 0; it < batch; ++it) {
    // pass A
    if (haveIf) {
      k_pack<<<small_grid(h->nIfFaces), kBlock, 0, s>>>(h->nIfFaces, h->ifFaceCells, PACK_CG_P,
                                                        h->r, h->rD, h->p0, h->p1, h->st,
                                                        h->sendbuf);
      ++kernels;
      halo_exchange(h, s);
    }
    Red ra = red_of(h, CTL_CG_A, !mr, h->gridA);
    if (haveIf) ra.store_only = 1;
    prof_mark(h, profile, 4 * it + 0, s);
    launch_passA(h, ra, s);
    prof_mark(h, profile, 4 * it + 1, s);
    ++kernels;
    if (haveIf) {
      wait_halo(h, s);
      Red ri = red_of(h, CTL_CG_A, !mr);
      const int ig = std::min(small_grid(h->nIfCells), h->maxParts - h->gridA);
      ri.slot_base = h->gridA;
      ri.total = h->gridA + ig;
      k_iface_cg<<<ig, kBlock, 0, s>>>(h->nIfCells, h->ifCell, h->ifCellPtr, h->ifFaceIdx,
                                       h->ifCoeffs, h->recvbuf, h->q, h->p0, h->p1, h->st, ri);
      ++kernels;
    }
    if (mr) allgather_ctl(h, CTL_CG_A, 1, s, kernels);
    // pass B
    prof_mark(h, profile, 4 * it + 2, s);
    k_cg_passB<false><<<h->grid, kBlock, 0, s>>>(h->n, h->rD, h->q, h->r, h->st, red_of(h, CTL_CG_B, !mr));
    prof_mark(h, profile, 4 * it + 3, s);
    ++kernels;
    if (mr) allgather_ctl(h, CTL_CG_B, 2, s, kernels);
  }
  return kernels;
}

long long enqueue_pipe_iters(ldu_handle h, int batch, cudaStream_t s, bool profile,
                             bool rrFirst = false) {
  long long kernels = 0;
  const bool mr = multi(h);
  if (mr && h->p2pOn && h->fusePipe && h->mrFuse) {  // ONE kernel per iteration (k_pipe_SU_mr)
    const bool haveIf = h->nIfFaces > 0;
    MrTail T{h->mrGapStart, haveIf ? h->mrGapLen : h->n, h->mrTailMeta, h->ifCellPtr, h->ifFaceIdx,
             h->ifCoeffs, h->ifFaceIf, h->nIfFaces};
    const bool pdl = h->pdl && h->trace.empty();
    if (h->mrFold && !rrFirst) {  // one kernel per iteration, control step in its last block
      for (int it = 0; it < batch; ++it) {
        trace_mark(h, it, 0, s);
        trace_mark(h, it, 1, s);
        prof_mark(h, profile, 4 * it + 0, s);
        prof_mark(h, profile, 4 * it + 1, s);
        prof_mark(h, profile, 4 * it + 2, s);
        Red ru = red_loop(h, CTL_NONE, false, h->gridSUmr);
        with_format(h, [&](auto A) {
          using Fmt = decltype(A);
          launch_pdl(pdl && it > 0 && !profile, k_pipe_SU_mr<Fmt, 0, 5, true>, h->gridSUmr, kBlock, s,
                     A, (const double*)h->rD, h->w, h->w2, h->z, h->s, h->p0, h->x, h->r, h->st,
                     ru, T, h->p2pDesc);
        });
        ++kernels;
        prof_mark(h, profile, 4 * it + 3, s);
        trace_mark(h, it, 2, s);
        trace_mark(h, it, 3, s);
        trace_mark(h, it, 4, s);
      }
      return kernels;
    }
    for (int it = 0; it < batch; ++it) {
      trace_mark(h, it, 0, s);
      launch_pdl(pdl && it > 0 && !profile, k_ctl_ll, 1, 64, s, h->st, h->p2pDesc,
                 (rrFirst && it == 0) ? 1 : 0);
      ++kernels;
      trace_mark(h, it, 1, s);
      prof_mark(h, profile, 4 * it + 0, s);
      prof_mark(h, profile, 4 * it + 1, s);
      prof_mark(h, profile, 4 * it + 2, s);
      Red ru = red_loop(h, CTL_NONE, false, h->gridSUmr);
      with_format(h, [&](auto A) {
        using Fmt = decltype(A);
        auto go = [&](auto kern) {
          launch_pdl(pdl && !profile, kern, h->gridSUmr, kBlock, s, A, (const double*)h->rD, h->w,
                     h->w2, h->z, h->s, h->p0, h->x, h->r, h->st, ru, T, h->p2pDesc);
        };
        if (h->mrPre == 8) go(k_pipe_SU_mr<Fmt, 8>);
        else if (h->mrPre == 4) go(k_pipe_SU_mr<Fmt, 4>);
        else go(k_pipe_SU_mr<Fmt, 0>);
      });
      ++kernels;
      prof_mark(h, profile, 4 * it + 3, s);
      trace_mark(h, it, 2, s);
      trace_mark(h, it, 3, s);
      trace_mark(h, it, 4, s);
    }
    return kernels;
  }
  if (mr && h->p2pOn && h->fusePipe) {  // fused S+U pass per iteration over peer memory
    // trip i: ctl_i (alpha_i, beta_i) -> k_pipe_SU over all rows (internal SpMV) -> [join the
    // halo stream] -> fix-up of the interface rows with exchange i (publishes the iteration's
    // single reduction) -> fork the pack of exchange i+1 (rD w_{i+1}) onto the halo stream, where
    // its NVLink stores and fences overlap ctl_{i+1} and the next fused pass.  Exchange 0 is sent
    // by the init; every batch ends joined.
    const bool haveIf = h->nIfFaces > 0;
    for (int it = 0; it < batch; ++it) {
      trace_mark(h, it, 0, s);
      const bool pdl = h->pdl && !profile && h->trace.empty() && (it > 0 || !haveIf);
      launch_pdl(pdl, k_ctl_p2p, 1, 32, s, (int)CTL_PIPE_NEXT, h->st, h->p2pDesc, haveIf ? 2 : 0);
      trace_mark(h, it, 1, s);
      trace_mark(h, it, 2, s);
      ++kernels;
      Red ru = red_loop(h, CTL_PIPE_NEXT, false, h->gridSU);
      if (haveIf) ru.store_only = 1;
      prof_mark(h, profile, 4 * it + 0, s);
      prof_mark(h, profile, 4 * it + 1, s);
      prof_mark(h, profile, 4 * it + 2, s);
      with_format(h, [&](auto A) {
        launch_pdl(h->pdl && !profile && h->trace.empty(), k_pipe_SU<decltype(A)>, h->gridSU,
                   kBlock, s, A, (const double*)h->rD, h->w, h->w2, h->z, h->s, h->p0, h->x,
                   h->r, h->st, ru);
      });
      prof_mark(h, profile, 4 * it + 3, s);
      trace_mark(h, it, 3, s);
      ++kernels;
      if (haveIf) {
        if (it > 0) p2p_join(h, s);
        Red ri = red_loop(h, CTL_PIPE_NEXT, false);
        const int ig = std::min(small_grid(h->nIfCells), h->maxParts - h->gridSU);
        ri.slot_base = h->gridSU;
        ri.total = h->gridSU + ig;
        launch_pdl(false, k_pipe_fixup_p2p,  // follows a cross-stream join: plain dependency
                   ig, kBlock, s, h->nIfCells, (const int*)h->ifCell, (const int*)h->ifCellPtr,
                   (const int*)h->ifFaceIdx, (const double*)h->ifCoeffs, (const double*)h->rD,
                   (const double*)h->r, h->z, h->w, h->w2, h->st, ri, h->p2pDesc, h->nIfFaces);
        p2p_pack_async(h, PACK_SCALED_W, nullptr, s, GATE_SNAP);
        kernels += 2;
      }
      trace_mark(h, it, 4, s);
    }
    if (haveIf) p2p_join(h, s);
    return kernels;
  }
  if (mr && h->p2pOn) {  // halo + the single reduction over NVLink peer memory
    const bool haveIf = h->nIfFaces > 0;
    for (int it = 0; it < batch; ++it) {
      if (haveIf) {
        p2p_pack_async(h, PACK_SCALED, h->w, s, GATE_LIVE);
        ++kernels;
      }
      prof_mark(h, profile, 4 * it + 0, s);
      launch_spmv_scaled(h, h->w, h->nv, s);  // overlaps the peers' reduction traffic
      prof_mark(h, profile, 4 * it + 1, s);
      ++kernels;
      if (haveIf) {
        p2p_join(h, s);
        k_iface_apply_p2p<<<small_grid(h->nIfCells), kBlock, 0, s>>>(
            h->nIfCells, h->ifCell, h->ifCellPtr, h->ifFaceIdx, h->ifCoeffs, h->nv, h->st,
            h->p2pDesc, h->nIfFaces);
        ++kernels;
      }
      k_ctl_p2p<<<1, 32, 0, s>>>(CTL_PIPE_NEXT, h->st, h->p2pDesc, haveIf ? 1 : 0);
      prof_mark(h, profile, 4 * it + 2, s);
      k_pipe_U<<<h->grid, kBlock, 0, s>>>(h->n, h->rD, h->nv, h->z, h->s, h->p0, h->x, h->r, h->w,
                                          h->st, red_loop(h, CTL_PIPE_NEXT, false));
      prof_mark(h, profile, 4 * it + 3, s);
      kernels += 2;
    }
    return kernels;
  }
  if (!mr && h->fusePipe) {  // one fused pass per iteration (profile: pass slot 1)
    for (int it = 0; it < batch; ++it) {
      prof_mark(h, profile, 4 * it + 0, s);
      prof_mark(h, profile, 4 * it + 1, s);
      prof_mark(h, profile, 4 * it + 2, s);
      with_format(h, [&](auto A) {
        using Fmt = decltype(A);
        const Red rd = red_of(h, CTL_PIPE_NEXT, true, h->gridSU);
        if (h->suMinB == 8)
          k_pipe_SU<Fmt, 8><<<h->gridSU, kBlock, 0, s>>>(A, h->rD, h->w, h->w2, h->z, h->s, h->p0, h->x, h->r, h->st, rd);
        else
          k_pipe_SU<Fmt><<<h->gridSU, kBlock, 0, s>>>(A, h->rD, h->w, h->w2, h->z, h->s, h->p0, h->x, h->r, h->st, rd);
      });
      prof_mark(h, profile, 4 * it + 3, s);
      ++kernels;
    }
    return kernels;
  }
  const bool haveIf = h->nIfFaces > 0;
  ldu_comm cm = h->comm;
  for (int it = 0; it < batch; ++it) {
    // the single fused reduction of the previous U (or init) runs on red_stream, overlapped
    // with the SpMV below ("global synchronization can be overlapped by the sparse
    // matrix-vector multiplication kernel")
    if (mr) {
      CUDA_CHECK(cudaEventRecord(h->ev_fork, s));
      CUDA_CHECK(cudaStreamWaitEvent(h->red_stream, h->ev_fork, 0));
      NCCL_CHECK(ncclAllGather(h->sums, h->gsums, kMaxVals, ncclDouble, cm->red, h->red_stream));
      CUDA_CHECK(cudaEventRecord(h->ev_red, h->red_stream));
    }
    if (haveIf) {
      k_pack<<<small_grid(h->nIfFaces), kBlock, 0, s>>>(h->nIfFaces, h->ifFaceCells, PACK_SCALED,
                                                        h->w, h->rD, nullptr, nullptr, h->st,
                                                        h->sendbuf);
      ++kernels;
      halo_exchange(h, s);
    }
    prof_mark(h, profile, 4 * it + 0, s);
    launch_spmv_scaled(h, h->w, h->nv, s);
    prof_mark(h, profile, 4 * it + 1, s);
    ++kernels;
    if (haveIf) {
      wait_halo(h, s);
      k_iface_apply<<<small_grid(h->nIfCells), kBlock, 0, s>>>(
          h->nIfCells, h->ifCell, h->ifCellPtr, h->ifFaceIdx, h->ifCoeffs, h->recvbuf, h->nv, h->st);
      ++kernels;
    }
    if (mr) {
      CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_red, 0));
      k_ctl<<<1, 32, 0, s>>>(CTL_PIPE_NEXT, h->st, h->gsums, cm->nRanks, 3);
      ++kernels;
    }
    // U: single rank runs the next top-of-iteration control in its last block
    prof_mark(h, profile, 4 * it + 2, s);
    k_pipe_U<<<h->grid, kBlock, 0, s>>>(h->n, h->rD, h->nv, h->z, h->s, h->p0, h->x, h->r, h->w,
                                        h->st, red_of(h, CTL_PIPE_NEXT, !mr));
    prof_mark(h, profile, 4 * it + 3, s);
    ++kernels;
  }
  return kernels;
}

// ---- residual replacement in the single-rank fused pipelined loop (NEXT-4) --------------------
// y = A x including the diagonal, skipped once the solve is done
template <class Fmt>
__global__ void __launch_bounds__(kBlock) k_amul_st(Fmt A, const double* __restrict__ diag,
                                                    const double* __restrict__ x,
                                                    double* __restrict__ y, const State* st) {
  if (st->done) return;
  GRID_STRIDE(c, A.n) {
    y[c] = row_apply(A, c, __ldg(diag + c) * __ldg(x + c), [&](int j) { return __ldg(x + j); });
  }
}

// r = b - A x
__global__ void __launch_bounds__(kBlock) k_rr_r(int n, const double* __restrict__ b,
                                                 const double* __restrict__ ax,
                                                 double* __restrict__ r, const State* st) {
  if (st->done) return;
  GRID_STRIDE(c, n) r[c] = b[c] - ax[c];
}

// w_{i+1} = A (rD . r) into the ping-pong half the next fused pass reads (k not yet advanced)
template <class Fmt>
__global__ void __launch_bounds__(kBlock) k_rr_w(Fmt A, const double* __restrict__ rD,
                                                 const double* __restrict__ r, double* w0,
                                                 double* w1, const State* st) {
  if (st->done) return;
  double* __restrict__ wn = (st->k & 1) ? w0 : w1;
  GRID_STRIDE(c, A.n) {
    wn[c] = row_apply(A, c, __ldg(r + c), [&](int j) { return __ldg(rD + j) * __ldg(r + j); });
  }
}

// w_{i+1} = y (A rD r incl. interfaces) into the ping-pong half the next fused pass reads
__global__ void __launch_bounds__(kBlock) k_rr_copy_w(int n, const double* __restrict__ y,
                                                      double* w0, double* w1, const State* st) {
  if (st->done) return;
  double* __restrict__ wn = (st->k & 1) ? w0 : w1;
  GRID_STRIDE(c, n) wn[c] = y[c];
}

// the iteration's fused reduction over the replaced vectors: [(r, rD.r), (w, rD.r), crit(r)]
__global__ void __launch_bounds__(kBlock) k_rr_dots(int n, const double* __restrict__ rD,
                                                    const double* __restrict__ r, const double* w0,
                                                    const double* w1, State* st, Red rd) {
  if (st->done) return;
  const double* __restrict__ w = (st->k & 1) ? w0 : w1;
  const bool l2 = st->norm == LDU_NORM_L2;
  double v[3] = {0.0, 0.0, 0.0};
  GRID_STRIDE(c, n) {
    const double rc = r[c], u = rD[c] * rc;
    v[0] = fma(rc, u, v[0]);
    v[1] = fma(w[c], u, v[1]);
    v[2] += l2 ? rc * rc : fabs(rc);
  }
  finish_reduction<3>(v, rd, st);
}

// One batch of `batch` fused pipelined iterations whose last one is followed by the residual
// replacement: its fused pass reduces without the control step, the vectors are recomputed from
// their definitions (r = b - A x, w = A rD r, s = A p, z = A rD s; Jacobi form of GV Sec. 4), and
// the reduction of the replaced vectors runs the control step of the next iteration.
long long enqueue_pipe_rr(ldu_handle h, int batch, cudaStream_t s, bool profile) {
  long long kernels = 0;
  for (int it = 0; it < batch; ++it) {
    const bool last = it == batch - 1;
    prof_mark(h, profile, 4 * it + 0, s);
    prof_mark(h, profile, 4 * it + 1, s);
    prof_mark(h, profile, 4 * it + 2, s);
    with_format(h, [&](auto A) {
      k_pipe_SU<<<h->gridSU, kBlock, 0, s>>>(A, h->rD, h->w, h->w2, h->z, h->s, h->p0, h->x, h->r,
                                              h->st, red_of(h, last ? CTL_NONE : CTL_PIPE_NEXT, true, h->gridSU));
    });
    prof_mark(h, profile, 4 * it + 3, s);
    ++kernels;
  }
  with_format(h, [&](auto A) {
    k_amul_st<<<h->gridA, kBlock, 0, s>>>(A, h->diag, h->x, h->ybuf, h->st);
    k_rr_r<<<h->grid, kBlock, 0, s>>>(h->n, h->bbuf, h->ybuf, h->r, h->st);
    k_rr_w<<<h->gridA, kBlock, 0, s>>>(A, h->rD, h->r, h->w, h->w2, h->st);
    k_amul_st<<<h->gridA, kBlock, 0, s>>>(A, h->diag, h->p0, h->s, h->st);
    k_spmv_scaled<<<h->gridA, kBlock, 0, s>>>(A, h->rD, h->s, h->z, h->st);
  });
  k_rr_dots<<<h->grid, kBlock, 0, s>>>(h->n, h->rD, h->r, h->w, h->w2, h->st,
                                       red_of(h, CTL_PIPE_NEXT, true));
  return kernels + 6;
}

// Multi-rank residual replacement (one-kernel loop): `batch` fused iterations, then r = b - A x,
// w = A rD r, s = A p, z = A rD s with their halo exchanges (amul_dev), the reduction of the
// replaced vectors (flag protocol; the next batch's first control step gathers it) and the halo
// of rD w sent as exchange 0 of the next batch -- the single-rank replacement with the
// interfaces included (GV 2014 Sec. 4 [ext]; reading Z7).
long long enqueue_pipe_rr_mr(ldu_handle h, int batch, cudaStream_t s, bool profile) {
  long long kernels = enqueue_pipe_iters(h, batch, s, profile, true);
  k_ctl_ll_drain<<<1, 64, 0, s>>>(h->st, h->p2pDesc);
  ++kernels;
  double* tmp = h->nv;
  // w_{i+1} lives in the ping-pong half the next pass reads: (k & 1) ? w : w2 after pass k; the
  // graph is fixed, so both halves are written in turn by parity-selecting kernels
  amul_dev(h, h->x, h->ybuf, s, kernels);
  k_rr_r<<<h->grid, kBlock, 0, s>>>(h->n, h->bbuf, h->ybuf, h->r, h->st);
  k_scale_rD<<<h->grid, kBlock, 0, s>>>(h->n, h->rD, h->r, tmp);
  amul_dev(h, tmp, h->ybuf, s, kernels);
  k_rr_copy_w<<<h->grid, kBlock, 0, s>>>(h->n, h->ybuf, h->w, h->w2, h->st);
  amul_dev(h, h->p0, h->s, s, kernels);
  k_scale_rD<<<h->grid, kBlock, 0, s>>>(h->n, h->rD, h->s, tmp);
  amul_dev(h, tmp, h->z, s, kernels);
  k_rr_dots<<<h->grid, kBlock, 0, s>>>(h->n, h->rD, h->r, h->w, h->w2, h->st,
                                       red_loop(h, CTL_NONE, false));
  kernels += 5;
  if (h->nIfFaces) {  // exchange of the replaced rD w for the next pass (LL words)
    p2p_pack(h, PACK_SCALED_LL_W, nullptr, s, GATE_LIVE);
    ++kernels;
  }
  return kernels;
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// public-internal entry points
// ---------------------------------------------------------------------------------------------
void amul(ldu_handle h, const double* x, double* y) {
  cudaStream_t s = h->own_stream;
  long long kernels = 0;
  h->stats = ldu_solve_stats{};
  if (h->stream != h->own_stream) {
    CUDA_CHECK(cudaEventRecord(h->ev_fork, h->stream));
    CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_fork, 0));
  }
  const bool xd = is_device_ptr(x), yd = is_device_ptr(y);
  const double* xin = x;
  double* yout = y;
  if (!xd) {
    ensure_vec(h->bbuf, h->n);
    CUDA_CHECK(cudaMemcpyAsync(h->bbuf, x, sizeof(double) * h->n, cudaMemcpyHostToDevice, s));
    h->stats.h2dBytes += 8LL * h->n;
    xin = h->bbuf;
  }
  if (!yd) {
    ensure_vec(h->ybuf, h->n);
    yout = h->ybuf;
  }
  amul_dev(h, xin, yout, s, kernels);
  if (!yd) {
    CUDA_CHECK(cudaMemcpyAsync(y, yout, sizeof(double) * h->n, cudaMemcpyDeviceToHost, s));
    h->stats.d2hBytes += 8LL * h->n;
  }
  if (h->stream != h->own_stream) {
    CUDA_CHECK(cudaEventRecord(h->ev_fork, s));
    CUDA_CHECK(cudaStreamWaitEvent(h->stream, h->ev_fork, 0));
  }
  CUDA_CHECK(cudaGetLastError());
  CUDA_CHECK(cudaStreamSynchronize(s));
  h->stats.kernels = kernels;
}

ldu_status solve(ldu_handle h, bool pipelined, const double* b, double* x, double tol,
                 int maxIter, const ldu_solve_opts* opts, int* nIter, double* finalRes) {
  if (!b || !x) fail_arg("b and x must not be NULL");
  if (!(tol >= 0.0)) fail_arg("tol must be >= 0");
  if (maxIter < 0) fail_arg("maxIter must be >= 0");
  ldu_solve_opts o{};
  if (opts) {
    o = *opts;
    if (o.reserved2[0] != 0.0 || o.reserved2[1] != 0.0)
      fail_arg("ldu_solve_opts.reserved2 must be zero");
  }
  if (!(o.relTol >= 0.0)) fail_arg("relTol must be >= 0");
  if (o.minIter < 0) fail_arg("minIter must be >= 0");
  if (o.norm != LDU_NORM_L2 && o.norm != LDU_NORM_OPENFOAM) fail_arg("unknown norm");
  if (o.batch < 0) fail_arg("batch must be >= 0");
  if (o.profile != 0 && o.profile != 1) fail_arg("profile must be 0 or 1");
  if (o.replaceEvery < 0) fail_arg("replaceEvery must be >= 0");
  const int rr = o.replaceEvery;
  if (rr && !pipelined) fail_arg("replaceEvery applies to pipelined CG only");
  if (rr && (!h->fusePipe || (multi(h) && !(h->p2pOn && h->mrFuse))))
    throw Error(LDU_ERR_STATE, "residual replacement needs the fused pipelined pass (single rank, "
                               "or the one-kernel multi-rank loop)");
  const bool profile = o.profile == 1;
  const int batch = rr ? rr : (o.batch ? o.batch : 32);

  ensure_work(h, pipelined);
  const int n = h->n;
  cudaStream_t s = h->own_stream;
  const bool mr = multi(h);
  h->stats = ldu_solve_stats{};
  long long kernels = 0;

  // order after the user's stream
  if (h->stream != h->own_stream) {
    CUDA_CHECK(cudaEventRecord(h->ev_fork, h->stream));
    CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_fork, 0));
  }
  CUDA_CHECK(cudaEventRecord(h->ev[0], s));

  // inputs
  const bool bd = is_device_ptr(b), xd = is_device_ptr(x);
  const double* bin = b;
  if (!bd) {
    ensure_vec(h->bbuf, n);
    CUDA_CHECK(cudaMemcpyAsync(h->bbuf, b, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    h->stats.h2dBytes += 8LL * n;
    bin = h->bbuf;
  }
  CUDA_CHECK(cudaMemcpyAsync(h->x, x, sizeof(double) * n, xd ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  if (!xd) h->stats.h2dBytes += 8LL * n;
  if (rr && bin != h->bbuf) {  // the replacement graph reads b from a fixed buffer
    ensure_vec(h->bbuf, n);
    CUDA_CHECK(cudaMemcpyAsync(h->bbuf, bin, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    bin = h->bbuf;
  }

  // history buffer
  if (o.recordHistory) {
    if (h->histCap < maxIter + 1) {
      dfree(h->hist);
      h->hist = nullptr;
      h->histCap = 0;
      h->hist = dmalloc<double>((size_t)maxIter + 1);
      h->histCap = maxIter + 1;
    }
  }
  h->histN = -1;

  // state
  State* sh = h->st_host;
  std::memset(sh, 0, sizeof(State));
  sh->tol = tol;
  sh->relTol = o.relTol;
  sh->minIter = o.minIter;
  sh->maxIter = maxIter;
  sh->norm = o.norm;
  sh->record = o.recordHistory ? 1 : 0;
  sh->hist = h->hist;
  sh->histCap = h->histCap;
  CUDA_CHECK(cudaMemcpyAsync(h->st, sh, sizeof(State), cudaMemcpyHostToDevice, s));
  CUDA_CHECK(cudaMemsetAsync(h->ticket, 0, 2 * sizeof(unsigned), s));
  if (h->tbuf) CUDA_CHECK(cudaMemsetAsync(h->tbuf, 0, sizeof(unsigned long long) * 256 * 16, s));
  if (pipelined) {
    CUDA_CHECK(cudaMemsetAsync(h->z, 0, sizeof(double) * n, s));
    CUDA_CHECK(cudaMemsetAsync(h->s, 0, sizeof(double) * n, s));
    CUDA_CHECK(cudaMemsetAsync(h->p0, 0, sizeof(double) * n, s));
  } else {
    CUDA_CHECK(cudaMemsetAsync(h->p0, 0, sizeof(double) * n, s));
    CUDA_CHECK(cudaMemsetAsync(h->p1, 0, sizeof(double) * n, s));
  }

  // ---- r0 = b - A x0 and the criterion scale ---------------------------------------------
  double* sumA = pipelined ? h->nv : h->q;
  if (o.norm == LDU_NORM_OPENFOAM) {
    k_fill<<<small_grid(n), kBlock, 0, s>>>(n, 1.0, h->r);
    ++kernels;
    amul_dev(h, h->r, sumA, s, kernels);  // sumA = A 1 incl. interfaces
    k_sum_x<<<h->grid, kBlock, 0, s>>>(n, h->x, h->st, red_loop(h, CTL_XBAR, !mr));
    ++kernels;
    if (mr) allgather_ctl(h, CTL_XBAR, 2, s, kernels);
  }
  amul_dev(h, h->x, h->ybuf, s, kernels);
  k_resid<<<h->grid, kBlock, 0, s>>>(n, bin, h->ybuf, sumA, h->rD, h->r, h->st,
                                     red_loop(h, pipelined ? CTL_PIPE_SCALE : CTL_CG_INIT, !mr));
  ++kernels;
  if (mr) allgather_ctl(h, pipelined ? CTL_PIPE_SCALE : CTL_CG_INIT, 3, s, kernels);
  if (pipelined && h->p2pOn && h->nIfFaces) {  // w0 = A (rD.r0) over the peer mailboxes
    p2p_pack_async(h, PACK_SCALED, h->r, s, GATE_NONE);
    launch_spmv_scaled(h, h->r, h->w, s);
    p2p_join(h, s);
    k_iface_apply_p2p<<<small_grid(h->nIfCells), kBlock, 0, s>>>(
        h->nIfCells, h->ifCell, h->ifCellPtr, h->ifFaceIdx, h->ifCoeffs, h->w, nullptr,
        h->p2pDesc, h->nIfFaces);
    k_p2p_halo_consumed<<<1, 32, 0, s>>>(h->p2pDesc);
    kernels += 4;
    h->stats.haloBytes += 8LL * h->nIfFaces;
    k_pipe_dots<<<h->grid, kBlock, 0, s>>>(n, h->rD, h->r, h->w, h->st, red_loop(h, CTL_PIPE_TOP, !mr));
    ++kernels;
    if (h->fusePipe) {  // exchange 0 of the fused loop (LL words for the one-kernel loop)
      p2p_pack(h, h->mrFuse ? PACK_SCALED_LL : PACK_SCALED, h->w, s, GATE_LIVE);
      ++kernels;
    }
  } else if (pipelined) {
    // w0 = A u0 with u0 = rD.r0 (incl. interfaces), then the first fused reduction
    if (h->nIfFaces) {
      k_pack<<<small_grid(h->nIfFaces), kBlock, 0, s>>>(h->nIfFaces, h->ifFaceCells, PACK_SCALED,
                                                        h->r, h->rD, nullptr, nullptr, h->st,
                                                        h->sendbuf);
      ++kernels;
      halo_exchange(h, s);
    }
    launch_spmv_scaled(h, h->r, h->w, s);
    ++kernels;
    if (h->nIfFaces) {
      wait_halo(h, s);
      k_iface_apply<<<small_grid(h->nIfCells), kBlock, 0, s>>>(
          h->nIfCells, h->ifCell, h->ifCellPtr, h->ifFaceIdx, h->ifCoeffs, h->recvbuf, h->w, h->st);
      ++kernels;
    }
    k_pipe_dots<<<h->grid, kBlock, 0, s>>>(n, h->rD, h->r, h->w, h->st, red_loop(h, CTL_PIPE_TOP, !mr));
    ++kernels;
    if (mr && h->p2pOn && h->fusePipe && h->nIfFaces) {  // exchange 0 of the fused loop
      p2p_pack(h, PACK_SCALED, h->w, s, GATE_LIVE);
      ++kernels;
    }
    // multi-rank: the allgather of these sums is issued by the first loop trip (overlapped)
  }
  CUDA_CHECK(cudaGetLastError());
  if (pipelined && mr) {
    // k = -1 so that CTL_PIPE_NEXT of the first iteration evaluates i = 0
    static const int minus_one = -1;
    CUDA_CHECK(cudaMemcpyAsync(&h->st->k, &minus_one, sizeof(int), cudaMemcpyHostToDevice, s));
    if (h->p2pOn && h->fusePipe && h->mrFuse) {
      k_mr_init<<<1, 32, 0, s>>>(h->p2pDesc, h->st);
      ++kernels;
      if (h->mrFold && !rr) {  // the folded loop starts at iteration 0 with alpha_0 known
        k_ctl_ll<<<1, 64, 0, s>>>(h->st, h->p2pDesc, 1);
        ++kernels;
      }
    }
  }
  CUDA_CHECK(cudaEventRecord(h->ev[1], s));

  // ---- single rank, persistent cooperative kernel (latency-bound sizes) --------------------
  if (!mr && h->persist && !rr) {
    if (!h->ppartials) h->ppartials = dmalloc<double>((size_t)2 * kMaxVals * h->gridP);
    CUDA_CHECK(cudaEventRecord(h->ev[1], s));
    long long launches = 0;
    const int trips = tol == 0.0 ? std::max(1, maxIter) : std::max(1, std::min(maxIter, 256));
    if (maxIter > 0) {
      for (;;) {
        int ld = h->gridP, mt = trips;
        void* args[13];
        int nargs = 0;
        if (pipelined) {
          with_format(h, [&](auto A) {
            using Fmt = decltype(A);
            static thread_local Fmt Ak;
            Ak = A;
            void* a[] = {&Ak, &h->rD, &h->w, &h->w2, &h->z, &h->s, &h->p0, &h->x, &h->r, &h->st,
                         &h->ppartials, &ld, &mt};
            nargs = 13;
            for (int i = 0; i < nargs; ++i) args[i] = a[i];
            CUDA_CHECK(cudaEventRecord(h->ev_fork, s));
            CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_pipe_persist<Fmt>, h->gridP,
                                                   kBlock, args, 0, s));
          });
        } else {
          with_format(h, [&](auto A) {
            using Fmt = decltype(A);
            static thread_local Fmt Ak;
            Ak = A;
            void* a[] = {&Ak, &h->rD, &h->r, &h->p0, &h->p1, &h->q, &h->x, &h->st, &h->ppartials,
                         &ld, &mt};
            nargs = 11;
            for (int i = 0; i < nargs; ++i) args[i] = a[i];
            CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_cg_persist<Fmt>, h->gridP,
                                                   kBlock, args, 0, s));
          });
        }
        ++launches;
        if (tol == 0.0 && trips >= maxIter) break;
        CUDA_CHECK(cudaMemcpyAsync(sh, h->st, sizeof(State), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        if (sh->done || launches * (long long)trips > (long long)maxIter + 2) break;
      }
    }
    CUDA_CHECK(cudaEventRecord(h->ev[2], s));
    h->stats.kernels = kernels + launches;
    // pending x update (classical) / x = 0 when b = 0, on the device: one host sync per solve
    k_cg_final<<<small_grid(n), kBlock, 0, s>>>(n, h->p0, h->p1, h->x, h->st);
    ++h->stats.kernels;
    CUDA_CHECK(cudaMemcpyAsync(sh, h->st, sizeof(State), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaMemcpyAsync(x, h->x, sizeof(double) * n, xd ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    if (!xd) h->stats.d2hBytes += 8LL * n;
    CUDA_CHECK(cudaEventRecord(h->ev[3], s));
    if (h->stream != h->own_stream) {
      CUDA_CHECK(cudaEventRecord(h->ev_fork, s));
      CUDA_CHECK(cudaStreamWaitEvent(h->stream, h->ev_fork, 0));
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[3]));
    h->stats.solveMs = ms;
    CUDA_CHECK(cudaEventElapsedTime(&ms, h->ev[1], h->ev[2]));
    h->stats.iterMs = ms;
    h->stats.iterations = sh->iter;
    h->stats.reductions = sh->nRed;
    if (profile) {  // no per-pass split inside the persistent kernel: whole iterations
      h->stats.passMs[pipelined ? 1 : 0] = ms;
      h->stats.passLaunches[pipelined ? 1 : 0] = sh->iter;
    }
    if (sh->record) h->histN = std::min(sh->iter + 1, h->histCap);
    if (!sh->done) sh->status = LDU_NOT_CONVERGED;
    if (nIter) *nIter = sh->iter;
    if (finalRes) *finalRes = sh->res;
    return (ldu_status)sh->status;
  }

  // ---- iteration batches as CUDA graphs ----------------------------------------------------
  ldu_handle_s::Graph& G = rr ? h->graphRR[profile ? 1 : 0] : h->graphs[pipelined ? 1 : 0][profile ? 1 : 0];
  if (profile && (int)h->prof_ev.size() < 4 * batch) {
    for (cudaEvent_t e : h->prof_ev) cudaEventDestroy(e);
    h->prof_ev.assign(4 * batch, nullptr);
    for (auto& e : h->prof_ev) CUDA_CHECK(cudaEventCreate(&e));
    if (h->graphs[0][1].exec) { cudaGraphExecDestroy(h->graphs[0][1].exec); h->graphs[0][1] = {}; }
    if (h->graphs[1][1].exec) { cudaGraphExecDestroy(h->graphs[1][1].exec); h->graphs[1][1] = {}; }
    if (h->graphRR[1].exec) { cudaGraphExecDestroy(h->graphRR[1].exec); h->graphRR[1] = {}; }
  }
  if (const char* tr = std::getenv("LDU_TRACE"); tr && std::atoi(tr) == 1 && (int)h->trace.size() < 5 * batch) {
    h->trace.assign(5 * batch, nullptr);
    for (auto& e : h->trace) CUDA_CHECK(cudaEventCreate(&e));
    for (auto& row : h->graphs)
      for (auto& GG : row)
        if (GG.exec) { cudaGraphExecDestroy(GG.exec); GG = {}; }
    for (auto& GG : h->graphRR)
      if (GG.exec) { cudaGraphExecDestroy(GG.exec); GG = {}; }
  }
  if (!G.exec || G.batch != batch) {
    if (G.exec) {
      cudaGraphExecDestroy(G.exec);
      G = {};
    }
    const ldu_solve_stats saved = h->stats;  // capture enqueues nothing that runs now
    cudaGraph_t g;
    CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    G.kernels = rr ? (mr ? enqueue_pipe_rr_mr(h, batch, s, profile) : enqueue_pipe_rr(h, batch, s, profile))
                   : pipelined ? enqueue_pipe_iters(h, batch, s, profile)
                               : enqueue_cg_iters(h, batch, s, profile);
    CUDA_CHECK(cudaStreamEndCapture(s, &g));
    CUDA_CHECK(cudaGraphInstantiate(&G.exec, g, 0));
    CUDA_CHECK(cudaGraphDestroy(g));
    G.batch = batch;
    h->stats = saved;
  }
  cudaGraphExec_t gexec = G.exec;
  const long long kpb = G.kernels;
  const long long haloPerIter = h->nIfFaces ? 8LL * h->nIfFaces : 0;
  long long launched = 0;
  int batches = 0;
  std::vector<float> passT;  // profile: [batch][it][2] elapsed ms
  std::vector<float> traceT;  // LDU_TRACE: [batch][it < batch-1][5]
  // multi-rank pipelined needs one more loop trip: the decision on r_i is taken by the
  // control kernel after the overlapped allgather of trip i (single rank: in U_{i-1}).
  const bool folded = pipelined && mr && h->p2pOn && h->fusePipe && h->mrFuse && h->mrFold && !rr;
  const long long trips = (long long)maxIter + ((pipelined && mr && !folded) ? 1 : 0);
  auto collect = [&]() {
    for (int it = 0; it < batch; ++it)
      for (int p = 0; p < 2; ++p) {
        float ms = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&ms, h->prof_ev[4 * it + 2 * p], h->prof_ev[4 * it + 2 * p + 1]));
        passT.push_back(ms);
      }
  };
  if (maxIter > 0) {
    if (tol == 0.0 && !profile && h->trace.empty()) {  // fixed iterations: only breakdown / r == 0 stop early
      const long long nb = (trips + batch - 1) / batch;
      for (long long i = 0; i < nb; ++i) CUDA_CHECK(cudaGraphLaunch(gexec, s));
      batches = (int)nb;
    } else {
      for (;;) {
        CUDA_CHECK(cudaGraphLaunch(gexec, s));
        ++batches;
        CUDA_CHECK(cudaMemcpyAsync(sh, h->st, sizeof(State), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        if (profile) collect();
        if (!h->trace.empty() && pipelined && mr)
          for (int it = 0; it + 1 < batch; ++it) {
            float a[5];
            for (int k = 0; k < 4; ++k) cudaEventElapsedTime(&a[k], h->trace[5 * it + k], h->trace[5 * it + k + 1]);
            cudaEventElapsedTime(&a[4], h->trace[5 * it + 4], h->trace[5 * (it + 1)]);
            cudaGetLastError();
            for (int k = 0; k < 5; ++k) traceT.push_back(a[k]);
          }
        if (sh->done) break;
        if ((long long)batches * batch >= trips + batch) break;  // safety net
      }
    }
  }
  launched = (long long)batches * kpb;
  h->stats.haloBytes += (long long)batches * batch * haloPerIter;
  CUDA_CHECK(cudaEventRecord(h->ev[2], s));

  // pending x update (classical) / x = 0 when b = 0, on the device: one host sync per solve
  k_cg_final<<<small_grid(n), kBlock, 0, s>>>(n, h->p0, h->p1, h->x, h->st);
  ++kernels;
  CUDA_CHECK(cudaMemcpyAsync(sh, h->st, sizeof(State), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaMemcpyAsync(x, h->x, sizeof(double) * n, xd ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  if (!xd) h->stats.d2hBytes += 8LL * n;
  CUDA_CHECK(cudaEventRecord(h->ev[3], s));
  if (h->stream != h->own_stream) {
    CUDA_CHECK(cudaEventRecord(h->ev_fork, s));
    CUDA_CHECK(cudaStreamWaitEvent(h->stream, h->ev_fork, 0));
  }
  CUDA_CHECK(cudaStreamSynchronize(s));
  CUDA_CHECK(cudaGetLastError());

  float ms = 0.f;
  CUDA_CHECK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[3]));
  h->stats.solveMs = ms;
  CUDA_CHECK(cudaEventElapsedTime(&ms, h->ev[1], h->ev[2]));
  h->stats.iterMs = ms;
  if (h->tbuf && pipelined && mr && sh->iter > 20) {  // device %globaltimer stamps (debug)
    std::vector<unsigned long long> tb(256 * 16);
    CUDA_CHECK(cudaMemcpy(tb.data(), h->tbuf, sizeof(unsigned long long) * tb.size(), cudaMemcpyDeviceToHost));
    double acc[11] = {0};
    int cnt = 0;
    for (int k = 5; k < std::min(sh->iter - 2, 250); ++k) {
      unsigned long long a[16], nx[16];
      for (int q = 0; q < 16; ++q) {
        a[q] = tb[k * 16 + q];
        nx[q] = tb[(k + 1) * 16 + q];
      }
      a[2] = ~a[2];  // min slots are stored complemented
      a[4] = ~a[4];
      acc[0] += (double)(a[1] - a[0]);   // ctl: gather wait
      acc[1] += (double)(a[2] - a[1]);   // ctl end -> SU first block
      acc[2] += (double)(a[3] - a[2]);   // SU
      acc[3] += (double)(a[4] - a[3]);   // SU last block -> fixup first block
      acc[4] += (double)(a[5] - a[4]);   // fixup halo wait
      acc[5] += (double)(a[6] - a[5]);   // fixup work
      acc[6] += (double)(a[7] - a[6]);   // fixup fence + reduction + publish
      acc[7] += (double)(nx[0] - a[7]);  // -> next ctl start
      acc[8] += (double)(a[8] - a[6]);   // blocks done -> last block past the ticket
      acc[9] += (double)(a[9] - a[8]);   // sum of partials
      acc[10] += (double)(a[10] - a[9]); // publish
      ++cnt;
    }
    if (cnt && h->mrFuse && h->fusePipe) {
      double m[9] = {0};
      int mc = 0;
      for (int k = 5; k < std::min(sh->iter - 2, 250); ++k) {
        unsigned long long a[16], nx0 = tb[(k + 1) * 16 + 0];
        for (int q = 0; q < 16; ++q) a[q] = tb[k * 16 + q];
        a[2] = ~a[2];
        a[4] = ~a[4];
        m[0] += (double)(a[1] - a[0]);    // ctl gather wait
        m[1] += (double)(a[2] - a[1]);    // ctl end -> first block past pdl_wait
        m[2] += (double)(a[3] - a[2]);    // -> last bulk end
        m[3] += (double)(a[6] - a[4]);    // first boundary row begin -> last boundary end
        m[4] += (double)(a[6] - a[2]);    // first block start -> last boundary end
        m[5] += (double)(a[7] - a[3]);    // last bulk end -> last block at its ticket
        m[6] += (double)(a[12] - a[7]);   // -> last block past the ticket
        m[7] += (double)(a[13] - a[12]);  // sum + publish
        m[8] += (double)(nx0 - a[13]);    // -> next ctl start
        ++mc;
      }
      if (mc)
        fprintf(stderr, "[ldu gtimer mr rank %d] us: ctlwait %.1f ->SU %.1f bulk %.1f boundary %.1f (from start %.1f) ->ticket %.1f ticket %.1f publish %.1f ->ctl %.1f\n",
                h->rank, m[0] / mc / 1e3, m[1] / mc / 1e3, m[2] / mc / 1e3, m[3] / mc / 1e3, m[4] / mc / 1e3,
                m[5] / mc / 1e3, m[6] / mc / 1e3, m[7] / mc / 1e3, m[8] / mc / 1e3);
    } else if (cnt)
      fprintf(stderr, "[ldu gtimer rank %d] us: ctlwait %.1f ->SU %.1f SU %.1f ->fix %.1f fixwait %.1f fixwork %.1f fixfin %.1f (ticket %.1f sum %.1f publish %.1f) ->ctl %.1f\n",
              h->rank, acc[0] / cnt / 1e3, acc[1] / cnt / 1e3, acc[2] / cnt / 1e3, acc[3] / cnt / 1e3,
              acc[4] / cnt / 1e3, acc[5] / cnt / 1e3, acc[6] / cnt / 1e3, acc[8] / cnt / 1e3,
              acc[9] / cnt / 1e3, acc[10] / cnt / 1e3, acc[7] / cnt / 1e3);
  }
  if (!h->trace.empty() && pipelined && mr) {  // segments of the real iterations (debug)
    double seg[5] = {0, 0, 0, 0, 0};
    int cnt = 0;
    const int per = batch - 1;
    for (size_t g = 0; g < traceT.size() / 5; ++g) {
      const long long trip = (long long)(g / per) * batch + g % per;
      if (trip < 2 || trip > sh->iter - 1) continue;
      for (int k = 0; k < 5; ++k) seg[k] += traceT[5 * g + k];
      ++cnt;
    }
    if (cnt)
      fprintf(stderr, "[ldu trace rank %d] %d iters, us/iter: ctl %.1f pack %.1f SU %.1f fixup %.1f gap %.1f\n",
              h->rank, cnt, 1e3 * seg[0] / cnt, 1e3 * seg[1] / cnt, 1e3 * seg[2] / cnt,
              1e3 * seg[3] / cnt, 1e3 * seg[4] / cnt);
  }
  h->stats.kernels = kernels + launched;
  h->stats.iterations = sh->iter;
  h->stats.reductions = sh->nRed;                      // counted on the device (run_ctl)
  h->stats.allreduces = mr ? (long long)sh->nRed : 0;  // every multi-rank control step gathers
  if (profile) {  // passes that did work: trips 0 .. iter-1 (multi-rank pipelined: 1 .. iter)
    const long long first = (pipelined && mr && !folded) ? 1 : 0;
    for (long long g = first; g < first + sh->iter && g < (long long)passT.size() / 2; ++g)
      for (int p = 0; p < 2; ++p) {
        h->stats.passMs[p] += passT[2 * g + p];
        h->stats.passLaunches[p] += 1;
      }
  }
  if (sh->record) h->histN = std::min(sh->iter + 1, h->histCap);
  if (!sh->done) {  // safety net: batches exhausted without a decision
    sh->status = LDU_NOT_CONVERGED;
  }
  if (nIter) *nIter = sh->iter;
  if (finalRes) *finalRes = sh->res;
  return (ldu_status)sh->status;
}

void release_work(ldu_handle h) {
  for (double** p : {&h->x, &h->r, &h->p0, &h->p1, &h->q, &h->w, &h->w2, &h->nv, &h->z, &h->s,
                     &h->ppartials,
                     &h->bbuf, &h->ybuf, &h->hist}) {
    dfree(*p);
    *p = nullptr;
  }
  for (auto& row : h->graphs)
    for (auto& G : row) {
      if (G.exec) cudaGraphExecDestroy(G.exec);
      G = {};
    }
  for (auto& G : h->graphRR) {
    if (G.exec) cudaGraphExecDestroy(G.exec);
    G = {};
  }
  for (cudaEvent_t e : h->prof_ev) cudaEventDestroy(e);
  h->prof_ev.clear();
}

// ---------------------------------------------------------------------------------------------
// NVLink peer-memory setup (collective over the comm): mailbox allocation, CUDA IPC handle and
// interface-table exchange with NCCL allgathers, peer mappings, the device descriptor.
// ---------------------------------------------------------------------------------------------
void p2p_setup(ldu_handle h) {
  ldu_comm cm = h->comm;
  const int R = cm->nRanks, me = cm->rank;
  if (R > kP2PMaxRanks || (int)h->ifaces.size() > kP2PMaxIf)
    throw Error(LDU_ERR_INVALID_ARG, "peer-memory path supports <= 64 ranks and <= 16 interfaces");
  cudaStream_t s = h->own_stream;
  const size_t bytes = MailboxLayout::bytes(h->nIfFaces);
  // a plain (never staggered) allocation: peers map it through its CUDA IPC handle, which
  // names the allocation base
  CUDA_CHECK(cudaMalloc((void**)&h->mailbox, bytes));
  CUDA_CHECK(cudaMemset(h->mailbox, 0, bytes));
  // interface index of every packed face
  std::vector<int> faceIf(std::max(1, h->nIfFaces), 0);
  for (size_t k = 0; k < h->ifaces.size(); ++k)
    for (int i = 0; i < h->ifaces[k].nFaces; ++i) faceIf[h->ifaces[k].offset + i] = (int)k;
  h->ifFaceIf = dmalloc<int>(faceIf.size());
  CUDA_CHECK(cudaMemcpy(h->ifFaceIf, faceIf.data(), sizeof(int) * faceIf.size(), cudaMemcpyHostToDevice));

  // exchange IPC handles and interface tables: table = [nIf, nIfFaces, (nb, nFaces, off) x 16]
  constexpr int TW = 2 + 3 * kP2PMaxIf;
  cudaIpcMemHandle_t mine;
  CUDA_CHECK(cudaIpcGetMemHandle(&mine, h->mailbox));
  std::vector<int> tbl(TW, 0);
  tbl[0] = (int)h->ifaces.size();
  tbl[1] = h->nIfFaces;
  for (size_t k = 0; k < h->ifaces.size(); ++k) {
    tbl[2 + 3 * k] = h->ifaces[k].neighbRank;
    tbl[3 + 3 * k] = h->ifaces[k].nFaces;
    tbl[4 + 3 * k] = h->ifaces[k].offset;
  }
  char* dbuf = dmalloc<char>((size_t)R * (sizeof(cudaIpcMemHandle_t) + sizeof(int) * TW) + 64);
  char* dsend = dbuf;
  const size_t rec = sizeof(cudaIpcMemHandle_t) + sizeof(int) * TW;
  std::vector<char> hsend(rec), hrecv(rec * R);
  std::memcpy(hsend.data(), &mine, sizeof(mine));
  std::memcpy(hsend.data() + sizeof(mine), tbl.data(), sizeof(int) * TW);
  if (cm->nccl()) {
    char* dall = dmalloc<char>(rec * R);
    CUDA_CHECK(cudaMemcpy(dsend, hsend.data(), rec, cudaMemcpyHostToDevice));
    NCCL_CHECK(ncclAllGather(dsend, dall, rec, ncclChar, cm->red, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    CUDA_CHECK(cudaMemcpy(hrecv.data(), dall, rec * R, cudaMemcpyDeviceToHost));
    dfree(dall);
  } else {
    host_allgather(cm, hsend.data(), hrecv.data(), rec);
  }
  dfree(dbuf);

  P2PDesc d{};
  d.rank = me;
  d.nRanks = R;
  d.nIf = (int)h->ifaces.size();
  h->peerMailbox.assign(R, nullptr);
  for (int r = 0; r < R; ++r) {
    if (r == me) {
      d.base[r] = h->mailbox;
      continue;
    }
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, hrecv.data() + rec * r, sizeof(hd));
    void* ptr = nullptr;
    CUDA_CHECK(cudaIpcOpenMemHandle(&ptr, hd, cudaIpcMemLazyEnablePeerAccess));
    h->peerMailbox[r] = static_cast<char*>(ptr);
    d.base[r] = static_cast<char*>(ptr);
  }
  auto peer_tbl = [&](int r) {
    return reinterpret_cast<const int*>(hrecv.data() + rec * r + sizeof(cudaIpcMemHandle_t));
  };
  for (int k = 0; k < d.nIf; ++k) {
    const DevInterface& it = h->ifaces[k];
    int ord = 0;  // ordinal of this interface among mine to the same neighbour (pairing, Z22)
    for (int j = 0; j < k; ++j) ord += h->ifaces[j].neighbRank == it.neighbRank;
    const int* pt = peer_tbl(it.neighbRank);
    int found = -1, seen = 0;
    for (int kk = 0; kk < pt[0]; ++kk)
      if (pt[2 + 3 * kk] == me && seen++ == ord) {
        found = kk;
        break;
      }
    if (found < 0 || pt[3 + 3 * found] != it.nFaces)
      throw Error(LDU_ERR_INVALID_ARG, "interface " + std::to_string(k) +
                                           ": no matching interface (same face count) on rank " +
                                           std::to_string(it.neighbRank));
    d.ifNeighbor[k] = it.neighbRank;
    d.ifLocalOff[k] = it.offset;
    d.ifNFaces[k] = it.nFaces;
    d.ifRemoteOff[k] = pt[4 + 3 * found];
    d.ifRemoteIdx[k] = found;
    d.ifRemoteTotal[k] = pt[1];
  }
  if (const char* tr = std::getenv("LDU_TRACE"); tr && std::atoi(tr) == 2) {
    h->tbuf = dmalloc<unsigned long long>(256 * 16);
    d.tbuf = h->tbuf;
  }
  h->p2pDesc = dmalloc<P2PDesc>(1);
  CUDA_CHECK(cudaMemcpy(h->p2pDesc, &d, sizeof(d), cudaMemcpyHostToDevice));
  if (h->nIfFaces > 0) {  // boundary-row metadata of the one-kernel pipelined loop
    const int L = h->n - h->mrGapLen;
    h->mrTailMeta = dmalloc<int4>(std::max(1, L));
    k_build_tail_meta<<<small_grid(L), kBlock, 0, s>>>(L, h->mrTailIf, h->ifCellPtr, h->ifFaceIdx,
                                                        h->ifFaceIf, h->p2pDesc, h->mrTailMeta);
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  // every rank's mailbox is mapped before anyone writes into it
  if (cm->nccl()) {
    int* flag = dmalloc<int>(1);
    NCCL_CHECK(ncclAllReduce(flag, flag, 1, ncclInt, ncclSum, cm->red, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    dfree(flag);
  } else {
    CUDA_CHECK(cudaDeviceSynchronize());
    char one = 1;
    std::vector<char> all(R);
    host_allgather(cm, &one, all.data(), 1);  // barrier
  }
  h->p2pOn = true;
}

// the caller's host all-gather of a host-bootstrapped comm (setup only, never inside a solve)
void host_allgather(ldu_comm cm, const void* send, void* recv, size_t bytes) {
  if (!cm->hostAllgather) throw Error(LDU_ERR_STATE, "comm has neither NCCL nor a host all-gather");
  if (cm->hostAllgather(cm->hostCtx, send, recv, (unsigned long long)bytes) != 0)
    throw Error(LDU_ERR_INVALID_ARG, "the host all-gather callback failed");
}

void p2p_release(ldu_handle h) {
  for (char* p : h->peerMailbox)
    if (p) cudaIpcCloseMemHandle(p);
  h->peerMailbox.clear();
  dfree(h->mailbox);
  dfree(h->p2pDesc);
  dfree(h->ifFaceIf);
  h->mailbox = nullptr;
  h->p2pDesc = nullptr;
  h->ifFaceIf = nullptr;
  h->p2pOn = false;
}

// Launch geometry: grid = SMs x resident blocks of the heaviest pass (multiple of the SM count).
void configure(ldu_handle h) {
  cudaDeviceProp prop;
  CUDA_CHECK(cudaGetDeviceProperties(&prop, h->device));
  // kernel variant of the SpMV-bearing passes (DIA layout): 0 generic, 1 hoisted, 2 hoisted x2
  h->variant = 7;  // measured fastest for classical pass A (profiles/r01_variants)
  if (const char* v = std::getenv("LDU_VARIANT")) h->variant = std::atoi(v);
  if (h->variant < 0 || h->variant > 7) h->variant = 0;
  h->chunkK = 2048;
  h->fusePipe = true;
  if (const char* v = std::getenv("LDU_PIPE_FUSE")) h->fusePipe = std::atoi(v) != 0;
  // PDL on the multi-rank fused pipelined chain is opt-in: measured +0.7 % at 256^3 / 4 ranks,
  // but at 512^3 / 4 ranks it produced a wrong iterate (BREAKDOWN after 18 iterations, then a
  // peer wait timeout) that LDU_PDL=0 does not (profiles/r01_amg/SUMMARY.md)
  h->pdl = true;  // multi-rank fused chains: control step -> pass with programmatic launch
  if (const char* v = std::getenv("LDU_PDL")) h->pdl = std::atoi(v) != 0;
  h->mrFuse = true;
  if (const char* v = std::getenv("LDU_MR_FUSE")) h->mrFuse = std::atoi(v) != 0;
  h->mrFold = true;
  if (const char* v = std::getenv("LDU_MR_FOLD")) h->mrFold = std::atoi(v) != 0;
  h->cgLL = true;  // classical multi-rank: LL reductions, control steps in the last blocks
  if (const char* v = std::getenv("LDU_CG_LL")) h->cgLL = std::atoi(v) != 0;
  h->mrPre = 4;
  if (const char* v = std::getenv("LDU_MR_PRE")) h->mrPre = std::atoi(v) >= 8 ? 8 : (std::atoi(v) >= 4 ? 4 : 0);
  // persistent cooperative kernels for single-rank, latency-bound sizes (LDU_PERSIST=0/1 forces)
  h->persist = !(h->comm && h->comm->nRanks > 1) && (long long)h->n * 80 < (long long)prop.l2CacheSize;
  if (const char* v = std::getenv("LDU_PERSIST")) h->persist = std::atoi(v) != 0 && !(h->comm && h->comm->nRanks > 1);
  if (const char* v = std::getenv("LDU_CHUNK")) h->chunkK = std::max(256, std::atoi(v) / 256 * 256);
  const long long need = ((long long)h->n + kBlock - 1) / kBlock;
  // multi-rank: SMs left free for the NCCL kernels that run concurrently with the passes
  // (only the NCCL fallback launches NCCL kernels inside the iteration loop)
  int reserve = 0;
  if (h->comm && h->comm->nRanks > 1) {
    const char* v = std::getenv("LDU_P2P");
    if (v && std::atoi(v) == 0) reserve = 4;
  }
  if (const char* v = std::getenv("LDU_RESERVE_SMS")) reserve = std::max(0, std::atoi(v));
  const int sms = std::max(1, prop.multiProcessorCount - reserve);
  auto grid_of = [&](const void* fn) {
    int o = 1;
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, kBlock, 0));
    long long g = (long long)sms * std::max(1, o);
    return (int)std::max(1LL, std::min(g, need));
  };
  h->grid = grid_of((const void*)k_cg_passB<false>);  // streaming passes
  // plane-marching geometry (DIA with one far offset D >= 4096 and near offsets <= 1024)
  h->marchOk = false;
  if (h->layout == LDU_LAYOUT_DIA_SYM && h->nd >= 2) {
    const int D = h->off[h->nd - 1], H = h->off[h->nd - 2];
    if (D >= 4096 && H <= kMarchHMax && H < D) {
      h->marchOk = true;
      h->mT = kMarchT;
      h->mH = H;
      h->mTiles = (D + h->mT - 1) / h->mT;
      h->mPlanes = (int)(((long long)h->n + D - 1) / D);
    }
  }
  // TMA plane march: one 512-thread block per SM, grid = tiles * chunks = #SMs, T even and
  // small enough that the shared footprint of the heaviest mode fits; D, H, n even (16 B copies)
  h->tmaOk = false;
  h->tL = 1;
  if (const char* v = std::getenv("LDU_TMA_L")) h->tL = std::atoi(v) == 2 ? 2 : 1;
  if (h->marchOk && h->off[h->nd - 1] % 2 == 0 && h->mH % 2 == 0 && h->n % 2 == 0) {
    with_dia(h, [&](auto A) {
      constexpr int ND = sizeof(A.off) / sizeof(int);
      if constexpr (ND >= 2) {
        const int D = h->off[h->nd - 1];
        const long long G = prop.multiProcessorCount;
        const long long maxSmem = prop.sharedMemPerBlockOptin - 2048;  // static smem headroom
        int bestTiles = 0, bestCh = 0;
        long long bestT = 0;
        bool bestStrict = false;
        for (long long ch = 1; ch <= G; ++ch) {
          if (G % ch) continue;
          const long long tiles = G / ch;
          long long T = (D + tiles - 1) / tiles;
          T += T & 1;
          const long long need = h->tL == 1 ? tma_smem_doubles<ND, MARCH_A, 1>(T, h->mH)
                                            : tma_smem_doubles<ND, MARCH_A, 2>(T, h->mH);
          if (8LL * need > maxSmem) continue;
          const bool strict = T >= 2LL * h->mH && T >= 256 && (h->mPlanes + ch - 1) / ch >= 8;
          // prefer strict geometries, then the largest tile (least halo re-read)
          if (!bestTiles || (strict && !bestStrict) || (strict == bestStrict && T > bestT)) {
            bestTiles = (int)tiles;
            bestCh = (int)ch;
            bestT = T;
            bestStrict = strict;
          }
        }
        if (bestTiles) {
          h->tmaOk = true;
          h->tmaStrict = bestStrict;
          h->tT = (int)bestT;
          h->tTiles = bestTiles;
          h->tChunk = (h->mPlanes + bestCh - 1) / bestCh;
          h->tGrid = bestTiles * ((h->mPlanes + h->tChunk - 1) / h->tChunk);
          const void* fns[6] = {(const void*)k_tma_march<ND, MARCH_AMUL, 1>, (const void*)k_tma_march<ND, MARCH_S, 1>,
                                (const void*)k_tma_march<ND, MARCH_A, 1>, (const void*)k_tma_march<ND, MARCH_AMUL, 2>,
                                (const void*)k_tma_march<ND, MARCH_S, 2>, (const void*)k_tma_march<ND, MARCH_A, 2>};
          const size_t sm[3] = {tma_smem<ND, MARCH_AMUL>(h), tma_smem<ND, MARCH_S>(h), tma_smem<ND, MARCH_A>(h)};
          for (int i = 0; i < 6; ++i)
            CUDA_CHECK(cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm[i % 3]));
        }
      }
    });
  }
  if (h->variant == 4 && !h->tmaOk) h->variant = 0;
  if (h->variant == 3 && !h->marchOk) h->variant = 0;
  if (use_march(h)) {
    with_dia(h, [&](auto A) {
      constexpr int ND = sizeof(A.off) / sizeof(int);
      if constexpr (ND >= 2) {
        const size_t smem = march_smem(h);
        const void* fns[3] = {(const void*)k_march<ND, MARCH_AMUL>, (const void*)k_march<ND, MARCH_S>,
                              (const void*)k_march<ND, MARCH_A>};
        int occ = 1 << 30;
        for (const void* fn : fns) {
          CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          int o = 1;
          CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, kBlock, smem));
          occ = std::min(occ, std::max(1, o));
        }
        // grid G = SMs * occ = tiles * chunks; the tile width T = ceil(D / tiles) <= kMarchT.
        // Largest chunk count (most parallel planes) keeping T <= kMarchT and >= 2H, and at
        // least 8 planes per chunk (prologue of 2 planes per chunk).
        const int D = h->off[h->nd - 1];
        const long long G = (long long)prop.multiProcessorCount * occ;
        int bestTiles = 0, bestCh = 0;
        for (long long ch = 1; ch <= G; ++ch) {
          if (G % ch) continue;
          const long long tiles = G / ch;
          const long long T = (D + tiles - 1) / tiles;
          if (T > kMarchT || T < 2LL * h->mH || T < kBlock) continue;
          if ((h->mPlanes + ch - 1) / ch < 8) continue;
          bestTiles = (int)tiles;
          bestCh = (int)ch;  // keep the largest ch (ascending loop)
        }
        h->marchStrict = bestTiles > 0;
        if (!bestTiles) {  // relaxed geometry (small meshes; only used when LDU_VARIANT=3)
          long long T = std::max<long long>({(D + G - 1) / G, 2LL * h->mH, 32LL});
          T = std::min<long long>(T, kMarchT);
          bestTiles = (int)((D + T - 1) / T);
          bestCh = (int)std::max(1LL, std::min<long long>(h->mPlanes, G / bestTiles));
        }
        h->mTiles = bestTiles;
        h->mT = (D + bestTiles - 1) / bestTiles;
        h->mChunk = (h->mPlanes + bestCh - 1) / bestCh;
        h->gridA = bestTiles * ((h->mPlanes + h->mChunk - 1) / h->mChunk);
      }
    });
  } else if (use_dia_kernels(h)) {
    with_dia(h, [&](auto A) {
      constexpr int ND = sizeof(A.off) / sizeof(int);
      h->gridA = h->variant == 2 ? grid_of((const void*)k_cg_passA_dia<ND, 2>)
                                 : grid_of((const void*)k_cg_passA_dia<ND, 1>);
    });
  } else {
    with_format(h, [&](auto A) {
      using Fmt = decltype(A);
      h->gridA = grid_of((const void*)k_cg_passA<Fmt>);
    });
  }
  if (use_tma(h)) h->gridA = h->tGrid;
  if (h->variant == 7) {  // the SpMV-bearing kernel of the split pass A is k_cg_passA2 (40 regs)
    with_format(h, [&](auto A) { h->gridA = grid_of((const void*)k_cg_passA2<decltype(A)>); });
  }
  // fused pipelined pass: 6 resident blocks per SM (LDU_SU_MINB=8 single rank: 8, measured slower)
  h->suMinB = 6;
  if (const char* v = std::getenv("LDU_SU_MINB")) h->suMinB = std::atoi(v) == 8 && !(h->comm && h->comm->nRanks > 1) ? 8 : 6;
  with_format(h, [&](auto A) {
    using Fmt = decltype(A);
    h->gridSU = h->suMinB == 8 ? grid_of((const void*)k_pipe_SU<Fmt, 8>) : grid_of((const void*)k_pipe_SU<Fmt>);
    h->gridSUmr = h->mrPre == 8 ? grid_of((const void*)k_pipe_SU_mr<Fmt, 8>)
                : h->mrPre == 4 ? grid_of((const void*)k_pipe_SU_mr<Fmt, 4>)
                                : grid_of((const void*)k_pipe_SU_mr<Fmt, 0>);
  });
  if (h->variant == 6 && h->layout == LDU_LAYOUT_DIA_SYM && h->off[0] == 1) {
    with_dia(h, [&](auto A) {
      constexpr int ND = sizeof(A.off) / sizeof(int);
      h->gridA = grid_of((const void*)k_cg_passA_shfl<ND>);
    });
  }
  if (h->variant == 5) {
    with_format(h, [&](auto A) {
      using Fmt = decltype(A);
      const void* fns[2] = {(const void*)k_cg_passA_chunk<Fmt>, (const void*)k_spmv_scaled_chunk<Fmt>};
      for (const void* fn : fns)  // all of the unified L1/shared storage as L1
        CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
      h->gridA = grid_of((const void*)k_cg_passA_chunk<Fmt>);
    });
  }
  if (h->persist) {  // co-resident grid for the cooperative launches
    int o1 = 1, o2 = 1;
    with_format(h, [&](auto A) {
      using Fmt = decltype(A);
      CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_pipe_persist<Fmt>, kBlock, 0));
      CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_cg_persist<Fmt>, kBlock, 0));
    });
    const long long g = (long long)prop.multiProcessorCount * std::max(1, std::min(o1, o2));
    h->gridP = (int)std::max(1LL, std::min(g, need));
  }
  h->maxParts = std::max({h->grid, h->gridA, h->gridSU, h->gridSUmr}) + 4096;
  h->partials = dmalloc<double>((size_t)kMaxVals * h->maxParts);
  h->ticket = dmalloc<unsigned>(2);  // [0] reductions, [1] halo pack (may run concurrently)
  CUDA_CHECK(cudaMemset(h->ticket, 0, 2 * sizeof(unsigned)));
  h->sums = dmalloc<double>(kMaxVals);
  h->gsums = dmalloc<double>((size_t)kMaxVals * std::max(1, h->nRanks));
  CUDA_CHECK(cudaMemset(h->gsums, 0, sizeof(double) * kMaxVals * std::max(1, h->nRanks)));
  h->st = dmalloc<State>(1);
  CUDA_CHECK(cudaMallocHost((void**)&h->st_host, sizeof(State)));
  if (h->comm && h->comm->nRanks > 1) {
    const char* v = std::getenv("LDU_P2P");
    if (!h->comm->nccl() || !v || std::atoi(v) != 0) p2p_setup(h);  // host comm: peer memory only
  }
}

double stream_triad(int device, long long n, int reps) {
  CUDA_CHECK(cudaSetDevice(device));
  n &= ~1LL;
  double *a = dmalloc<double>(n), *b = dmalloc<double>(n), *c = dmalloc<double>(n);
  cudaStream_t s;
  CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CUDA_CHECK(cudaEventCreate(&e0));
  CUDA_CHECK(cudaEventCreate(&e1));
  CUDA_CHECK(cudaMemsetAsync(b, 0, 8 * n, s));
  CUDA_CHECK(cudaMemsetAsync(c, 0, 8 * n, s));
  cudaDeviceProp prop;
  CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
  const int grid = prop.multiProcessorCount * 8;
  double best = 0.0;
  for (int r = 0; r < reps + 1; ++r) {
    CUDA_CHECK(cudaEventRecord(e0, s));
    k_triad<<<grid, 256, 0, s>>>(n, a, b, c, 3.0);
    CUDA_CHECK(cudaEventRecord(e1, s));
    CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    if (r > 0) best = std::max(best, 24.0 * n / (ms * 1e-3) / 1e9);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(s);
  dfree(a);
  dfree(b);
  dfree(c);
  return best;
}

}  // namespace ldu

// aggregation-AMG V-cycle and AMG-preconditioned solvers (NEXT-2), same translation unit
#include "ldu_amg_solve.cuh"
