// ldu_amg_solve.cuh -- V-cycle and AMG-preconditioned CG / pipelined CG (NEXT-2; P:236,
// Table 2).  Included at the end of ldu_solve.cu: it shares that translation unit's
// helpers (layout dispatch, reductions, r0, graph plumbing).
//
// V-cycle z = B f (reading Z32), level l < L with A_l, P_l, R_l, w_l, rD_l:
//   K1  r_l = f_l - A_l (w rD f_l)                 pre-sweep from x = 0 fused with the residual
//   K2  f_{l+1} = R_l r_l                          restriction
//       ... level l+1 ...   (level L: z_L = A_L^-1 f_L, dense inverse)
//   K3  x_l = w rD f_l + P_l z_{l+1}               prolongation added to the pre-sweep iterate
//   K4  z_l = x_l + w rD (f_l - A_l x_l)           post-sweep
// Level 0 runs K1 / K4 on the handle's own layout (DIA / SELL-32, one row per thread); coarser
// levels and every P / R are CSR with a sub-warp of `group` lanes per row (fixed-order shuffle
// reduction: deterministic).
//
// AMG-PCG, iteration k (SURVEY §8(c) c2 with z = B r):
//   V-cycle z_k = B r_k, K4 of level 0 carries the partial (z_k, r_k)   -> ctl: beta_k
//   pass A: x += alpha_{k-1} p_{k-1}; p_k = z_k + beta_k p_{k-1} (recomputed at the neighbours,
//           ping-pong); q = A p_k; partial (p_k, q)                       -> ctl: alpha_k
//   pass B: r -= alpha_k q; partial crit(r)                                -> ctl: test
// AMG-PipeCG, iteration i (c3 literal Ghysels-Vanroose, u = B r, m = B w):
//   V-cycle m_i = B w_i
//   pass SU: n = A m (row by row, never stored); z = n + b z; q = m + b q; s = w + b s;
//            p = u + b p; x += a p; r -= a s; u -= a q; w -= a z; partials (r,u), (w,u), crit(r)
//                                                                          -> ctl: a, b, test
#pragma once

#include "ldu_amg.cuh"

namespace ldu {
namespace {

// ---- CSR-vector rows: `G` lanes per row, grid-stride over warps -------------------------------
// Each lane sums the entries k = start + sub, + G, + 2G, ... of its row in that order (U of them
// per trip, loads issued together for memory-level parallelism), then the G lanes combine in a
// fixed xor-butterfly: deterministic.  G is chosen per matrix so that a lane holds ~U entries.
template <int G, class Epi>
__global__ void __launch_bounds__(kBlock) k_csr_vec(CsrView A, Epi e, const State* st) {
  if (st && st->done) return;
  constexpr int kCsrU = G == 1 ? 4 : 8;  // entries per lane per trip (see group_of)
  constexpr int RPW = 32 / G;  // rows per warp
  const int lane = threadIdx.x & 31, sub = lane & (G - 1);
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long base = warp * RPW; base < A.n; base += nwarps * RPW) {
    const int row = (int)(base + lane / G);
    double s = 0.0;
    if (row < A.n) {
      const int end = __ldg(A.ptr + row + 1);
      for (int k = __ldg(A.ptr + row) + sub; k < end; k += kCsrU * G) {
        int c[kCsrU];
        double v[kCsrU], x[kCsrU];
#pragma unroll
        for (int u = 0; u < kCsrU; ++u) {
          const int kk = k + u * G;
          const bool ok = kk < end;
          c[u] = ok ? __ldg(A.col + kk) : 0;
          v[u] = ok ? __ldg(A.val + kk) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kCsrU; ++u) x[u] = e.in(c[u]);
#pragma unroll
        for (int u = 0; u < kCsrU; ++u)
          if (k + u * G < end) s = fma(v[u], x[u], s);
      }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (sub == 0 && row < A.n) e.out(row, s);
  }
}

struct EpiPre {  // K1 at level >= 1: r = f - A xpre, xpre = w rD f stored by the restriction
  const double* __restrict__ xpre;
  const double* __restrict__ f;
  double* __restrict__ r;
  __device__ __forceinline__ double in(int j) const { return __ldg(xpre + j); }
  __device__ __forceinline__ void out(int i, double s) const { r[i] = f[i] - s; }
};
struct EpiRestrict {  // K2: f_c = R r; and the next level's pre-sweep iterate w_c rD_c f_c
  const double* __restrict__ r;
  double* __restrict__ fc;
  double* __restrict__ xpre;  // nullptr for the coarsest level
  double w;
  const double* __restrict__ rDc;
  __device__ __forceinline__ double in(int j) const { return __ldg(r + j); }
  __device__ __forceinline__ void out(int i, double s) const {
    fc[i] = s;
    if (xpre) xpre[i] = w * rDc[i] * s;
  }
};
struct EpiProlong0 {  // K3 at level 0: x = w rD f + P xc
  double w;
  const double* __restrict__ rD;
  const double* __restrict__ f;
  const double* __restrict__ xc;
  double* __restrict__ x;
  __device__ __forceinline__ double in(int j) const { return __ldg(xc + j); }
  __device__ __forceinline__ void out(int i, double s) const { x[i] = w * rD[i] * f[i] + s; }
};
struct EpiProlong {  // K3 at level >= 1: x = xpre + P xc (in place over xpre)
  const double* __restrict__ xc;
  double* x;
  __device__ __forceinline__ double in(int j) const { return __ldg(xc + j); }
  __device__ __forceinline__ void out(int i, double s) const { x[i] = x[i] + s; }
};
struct EpiPost {  // K4: z = x + w rD (f - A x)
  double w;
  const double* __restrict__ rD;
  const double* __restrict__ f;
  const double* __restrict__ x;
  double* __restrict__ z;
  __device__ __forceinline__ double in(int j) const { return __ldg(x + j); }
  __device__ __forceinline__ void out(int i, double s) const { z[i] = x[i] + w * rD[i] * (f[i] - s); }
};

// SELL-32 rows (coarse A_l, see attach_sell): one row per thread, lane-interleaved pairs, 4 pair
// loads in flight per trip; padding is (a column of the row, 0): no data-dependent exit
template <class Epi>
__global__ void __launch_bounds__(kBlock) k_sell_rows(SellView A, Epi e, const State* st) {
  if (st && st->done) return;
  GRID_STRIDE(c, A.n) {
    const int slice = c >> 5, lane = c & 31;
    const long long base = __ldg(A.slicePtr + slice);
    const int np = __ldg(A.npairs + slice);
    double s = 0.0;
    int jj = 0;
    for (; jj + 4 <= np; jj += 4) {
      int2 cc[4];
      double2 vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const long long q = (base + jj + u) * 32 + lane;
        cc[u] = __ldg(A.col + q);
        vv[u] = __ldg(A.val + q);
      }
      double x0[4], x1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x0[u] = e.in(cc[u].x);
        x1[u] = e.in(cc[u].y);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s = fma(vv[u].x, x0[u], s);
        s = fma(vv[u].y, x1[u], s);
      }
    }
    for (; jj < np; ++jj) {
      const long long q = (base + jj) * 32 + lane;
      const int2 cc = __ldg(A.col + q);
      const double2 vv = __ldg(A.val + q);
      s = fma(vv.x, e.in(cc.x), s);
      s = fma(vv.y, e.in(cc.y), s);
    }
    e.out(c, s);
  }
}

int csr_grid(long long rows, int G) {
  const long long warps = (rows + 32 / G - 1) / (32 / G);
  const long long b = (warps * 32 + kBlock - 1) / kBlock;
  return (int)std::max(1LL, std::min(b, 148LL * 16));
}

template <class Epi>
void launch_csr(const CsrMat& M, const Epi& e, const State* st, cudaStream_t s) {
  if (M.useSell) {
    const long long b = ((long long)M.nrows + kBlock - 1) / kBlock;
    k_sell_rows<<<(int)std::max(1LL, std::min(b, 148LL * 8)), kBlock, 0, s>>>(sell_view(M), e, st);
    return;
  }
  const CsrView v = view(M);
  const int g = csr_grid(M.nrows, M.group);
  switch (M.group) {
    case 1: k_csr_vec<1><<<g, kBlock, 0, s>>>(v, e, st); break;
    case 2: k_csr_vec<2><<<g, kBlock, 0, s>>>(v, e, st); break;
    case 4: k_csr_vec<4><<<g, kBlock, 0, s>>>(v, e, st); break;
    case 8: k_csr_vec<8><<<g, kBlock, 0, s>>>(v, e, st); break;
    case 16: k_csr_vec<16><<<g, kBlock, 0, s>>>(v, e, st); break;
    default: k_csr_vec<32><<<g, kBlock, 0, s>>>(v, e, st); break;
  }
}

// ---- level 0 on the handle's layout -----------------------------------------------------------
template <class Fmt>
__global__ void __launch_bounds__(kBlock) k_vc_pre(Fmt A, const double* __restrict__ diag,
                                                   const double* __restrict__ rD, double w,
                                                   const double* __restrict__ f,
                                                   double* __restrict__ r, const State* st) {
  if (st && st->done) return;
  GRID_STRIDE(c, A.n) {
    const double fc = __ldg(f + c);
    const double xc = w * __ldg(rD + c) * fc;
    const double ax = row_apply(A, c, __ldg(diag + c) * xc,
                                [&](int j) { return w * __ldg(rD + j) * __ldg(f + j); });
    r[c] = fc - ax;
  }
}

// K4 at level 0; RHO: partial (z, f) for the classical control step
template <class Fmt, bool RHO>
__global__ void __launch_bounds__(kBlock) k_vc_post(Fmt A, const double* __restrict__ diag,
                                                    const double* __restrict__ rD, double w,
                                                    const double* __restrict__ f,
                                                    const double* __restrict__ x,
                                                    double* __restrict__ z, State* st, Red rd) {
  if (st && st->done) return;
  double v[1] = {0.0};
  GRID_STRIDE(c, A.n) {
    const double xc = __ldg(x + c), fc = __ldg(f + c);
    const double ax = row_apply(A, c, __ldg(diag + c) * xc, [&](int j) { return __ldg(x + j); });
    const double zc = xc + w * __ldg(rD + c) * (fc - ax);
    z[c] = zc;
    if (RHO) v[0] = fma(zc, fc, v[0]);
  }
  if (RHO) finish_reduction<1>(v, rd, st);
}

// coarsest level: z = Ainv f, one warp per row
__global__ void __launch_bounds__(kBlock) k_dense_mv(int n, const double* __restrict__ Ainv,
                                                     const double* __restrict__ f,
                                                     double* __restrict__ z, const State* st) {
  if (st && st->done) return;
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long i = warp; i < n; i += nwarps) {
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s = fma(Ainv[i * n + j], f[j], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) z[i] = s;
  }
}

// (a, b) partial -> control step (used when the hierarchy has no level below 0)
__global__ void __launch_bounds__(kBlock) k_amg_dot(int n, const double* __restrict__ a,
                                                    const double* __restrict__ b, State* st,
                                                    Red rd) {
  if (st->done) return;
  double v[1] = {0.0};
  GRID_STRIDE(c, n) v[0] = fma(a[c], b[c], v[0]);
  finish_reduction<1>(v, rd, st);
}

// ---- Krylov passes ----------------------------------------------------------------------------
template <class Fmt>
__global__ void __launch_bounds__(kBlock, 8) k_amg_passA(Fmt A, const double* __restrict__ diag,
                                                      const double* __restrict__ z, double* p0,
                                                      double* p1, double* __restrict__ q,
                                                      double* __restrict__ x, State* st, Red rd) {
  if (st->done) return;
  const int k = st->k;
  const double beta = st->beta, alpha = st->alpha;
  const double* __restrict__ pold = (k & 1) ? p0 : p1;
  double* __restrict__ pnew = (k & 1) ? p1 : p0;
  double v[1] = {0.0};
  GRID_STRIDE(c, A.n) {
    const double po = __ldg(pold + c);
    const double pc = fma(beta, po, __ldg(z + c));
    const double qc = row_apply(A, c, __ldg(diag + c) * pc,
                                [&](int j) { return fma(beta, __ldg(pold + j), __ldg(z + j)); });
    pnew[c] = pc;
    q[c] = qc;
    x[c] = fma(alpha, po, x[c]);
    v[0] = fma(pc, qc, v[0]);
  }
  finish_reduction<1>(v, rd, st);
}

__global__ void __launch_bounds__(kBlock) k_amg_passB(int n, const double* __restrict__ q,
                                                      double* __restrict__ r, State* st, Red rd) {
  if (st->done) return;
  const double alpha = st->alpha;
  const bool l2 = st->norm == LDU_NORM_L2;
  double v[1] = {0.0};
  GRID_STRIDE(c, n) {
    const double rc = fma(-alpha, q[c], r[c]);
    r[c] = rc;
    v[0] += l2 ? rc * rc : fabs(rc);
  }
  finish_reduction<1>(v, rd, st);
}

// pipelined: partials [gamma = (r, u), delta = (w, u), crit(r)]
__global__ void __launch_bounds__(kBlock) k_amg_pipe_dots(int n, const double* __restrict__ r,
                                                          const double* __restrict__ u,
                                                          const double* __restrict__ w, State* st,
                                                          Red rd) {
  if (st->done) return;
  const bool l2 = st->norm == LDU_NORM_L2;
  double v[3] = {0.0, 0.0, 0.0};
  GRID_STRIDE(c, n) {
    const double rc = r[c], uc = u[c];
    v[0] = fma(rc, uc, v[0]);
    v[1] = fma(w[c], uc, v[1]);
    v[2] += l2 ? rc * rc : fabs(rc);
  }
  finish_reduction<3>(v, rd, st);
}

template <class Fmt>
__global__ void __launch_bounds__(kBlock, 6) k_amg_pipe_SU(
    Fmt A, const double* __restrict__ diag, const double* __restrict__ m, double* __restrict__ z,
    double* __restrict__ q, double* __restrict__ s, double* __restrict__ p, double* __restrict__ x,
    double* __restrict__ r, double* __restrict__ u, double* __restrict__ w, State* st, Red rd) {
  if (st->done) return;
  const double a = st->pa, b = st->pb;
  const bool l2 = st->norm == LDU_NORM_L2;
  double v[3] = {0.0, 0.0, 0.0};
  GRID_STRIDE(c, A.n) {
    const double mc = __ldg(m + c);
    const double nc = row_apply(A, c, __ldg(diag + c) * mc, [&](int j) { return __ldg(m + j); });
    const double zc = fma(b, z[c], nc);
    const double qc = fma(b, q[c], mc);
    const double sc = fma(b, s[c], w[c]);
    const double pc = fma(b, p[c], u[c]);
    z[c] = zc;
    q[c] = qc;
    s[c] = sc;
    p[c] = pc;
    x[c] = fma(a, pc, x[c]);
    const double rc = fma(-a, sc, r[c]);
    const double uc = fma(-a, qc, u[c]);
    const double wc = fma(-a, zc, w[c]);
    r[c] = rc;
    u[c] = uc;
    w[c] = wc;
    v[0] = fma(rc, uc, v[0]);
    v[1] = fma(wc, uc, v[1]);
    v[2] += l2 ? rc * rc : fabs(rc);
  }
  finish_reduction<3>(v, rd, st);
}

// multi-rank classical: x += alpha_{k-1} p_{k-1}; p_k = z_k + beta_k p_{k-1} in place (the SpMV
// with its halo exchange follows as a separate step)
__global__ void __launch_bounds__(kBlock) k_amg_p(int n, const double* __restrict__ z,
                                                  double* __restrict__ p, double* __restrict__ x,
                                                  const State* st) {
  if (st->done) return;
  const double beta = st->beta, alpha = st->alpha;
  GRID_STRIDE(c, n) {
    const double po = p[c];
    x[c] = fma(alpha, po, x[c]);
    p[c] = fma(beta, po, z[c]);
  }
}

// multi-rank pipelined: the GV recurrences with n = A m (incl. interfaces) already in nv
__global__ void __launch_bounds__(kBlock) k_amg_pipe_U(
    int n, const double* __restrict__ m, const double* __restrict__ nv, double* __restrict__ z,
    double* __restrict__ q, double* __restrict__ s, double* __restrict__ p, double* __restrict__ x,
    double* __restrict__ r, double* __restrict__ u, double* __restrict__ w, State* st, Red rd) {
  if (st->done) return;
  const double a = st->pa, b = st->pb;
  const bool l2 = st->norm == LDU_NORM_L2;
  double v[3] = {0.0, 0.0, 0.0};
  GRID_STRIDE(c, n) {
    const double mc = m[c];
    const double zc = fma(b, z[c], nv[c]);
    const double qc = fma(b, q[c], mc);
    const double sc = fma(b, s[c], w[c]);
    const double pc = fma(b, p[c], u[c]);
    z[c] = zc;
    q[c] = qc;
    s[c] = sc;
    p[c] = pc;
    x[c] = fma(a, pc, x[c]);
    const double rc = fma(-a, sc, r[c]);
    const double uc = fma(-a, qc, u[c]);
    const double wc = fma(-a, zc, w[c]);
    r[c] = rc;
    u[c] = uc;
    w[c] = wc;
    v[0] = fma(rc, uc, v[0]);
    v[1] = fma(wc, uc, v[1]);
    v[2] += l2 ? rc * rc : fabs(rc);
  }
  finish_reduction<3>(v, rd, st);
}

// resident blocks per SM x SMs, capped by the rows (grid-stride kernels)
int occ_grid(ldu_handle h, const void* fn) {
  int dev = 0, sms = 1, o = 1;
  CUDA_CHECK(cudaGetDevice(&dev));
  CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, kBlock, 0));
  const long long need = ((long long)h->n + kBlock - 1) / kBlock;
  return (int)std::max(1LL, std::min((long long)sms * std::max(1, o), need));
}

void amg_grids(ldu_handle h) {
  AmgHierarchy* H = h->amg;
  if (H->gPre) return;
  with_format(h, [&](auto A) {
    using Fmt = decltype(A);
    H->gPre = occ_grid(h, (const void*)k_vc_pre<Fmt>);
    H->gPost = std::min(occ_grid(h, (const void*)k_vc_post<Fmt, true>),
                        occ_grid(h, (const void*)k_vc_post<Fmt, false>));
    H->gPassA = occ_grid(h, (const void*)k_amg_passA<Fmt>);
    H->gPipe = occ_grid(h, (const void*)k_amg_pipe_SU<Fmt>);
  });
  if (std::max({H->gPre, H->gPost, H->gPassA, H->gPipe}) > h->maxParts)
    throw Error(LDU_ERR_STATE, "AMG grid exceeds the reduction slots");
}

// ---- DIC preconditioner (NEXT-1, reading Z35): level-scheduled triangular sweeps --------------
// forward:  z_c = rD_c (f_c - sum_{lower j} a_cj z_j)      levels ascending
// backward: z_c -= rD_c sum_{upper j} a_cj z_j              levels descending
// One thread per cell of the level; the level's cells read only z of earlier launches.
__global__ void __launch_bounds__(kBlock) k_dic_fwd(int beg, int end, const int* __restrict__ perm,
                                                    const int* __restrict__ ptr,
                                                    const int* __restrict__ col,
                                                    const double* __restrict__ val,
                                                    const double* __restrict__ rD,
                                                    const double* __restrict__ f, double* z,
                                                    const State* st) {
  if (st && st->done) return;
  for (int k = beg + blockIdx.x * blockDim.x + threadIdx.x; k < end; k += gridDim.x * blockDim.x) {
    const int c = __ldg(perm + k);
    if (c < 0) continue;
    double s = __ldg(f + c);
    const int j1 = __ldg(ptr + k + 1);
    for (int j = __ldg(ptr + k); j < j1; ++j) s = fma(-__ldg(val + j), z[__ldg(col + j)], s);
    z[c] = __ldg(rD + c) * s;
  }
}

__global__ void __launch_bounds__(kBlock) k_dic_bwd(int beg, int end, const int* __restrict__ perm,
                                                    const int* __restrict__ ptr,
                                                    const int* __restrict__ col,
                                                    const double* __restrict__ val,
                                                    const double* __restrict__ rD, double* z,
                                                    const State* st) {
  if (st && st->done) return;
  for (int k = beg + blockIdx.x * blockDim.x + threadIdx.x; k < end; k += gridDim.x * blockDim.x) {
    const int c = __ldg(perm + k);
    if (c < 0) continue;
    double s = 0.0;
    const int j1 = __ldg(ptr + k + 1);
    for (int j = __ldg(ptr + k); j < j1; ++j) s = fma(__ldg(val + j), z[__ldg(col + j)], s);
    if (j1 > __ldg(ptr + k)) z[c] = fma(-__ldg(rD + c), s, z[c]);
  }
}

// Sync-free variant (opt-in, LDU_DIC_SF): ONE persistent launch per sweep.  Blocks take 256-position chunks
// of the (warp-aligned) level order from a ticket counter, so a chunk only ever waits for chunks
// taken earlier by running blocks (no deadlock, any grid size), and no warp waits on itself
// (levels start on warp boundaries).  A cell spins until each neighbour it reads carries this
// sweep's epoch tag (fence + volatile tag store after its z store; volatile polls with
// __nanosleep back-off, then a fence before the reads), i.e. the
// dependency is per cell, not per level: the critical path is one flag hand-off per level.

template <bool FWD, int SLEEP_NS>
__global__ void __launch_bounds__(kBlock) k_dic_sweep_sf(int nPad, const int* __restrict__ perm,
                                                         const int* __restrict__ ptr,
                                                         const int* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ rD,
                                                         const double* __restrict__ f, double* z,
                                                         unsigned* flag, unsigned* ctl,
                                                         const State* st) {
  if (st && st->done) return;
  __shared__ int chunk;
  const unsigned tag = 2u * ctl[0] + (FWD ? 1u : 2u);
  unsigned* ticket = ctl + (FWD ? 1 : 2);
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) chunk = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    const long long base = (long long)chunk * kBlock;
    if (base >= nPad) return;
    const long long q = base + threadIdx.x;
    if (q >= nPad) continue;
    const int k = FWD ? (int)q : nPad - 1 - (int)q;
    const int c = __ldg(perm + k);
    if (c < 0) continue;
    const int j0 = __ldg(ptr + k), j1 = __ldg(ptr + k + 1);
    double s = FWD ? __ldg(f + c) : 0.0;
    // wait (relaxed polls with back-off) for every neighbour, then one acquire fence
    for (int j = j0; j < j1; ++j) {
      const volatile unsigned* fl = flag + __ldg(col + j);
      while (*fl != tag) __nanosleep(SLEEP_NS);
    }
    __threadfence();
    for (int j = j0; j < j1; ++j) {
      const double v = __ldg(val + j) * __ldcg(z + __ldg(col + j));
      s = FWD ? s - v : s + v;
    }
    if (FWD) {
      z[c] = __ldg(rD + c) * s;
    } else if (j1 > j0) {
      z[c] = fma(-__ldg(rD + c), s, __ldcg(z + c));
    }
    __threadfence();
    *(volatile unsigned*)(flag + c) = tag;
  }
}

// next epoch, tickets back to 0 (stream-ordered after both sweeps)
__global__ void k_dic_bump(unsigned* ctl, const State* st) {
  if (st && st->done) return;
  ctl[0] += 1u;
  ctl[1] = 0u;
  ctl[2] = 0u;
}

// ELL sweeps with programmatic dependent launch: the level's row data (constant since the setup)
// is loaded before griddepcontrol.wait, so it overlaps the previous level's execution and the
// launch gap; f and z (produced by earlier kernels) are read only after the wait.  The grid covers the
// level exactly.  W = padded row width (column -1 = no entry).
template <int W, bool FWD>
__global__ void __launch_bounds__(kBlock) k_dic_ell(int beg, int end, int nPad,
                                                    const int* __restrict__ perm,
                                                    const int* __restrict__ ecol,
                                                    const double* __restrict__ eval,
                                                    const double* __restrict__ rD,
                                                    const double* f, double* z, const State* st) {
  const int k = beg + blockIdx.x * blockDim.x + threadIdx.x;
  int c = -1;
  int cj[W];
  double a[W];
  double rc = 0.0;
  if (k < end) {
    c = __ldg(perm + k);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      cj[w] = __ldg(ecol + (size_t)w * nPad + k);
      a[w] = __ldg(eval + (size_t)w * nPad + k);
    }
    if (c >= 0) rc = __ldg(rD + c);
  }
  pdl_wait();     // the previous level (and, transitively, every earlier kernel) is complete
  pdl_trigger();  // after the wait: at most one level of look-ahead is resident
  if ((st && st->done) || c < 0) return;
  double s = FWD ? f[c] : 0.0;
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (cj[w] >= 0) s = FWD ? fma(-a[w], z[cj[w]], s) : fma(a[w], z[cj[w]], s);
  if (FWD)
    z[c] = rc * s;
  else if (cj[0] >= 0)
    z[c] = fma(-rc, s, z[c]);
}

// A run of consecutive narrow levels (each <= kRun positions) in ONE block: __syncthreads between
// levels (global writes before the barrier are visible to the block after it) instead of a launch
// per level.  Levels [l0, l1) ascending (FWD) or descending (!FWD).
constexpr int kRun = 1024;
template <int W, bool FWD>
__global__ void __launch_bounds__(kRun) k_dic_ell_run(int l0, int l1, const int* __restrict__ levPtr,
                                                      int nPad, const int* __restrict__ perm,
                                                      const int* __restrict__ ecol,
                                                      const double* __restrict__ eval,
                                                      const double* __restrict__ rD,
                                                      const double* f, double* z, const State* st) {
  pdl_wait();
  pdl_trigger();
  if (st && st->done) return;
  for (int i = 0; i < l1 - l0; ++i) {
    const int l = FWD ? l0 + i : l1 - 1 - i;
    const int k = __ldg(levPtr + l) + threadIdx.x;
    if (k < __ldg(levPtr + l + 1)) {
      const int c = __ldg(perm + k);
      if (c >= 0) {
        double s = FWD ? f[c] : 0.0;
        bool any = false;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const int cj = __ldg(ecol + (size_t)w * nPad + k);
          if (cj >= 0) {
            const double a = __ldg(eval + (size_t)w * nPad + k);
            s = FWD ? fma(-a, z[cj], s) : fma(a, z[cj], s);
            any = true;
          }
        }
        if (FWD)
          z[c] = __ldg(rD + c) * s;
        else if (any)
          z[c] = fma(-__ldg(rD + c), s, z[c]);
      }
    }
    __syncthreads();
  }
}

template <bool FWD>
void launch_dic_run(int W, bool pdl, int l0, int l1, const int* levPtr, int nPad, const int* perm,
                    const int* ecol, const double* eval, const double* rD, const double* f,
                    double* z, const State* st, cudaStream_t s) {
#define LDU_DIC_RUN(WW)                                                                          \
  launch_pdl(pdl, k_dic_ell_run<WW, FWD>, 1, kRun, s, l0, l1, levPtr, nPad, perm, ecol, eval, rD, \
             f, z, st);                                                                          \
  return;
  switch (W) {
    case 1: LDU_DIC_RUN(1)
    case 2: LDU_DIC_RUN(2)
    case 3: LDU_DIC_RUN(3)
    case 4: LDU_DIC_RUN(4)
    case 5: case 6: LDU_DIC_RUN(6)
    default: LDU_DIC_RUN(8)
  }
#undef LDU_DIC_RUN
}

template <bool FWD>
void launch_dic_ell(int W, bool pdl, int b, int e, int nPad, const int* perm, const int* ecol,
                    const double* eval, const double* rD, const double* f, double* z,
                    const State* st, cudaStream_t s) {
  const int g = std::max(1, (e - b + kBlock - 1) / kBlock);
#define LDU_DIC_ELL(WW)                                                                         \
  launch_pdl(pdl, k_dic_ell<WW, FWD>, g, kBlock, s, b, e, nPad, perm, ecol, eval, rD, f, z, st); \
  return;
  switch (dic_ell_width(W)) {  // the setup stored exactly this width (same helper)
    case 1: LDU_DIC_ELL(1)
    case 2: LDU_DIC_ELL(2)
    case 3: LDU_DIC_ELL(3)
    case 4: LDU_DIC_ELL(4)
    case 6: LDU_DIC_ELL(6)
    case 8: LDU_DIC_ELL(8)
    default: throw Error(LDU_ERR_STATE, "DIC ELL width " + std::to_string(W) + " has no sweep kernel");
  }
#undef LDU_DIC_ELL
}

long long enqueue_dic(ldu_handle h, const double* f0, double* z0, cudaStream_t s, State* st,
                      const Red* rho) {
  const DicFactor& D = h->amg->dic;
  auto grid = [](int m) { return (int)std::max(1, std::min((m + kBlock - 1) / kBlock, 148 * 8)); };
  long long kernels = 0;
  // LDU_DIC_SF = back-off in ns of the sync-free sweeps (0 = one launch per level, the default)
  static const int sf = std::getenv("LDU_DIC_SF") ? std::atoi(std::getenv("LDU_DIC_SF")) : 0;
  static const int sfBlocks = std::getenv("LDU_DIC_SF_BLOCKS") ? std::atoi(std::getenv("LDU_DIC_SF_BLOCKS")) : 148 * 4;
  static const bool useEll = !(std::getenv("LDU_DIC_ELL") && std::atoi(std::getenv("LDU_DIC_ELL")) == 0);
  static const bool ellPdl = !(std::getenv("LDU_DIC_PDL") && std::atoi(std::getenv("LDU_DIC_PDL")) == 0);
  if (!sf && useEll && D.eLoCol && (D.nLev < 2 || D.eUpCol)) {
    // one launch per level and sweep, ELL rows, PDL between consecutive launches (default).
    // LDU_DIC_RUN = m > 0: runs of >= m narrow levels (<= kRun positions) in one single-block
    // launch each -- measured slower inside the solver's graphs (profiles/r01_dic), so opt-in
    static const int minRun = std::getenv("LDU_DIC_RUN") ? std::atoi(std::getenv("LDU_DIC_RUN")) : 0;
    auto narrow = [&](int l) { return D.levPtr[l + 1] - D.levPtr[l] <= kRun; };
    long long launches = 0;
    for (int l = 0; l < D.nLev;) {  // forward, levels ascending
      int e = l;
      while (minRun > 0 && e < D.nLev && narrow(e)) ++e;
      if (minRun > 0 && e - l >= minRun) {
        launch_dic_run<true>(D.wLo, ellPdl && launches > 0, l, e, D.dLevPtr, D.nPad, D.perm,
                             D.eLoCol, D.eLoVal, D.rD, f0, z0, st, s);
        l = e;
      } else {
        launch_dic_ell<true>(D.wLo, ellPdl && launches > 0, D.levPtr[l], D.levPtr[l + 1], D.nPad,
                             D.perm, D.eLoCol, D.eLoVal, D.rD, f0, z0, st, s);
        ++l;
      }
      ++launches;
    }
    for (int l = D.nLev - 2; l >= 0;) {  // backward, levels descending
      int b = l;
      while (minRun > 0 && b >= 0 && narrow(b)) --b;
      if (minRun > 0 && l - b >= minRun) {
        launch_dic_run<false>(D.wUp, ellPdl, b + 1, l + 1, D.dLevPtr, D.nPad, D.perm, D.eUpCol,
                              D.eUpVal, D.rD, f0, z0, st, s);
        l = b;
      } else {
        launch_dic_ell<false>(D.wUp, ellPdl, D.levPtr[l], D.levPtr[l + 1], D.nPad, D.perm,
                              D.eUpCol, D.eUpVal, D.rD, f0, z0, st, s);
        --l;
      }
      ++launches;
    }
    kernels += launches;
  } else if (!sf) {  // one launch per level and sweep, CSR rows (measured reference variant)
    for (int l = 0; l < D.nLev; ++l) {
      const int b = D.levPtr[l], e = D.levPtr[l + 1];
      k_dic_fwd<<<grid(e - b), kBlock, 0, s>>>(b, e, D.perm, D.loPtr, D.loCol, D.loVal, D.rD, f0,
                                               z0, st);
    }
    // the last level has no upper neighbours: the backward sweep starts one level down
    for (int l = D.nLev - 2; l >= 0; --l) {
      const int b = D.levPtr[l], e = D.levPtr[l + 1];
      k_dic_bwd<<<grid(e - b), kBlock, 0, s>>>(b, e, D.perm, D.upPtr, D.upCol, D.upVal, D.rD, z0,
                                               st);
    }
    kernels += D.nLev + std::max(0, D.nLev - 1);
  } else {
    // the backward sweep's first cell (highest level) sets its tag without waiting; every
    // upper neighbour it reads was tagged earlier in the same sweep
    const int g = std::max(1, std::min(sfBlocks, (D.nPad + kBlock - 1) / kBlock));
    auto sweeps = [&](auto fwd, auto bwd) {
      fwd<<<g, kBlock, 0, s>>>(D.nPad, D.perm, D.loPtr, D.loCol, D.loVal, D.rD, f0, z0, D.flag,
                               D.ctl, st);
      bwd<<<g, kBlock, 0, s>>>(D.nPad, D.perm, D.upPtr, D.upCol, D.upVal, D.rD, f0, z0, D.flag,
                               D.ctl, st);
    };
    if (sf >= 256) sweeps(k_dic_sweep_sf<true, 256>, k_dic_sweep_sf<false, 256>);
    else if (sf >= 64) sweeps(k_dic_sweep_sf<true, 64>, k_dic_sweep_sf<false, 64>);
    else sweeps(k_dic_sweep_sf<true, 16>, k_dic_sweep_sf<false, 16>);
    k_dic_bump<<<1, 1, 0, s>>>(D.ctl, st);
    kernels += 3;
  }
  if (rho) {
    k_amg_dot<<<h->grid, kBlock, 0, s>>>(h->n, z0, f0, st, *rho);
    ++kernels;
  }
  return kernels;
}

// ---- V-cycle enqueue --------------------------------------------------------------------------
// z0 = B f0 on stream s.  st != nullptr: every kernel exits at entry once the solve is done.
// rho != nullptr: level-0 post-sweep (or the direct solve) also reduces (z0, f0) into rho's control.
long long enqueue_vcycle(ldu_handle h, const double* f0, double* z0, cudaStream_t s, State* st,
                         const Red* rho) {
  AmgHierarchy* H = h->amg;
  if (H->kind == PREC_DIC) return enqueue_dic(h, f0, z0, s, st, rho);
  long long kernels = 0;
  const int L = H->L;
  for (int l = 0; l < L; ++l) {
    AmgLevel& Lv = H->lv[l];
    const double* f = l ? Lv.f : f0;
    if (l == 0) {
      with_format(h, [&](auto A) {
        k_vc_pre<<<H->gPre, kBlock, 0, s>>>(A, Lv.diag, Lv.rD, Lv.omega, f, Lv.r, st);
      });
    } else {
      launch_csr(Lv.A, EpiPre{Lv.x, f, Lv.r}, st, s);
    }
    if (l + 1 < L) {
      AmgLevel& Nx = H->lv[l + 1];
      launch_csr(Lv.R, EpiRestrict{Lv.r, Nx.f, Nx.x, Nx.omega, Nx.rD}, st, s);
    } else {
      launch_csr(Lv.R, EpiRestrict{Lv.r, H->fL, nullptr, 0.0, nullptr}, st, s);
    }
    kernels += 2;
  }
  {
    const double* f = L ? H->fL : f0;
    double* z = L ? H->zL : z0;
    const int g = (int)std::min<long long>(148LL * 8, ((long long)H->nc * 32 + kBlock - 1) / kBlock);
    k_dense_mv<<<std::max(1, g), kBlock, 0, s>>>(H->nc, H->Ainv, f, z, st);
    ++kernels;
    if (L == 0 && rho) {
      k_amg_dot<<<h->grid, kBlock, 0, s>>>(h->n, z0, f0, st, *rho);
      ++kernels;
    }
  }
  for (int l = L - 1; l >= 0; --l) {
    AmgLevel& Lv = H->lv[l];
    const double* f = l ? Lv.f : f0;
    const double* xc = (l + 1 == L) ? H->zL : H->lv[l + 1].z;
    if (l == 0) {
      launch_csr(Lv.P, EpiProlong0{Lv.omega, Lv.rD, f, xc, Lv.x}, st, s);
      with_format(h, [&](auto A) {
        if (rho)
          k_vc_post<decltype(A), true><<<H->gPost, kBlock, 0, s>>>(A, Lv.diag, Lv.rD, Lv.omega, f,
                                                                   Lv.x, z0, st, *rho);
        else
          k_vc_post<decltype(A), false><<<H->gPost, kBlock, 0, s>>>(A, Lv.diag, Lv.rD, Lv.omega, f,
                                                                    Lv.x, z0, st, Red{});
      });
    } else {
      launch_csr(Lv.P, EpiProlong{xc, Lv.x}, st, s);
      launch_csr(Lv.A, EpiPost{Lv.omega, Lv.rD, f, Lv.x, Lv.z}, st, s);
    }
    kernels += 2;
  }
  return kernels;
}

void ensure_amg_work(ldu_handle h, bool pipelined) {
  AmgHierarchy* H = h->amg;
  const int n = h->n;
  ensure_vec(h->x, n);
  ensure_vec(h->r, n);
  ensure_vec(h->ybuf, n);
  ensure_vec(h->p0, n);
  if (!pipelined) {
    ensure_vec(h->p1, n);
    ensure_vec(h->q, n);
    ensure_vec(H->zk, n);
  } else {
    ensure_vec(h->w, n);
    ensure_vec(h->z, n);
    ensure_vec(h->s, n);
    ensure_vec(h->nv, n);  // sumA of the OpenFOAM norm
    ensure_vec(H->u, n);
    ensure_vec(H->m, n);
    ensure_vec(H->qk, n);
  }
}

// Multi-rank (block-Jacobi, reading Z33): the V-cycle is local; the SpMV exchanges the halo
// (amul_dev) and every reduction is a cross-rank gather of the local sums + the control kernel,
// both over the peer mailboxes by default (the reducing kernel's last block publishes its sums,
// red_loop) or over NCCL (LDU_P2P=0).  Pipelined: the gather of iteration i's fused sums is
// overlapped with the V-cycle m_i = B w_i and n_i = A m_i (neither needs alpha_i, beta_i): P:97.
long long enqueue_amg_iters_mr(ldu_handle h, bool pipelined, int batch, cudaStream_t s,
                               bool profile) {
  AmgHierarchy* H = h->amg;
  ldu_comm cm = h->comm;
  long long kernels = 0;
  for (int it = 0; it < batch; ++it) {
    prof_mark(h, profile, 4 * it + 0, s);
    if (!pipelined) {
      const Red rr = red_loop(h, CTL_NONE, false, H->L ? H->gPost : h->grid);
      kernels += enqueue_vcycle(h, h->r, H->zk, s, h->st, &rr);
      prof_mark(h, profile, 4 * it + 1, s);
      allgather_ctl(h, CTL_AMG_RHO, 1, s, kernels);
      prof_mark(h, profile, 4 * it + 2, s);
      k_amg_p<<<h->grid, kBlock, 0, s>>>(h->n, H->zk, h->p0, h->x, h->st);
      ++kernels;
      amul_dev(h, h->p0, h->q, s, kernels);
      k_amg_dot<<<h->grid, kBlock, 0, s>>>(h->n, h->p0, h->q, h->st, red_loop(h, CTL_NONE, false));
      ++kernels;
      allgather_ctl(h, CTL_CG_A, 1, s, kernels);
      k_amg_passB<<<h->grid, kBlock, 0, s>>>(h->n, h->q, h->r, h->st, red_loop(h, CTL_NONE, false));
      ++kernels;
      allgather_ctl(h, CTL_AMG_B, 1, s, kernels);
    } else if (h->p2pOn) {  // the sums published by the previous U (or the init) wait in the mailboxes
      kernels += enqueue_vcycle(h, h->w, H->m, s, h->st, nullptr);
      amul_dev(h, H->m, h->nv, s, kernels);
      prof_mark(h, profile, 4 * it + 1, s);
      k_ctl_p2p<<<1, 32, 0, s>>>(CTL_PIPE_NEXT, h->st, h->p2pDesc, 0);
      prof_mark(h, profile, 4 * it + 2, s);
      k_amg_pipe_U<<<h->grid, kBlock, 0, s>>>(h->n, H->m, h->nv, h->z, H->qk, h->s, h->p0, h->x,
                                              h->r, H->u, h->w, h->st, red_loop(h, CTL_NONE, false));
      kernels += 2;
    } else {
      CUDA_CHECK(cudaEventRecord(h->ev_fork, s));
      CUDA_CHECK(cudaStreamWaitEvent(h->red_stream, h->ev_fork, 0));
      NCCL_CHECK(ncclAllGather(h->sums, h->gsums, kMaxVals, ncclDouble, cm->red, h->red_stream));
      CUDA_CHECK(cudaEventRecord(h->ev_red, h->red_stream));
      kernels += enqueue_vcycle(h, h->w, H->m, s, h->st, nullptr);
      amul_dev(h, H->m, h->nv, s, kernels);
      prof_mark(h, profile, 4 * it + 1, s);
      CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_red, 0));
      k_ctl<<<1, 32, 0, s>>>(CTL_PIPE_NEXT, h->st, h->gsums, cm->nRanks, 3);
      prof_mark(h, profile, 4 * it + 2, s);
      k_amg_pipe_U<<<h->grid, kBlock, 0, s>>>(h->n, H->m, h->nv, h->z, H->qk, h->s, h->p0, h->x,
                                              h->r, H->u, h->w, h->st, red_of(h, CTL_NONE, false));
      kernels += 2;
    }
    prof_mark(h, profile, 4 * it + 3, s);
  }
  return kernels;
}

long long enqueue_amg_iters(ldu_handle h, bool pipelined, int batch, cudaStream_t s, bool profile) {
  if (multi(h)) return enqueue_amg_iters_mr(h, pipelined, batch, s, profile);
  AmgHierarchy* H = h->amg;
  long long kernels = 0;
  for (int it = 0; it < batch; ++it) {
    prof_mark(h, profile, 4 * it + 0, s);
    if (!pipelined) {
      const Red rr = red_of(h, CTL_AMG_RHO, true, H->L ? H->gPost : h->grid);
      kernels += enqueue_vcycle(h, h->r, H->zk, s, h->st, &rr);
      prof_mark(h, profile, 4 * it + 1, s);
      prof_mark(h, profile, 4 * it + 2, s);
      with_format(h, [&](auto A) {
        k_amg_passA<<<H->gPassA, kBlock, 0, s>>>(A, h->diag, H->zk, h->p0, h->p1, h->q, h->x,
                                                 h->st, red_of(h, CTL_CG_A, true, H->gPassA));
      });
      k_amg_passB<<<h->grid, kBlock, 0, s>>>(h->n, h->q, h->r, h->st, red_of(h, CTL_AMG_B, true));
      kernels += 2;
    } else {
      kernels += enqueue_vcycle(h, h->w, H->m, s, h->st, nullptr);
      prof_mark(h, profile, 4 * it + 1, s);
      prof_mark(h, profile, 4 * it + 2, s);
      with_format(h, [&](auto A) {
        k_amg_pipe_SU<<<H->gPipe, kBlock, 0, s>>>(A, h->diag, H->m, h->z, H->qk, h->s, h->p0, h->x,
                                                  h->r, H->u, h->w, h->st,
                                                  red_of(h, CTL_PIPE_NEXT, true, H->gPipe));
      });
      ++kernels;
    }
    prof_mark(h, profile, 4 * it + 3, s);
  }
  return kernels;
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// public-internal entry points
// ---------------------------------------------------------------------------------------------
static void check_prec(ldu_handle h, int kind) {
  if (!h->amg || h->amg->kind != kind)
    throw Error(LDU_ERR_STATE, kind == PREC_DIC ? "no DIC factor (call ldu_dic_setup)"
                                                : "no AMG hierarchy (call ldu_amg_setup)");
}

void amg_vcycle(ldu_handle h, const double* r, double* z, int kind) {
  check_prec(h, kind);
  amg_grids(h);
  if (!r || !z) fail_arg("r and z must not be NULL");
  cudaStream_t s = h->own_stream;
  h->stats = ldu_solve_stats{};
  if (h->stream != h->own_stream) {
    CUDA_CHECK(cudaEventRecord(h->ev_fork, h->stream));
    CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_fork, 0));
  }
  const int n = h->n;
  const bool rd = is_device_ptr(r), zd = is_device_ptr(z);
  const double* rin = r;
  double* zout = z;
  if (!rd) {
    ensure_vec(h->bbuf, n);
    CUDA_CHECK(cudaMemcpyAsync(h->bbuf, r, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    h->stats.h2dBytes += 8LL * n;
    rin = h->bbuf;
  }
  if (!zd) {
    ensure_vec(h->ybuf, n);
    zout = h->ybuf;
  }
  CUDA_CHECK(cudaEventRecord(h->ev[0], s));
  h->stats.kernels = enqueue_vcycle(h, rin, zout, s, nullptr, nullptr);
  CUDA_CHECK(cudaEventRecord(h->ev[1], s));
  if (!zd) {
    CUDA_CHECK(cudaMemcpyAsync(z, zout, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    h->stats.d2hBytes += 8LL * n;
  }
  if (h->stream != h->own_stream) {
    CUDA_CHECK(cudaEventRecord(h->ev_fork, s));
    CUDA_CHECK(cudaStreamWaitEvent(h->stream, h->ev_fork, 0));
  }
  CUDA_CHECK(cudaGetLastError());
  CUDA_CHECK(cudaStreamSynchronize(s));
  float ms = 0.f;
  CUDA_CHECK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
  h->stats.solveMs = ms;
  h->stats.iterMs = ms;
}

ldu_status amg_solve(ldu_handle h, int kind, bool pipelined, const double* b, double* x,
                     double tol, int maxIter, const ldu_solve_opts* opts, int* nIter,
                     double* finalRes) {
  check_prec(h, kind);
  AmgHierarchy* H = h->amg;
  if (!b || !x) fail_arg("b and x must not be NULL");
  if (!(tol >= 0.0)) fail_arg("tol must be >= 0");
  if (maxIter < 0) fail_arg("maxIter must be >= 0");
  ldu_solve_opts o{};
  if (opts) {
    o = *opts;
    if (o.replaceEvery) fail_arg("replaceEvery is not supported by the AMG / DIC solvers");
    if (o.reserved2[0] != 0.0 || o.reserved2[1] != 0.0)
      fail_arg("ldu_solve_opts.reserved2 must be zero");
  }
  if (!(o.relTol >= 0.0)) fail_arg("relTol must be >= 0");
  if (o.minIter < 0) fail_arg("minIter must be >= 0");
  if (o.norm != LDU_NORM_L2 && o.norm != LDU_NORM_OPENFOAM) fail_arg("unknown norm");
  if (o.batch < 0) fail_arg("batch must be >= 0");
  if (o.profile != 0 && o.profile != 1) fail_arg("profile must be 0 or 1");
  const bool profile = o.profile == 1;
  const int batch = o.batch ? o.batch : (kind == PREC_DIC ? 2 : 8);  // DIC: ~2 nLev nodes/iter

  ensure_amg_work(h, pipelined);
  amg_grids(h);
  const int n = h->n;
  const bool mr = multi(h);
  if (mr && pipelined) ensure_vec(h->nv, n);
  cudaStream_t s = h->own_stream;
  h->stats = ldu_solve_stats{};
  long long kernels = 0;
  if (h->stream != h->own_stream) {
    CUDA_CHECK(cudaEventRecord(h->ev_fork, h->stream));
    CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_fork, 0));
  }
  CUDA_CHECK(cudaEventRecord(h->ev[0], s));
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
  if (o.recordHistory && h->histCap < maxIter + 1) {
    dfree(h->hist);
    h->hist = nullptr;
    h->histCap = 0;
    h->hist = dmalloc<double>((size_t)maxIter + 1);
    h->histCap = maxIter + 1;
  }
  h->histN = -1;
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
  CUDA_CHECK(cudaMemsetAsync(h->p0, 0, sizeof(double) * n, s));
  if (!pipelined) {
    CUDA_CHECK(cudaMemsetAsync(h->p1, 0, sizeof(double) * n, s));
  } else {
    CUDA_CHECK(cudaMemsetAsync(h->z, 0, sizeof(double) * n, s));
    CUDA_CHECK(cudaMemsetAsync(h->s, 0, sizeof(double) * n, s));
    CUDA_CHECK(cudaMemsetAsync(H->qk, 0, sizeof(double) * n, s));
  }

  // ---- r0 = b - A x0 and the criterion scale ---------------------------------------------
  double* sumA = pipelined ? h->nv : h->q;
  double* Ax0 = h->ybuf;
  if (o.norm == LDU_NORM_OPENFOAM) {
    k_fill<<<small_grid(n), kBlock, 0, s>>>(n, 1.0, h->r);
    ++kernels;
    amul_dev(h, h->r, sumA, s, kernels);
    k_sum_x<<<h->grid, kBlock, 0, s>>>(n, h->x, h->st, red_loop(h, CTL_XBAR, !mr));
    ++kernels;
    if (mr) allgather_ctl(h, CTL_XBAR, 2, s, kernels);
  }
  amul_dev(h, h->x, Ax0, s, kernels);
  k_resid<<<h->grid, kBlock, 0, s>>>(n, bin, Ax0, sumA, h->rD, h->r, h->st,
                                     red_loop(h, pipelined ? CTL_PIPE_SCALE : CTL_CG_INIT, !mr));
  ++kernels;
  if (mr) allgather_ctl(h, pipelined ? CTL_PIPE_SCALE : CTL_CG_INIT, 3, s, kernels);
  if (pipelined) {  // u0 = B r0; w0 = A u0; first fused reduction
    kernels += enqueue_vcycle(h, h->r, H->u, s, h->st, nullptr);
    amul_dev(h, H->u, h->w, s, kernels);
    k_amg_pipe_dots<<<h->grid, kBlock, 0, s>>>(n, h->r, H->u, h->w, h->st,
                                               red_loop(h, CTL_PIPE_TOP, !mr));
    ++kernels;
    if (mr) {  // its allgather is issued by the first loop trip; k = -1 so that trip evaluates i = 0
      static const int minus_one = -1;
      CUDA_CHECK(cudaMemcpyAsync(&h->st->k, &minus_one, sizeof(int), cudaMemcpyHostToDevice, s));
    }
  }
  CUDA_CHECK(cudaGetLastError());
  CUDA_CHECK(cudaEventRecord(h->ev[1], s));

  // ---- iteration batches as CUDA graphs (one per solver; rebuilt with the hierarchy) -------
  const int gi = (pipelined ? 1 : 0) + (profile ? 2 : 0);
  if (profile && (int)h->prof_ev.size() < 4 * batch) {
    for (cudaEvent_t e : h->prof_ev) cudaEventDestroy(e);
    h->prof_ev.assign(4 * batch, nullptr);
    for (auto& e : h->prof_ev) CUDA_CHECK(cudaEventCreate(&e));
    for (int k = 2; k < 4; ++k)
      if (H->graph[k]) { cudaGraphExecDestroy(H->graph[k]); H->graph[k] = nullptr; }
    if (h->graphs[0][1].exec) { cudaGraphExecDestroy(h->graphs[0][1].exec); h->graphs[0][1] = {}; }
    if (h->graphs[1][1].exec) { cudaGraphExecDestroy(h->graphs[1][1].exec); h->graphs[1][1] = {}; }
  }
  if (!H->graph[gi] || H->graphBatch[gi] != batch) {
    if (H->graph[gi]) cudaGraphExecDestroy(H->graph[gi]);
    H->graph[gi] = nullptr;
    cudaGraph_t g;
    CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    H->graphKernels[gi] = enqueue_amg_iters(h, pipelined, batch, s, profile);
    CUDA_CHECK(cudaStreamEndCapture(s, &g));
    CUDA_CHECK(cudaGraphInstantiate(&H->graph[gi], g, 0));
    CUDA_CHECK(cudaGraphDestroy(g));
    H->graphBatch[gi] = batch;
  }
  std::vector<float> passT;
  int batches = 0;
  // multi-rank pipelined needs one more trip: the decision on r_i is taken after trip i's allgather
  const long long trips = (long long)maxIter + ((pipelined && mr) ? 1 : 0);
  if (maxIter > 0) {
    for (;;) {
      CUDA_CHECK(cudaGraphLaunch(H->graph[gi], s));
      ++batches;
      if (tol == 0.0 && !profile && o.relTol == 0.0) {  // fixed iterations: sync at the end only
        if ((long long)batches * batch >= trips) break;
        continue;
      }
      CUDA_CHECK(cudaMemcpyAsync(sh, h->st, sizeof(State), cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      if (profile)
        for (int it = 0; it < batch; ++it)
          for (int p = 0; p < 2; ++p) {
            float ms = 0.f;
            CUDA_CHECK(cudaEventElapsedTime(&ms, h->prof_ev[4 * it + 2 * p], h->prof_ev[4 * it + 2 * p + 1]));
            passT.push_back(ms);
          }
      if (sh->done) break;
      if ((long long)batches * batch >= trips + batch) break;  // safety net
    }
  }
  CUDA_CHECK(cudaEventRecord(h->ev[2], s));
  // pending x update (classical; multi-rank keeps p in place in p0) / x = 0 when b = 0
  k_cg_final<<<small_grid(n), kBlock, 0, s>>>(n, h->p0, mr ? h->p0 : h->p1, h->x, h->st);
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
  h->stats.kernels = kernels + (long long)batches * H->graphKernels[gi];
  h->stats.allreduces = mr ? (long long)sh->nRed : 0;  // counted on the device (run_ctl)
  h->stats.reductions = sh->nRed;
  h->stats.iterations = sh->iter;
  if (profile)  // pass 0 = V-cycle, pass 1 = Krylov passes, over the iterations that did work
    for (long long g = (pipelined && mr) ? 1 : 0;
         g < sh->iter + ((pipelined && mr) ? 1 : 0) && g < (long long)passT.size() / 2; ++g)
      for (int p = 0; p < 2; ++p) {
        h->stats.passMs[p] += passT[2 * g + p];
        h->stats.passLaunches[p] += 1;
      }
  if (sh->record) h->histN = std::min(sh->iter + 1, h->histCap);
  if (!sh->done) sh->status = LDU_NOT_CONVERGED;
  if (nIter) *nIter = sh->iter;
  if (finalRes) *finalRes = sh->res;
  return (ldu_status)sh->status;
}

}  // namespace ldu
