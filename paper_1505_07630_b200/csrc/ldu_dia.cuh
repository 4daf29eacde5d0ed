// ldu_dia.cuh -- SpMV-bearing passes specialised for the symmetric diagonal (DIA) layout.
//
// Every load a row needs (own operand, the operand at the 2*ND neighbours, the ND upper and ND
// lower coefficients, x) is issued before any arithmetic, with clamped instead of predicated
// addresses, so a warp keeps ~30 independent 8-byte loads in flight (v0 issued them in small
// dependent groups and was long-scoreboard bound, profiles/r01_v0).  ROWS rows per thread
// (rows t and t + 256 of a 512-row block tile) double the loads in flight per thread.
//
// Boundary handling without predicates: an upper neighbour c + d >= n has U[k][c] == 0 by
// construction, a lower neighbour c - d < 0 gets its coefficient forced to 0; both read the
// operand at the clamped index c (finite), so the contribution fma(0, v, s) == s exactly.
#pragma once

#include "ldu_kernels.cuh"

namespace ldu {

// Operand values of one row position.  NA arrays per position.
struct OpX {  // op(j) = x[j]
  static constexpr int NA = 1;
  const double* __restrict__ x;
  __device__ __forceinline__ void load(int j, double (&v)[1]) const { v[0] = __ldg(x + j); }
  __device__ __forceinline__ double eval(const double (&v)[1]) const { return v[0]; }
};

struct OpScaled {  // op(j) = rD[j] * w[j]
  static constexpr int NA = 2;
  const double* __restrict__ rD;
  const double* __restrict__ w;
  __device__ __forceinline__ void load(int j, double (&v)[2]) const {
    v[0] = __ldg(rD + j);
    v[1] = __ldg(w + j);
  }
  __device__ __forceinline__ double eval(const double (&v)[2]) const { return v[0] * v[1]; }
};

struct OpCgP {  // op(j) = rD[j] * r[j] + beta * p_old[j]   (p_k of classical CG)
  static constexpr int NA = 3;
  const double* __restrict__ rD;
  const double* __restrict__ r;
  const double* __restrict__ pold;
  double beta;
  __device__ __forceinline__ void load(int j, double (&v)[3]) const {
    v[0] = __ldg(rD + j);
    v[1] = __ldg(r + j);
    v[2] = __ldg(pold + j);
  }
  __device__ __forceinline__ double eval(const double (&v)[3]) const {
    return fma(beta, v[2], v[0] * v[1]);
  }
};

// All loads of one row.
template <int ND, class Op>
struct DiaRow {
  double own[Op::NA];
  double lo[ND][Op::NA], up[ND][Op::NA];
  double Ulo[ND], Uup[ND];

  __device__ __forceinline__ void load(const DiaView<ND>& A, const Op& op, int c) {
    op.load(c, own);
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      const int jl = c - A.off[k];
      const int ju = c + A.off[k];
      const bool okl = jl >= 0;
      const int jlc = okl ? jl : c;
      const int juc = ju < A.n ? ju : c;
      Ulo[k] = __ldg(A.U[k] + jlc);
      Uup[k] = __ldg(A.U[k] + c);
      if (!okl) Ulo[k] = 0.0;  // select after the (unconditional) load
      op.load(jlc, lo[k]);
      op.load(juc, up[k]);
    }
  }

  // s = init + sum_j a_cj op(j), ascending columns
  __device__ __forceinline__ double apply(const Op& op, double s) const {
#pragma unroll
    for (int k = ND - 1; k >= 0; --k) s = fma(Ulo[k], op.eval(lo[k]), s);
#pragma unroll
    for (int k = 0; k < ND; ++k) s = fma(Uup[k], op.eval(up[k]), s);
    return s;
  }
};

// Row tiles of ROWS * blockDim.x consecutive rows, grid-stride over tiles (wavefront order).
#define DIA_TILE_LOOP(base, n, ROWS) \
  for (long long base = (long long)blockIdx.x * ROWS * blockDim.x; base < (n); \
       base += (long long)gridDim.x * ROWS * blockDim.x)

template <int ND, int ROWS>
__global__ void __launch_bounds__(kBlock) k_amul_dia(DiaView<ND> A, const double* __restrict__ diag,
                                                     const double* __restrict__ x,
                                                     double* __restrict__ y) {
  const OpX op{x};
  DIA_TILE_LOOP(base, A.n, ROWS) {
    DiaRow<ND, OpX> row[ROWS];
    double dg[ROWS];
#pragma unroll
    for (int u = 0; u < ROWS; ++u) {
      const int c = (int)min(base + u * blockDim.x + threadIdx.x, (long long)A.n - 1);
      row[u].load(A, op, c);
      dg[u] = __ldg(diag + c);
    }
#pragma unroll
    for (int u = 0; u < ROWS; ++u) {
      const long long c = base + u * blockDim.x + threadIdx.x;
      if (c < A.n) y[c] = row[u].apply(op, dg[u] * op.eval(row[u].own));
    }
  }
}

// pipelined pass S: n = A (rD.w); the diagonal term diag*rD*w is taken as w exactly.
template <int ND, int ROWS>
__global__ void __launch_bounds__(kBlock) k_spmv_scaled_dia(DiaView<ND> A,
                                                            const double* __restrict__ rD,
                                                            const double* __restrict__ in,
                                                            double* __restrict__ out,
                                                            const State* st) {
  if (st->done) return;
  const OpScaled op{rD, in};
  DIA_TILE_LOOP(base, A.n, ROWS) {
    DiaRow<ND, OpScaled> row[ROWS];
#pragma unroll
    for (int u = 0; u < ROWS; ++u) {
      const int c = (int)min(base + u * blockDim.x + threadIdx.x, (long long)A.n - 1);
      row[u].load(A, op, c);
    }
#pragma unroll
    for (int u = 0; u < ROWS; ++u) {
      const long long c = base + u * blockDim.x + threadIdx.x;
      if (c < A.n) out[c] = row[u].apply(op, row[u].own[1]);
    }
  }
}

}  // namespace ldu
