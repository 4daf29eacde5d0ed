// ldu_persist.cuh -- persistent cooperative CG kernels (single rank; latency-bound sizes).
//
// One cooperative launch runs up to `maxTrips` iterations.  Between the passes of an iteration a
// grid barrier (cooperative_groups grid.sync) replaces the kernel boundary; after it, EVERY block
// sums all blocks' partials in the same fixed order and runs the control step on its own
// shared-memory copy of the State, so all blocks take bit-identical decisions without a second
// barrier.  Block 0 alone records history and writes the State back at exit.  Partials are
// double-buffered so a fast block can start the next pass while slow blocks still read them.
// Pipelined CG: 1 grid barrier per iteration; classical: 2.  (persistent kernel
// for the latency-bound configs 1 and 2.)
#pragma once

#include <cooperative_groups.h>

#include "ldu_kernels.cuh"

namespace ldu {

namespace cg = cooperative_groups;

// Fixed-order sum of the G block partials (NV values, slot layout [NV][ld]) -> out[] in every
// block (same tree in every block => identical results).
template <int NV>
__device__ __forceinline__ void persist_sum(const double* partials, int ld, int G, double* out) {
  __shared__ double sm[NV][32];
  double v[NV];
  sum_slots<NV>(partials, ld, G, v);
  block_reduce<NV>(v, sm);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) out[k] = v[k];
}

template <int NV>
__device__ __forceinline__ void persist_store(double (&v)[NV], double* partials, int ld) {
  __shared__ double sm[NV][32];
  block_reduce<NV>(v, sm);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) partials[k * ld + blockIdx.x] = v[k];
}

// Pipelined CG, fused S+U pass per iteration (as k_pipe_SU), persistent.
template <class Fmt>
__global__ void __launch_bounds__(kBlock) k_pipe_persist(Fmt A, const double* __restrict__ rD,
                                                         double* w0, double* w1, double* z,
                                                         double* s, double* p, double* x,
                                                         double* r, State* gst, double* partials,
                                                         int ld, int maxTrips) {
  cg::grid_group grid = cg::this_grid();
  __shared__ State st;
  __shared__ double sums[kMaxVals];
  if (threadIdx.x == 0) {
    st = *gst;
    if (blockIdx.x != 0) st.record = 0;
  }
  __syncthreads();
  for (int trip = 0; trip < maxTrips && !st.done; ++trip) {
    const double a = st.pa, b = st.pb;
    const bool l2 = st.norm == LDU_NORM_L2;
    const double* __restrict__ w = (st.k & 1) ? w1 : w0;
    double* __restrict__ wn = (st.k & 1) ? w0 : w1;
    double* part = partials + (size_t)(st.k & 1) * kMaxVals * ld;
    double v[3] = {0.0, 0.0, 0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < A.n; c += gridDim.x * blockDim.x) {
      const double wc0 = w[c];
      const double nc = row_apply(A, c, wc0, [&](int j) { return __ldg(rD + j) * w[j]; });
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
    persist_store<3>(v, part, ld);
    grid.sync();
    persist_sum<3>(part, ld, gridDim.x, sums);
    if (threadIdx.x == 0) {
      st.k += 1;
      st.nRed += 1;
      ctl_pipe_top(&st, sums);
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *gst = st;
}

// Classical Jacobi-PCG, passes A and B (as k_cg_passA / k_cg_passB), persistent.
template <class Fmt>
__global__ void __launch_bounds__(kBlock) k_cg_persist(Fmt A, const double* __restrict__ rD,
                                                       double* r, double* p0, double* p1,
                                                       double* q, double* x, State* gst,
                                                       double* partials, int ld, int maxTrips) {
  cg::grid_group grid = cg::this_grid();
  __shared__ State st;
  __shared__ double sums[kMaxVals];
  if (threadIdx.x == 0) {
    st = *gst;
    if (blockIdx.x != 0) st.record = 0;
  }
  __syncthreads();
  double* partA = partials;
  double* partB = partials + (size_t)kMaxVals * ld;
  for (int trip = 0; trip < maxTrips && !st.done; ++trip) {
    {  // pass A_k
      const int k = st.k;
      const double beta = st.beta, alpha = st.alpha;
      const double* __restrict__ pold = (k & 1) ? p0 : p1;
      double* __restrict__ pnew = (k & 1) ? p1 : p0;
      double v[1] = {0.0};
      for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < A.n; c += gridDim.x * blockDim.x) {
        auto op = [&](int j) { return fma(beta, pold[j], __ldg(rD + j) * r[j]); };
        const double po = pold[c];
        const double pc = fma(beta, po, __ldg(rD + c) * r[c]);
        const double qc = row_apply(A, c, pc / __ldg(rD + c), op);
        pnew[c] = pc;
        q[c] = qc;
        x[c] = fma(alpha, po, x[c]);
        v[0] = fma(pc, qc, v[0]);
      }
      persist_store<1>(v, partA, ld);
      grid.sync();
      persist_sum<1>(partA, ld, gridDim.x, sums);
      if (threadIdx.x == 0) {
        st.nRed += 1;
        ctl_cg_A(&st, sums);
      }
      __syncthreads();
      if (st.done) break;
    }
    {  // pass B_k
      const double alpha = st.alpha;
      const bool l2 = st.norm == LDU_NORM_L2;
      double v[2] = {0.0, 0.0};
      for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < A.n; c += gridDim.x * blockDim.x) {
        const double rc = fma(-alpha, q[c], r[c]);
        r[c] = rc;
        v[0] = fma(rc, __ldg(rD + c) * rc, v[0]);
        v[1] += l2 ? rc * rc : fabs(rc);
      }
      persist_store<2>(v, partB, ld);
      grid.sync();
      persist_sum<2>(partB, ld, gridDim.x, sums);
      if (threadIdx.x == 0) {
        st.nRed += 1;
        ctl_cg_B(&st, sums);
      }
      __syncthreads();
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *gst = st;
}

}  // namespace ldu
