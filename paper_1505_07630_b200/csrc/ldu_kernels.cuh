// ldu_kernels.cuh -- device code of the CG hot path.
//
// Every streaming pass walks the rows in a grid-stride wavefront (block b handles rows
// b*256 + t, then + gridDim*256, ...), so all blocks sweep the vectors together and the
// neighbour gathers at +-nx*ny rows hit L2 instead of HBM; the grid is a multiple of the SM
// count (occupancy-derived).  Reductions are deterministic: warp xor-butterfly, fixed-order block
// tree, per-block partials in a fixed slot, and the last block to arrive sums the slots in index
// order (no floating-point atomics anywhere).
#pragma once

#include "ldu_impl.cuh"
#include "ldu_p2p.cuh"

namespace ldu {

// ---------------------------------------------------------------------------------------------
// row operators: s = init + sum_j a_cj * op(j) in ascending column order (diag term is `init`)
// ---------------------------------------------------------------------------------------------
template <int ND, class Op>
__device__ __forceinline__ double row_apply(const DiaView<ND>& A, int c, double s, Op op) {
#pragma unroll
  for (int k = ND - 1; k >= 0; --k) {  // lower side: columns c - off[ND-1] < ... < c - off[0]
    int j = c - A.off[k];
    if (j >= 0) s = fma(__ldg(A.U[k] + j), op(j), s);
  }
#pragma unroll
  for (int k = 0; k < ND; ++k) {  // upper side: columns c + off[0] < ... < c + off[ND-1]
    int j = c + A.off[k];
    if (j < A.n) s = fma(__ldg(A.U[k] + c), op(j), s);
  }
  return s;
}

// SELL-32 row: the slice's pair loads are issued kSellBatch at a time before any gather (no
// data-dependent exit: a padding entry (col -1, value 0) gathers the row's own operand and adds
// an exact 0, so the sum of the real entries keeps its order).  One dependent load chain per
// batch instead of one per pair.
constexpr int kSellBatch = 4;
template <class Op>
__device__ __forceinline__ double row_apply(const SellView& A, int c, double s, Op op) {
  const int slice = c >> 5, lane = c & 31;
  const long long base = __ldg(A.slicePtr + slice);
  const int np = __ldg(A.npairs + slice);
  int jj = 0;
  for (; jj + kSellBatch <= np; jj += kSellBatch) {
    int2 cc[kSellBatch];
    double2 vv[kSellBatch];
#pragma unroll
    for (int u = 0; u < kSellBatch; ++u) {
      const long long e = (base + jj + u) * 32 + lane;
      cc[u] = __ldg(A.col + e);
      vv[u] = __ldg(A.val + e);
    }
    double x0[kSellBatch], x1[kSellBatch];
#pragma unroll
    for (int u = 0; u < kSellBatch; ++u) {
      x0[u] = op(cc[u].x < 0 ? c : cc[u].x);
      x1[u] = op(cc[u].y < 0 ? c : cc[u].y);
    }
#pragma unroll
    for (int u = 0; u < kSellBatch; ++u) {
      s = fma(vv[u].x, x0[u], s);
      s = fma(vv[u].y, x1[u], s);
    }
  }
  for (; jj < np; ++jj) {
    const long long e = (base + jj) * 32 + lane;
    const int2 cc = __ldg(A.col + e);
    const double2 vv = __ldg(A.val + e);
    const double x0 = op(cc.x < 0 ? c : cc.x), x1 = op(cc.y < 0 ? c : cc.y);
    s = fma(vv.x, x0, s);
    s = fma(vv.y, x1, s);
  }
  return s;
}

// ---------------------------------------------------------------------------------------------
// programmatic dependent launch (PDL): a kernel launched with programmatic stream serialisation
// may start while its predecessor drains; it must wait before touching the predecessor's data.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------------------------------------
// deterministic reductions
// ---------------------------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ void warp_allreduce(double (&v)[NV]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
}

// Sum over the block in a fixed tree; result in every lane of warp 0.
template <int NV>
__device__ __forceinline__ void block_reduce(double (&v)[NV], double (*sm)[32]) {
  warp_allreduce<NV>(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) sm[k][wid] = v[k];
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = lane < (int)(blockDim.x >> 5) ? sm[k][lane] : 0.0;
    warp_allreduce<NV>(v);
  }
}

// Block partial -> partials[k*ld + slot]; returns true in every thread of the last block to
// arrive (of `nblocks` participating blocks).
template <int NV>
__device__ __forceinline__ bool store_partial_is_last(double (&v)[NV], double* partials, int ld,
                                                      int slot, unsigned* ticket,
                                                      unsigned nblocks) {
  __shared__ double sm[NV][32];
  __shared__ bool last;
  block_reduce<NV>(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) partials[k * ld + slot] = v[k];
    __threadfence();
    const unsigned t = atomicAdd(ticket, 1u);
    last = (t == nblocks - 1);
  }
  __syncthreads();
  return last;
}

// Fixed-order sum of partial slots [k*ld + 0 .. total): thread t owns slots t, t + B, ...; its
// loads are issued 8 at a time (independent) before they are added in slot order, then the block
// tree.  (A dependent load-add chain per thread cost ~5 us of L2 latency for ~1300 slots.)
template <int NV>
__device__ __forceinline__ void sum_slots(const double* partials, int ld, int total,
                                          double (&v)[NV]) {
  const int B = blockDim.x;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = 0.0;
  for (int i0 = threadIdx.x; i0 < total; i0 += 8 * B) {
    double t[NV][8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = i0 + j * B;
#pragma unroll
      for (int k = 0; k < NV; ++k) t[k][j] = i < total ? __ldcg(partials + k * ld + i) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int k = 0; k < NV; ++k) v[k] += t[k][j];
  }
}

// In the last block: out[k] = sum of partials[k*ld + 0 .. total) in a fixed order.
template <int NV>
__device__ __forceinline__ void sum_partials(const double* partials, int ld, int total,
                                             double* out, unsigned* ticket) {
  __shared__ double sm[NV][32];
  __threadfence();
  double v[NV];
  sum_slots<NV>(partials, ld, total, v);
  block_reduce<NV>(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) out[k] = v[k];
    *ticket = 0u;
  }
}

// ---------------------------------------------------------------------------------------------
// control steps (one thread; readings Z1-Z3, Z19)
// ---------------------------------------------------------------------------------------------
// stopping test after `it` x-updates (readings Z2, Z2', Z26)
__device__ __forceinline__ bool converged(const State* st, double res, int it) {
  if (it < st->minIter) return false;
  return res < st->tol || res == 0.0 || (st->relTol > 0.0 && res < st->relTol * st->res0);
}

__device__ __forceinline__ double crit_value(const State* st, double v) {
  return st->norm == LDU_NORM_L2 ? sqrt(v) / st->scale : v / st->scale;
}

__device__ __forceinline__ void record(State* st, int i, double res) {
  st->res = res;
  if (st->record && i < st->histCap) st->hist[i] = res;
}

__device__ __forceinline__ void finish(State* st, int status, int iter) {
  st->done = 1;
  st->status = status;
  st->iter = iter;
}

// criterion scale from s0 = sum b^2 (L2) or the OpenFOAM normFactor sum
__device__ __forceinline__ void ctl_scale(State* st, double s0) {
  if (st->norm == LDU_NORM_L2) {
    st->scale = sqrt(s0);
    if (st->scale == 0.0) {  // b = 0 => x = 0 (reading Z1)
      st->zero_x = 1;
      record(st, 0, 0.0);
      finish(st, LDU_OK, 0);
    }
  } else {
    st->scale = s0 + 1e-20;
  }
}

// classical, after r0: s = [scale piece, (r0, z0), crit piece(r0)]
__device__ __forceinline__ void ctl_cg_init(State* st, const double* s) {
  ctl_scale(st, s[0]);
  if (st->done) return;
  const double res = crit_value(st, s[2]);
  record(st, 0, res);
  st->res0 = res;
  st->iter = 0;
  st->k = 0;
  st->rho = s[1];
  st->alpha = 0.0;
  st->beta = 0.0;
  st->xpending = 0;
  if (converged(st, res, 0)) finish(st, LDU_OK, 0);
  else if (st->maxIter == 0) finish(st, LDU_NOT_CONVERGED, 0);
}

// classical, after pass A_k: s = [(p_k, A p_k)]
__device__ __forceinline__ void ctl_cg_A(State* st, const double* s) {
  const double pq = s[0];
  st->xpending = 0;  // pass A_k applied alpha_{k-1} p_{k-1}: x = x_k
  if (!(pq > 0.0) || !isfinite(pq)) {
    finish(st, LDU_BREAKDOWN, st->k);
    return;
  }
  st->alpha = st->rho / pq;
}

// classical, after pass B_k: s = [(r_{k+1}, z_{k+1}), crit piece(r_{k+1})]
__device__ __forceinline__ void ctl_cg_B(State* st, const double* s) {
  const int it = st->k + 1;
  st->iter = it;
  st->xpending = 1;  // alpha_k p_k still to be added to x
  const double res = crit_value(st, s[1]);
  record(st, it, res);
  if (converged(st, res, it)) finish(st, LDU_OK, it);
  else if (it >= st->maxIter) finish(st, LDU_NOT_CONVERGED, it);
  else {
    st->beta = s[0] / st->rho;
    st->rho = s[0];
    st->k = it;
  }
}

// pipelined, top of iteration i = st->k: s = [gamma_i, delta_i, crit piece(r_i)]
__device__ __forceinline__ void ctl_pipe_top(State* st, const double* s) {
  const int i = st->k;
  const double res = crit_value(st, s[2]);
  record(st, i, res);
  if (i == 0) st->res0 = res;
  st->iter = i;
  if (converged(st, res, i)) { finish(st, LDU_OK, i); return; }
  if (i >= st->maxIter) { finish(st, LDU_NOT_CONVERGED, i); return; }
  const double g = s[0], d = s[1];
  double a, b;
  if (i == 0) {
    b = 0.0;
    if (!(d > 0.0) || !isfinite(d)) { finish(st, LDU_BREAKDOWN, i); return; }
    a = g / d;
  } else {
    b = g / st->gamma_old;
    const double den = d - b * g / st->alpha_old;
    if (!(den > 0.0) || !isfinite(den)) { finish(st, LDU_BREAKDOWN, i); return; }
    a = g / den;
  }
  st->pa = a;
  st->pb = b;
  st->gamma_old = g;
  st->alpha_old = a;
}

// AMG-PCG (NEXT-2), after the V-cycle z_k = B r_k: s = [(z_k, r_k)]; beta_0 = 0 (p_0 = z_0)
__device__ __forceinline__ void ctl_amg_rho(State* st, const double* s) {
  const double rho = s[0];
  st->beta = (st->k == 0) ? 0.0 : rho / st->rho;
  st->rho = rho;
}

// AMG-PCG, after r_{k+1} = r_k - alpha_k q_k: s = [crit piece(r_{k+1})]
__device__ __forceinline__ void ctl_amg_B(State* st, const double* s) {
  const int it = st->k + 1;
  st->iter = it;
  st->xpending = 1;  // alpha_k p_k still to be added to x
  const double res = crit_value(st, s[0]);
  record(st, it, res);
  if (converged(st, res, it)) finish(st, LDU_OK, it);
  else if (it >= st->maxIter) finish(st, LDU_NOT_CONVERGED, it);
  else st->k = it;
}

// control selector for the "last block" epilogue of a pass (single rank) or the ctl kernel
enum Ctl : int { CTL_NONE = 0, CTL_CG_INIT, CTL_PIPE_SCALE, CTL_XBAR, CTL_CG_A, CTL_CG_B,
                 CTL_PIPE_TOP, CTL_PIPE_NEXT, CTL_AMG_RHO, CTL_AMG_B };

__device__ __forceinline__ void run_ctl(int ctl, State* st, const double* s) {
  if (ctl != CTL_NONE) st->nRed += 1;  // device-side reduction count (ldu_solve_stats)
  switch (ctl) {
    case CTL_CG_INIT: ctl_cg_init(st, s); break;
    case CTL_PIPE_SCALE: ctl_scale(st, s[0]); break;
    case CTL_XBAR: st->xbar = s[0] / s[1]; break;
    case CTL_CG_A: ctl_cg_A(st, s); break;
    case CTL_CG_B: ctl_cg_B(st, s); break;
    case CTL_PIPE_TOP: ctl_pipe_top(st, s); break;
    case CTL_PIPE_NEXT: st->k += 1; ctl_pipe_top(st, s); break;
    case CTL_AMG_RHO: ctl_amg_rho(st, s); break;
    case CTL_AMG_B: ctl_amg_B(st, s); break;
    default: break;
  }
}

struct Red {  // reduction plumbing of one pass
  double* partials;
  int ld;
  unsigned* ticket;
  double* sums;
  int ctl;         // control step run by the last block (single rank) or CTL_NONE
  int slot_base;   // first partial slot of this kernel
  int total;       // slots summed by the last block
  int store_only;  // 1: store partials only (a later kernel finishes the reduction)
  P2PDesc* p2p;    // multi-rank over peer memory: publish the local sums to every rank
  int llctl;       // != 0 (multi-rank, peer memory): publish the sums as LL words, gather every
                   // rank's in the same last block and run this control step there (no flag, no
                   // fence, no control kernel)
  int llHalo;      // halo exchanges consumed by this pass (retired by that control step)
};

// Last block of an LL-reducing pass: the sums (NV <= 4) to every rank's mailbox as LL words
// (lane q -> rank q), every rank's sums back from this rank's mailbox, summed in rank order,
// the control step.  Out of line: the streaming loops of the kernels that inline
// finish_reduction keep their registers.
template <int NV>
__device__ __noinline__ void ll_reduce_ctl(const Red& rd, State* st) {
  P2PDesc* d = rd.p2p;
  __shared__ double part[kP2PMaxRanks][NV];
  const unsigned long long sq = d->seqRed + 1;
  const int par = (int)(sq & 1);
  __syncthreads();
  for (int q = threadIdx.x; q < d->nRanks; q += blockDim.x) {
    uint64_t* dst = mb_redll(d->base[q], par, d->rank);
#pragma unroll
    for (int m = 0; m < NV; ++m) ll_store(dst + 2 * m, __ldcg(rd.sums + m), (uint32_t)sq);
  }
  char* me = d->base[d->rank];
  for (int q = threadIdx.x; q < d->nRanks; q += blockDim.x) {
    const uint64_t* src = mb_redll(me, par, q);
#pragma unroll
    for (int m = 0; m < NV; ++m) part[q][m] = ll_load(src + 2 * m, (uint32_t)sq);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sums[kMaxVals] = {0.0, 0.0, 0.0, 0.0};
    for (int q = 0; q < d->nRanks; ++q)
      for (int m = 0; m < NV; ++m) sums[m] += part[q][m];
    d->seqRed = sq;
    d->seqHalo += rd.llHalo;
    run_ctl(rd.llctl, st, sums);
  }
}

template <int NV>
__device__ __forceinline__ void finish_reduction(double (&v)[NV], const Red& rd, State* st) {
  if (rd.store_only) {
    __shared__ double sm[NV][32];
    block_reduce<NV>(v, sm);
    if (threadIdx.x == 0)
#pragma unroll
      for (int k = 0; k < NV; ++k) rd.partials[k * rd.ld + rd.slot_base + blockIdx.x] = v[k];
    return;
  }
  if (store_partial_is_last<NV>(v, rd.partials, rd.ld, rd.slot_base + blockIdx.x, rd.ticket,
                                gridDim.x)) {
    if (threadIdx.x == 0) tstamp(rd.p2p, st->k, 8, 0);
    sum_partials<NV>(rd.partials, rd.ld, rd.total, rd.sums, rd.ticket);
    if (threadIdx.x == 0) tstamp(rd.p2p, st->k, 9, 0);
    if (threadIdx.x == 0 && rd.ctl != CTL_NONE) run_ctl(rd.ctl, st, rd.sums);
    if (threadIdx.x == 0 && rd.p2p) p2p_publish_sums<NV>(rd.p2p, rd.sums);
    if (threadIdx.x == 0) tstamp(rd.p2p, st->k, 10, 0);
  }
}

// finish_reduction for the LL multi-rank passes (classical CG's fix-up and pass B): only those
// kernels instantiate it, so the single-rank passes keep their register allocation
template <int NV>
__device__ __forceinline__ void finish_reduction_ll(double (&v)[NV], const Red& rd, State* st) {
  if (store_partial_is_last<NV>(v, rd.partials, rd.ld, rd.slot_base + blockIdx.x, rd.ticket,
                                gridDim.x)) {
    sum_partials<NV>(rd.partials, rd.ld, rd.total, rd.sums, rd.ticket);
    ll_reduce_ctl<NV>(rd, st);
  }
}

}  // namespace ldu
