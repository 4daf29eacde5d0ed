// ldu_march.cuh -- plane-marching SpMV passes for the DIA layout (3-D stencil-like bands).
//
// Rows are viewed as planes of D = off[ND-1] consecutive rows (the far offset, nx*ny for a 3-D
// hex mesh); the near offsets off[0..ND-2] <= H.  Block b owns tile t (rows t*T .. t*T+T of every
// plane) and marches over a contiguous chunk of planes.  A 3-deep shared-memory ring holds the
// SpMV operand op(j) for the previous, current and next plane tile (current one with an H-row
// halo on both sides), so per row:
//   * the operand (classical CG: p_k = rD r + beta p_{k-1}) is computed ONCE, from one coalesced
//     load of each input array -- v0 recomputed it at all 2*ND neighbours through L1/L2;
//   * near neighbours (+-1, +-nx) come from shared memory, far neighbours (+-nx*ny) from the
//     ring instead of L2 gathers.
// HBM traffic stays at the layout minimum (each array once) plus the ring prologue of two planes
// per chunk.  Summation order per row is the same ascending-column order as row_apply.
#pragma once

#include "ldu_kernels.cuh"

namespace ldu {

enum MarchMode : int { MARCH_AMUL = 0, MARCH_S = 1, MARCH_A = 2 };

constexpr int kMarchT = 1024;                 // tile rows
constexpr int kMarchRows = kMarchT / kBlock;  // rows per thread per plane step
constexpr int kMarchHMax = 512;               // max near offset (halo rows)
constexpr int kMarchSR = (kMarchT + 2 * kMarchHMax + kBlock - 1) / kBlock;  // staged rows/thread

struct MarchGeom {
  int T;              // tile rows
  int H;              // halo rows = max near offset
  int tilesPerPlane;  // ceil(D / T)
  int planes;         // ceil(n / D)
  int chunk;          // planes per chunk
};

template <int ND, int MODE>
struct MarchArgs {
  DiaView<ND> A;
  MarchGeom g;
  // operand inputs: AMUL: in0 = x; S: in0 = rD, in1 = w; A: in0 = rD, in1 = r, (p0, p1 by parity)
  const double* __restrict__ in0;
  const double* __restrict__ in1;
  double* p0;
  double* p1;
  const double* __restrict__ diag;  // AMUL
  double* __restrict__ out;         // y / n / q
  double* __restrict__ x;           // A: x += alpha p_{k-1}
};

template <int ND, int MODE>
__global__ void __launch_bounds__(kBlock) k_march(MarchArgs<ND, MODE> a, State* st, Red rd) {
  extern __shared__ double ring[];  // 3 x W, W = T + 2H
  if (MODE != MARCH_AMUL && st->done) return;
  const int n = a.A.n;
  const int D = a.A.off[ND - 1];
  const int T = a.g.T, H = a.g.H, W = T + 2 * H;
  // Block b owns tile b % tiles of plane chunk b / tiles: all tiles of a chunk march in lockstep,
  // so the halo rows a block stages were staged as own rows by its neighbour tile moments
  // earlier (L2 hits).  Grid = tiles * chunks = SMs * occupancy (one wave).
  const int tile = blockIdx.x % a.g.tilesPerPlane;
  const int chunkId = blockIdx.x / a.g.tilesPerPlane;

  double beta = 0.0, alpha = 0.0;
  const double* pold = nullptr;
  double* pnew = nullptr;
  if (MODE == MARCH_A) {
    const int k = st->k;
    beta = st->beta;
    alpha = st->alpha;
    pold = (k & 1) ? a.p0 : a.p1;
    pnew = (k & 1) ? a.p1 : a.p0;
  }
  auto op = [&](long long j) -> double {
    if (MODE == MARCH_AMUL) return __ldg(a.in0 + j);
    if (MODE == MARCH_S) return __ldg(a.in0 + j) * __ldg(a.in1 + j);
    return fma(beta, __ldg(pold + j), __ldg(a.in0 + j) * __ldg(a.in1 + j));
  };
  // Staging of plane `plane`: stage_load issues every load of this thread into v (op(row) for
  // row = plane*D + tileOff - H + i, 0 outside [0, n) or the plane range); stage_store writes v
  // to the ring slot.  Split so a step issues ALL its global loads before the first barrier.
  auto stage_load = [&](int plane, int tileOff, int tileLen, double (&v)[kMarchSR]) {
    const long long base = (long long)plane * D + tileOff - H;
    const bool pin = plane >= 0 && plane < a.g.planes;
    const int len = tileLen + 2 * H;
#pragma unroll
    for (int u = 0; u < kMarchSR; ++u) {
      const int i = threadIdx.x + u * kBlock;
      const long long row = base + i;
      const bool ok = pin && i < len && row >= 0 && row < n;
      v[u] = op(ok ? row : 0);
      if (!ok) v[u] = 0.0;
    }
  };
  auto stage_store = [&](const double (&v)[kMarchSR], int tileLen, double* buf) {
    const int len = tileLen + 2 * H;
#pragma unroll
    for (int u = 0; u < kMarchSR; ++u) {
      const int i = threadIdx.x + u * kBlock;
      if (i < len) buf[i] = v[u];
    }
  };
  auto slot = [&](int plane) { return ring + ((plane % 3 + 3) % 3) * W; };

  double acc[1] = {0.0};
  {
    const int pBeg = chunkId * a.g.chunk;
    const int pEnd = min(pBeg + a.g.chunk, a.g.planes);
    const int tileOff = tile * T;
    const int tileLen = max(0, min(T, D - tileOff));
    {
      double v[kMarchSR];
      stage_load(pBeg - 1, tileOff, tileLen, v);
      stage_store(v, tileLen, slot(pBeg - 1));
      stage_load(pBeg, tileOff, tileLen, v);
      stage_store(v, tileLen, slot(pBeg));
    }
    for (int p = pBeg; p < pEnd; ++p) {
      double v[kMarchSR];
      stage_load(p + 1, tileOff, tileLen, v);
      const double* prv = slot(p - 1);
      const double* cur = slot(p);
      const double* nxt = slot(p + 1);
      const long long rowBase = (long long)p * D + tileOff;
      // phase 1: every global load of this thread's kMarchRows rows
      double uf[kMarchRows], ul[kMarchRows][ND - 1], uu[kMarchRows][ND], dg[kMarchRows],
          po[kMarchRows], xo[kMarchRows];
#pragma unroll
      for (int u = 0; u < kMarchRows; ++u) {
        const int i = threadIdx.x + u * kBlock;
        const long long c = min(rowBase + min(i, tileLen - 1), (long long)n - 1);
        uf[u] = __ldg(a.A.U[ND - 1] + (c >= D ? c - D : c));
        if (c < D) uf[u] = 0.0;
#pragma unroll
        for (int k = 0; k < ND - 1; ++k) {
          const int d = a.A.off[k];
          ul[u][k] = __ldg(a.A.U[k] + (c >= d ? c - d : c));
          if (c < d) ul[u][k] = 0.0;
        }
#pragma unroll
        for (int k = 0; k < ND; ++k) uu[u][k] = __ldg(a.A.U[k] + c);
        if (MODE == MARCH_AMUL) dg[u] = __ldg(a.diag + c);
        else if (MODE == MARCH_S) dg[u] = __ldg(a.in1 + c);
        else dg[u] = __ldg(a.in0 + c);
        if (MODE == MARCH_A) {
          po[u] = __ldg(pold + c);
          xo[u] = a.x[c];
        }
      }
      stage_store(v, tileLen, slot(p + 1));
      __syncthreads();
      // phase 2: arithmetic from registers and the shared ring, then the stores
#pragma unroll
      for (int u = 0; u < kMarchRows; ++u) {
        const int i = threadIdx.x + u * kBlock;
        const long long c = rowBase + i;
        if (i >= tileLen || c >= n) continue;
        const double pc = cur[H + i];
        double s;
        if (MODE == MARCH_AMUL) s = dg[u] * pc;
        else if (MODE == MARCH_S) s = dg[u];  // diag * rD * w taken as w (Z24)
        else s = pc / dg[u];                  // diag * p as p / rD (Z25)
        // lower far, lower near (descending offsets), upper near, upper far: ascending columns
        s = fma(uf[u], prv[H + i], s);
#pragma unroll
        for (int k = ND - 2; k >= 0; --k) s = fma(ul[u][k], cur[H + i - a.A.off[k]], s);
#pragma unroll
        for (int k = 0; k < ND - 1; ++k) s = fma(uu[u][k], cur[H + i + a.A.off[k]], s);
        s = fma(uu[u][ND - 1], nxt[H + i], s);
        a.out[c] = s;
        if (MODE == MARCH_A) {
          pnew[c] = pc;
          a.x[c] = fma(alpha, po[u], xo[u]);
          acc[0] = fma(pc, s, acc[0]);
        }
      }
      __syncthreads();
    }
  }
  if (MODE == MARCH_A) finish_reduction<1>(acc, rd, st);
}

}  // namespace ldu
