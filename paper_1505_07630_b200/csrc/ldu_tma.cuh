// ldu_tma.cuh -- plane-marching SpMV passes fed by TMA bulk copies (DIA layout).
//
// Same plane march as ldu_march.cuh (block = tile x plane chunk, all tiles of a chunk in
// lockstep, 3-deep shared ring of the SpMV operand), but every global input of a plane is moved
// into shared memory by the Tensor Memory Accelerator (cp.async.bulk global->shared, completion
// on an mbarrier) kTmaLookahead planes ahead of its use, so the following planes stream in while
// the threads compute the current one from shared memory.  One 512-thread block per SM; threads
// issue no global loads at all -- only the coalesced stores of the results.
//
// Plane slot q (one mbarrier; rows r0 = q*D + tileOff .. r0 + len):
//   the NR operand arrays over [r0 - H, r0 + len + H), the near coefficients U_k (k < ND-1) over
//   [r0 - H, r0 + len), the far coefficient U_{ND-1} and the extra own-row array (AMUL: diag,
//   A: x) over [r0, r0 + len).
// Step p: issue plane p+1+L; wait plane p+1 -> operand ring (p+1); compute the rows of plane p
// from slots p (own), p-1 (far-lower coefficient) and the ring.
// Requirements (checked on the host): D, H, T, n even (16-byte aligned bulk copies).
#pragma once

#include <cstdint>

#include "ldu_march.cuh"

namespace ldu {

constexpr int kTmaThreads = 512;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// Spin on the phase parity.  Bounded: a lost transaction traps (kernel error) instead of
// hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  for (long long spin = 0; spin < (1LL << 26); ++spin) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
  }
  __trap();
}

__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int MODE>
struct TmaTraits {
  static constexpr int NR = MODE == MARCH_AMUL ? 1 : (MODE == MARCH_S ? 2 : 3);
  static constexpr bool EXTRA = MODE != MARCH_S;
};

// Doubles of one plane slot: NR operand arrays over T+2H rows, ND-1 near coefficient arrays over
// T+H rows, the far coefficient and the extra array over T rows.
template <int ND, int MODE>
__host__ __device__ constexpr long long tma_slot_doubles(long long T, long long H) {
  return TmaTraits<MODE>::NR * (T + 2 * H) + (ND - 1) * (T + H) + T +
         (TmaTraits<MODE>::EXTRA ? T : 0);
}

// Shared-memory footprint in doubles for tile T, halo H, lookahead L (L + 3 plane slots).
template <int ND, int MODE, int L>
__host__ __device__ constexpr long long tma_smem_doubles(long long T, long long H) {
  return (L + 3) * tma_slot_doubles<ND, MODE>(T, H) + 3LL * (T + 2 * H);
}

template <int ND, int MODE, int L>
__global__ void __launch_bounds__(kTmaThreads, 1)
    k_tma_march(MarchArgs<ND, MODE> a, State* st, Red rd) {
  constexpr int kTmaLookahead = L;      // planes in flight beyond the one being consumed
  constexpr int kTmaSlots = L + 3;      // + plane p-1 (far-lower U), p, p+1
  using Tr = TmaTraits<MODE>;
  constexpr int NR = Tr::NR;
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar[kTmaSlots];
  if (MODE != MARCH_AMUL && st->done) return;

  const int n = a.A.n;
  const int D = a.A.off[ND - 1];
  const int T = a.g.T, H = a.g.H, W = T + 2 * H;
  const int tile = blockIdx.x % a.g.tilesPerPlane;
  const int chunkId = blockIdx.x / a.g.tilesPerPlane;
  const int pBeg = chunkId * a.g.chunk;
  const int pEnd = min(pBeg + a.g.chunk, a.g.planes);
  const int tileOff = tile * T;
  const int len = max(0, min(T, D - tileOff));
  const int slotD = (int)tma_slot_doubles<ND, MODE>(T, H);
  // slot layout: R[NR][W] | Un[ND-1][T+H] | Uf[T] | Ex[T]
  const int oUn = NR * W, oUf = oUn + (ND - 1) * (T + H), oEx = oUf + T;
  double* ring = sm + kTmaSlots * slotD;  // [3][W]
  auto slotOf = [](int q) { return ((q % kTmaSlots) + kTmaSlots) % kTmaSlots; };
  auto mod3 = [](int q) { return (q % 3 + 3) % 3; };
  auto plane = [&](int q) { return sm + slotOf(q) * slotD; };

  double beta = 0.0, alpha = 0.0;
  const double* pold = nullptr;
  double* pnew = nullptr;
  const double* R[3] = {a.in0, a.in1, nullptr};
  if (MODE == MARCH_A) {
    const int k = st->k;
    beta = st->beta;
    alpha = st->alpha;
    pold = (k & 1) ? a.p0 : a.p1;
    pnew = (k & 1) ? a.p1 : a.p0;
    R[2] = pold;
  }
  const double* exSrc = MODE == MARCH_AMUL ? a.diag : a.x;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kTmaSlots; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // rows [lo, hi) of src, clamped to [0, n), to dst (dst[0] = row lo)
  auto copy_rows = [&](double* dst, const double* src, int lo, int hi, uint64_t* b) {
    const int l = max(lo, 0), h = min(hi, n);
    if (h > l) tma_load_1d(dst + (l - lo), src + l, (uint32_t)(h - l) * 8u, b);
  };
  auto span = [&](int lo, int hi) {
    const int l = max(lo, 0), h = min(hi, n);
    return h > l ? (uint32_t)(h - l) * 8u : 0u;
  };
  // one elected thread: arm plane q's barrier with its byte total, then issue its copies
  auto issue = [&](int q) {
    uint64_t* b = &bar[slotOf(q)];
    const bool in = q >= 0 && q < a.g.planes && len > 0;
    const int r0 = q * D + tileOff;  // rows fit in int (nCells is an int)
    uint32_t bytes = 0;
    if (in)
      bytes = NR * span(r0 - H, r0 + len + H) + (ND - 1) * span(r0 - H, r0 + len) +
              (Tr::EXTRA ? 2 : 1) * span(r0, r0 + len);
    mbar_arrive_expect_tx(b, bytes);
    if (!in) return;
    double* ps = plane(q);
    for (int k = 0; k < NR; ++k) copy_rows(ps + k * W, R[k], r0 - H, r0 + len + H, b);
    for (int k = 0; k < ND - 1; ++k) copy_rows(ps + oUn + k * (T + H), a.A.U[k], r0 - H, r0 + len, b);
    copy_rows(ps + oUf, a.A.U[ND - 1], r0, r0 + len, b);
    if (Tr::EXTRA) copy_rows(ps + oEx, exSrc, r0, r0 + len, b);
  };
  uint32_t ph[kTmaSlots];
#pragma unroll
  for (int i = 0; i < kTmaSlots; ++i) ph[i] = 0u;
  // Warp 0 spins on the plane's mbarrier while the other warps sleep in bar.sync; afterwards
  // every thread performs one (already satisfied) try_wait to acquire the TMA writes.
  auto wait = [&](int q) {
    const int sl = slotOf(q);
    uint32_t par = 0;
#pragma unroll
    for (int i = 0; i < kTmaSlots; ++i)
      if (i == sl) par = ph[i];
    if (threadIdx.x < 32) mbar_wait(&bar[sl], par);
    __syncthreads();
    mbar_wait(&bar[sl], par);
#pragma unroll
    for (int i = 0; i < kTmaSlots; ++i)
      if (i == sl) ph[i] ^= 1u;
  };
  // operand of plane q from its slot into the ring (0 outside [0, n) / the plane range)
  auto build_ring = [&](int q) {
    const double* rs = plane(q);
    double* dst = ring + mod3(q) * W;
    const int base = q * D + tileOff - H;
    const bool in = q >= 0 && q < a.g.planes;
    for (int i = threadIdx.x; i < len + 2 * H; i += kTmaThreads) {
      const int row = base + i;
      double v = 0.0;
      if (in && row >= 0 && row < n) {
        if (MODE == MARCH_AMUL) v = rs[i];
        else if (MODE == MARCH_S) v = rs[i] * rs[W + i];
        else v = fma(beta, rs[2 * W + i], rs[i] * rs[W + i]);
      }
      dst[i] = v;
    }
  };

  double acc[1] = {0.0};
  if (pBeg < pEnd && len > 0) {
    if (threadIdx.x == 0)
      for (int q = pBeg - 1; q <= pBeg + kTmaLookahead; ++q) issue(q);
    wait(pBeg - 1);
    build_ring(pBeg - 1);
    wait(pBeg);
    build_ring(pBeg);
    __syncthreads();
    for (int p = pBeg; p < pEnd; ++p) {
      // plane p + 1 + L reuses the slot of plane p - 2 (released by the last barrier); planes
      // p + 2 .. p + 1 + L stay in flight while plane p + 1 is consumed
      if (threadIdx.x == 0) issue(p + 1 + kTmaLookahead);
      wait(p + 1);
      build_ring(p + 1);
      __syncthreads();
      const double* prv = ring + mod3(p - 1) * W;
      const double* cur = ring + mod3(p) * W;
      const double* nxt = ring + mod3(p + 1) * W;
      const double* ps = plane(p);
      const double* un = ps + oUn;
      const double* ufc = ps + oUf;
      const double* ufp = plane(p - 1) + oUf;
      const double* ex = ps + oEx;
      const int rowBase = p * D + tileOff;
      for (int i = threadIdx.x; i < len; i += kTmaThreads) {
        const int c = rowBase + i;
        if (c >= n) break;
        const double pc = cur[H + i];
        double s;
        if (MODE == MARCH_AMUL) s = ex[i] * pc;
        else if (MODE == MARCH_S) s = ps[W + H + i];  // diag * rD * w taken as w (Z24)
        else s = pc / ps[H + i];                      // diag * p as p / rD (Z25)
        // lower far, lower near (descending offsets), upper near, upper far: ascending columns
        s = fma(c >= D ? ufp[i] : 0.0, prv[H + i], s);
#pragma unroll
        for (int k = ND - 2; k >= 0; --k) {
          const int d = a.A.off[k];
          s = fma(c >= d ? un[k * (T + H) + H + i - d] : 0.0, cur[H + i - d], s);
        }
#pragma unroll
        for (int k = 0; k < ND - 1; ++k) s = fma(un[k * (T + H) + H + i], cur[H + i + a.A.off[k]], s);
        s = fma(ufc[i], nxt[H + i], s);
        a.out[c] = s;
        if (MODE == MARCH_A) {
          pnew[c] = pc;
          a.x[c] = fma(alpha, ps[2 * W + H + i], ex[i]);
          acc[0] = fma(pc, s, acc[0]);
        }
      }
      __syncthreads();
    }
    // drain: planes issued beyond pEnd must land before the block's shared memory is released
    for (int q = pEnd + 1; q <= pEnd + kTmaLookahead; ++q) wait(q);
  }
  if (MODE == MARCH_A) finish_reduction<1>(acc, rd, st);
}

}  // namespace ldu
