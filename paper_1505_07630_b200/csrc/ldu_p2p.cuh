// ldu_p2p.cuh -- NVLink peer-memory communication fused into the CG kernels (multi-rank).
//
// Every rank owns one "mailbox" allocation that its peers write into over NVLink (CUDA IPC
// mappings, one process per GPU):
//   redFlag[2][kP2PMaxRanks]  u64   reduction flags, slot [parity][source rank]
//   haloFlag[2][kP2PMaxIf]    u64   halo flags, slot [parity][receiving interface]
//   red[2][kP2PMaxRanks][4]   f64   the fused partial sums, slot [parity][source rank]
//   recv[2][nIfFaces]         f64   halo values, double-buffered by exchange parity
// Messages carry a sequence number (per handle, identical on every rank because all ranks run
// the same sequence of collective steps).  Producers store data, __threadfence_system(), then
// store the flag = seq; consumers spin (bounded, then trap) until flag >= seq and read with
// L1-bypassing loads.  Parity double-buffering is sufficient: a peer can run at most one
// exchange ahead because it needs this rank's reduction contribution to proceed.
#pragma once

#include <cstdint>

#include "ldu_impl.cuh"

namespace ldu {

constexpr int kP2PMaxRanks = 64;
constexpr int kP2PMaxIf = 16;

struct MailboxLayout {
  static constexpr size_t redFlag = 0;
  static constexpr size_t haloFlag = redFlag + sizeof(uint64_t) * 2 * kP2PMaxRanks;
  static constexpr size_t red = haloFlag + sizeof(uint64_t) * 2 * kP2PMaxIf;
  // low-latency (LL) slots of the one-kernel pipelined loop: every 8-byte word carries 32 bits
  // of payload and the 32-bit sequence number of its message, so a reader that sees the
  // expected sequence number in a word has its payload -- no fence, no separate flag.
  // redLL: [parity][source rank][4 values][2 words]; haloLL: [parity][face][2 words]
  static constexpr size_t redLL = red + sizeof(double) * 2 * kP2PMaxRanks * 4;
  static constexpr size_t recv = redLL + sizeof(uint64_t) * 2 * kP2PMaxRanks * 4 * 2;
  __host__ __device__ static size_t haloLL(int nIfFaces) { return recv + sizeof(double) * 2 * (size_t)nIfFaces; }
  __host__ __device__ static size_t bytes(int nIfFaces) { return haloLL(nIfFaces) + sizeof(uint64_t) * 2 * 2 * (size_t)nIfFaces; }
};

// Device-resident descriptor (one per handle).
struct P2PDesc {
  int rank, nRanks, nIf;
  unsigned long long seqRed, seqHalo;   // last consumed sequence numbers (device state)
  unsigned long long seqHaloSend;       // last sent halo exchange (advanced only by the pack)
  // Fused pipelined loop: (k, done) of the State as the fix-up of iteration i saw them.  The pack
  // of exchange i+1 runs on the halo stream concurrently with the control step of iteration
  // i+1, which advances k and may set done; the pack reads this snapshot instead of the live
  // State, so its buffer choice and its send/skip decision match what the consumer side assumes
  // (the control step retires an exchange exactly when the snapshot said it was sent).
  int snapK, snapDone;
  char* base[kP2PMaxRanks];             // mailbox of every rank (own = local pointer)
  int ifNeighbor[kP2PMaxIf];            // peer rank of my interface k
  int ifLocalOff[kP2PMaxIf];            // my packed face offset of interface k
  int ifNFaces[kP2PMaxIf];
  int ifRemoteOff[kP2PMaxIf];           // offset in the peer's recv of its interface back to me
  int ifRemoteIdx[kP2PMaxIf];           // the peer's interface index (its halo flag slot)
  int ifRemoteTotal[kP2PMaxIf];         // the peer's packed interface face count (recv stride)
  unsigned long long* tbuf;             // LDU_TRACE: [iteration % 256][16] %globaltimer stamps
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// stamp slot `s` of iteration k: mode 0 store, 1 min, 2 max
__device__ __forceinline__ void tstamp(P2PDesc* d, int k, int s, int mode) {
  if (!d || !d->tbuf || k < 0) return;
  unsigned long long* p = d->tbuf + (k & 255) * 16 + s;
  const unsigned long long t = gtimer();
  if (mode == 0) *p = t;
  else if (mode == 1) atomicMax(p, ~t);  // min, stored complemented (buffer zeroed per solve)
  else atomicMax(p, t);
}

__device__ __forceinline__ uint64_t* mb_redflag(char* b, int par, int src) {
  return reinterpret_cast<uint64_t*>(b + MailboxLayout::redFlag) + par * kP2PMaxRanks + src;
}
__device__ __forceinline__ uint64_t* mb_haloflag(char* b, int par, int k) {
  return reinterpret_cast<uint64_t*>(b + MailboxLayout::haloFlag) + par * kP2PMaxIf + k;
}
__device__ __forceinline__ double* mb_red(char* b, int par, int src) {
  return reinterpret_cast<double*>(b + MailboxLayout::red) + (par * kP2PMaxRanks + src) * 4;
}
__device__ __forceinline__ double* mb_recv(char* b, int par, int nIfFaces) {
  return reinterpret_cast<double*>(b + MailboxLayout::recv) + (size_t)par * nIfFaces;
}

// LL slots of the mailbox `b` (whose owner has nIfFaces packed interface faces)
__device__ __forceinline__ uint64_t* mb_redll(char* b, int par, int src) {
  return reinterpret_cast<uint64_t*>(b + MailboxLayout::redLL) + (size_t)(par * kP2PMaxRanks + src) * 8;
}
__device__ __forceinline__ uint64_t* mb_haloll(char* b, int par, int nIfFaces) {
  return reinterpret_cast<uint64_t*>(b + MailboxLayout::haloLL(nIfFaces)) + (size_t)par * nIfFaces * 2;
}

// One fp64 value as two LL words (NCCL's LL protocol): each aligned 8-byte word is single-copy
// atomic, so a reader that sees `flag` in both words holds both halves of this message's value.
__device__ __forceinline__ void ll_store(uint64_t* p, double v, uint32_t flag) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  const unsigned long long f = (unsigned long long)flag << 32;
  const unsigned long long w0 = f | (bits & 0xffffffffull), w1 = f | (bits >> 32);
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
__device__ __forceinline__ bool ll_try(const uint64_t* p, uint32_t flag, double& v) {
  unsigned long long w0, w1;
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
  if ((uint32_t)(w0 >> 32) != flag || (uint32_t)(w1 >> 32) != flag) return false;
  v = __longlong_as_double((long long)((w1 << 32) | (w0 & 0xffffffffull)));
  return true;
}
// Bounded spin (~4 s at 2 GHz), as spin_until_geq.
__device__ __forceinline__ double ll_load(const uint64_t* p, uint32_t flag) {
  double v;
  if (ll_try(p, flag, v)) return v;
  const long long t0 = clock64();
  while (!ll_try(p, flag, v)) {
    if (clock64() - t0 > 8000000000LL) __trap();
    __nanosleep(32);
  }
  return v;
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Flag store after ONE preceding __threadfence_system() that already ordered the data: each
// st.release.sys is its own system-scope release (serialised, several us apiece over NVLink).
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Bounded spin (~4 s at 2 GHz): a lost peer turns into a kernel error, not a hung GPU.
__device__ __forceinline__ void spin_until_geq(const uint64_t* p, uint64_t seq) {
  const long long t0 = clock64();
  while (ld_acquire_sys(p) < seq) {
    if (clock64() - t0 > 8000000000LL) __trap();
    __nanosleep(64);
  }
}

// Last block of a reducing pass: publish the local sums to every rank's mailbox (incl. self).
template <int NV>
__device__ __forceinline__ void p2p_publish_sums(P2PDesc* d, const double* sums) {
  const uint64_t seq = d->seqRed + 1;
  const int par = (int)(seq & 1);
  for (int r = 0; r < d->nRanks; ++r) {
    double* dst = mb_red(d->base[r], par, d->rank);
#pragma unroll
    for (int k = 0; k < NV; ++k) dst[k] = sums[k];
  }
  __threadfence_system();  // one system fence orders all data stores before every flag
  for (int r = 0; r < d->nRanks; ++r) st_relaxed_sys(mb_redflag(d->base[r], par, d->rank), seq);
}

// Raise the halo flags of exchange `seq` on every neighbour (after all blocks' remote stores
// were fenced at system scope and counted by the caller's ticket).
__device__ __forceinline__ void p2p_release_halo(P2PDesc* d, uint64_t seq) {
  const int par = (int)(seq & 1);
  __threadfence_system();
  for (int k = 0; k < d->nIf; ++k)
    st_relaxed_sys(mb_haloflag(d->base[d->ifNeighbor[k]], par, d->ifRemoteIdx[k]), seq);
}

// Control kernel side: wait for every rank's sums of the next sequence number, sum them in
// rank order into s[], advance the sequence.
template <int NV>
__device__ __forceinline__ void p2p_gather_sums(P2PDesc* d, double* s) {
  const uint64_t seq = d->seqRed + 1;
  const int par = (int)(seq & 1);
  char* me = d->base[d->rank];
  for (int k = 0; k < NV; ++k) s[k] = 0.0;
  for (int r = 0; r < d->nRanks; ++r) {
    spin_until_geq(mb_redflag(me, par, r), seq);
    const double* src = mb_red(me, par, r);
#pragma unroll
    for (int k = 0; k < NV; ++k) s[k] += __ldcv(src + k);
  }
  d->seqRed = seq;
}

}  // namespace ldu
