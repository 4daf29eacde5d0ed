// ldu_amg_setup.cu -- device-side setup of the aggregation-AMG hierarchy (NEXT-2).
//
// Per level l (readings Z27-Z32):
//   1. graph of A_l = its off-diagonal pattern (all couplings strong, Z29);
//   2. distance-2 MIS by parallel local-minimum rounds in key order: a node becomes a root when
//      its key is the smallest among the undecided nodes within distance 2; the roots and all
//      nodes within distance 2 of them are then decided.  This is exactly the greedy
//      (lexicographically first) MIS-2 in key order (Z30); aggregates are numbered by root index,
//      a node next to roots joins the smallest-key adjacent root, the rest join the aggregate of
//      their smallest-key adjacent step-3 node;
//   3. w_l = (4/3) / (1.05 x largest Ritz value of `lanczosSteps` Lanczos steps on
//      D^-1/2 A D^-1/2 from v0_i = mix32(i)/2^32 - 1/2) (Z27);
//   4. P = T - diag(w / a_ii) (A T) (smoothed aggregation, Z27), R = P^T, A_{l+1} = P^T (A P)
//      (Galerkin, Z32) -- each sparse product is expanded into (row, col, value) triples in a
//      fixed order, radix-sorted by (row, col) (stable), and equal keys are summed sequentially in
//      expansion order: deterministic, no floating-point atomics.  Exact zeros produced by the
//      products are dropped (as a sparse product does);
//   5. the coarsest matrix is inverted densely by Gauss-Jordan elimination (SPD: no pivoting).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <type_traits>

#include "ldu_amg.cuh"
#include "ldu_kernels.cuh"

namespace ldu {

namespace {

constexpr int kSB = 256;
constexpr unsigned long long kInfKey = ~0ULL;

int nblk(long long n) {
  long long b = (n + kSB - 1) / kSB;
  return (int)std::max(1LL, std::min(b, 148LL * 64));
}

#define GSTRIDE(i, n)                                                                 \
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)(n); \
       i += (long long)gridDim.x * blockDim.x)

// Setup memory.  The setup allocates and frees tens of GB of temporaries level after level, all
// on one in-order stream.  Measured on B200 (profiles/r02_amg/malloc_probe.txt): growing the
// stream-ordered pool (cudaMallocAsync beyond its reserve) costs 6-17 ms per GB with spikes to
// 200 ms, and trimming it as much again, while a plain cudaMalloc of 3 GB takes ~1 ms.  So inside
// amg_setup a ScratchCache hands out cudaMalloc'd blocks and takes them back when a Scratch goes
// out of scope: a later request on the same stream reuses a free block (safe: every earlier user
// of the block is ordered before it on s).  It is also the AllocHook for the setup's dmalloc /
// dfree: the previous hierarchy's buffers (amg_setup releases it under the hook) and the
// intermediate products the setup frees become reusable blocks, and outputs may take one
// (ownership passes to the hierarchy).  Whatever is left is freed at the end.  Outside a cache
// (single-stage test entry points) Scratch uses the stream-ordered pool.
struct ScratchCache : AllocHook {
  std::multimap<size_t, void*> avail;  // free blocks by size
  std::set<void*> owned;               // every block the cache owns (free or lent to a Scratch)
  static size_t granule(size_t bytes) {
    return (bytes + (2u << 20) - 1) & ~(size_t)((2u << 20) - 1);  // 2 MB granules
  }
  void* find(size_t bytes) {
    auto it = avail.lower_bound(bytes);
    if (it == avail.end() || it->first > 2 * bytes + (8u << 20)) return nullptr;
    void* q = it->second;
    avail.erase(it);
    return q;
  }
  void* get(size_t bytes) {  // lent to a Scratch, returned by put
    bytes = granule(bytes);
    if (void* q = find(bytes)) return q;
    void* q = nullptr;
    try {
      q = dmalloc_raw(bytes);
    } catch (const Error&) {  // device full: free the idle blocks and retry once
      trim();
      q = dmalloc_raw(bytes);
    }
    owned.insert(q);
    return q;
  }
  void put(void* q) { avail.emplace(alloc_size(q), q); }
  void* take(size_t bytes) override {  // an output: ownership passes to the caller
    void* q = find(bytes);
    if (q) owned.erase(q);
    return q;
  }
  bool give(void* p, size_t bytes) override {
    if (!owned.insert(p).second) return true;  // already cached (a repeated free): keep one entry
    avail.emplace(bytes, p);
    return true;
  }
  void trim() {
    cudaDeviceSynchronize();
    for (auto& kv : avail) {
      owned.erase(kv.second);
      dfree_raw(kv.second);
    }
    avail.clear();
  }
  void release(cudaStream_t s) {
    cudaStreamSynchronize(s);
    for (void* q : owned) dfree_raw(q);
    owned.clear();
    avail.clear();
  }
};
thread_local ScratchCache* g_scratch = nullptr;

struct ScratchScope {  // installs a cache (and the dmalloc / dfree hook) for one setup
  ScratchCache c;
  ScratchCache* prev;
  AllocHook* prevHook;
  cudaStream_t s;
  explicit ScratchScope(cudaStream_t st) : prev(g_scratch), prevHook(alloc_hook()), s(st) {
    g_scratch = &c;
    alloc_hook() = &c;
  }
  ~ScratchScope() {
    g_scratch = prev;
    alloc_hook() = prevHook;
    c.release(s);
  }
};

struct Scratch {
  cudaStream_t s;
  ScratchCache* cache;
  std::vector<void*> p;
  explicit Scratch(cudaStream_t st) : s(st), cache(g_scratch) {}
  template <class T>
  T* get(size_t n) {
    void* q = nullptr;
    const size_t bytes = std::max<size_t>(1, n) * sizeof(T);
    if (cache) {
      q = cache->get(bytes);
    } else if (cudaMallocAsync(&q, bytes, s) != cudaSuccess) {
      cudaGetLastError();
      throw Error(LDU_ERR_OOM, "cudaMallocAsync of " + std::to_string(bytes) + " bytes failed");
    }
    p.push_back(q);
    return static_cast<T*>(q);
  }
  ~Scratch() {
    for (void* q : p) {
      if (cache) cache->put(q);
      else cudaFreeAsync(q, s);
    }
  }
};

template <class T>
T d2h(const T* d, cudaStream_t s) {
  T v;
  CUDA_CHECK(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  return v;
}

// exclusive scan of in[0..n) into out[0..n] (out[n] = total)
template <class T>
void exclusive_scan(const T* in, T* out, long long n, cudaStream_t s) {
  Scratch sc(s);
  T* tmp = sc.get<T>(n + 1);
  CUDA_CHECK(cudaMemsetAsync(tmp + n, 0, sizeof(T), s));
  if (n) CUDA_CHECK(cudaMemcpyAsync(tmp, in, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
  size_t bytes = 0;
  CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, tmp, out, n + 1, s));
  void* ws = sc.get<char>(bytes);
  CUDA_CHECK(cub::DeviceScan::ExclusiveSum(ws, bytes, tmp, out, n + 1, s));
}

// lanes per row of the CSR-vector kernels: one trip of kCsrU entries per lane covers an average
// row (kCsrU = 4 for one lane per row, 8 otherwise; ldu_amg_solve.cuh)
double env_double(const char* name, double dflt) {
  const char* e = std::getenv(name);
  return e ? std::atof(e) : dflt;
}

int group_of(long long nnz, int rows) {
  static const double per = env_double("LDU_AMG_LANE_ENTRIES", 16.0);  // measured: 8 -> 16 -1.5 %
  const double avg = rows ? (double)nnz / rows : 1.0;
  int g = 1;
  while (g < 32 && (g == 1 ? 4.0 : per * g) < avg) g <<= 1;
  return g;
}

// ---------------------------------------------------------------------------------------------
// sparse assembly: triples (key = row * ncols + col, value) -> CSR, duplicates summed in order
// ---------------------------------------------------------------------------------------------
__global__ void k_seg_sum(long long m, const unsigned long long* __restrict__ key,
                          double* __restrict__ val, long long* __restrict__ keep, int drop) {
  GSTRIDE(k, m) {
    const unsigned long long kk = key[k];
    const bool head = (k == 0) || key[k - 1] != kk;
    long long flag = 0;
    if (head) {
      double s = val[k];
      for (long long t = k + 1; t < m && key[t] == kk; ++t) s += val[t];
      val[k] = s;  // only this thread touches slots [k, next head)
      flag = (!drop || s != 0.0) ? 1 : 0;
    }
    keep[k] = flag;
  }
}

__global__ void k_emit(long long m, int ncols, const unsigned long long* __restrict__ key,
                       const double* __restrict__ val, const long long* __restrict__ keep,
                       const long long* __restrict__ pos, int* __restrict__ col,
                       double* __restrict__ out, int* __restrict__ rowcnt) {
  GSTRIDE(k, m) {
    if (!keep[k]) continue;
    const unsigned long long kk = key[k];
    const long long p = pos[k];
    col[p] = (int)(kk % (unsigned long long)ncols);
    out[p] = val[k];
    atomicAdd(rowcnt + (kk / (unsigned long long)ncols), 1);  // integer: order-independent
  }
}

int bits_for(unsigned long long v) {
  int b = 1;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

// keys / vals [m] are consumed (clobbered).  (A per-row stable segmented sort measured 1.6-4.8x
// slower than this global radix sort at 256^3.)
CsrMat assemble(int nrows, int ncols, long long m, unsigned long long* keys, double* vals,
                bool drop, cudaStream_t s) {
  Scratch sc(s);
  CsrMat out;
  out.nrows = nrows;
  out.ncols = ncols;
  unsigned long long* k2 = sc.get<unsigned long long>(m);
  double* v2 = sc.get<double>(m);
  const int endbit = bits_for((unsigned long long)nrows * (unsigned long long)ncols);
  if (m > 0) {
    size_t bytes = 0;
    CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, k2, vals, v2, m, 0, endbit, s));
    void* ws = sc.get<char>(bytes);
    CUDA_CHECK(cub::DeviceRadixSort::SortPairs(ws, bytes, keys, k2, vals, v2, m, 0, endbit, s));
  }
  long long* keep = sc.get<long long>(m + 1);
  long long* pos = sc.get<long long>(m + 1);
  if (m > 0) k_seg_sum<<<nblk(m), kSB, 0, s>>>(m, k2, v2, keep, drop ? 1 : 0);
  exclusive_scan<long long>(keep, pos, m, s);
  const long long nnz = d2h(pos + m, s);
  if (nnz >= (1LL << 31) - 1) throw Error(LDU_ERR_OOM, "AMG level exceeds 2^31 stored entries");
  out.nnz = nnz;
  out.col = dmalloc<int>(nnz);
  out.val = dmalloc<double>(nnz);
  int* rowcnt = sc.get<int>(nrows + 1);
  CUDA_CHECK(cudaMemsetAsync(rowcnt, 0, sizeof(int) * (nrows + 1), s));
  if (m > 0) k_emit<<<nblk(m), kSB, 0, s>>>(m, ncols, k2, v2, keep, pos, out.col, out.val, rowcnt);
  out.ptr = dmalloc<int>(nrows + 1);
  exclusive_scan<int>(rowcnt, out.ptr, nrows, s);
  CUDA_CHECK(cudaGetLastError());
  out.group = group_of(out.nnz, nrows);
  return out;
}

// expansion entries per chunk of the row-wise assembly (LDU_AMG_CHUNK overrides; tests use tiny
// chunks to check that chunking does not change a single bit)
long long chunk_budget() {
  static long long v = [] {
    const char* e = std::getenv("LDU_AMG_CHUNK");
    const long long b = e ? std::atoll(e) : 0;
    return b > 0 ? b : (1LL << 28);
  }();
  return v;
}

__global__ void k_l2i(long long n, const long long* __restrict__ a, int* __restrict__ b) {
  GSTRIDE(i, n) b[i] = (int)a[i];
}

__global__ void k_ptr_shift(int rows, const int* __restrict__ src, int add, int* __restrict__ dst) {
  GSTRIDE(i, rows) dst[i] = src[i] + add;
}

// Row-wise sparse assembly in chunks of whole rows: count(cnt) writes every row's expansion size;
// fill(r0, r1, off, key, val) writes the triples of rows [r0, r1) with keys (r - r0) * ncols + col
// starting at off[r] - off[r0], in a fixed order.  Rows never straddle chunks and each chunk is
// sorted (stable) and summed on its own, so the result is bitwise the one-shot assembly's while
// the scratch stays bounded by the chunk budget.
template <class Count, class Fill>
CsrMat assemble_rows(int nrows, int ncols, bool drop, cudaStream_t s, Count count, Fill fill) {
  Scratch sc(s);
  long long* cnt = sc.get<long long>(nrows + 1);
  long long* off = sc.get<long long>(nrows + 1);
  count(cnt);
  exclusive_scan<long long>(cnt, off, nrows, s);
  const long long total = d2h(off + nrows, s);
  const long long budget = chunk_budget();
  if (total <= budget) {
    Scratch c(s);
    unsigned long long* key = c.get<unsigned long long>(total);
    double* val = c.get<double>(total);
    fill(0, nrows, off, key, val);
    CUDA_CHECK(cudaGetLastError());
    return assemble(nrows, ncols, total, key, val, drop, s);
  }
  std::vector<CsrMat> pieces;
  std::vector<int> starts;
  try {
    for (int r0 = 0; r0 < nrows;) {
      const long long base = d2h(off + r0, s);
      int lo = r0 + 1, hi = nrows;  // largest r1 with off[r1] - base <= budget (at least r0 + 1)
      while (lo < hi) {
        const int mid = lo + (hi - lo + 1) / 2;
        if (d2h(off + mid, s) - base <= budget) lo = mid;
        else hi = mid - 1;
      }
      const int r1 = lo;
      const long long m = d2h(off + r1, s) - base;
      Scratch c(s);
      unsigned long long* key = c.get<unsigned long long>(m);
      double* val = c.get<double>(m);
      fill(r0, r1, off, key, val);
      CUDA_CHECK(cudaGetLastError());
      pieces.push_back(assemble(r1 - r0, ncols, m, key, val, drop, s));
      starts.push_back(r0);
      r0 = r1;
    }
    CsrMat out;
    out.nrows = nrows;
    out.ncols = ncols;
    for (const CsrMat& pc : pieces) out.nnz += pc.nnz;
    if (out.nnz >= (1LL << 31) - 1) throw Error(LDU_ERR_OOM, "AMG level exceeds 2^31 stored entries");
    out.ptr = dmalloc<int>(nrows + 1);
    out.col = dmalloc<int>(out.nnz);
    out.val = dmalloc<double>(out.nnz);
    long long at = 0;
    for (size_t k = 0; k < pieces.size(); ++k) {
      const CsrMat& pc = pieces[k];
      if (pc.nnz) {
        CUDA_CHECK(cudaMemcpyAsync(out.col + at, pc.col, sizeof(int) * pc.nnz, cudaMemcpyDeviceToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(out.val + at, pc.val, sizeof(double) * pc.nnz, cudaMemcpyDeviceToDevice, s));
      }
      k_ptr_shift<<<nblk(pc.nrows), kSB, 0, s>>>(pc.nrows, pc.ptr, (int)at, out.ptr + starts[k]);
      at += pc.nnz;
    }
    const int last = (int)out.nnz;
    CUDA_CHECK(cudaMemcpyAsync(out.ptr + nrows, &last, sizeof(int), cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    for (CsrMat& pc : pieces) pc.release();
    out.group = group_of(out.nnz, nrows);
    return out;
  } catch (...) {
    for (CsrMat& pc : pieces) pc.release();
    throw;
  }
}

// ---------------------------------------------------------------------------------------------
// level 0: CSR (diag included) from the handle's layout
// ---------------------------------------------------------------------------------------------
// f(j, a) for the off-diagonal entries of row c in ascending column order.  DIA: a coefficient
// that is exactly 0 is not a coupling (reading Z34: the layout stores 0 where there is no face).
template <int ND, class F>
__device__ __forceinline__ void for_row(const DiaView<ND>& A, int c, F f) {
#pragma unroll
  for (int k = ND - 1; k >= 0; --k) {
    const int j = c - A.off[k];
    if (j >= 0) {
      const double a = A.U[k][j];
      if (a != 0.0) f(j, a);
    }
  }
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    const int j = c + A.off[k];
    if (j < A.n) {
      const double a = A.U[k][c];
      if (a != 0.0) f(j, a);
    }
  }
}

template <class F>
__device__ __forceinline__ void for_row(const SellView& A, int c, F f) {
  const int slice = c >> 5, lane = c & 31;
  const long long base = A.slicePtr[slice];
  const int np = A.npairs[slice];
  for (int jj = 0; jj < np; ++jj) {
    const long long e = (base + jj) * 32 + lane;
    const int2 cc = A.col[e];
    const double2 vv = A.val[e];
    if (cc.x < 0) break;
    f(cc.x, vv.x);
    if (cc.y < 0) break;
    f(cc.y, vv.y);
  }
}

// The same visit order for a matrix-vector product: zero DIA coefficients are visited too (they
// add an exact 0), so no load waits on a value test and the row's loads issue together.
template <int ND, class F>
__device__ __forceinline__ void for_row_mv(const DiaView<ND>& A, int c, F f) {
#pragma unroll
  for (int k = ND - 1; k >= 0; --k) {
    const int j = c - A.off[k];
    if (j >= 0) f(j, A.U[k][j]);
  }
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    const int j = c + A.off[k];
    if (j < A.n) f(j, A.U[k][c]);
  }
}
template <class F>
__device__ __forceinline__ void for_row_mv(const SellView& A, int c, F f) {
  for_row(A, c, f);
}

template <class Fmt>
__global__ void k_l0_count(Fmt A, long long* __restrict__ cnt) {
  GSTRIDE(c, A.n) {
    long long k = 1;
    for_row(A, (int)c, [&](int, double) { ++k; });
    cnt[c] = k;
  }
}

template <class Fmt>
__global__ void k_l0_fill(Fmt A, const double* __restrict__ diag, int r0, int r1,
                          const long long* __restrict__ off, unsigned long long* __restrict__ key,
                          double* __restrict__ val) {
  GSTRIDE(cc, r1 - r0) {
    const long long c = r0 + cc;
    long long o = off[c] - off[r0];
    const unsigned long long rowk = (unsigned long long)cc * (unsigned long long)A.n;
    bool diagDone = false;
    for_row(A, (int)c, [&](int j, double a) {
      if (!diagDone && j > c) {
        key[o] = rowk + c;
        val[o++] = diag[c];
        diagDone = true;
      }
      key[o] = rowk + j;
      val[o++] = a;
    });
    if (!diagDone) {
      key[o] = rowk + c;
      val[o] = diag[c];
    }
  }
}

template <class F>
void with_layout(ldu_handle h, F&& f) {
  if (h->layout == LDU_LAYOUT_SELL32) {
    f(SellView{h->n, h->slicePtr, h->npairs, h->col, h->val});
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

// DIA rows come out in ascending column order without duplicates: written in place, no sort
template <int ND>
__global__ void k_l0_direct(DiaView<ND> A, const double* __restrict__ diag,
                            const long long* __restrict__ off, int* __restrict__ col,
                            double* __restrict__ val) {
  GSTRIDE(c, A.n) {
    long long o = off[c];
    bool diagDone = false;
    for_row(A, (int)c, [&](int j, double a) {
      if (!diagDone && j > c) {
        col[o] = (int)c;
        val[o++] = diag[c];
        diagDone = true;
      }
      col[o] = j;
      val[o++] = a;
    });
    if (!diagDone) {
      col[o] = (int)c;
      val[o] = diag[c];
    }
  }
}

CsrMat level0_csr(ldu_handle h, cudaStream_t s) {
  const int n = h->n;
  if (h->layout == LDU_LAYOUT_DIA_SYM && !std::getenv("LDU_AMG_SORT_L0")) {
    Scratch sc(s);
    long long* cnt = sc.get<long long>(n + 1);
    long long* off = sc.get<long long>(n + 1);
    CsrMat out;
    with_layout(h, [&](auto A) {
      k_l0_count<<<nblk(n), kSB, 0, s>>>(A, cnt);
      exclusive_scan<long long>(cnt, off, n, s);
      out.nrows = out.ncols = n;
      out.nnz = d2h(off + n, s);
      out.ptr = dmalloc<int>(n + 1);
      out.col = dmalloc<int>(out.nnz);
      out.val = dmalloc<double>(out.nnz);
      k_l2i<<<nblk(n + 1), kSB, 0, s>>>(n + 1, off, out.ptr);
      if constexpr (!std::is_same<decltype(A), SellView>::value)
        k_l0_direct<<<nblk(n), kSB, 0, s>>>(A, h->diag, off, out.col, out.val);
    });
    CUDA_CHECK(cudaGetLastError());
    out.group = group_of(out.nnz, n);
    return out;
  }
  return assemble_rows(
      n, n, false, s,
      [&](long long* cnt) { with_layout(h, [&](auto A) { k_l0_count<<<nblk(n), kSB, 0, s>>>(A, cnt); }); },
      [&](int r0, int r1, const long long* off, unsigned long long* key, double* val) {
        with_layout(h, [&](auto A) {
          k_l0_fill<<<nblk(r1 - r0), kSB, 0, s>>>(A, h->diag, r0, r1, off, key, val);
        });
      });
}

// ---------------------------------------------------------------------------------------------
// distance-2 MIS aggregation (reading Z30)
// ---------------------------------------------------------------------------------------------
__global__ void k_mis_min1(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                           const unsigned char* __restrict__ und, int hashed,
                           unsigned long long* __restrict__ m1) {
  GSTRIDE(i, n) {
    unsigned long long m = und[i] ? amg_key((int)i, hashed) : kInfKey;
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
      const int j = col[k];
      if (j != i && und[j]) m = min(m, amg_key(j, hashed));
    }
    m1[i] = m;
  }
}

__global__ void k_mis_min2(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                           const unsigned char* __restrict__ und, int hashed,
                           const unsigned long long* __restrict__ m1,
                           unsigned char* __restrict__ fresh, unsigned char* __restrict__ root) {
  GSTRIDE(i, n) {
    unsigned long long m = m1[i];
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) m = min(m, m1[col[k]]);
    const bool nr = und[i] && m == amg_key((int)i, hashed);
    fresh[i] = nr ? 1 : 0;
    if (nr) root[i] = 1;
  }
}

// d[i] = src[i] or any src[j] over the neighbours
__global__ void k_mis_spread(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                             const unsigned char* __restrict__ src, unsigned char* __restrict__ d) {
  GSTRIDE(i, n) {
    unsigned char v = src[i];
    for (int k = ptr[i]; k < ptr[i + 1] && !v; ++k) v = src[col[k]];
    d[i] = v;
  }
}

__global__ void k_mis_retire(int n, const unsigned char* __restrict__ d2,
                             unsigned char* __restrict__ und, int* __restrict__ left) {
  int cnt = 0;
  GSTRIDE(i, n) {
    if (und[i] && d2[i]) und[i] = 0;
    cnt += und[i];
  }
  if (cnt) atomicAdd(left, cnt);
}

__global__ void k_root_flags(int n, const unsigned char* __restrict__ root, int* __restrict__ f) {
  GSTRIDE(i, n) f[i] = root[i];
}

// step 3: a1[i] = own aggregate (root) or that of the smallest-key adjacent root, else -1
__global__ void k_agg_step3(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                            const unsigned char* __restrict__ root, const int* __restrict__ rootIdx,
                            int hashed, int* __restrict__ a1) {
  GSTRIDE(i, n) {
    int a = -1;
    if (root[i]) {
      a = rootIdx[i];
    } else {
      unsigned long long best = kInfKey;
      for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
        const int j = col[k];
        if (j != i && root[j]) {
          const unsigned long long kj = amg_key(j, hashed);
          if (kj < best) {
            best = kj;
            a = rootIdx[j];
          }
        }
      }
    }
    a1[i] = a;
  }
}

// step 4: the rest join the aggregate of their smallest-key adjacent step-3 node
__global__ void k_agg_step4(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                            const int* __restrict__ a1, int hashed, int* __restrict__ agg,
                            int* __restrict__ orphan) {
  GSTRIDE(i, n) {
    int a = a1[i];
    if (a < 0) {
      unsigned long long best = kInfKey;
      for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
        const int j = col[k];
        if (j != i && a1[j] >= 0) {
          const unsigned long long kj = amg_key(j, hashed);
          if (kj < best) {
            best = kj;
            a = a1[j];
          }
        }
      }
    }
    agg[i] = a;
    if (a < 0) atomicAdd(orphan, 1);
  }
}

int g_mis_rounds = 0;  // rounds of the last aggregation (LDU_AMG_TRACE)

int mis2_aggregate(const CsrMat& A, int hashed, int* agg, cudaStream_t s) {
  Scratch sc(s);
  const int n = A.nrows;
  unsigned char* und = sc.get<unsigned char>(n);
  unsigned char* root = sc.get<unsigned char>(n);
  unsigned char* fresh = sc.get<unsigned char>(n);
  unsigned char* d1 = sc.get<unsigned char>(n);
  unsigned char* d2 = sc.get<unsigned char>(n);
  unsigned long long* m1 = sc.get<unsigned long long>(n);
  int* left = sc.get<int>(2);
  CUDA_CHECK(cudaMemsetAsync(und, 1, n, s));
  CUDA_CHECK(cudaMemsetAsync(root, 0, n, s));
  for (int round = 0; round <= n; ++round) {
    k_mis_min1<<<nblk(n), kSB, 0, s>>>(n, A.ptr, A.col, und, hashed, m1);
    k_mis_min2<<<nblk(n), kSB, 0, s>>>(n, A.ptr, A.col, und, hashed, m1, fresh, root);
    k_mis_spread<<<nblk(n), kSB, 0, s>>>(n, A.ptr, A.col, fresh, d1);
    k_mis_spread<<<nblk(n), kSB, 0, s>>>(n, A.ptr, A.col, d1, d2);
    CUDA_CHECK(cudaMemsetAsync(left, 0, sizeof(int), s));
    k_mis_retire<<<nblk(n), kSB, 0, s>>>(n, d2, und, left);
    CUDA_CHECK(cudaGetLastError());
    g_mis_rounds = round + 1;
    if (d2h(left, s) == 0) break;
  }
  int* rf = sc.get<int>(n + 1);
  int* ridx = sc.get<int>(n + 1);
  k_root_flags<<<nblk(n), kSB, 0, s>>>(n, root, rf);
  exclusive_scan<int>(rf, ridx, n, s);
  const int nAgg = d2h(ridx + n, s);
  int* a1 = sc.get<int>(n);
  k_agg_step3<<<nblk(n), kSB, 0, s>>>(n, A.ptr, A.col, root, ridx, hashed, a1);
  CUDA_CHECK(cudaMemsetAsync(left + 1, 0, sizeof(int), s));
  k_agg_step4<<<nblk(n), kSB, 0, s>>>(n, A.ptr, A.col, a1, hashed, agg, left + 1);
  CUDA_CHECK(cudaGetLastError());
  if (d2h(left + 1, s) != 0) throw Error(LDU_ERR_STATE, "MIS-2 aggregation left a node unassigned");
  return nAgg;
}

// ---------------------------------------------------------------------------------------------
// Lanczos estimate of rho(D^-1 A) (reading Z27)
// ---------------------------------------------------------------------------------------------
// fixed-order dot products: per-block partials, then one block sums them in index order
template <int NV>
__device__ __forceinline__ void block_store(double (&v)[NV], double* part) {
  __shared__ double sm[NV][32];
  block_reduce<NV>(v, sm);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) part[k * gridDim.x + blockIdx.x] = v[k];
}

__global__ void k_sum_parts(const double* __restrict__ part, int nparts, double* __restrict__ out) {
  __shared__ double sm[1][32];
  double v[1];
  sum_slots<1>(part, nparts, nparts, v);
  block_reduce<1>(v, sm);
  if (threadIdx.x == 0) out[0] = v[0];
}

// v0_i = mix32(i) / 2^32 - 1/2; s_i = 1 / sqrt(a_ii); partial sum v^2
__global__ void k_lz_init(int n, const double* __restrict__ diag, double* __restrict__ v,
                          double* __restrict__ sd, double* part) {
  double a[1] = {0.0};
  GSTRIDE(i, n) {
    const double vi = (double)amg_mix32((unsigned)i) / 4294967296.0 - 0.5;
    v[i] = vi;
    sd[i] = 1.0 / sqrt(diag[i]);
    a[0] += vi * vi;
  }
  block_store<1>(a, part);
}

__global__ void k_lz_scale(int n, double* __restrict__ v, const double* __restrict__ nrm2) {
  const double nr = sqrt(*nrm2);
  GSTRIDE(i, n) v[i] = v[i] / nr;
}

// The Lanczos steps run without a host round trip: lz[0] = stopped (beta_j == 0), lz[1] = the
// number of completed steps m; every kernel of a later step returns at once when stopped.
__global__ void k_lz_sum_ctl(const double* __restrict__ part, int nparts, double* __restrict__ out,
                             const int* lz) {
  if (lz[0]) return;
  __shared__ double sm[1][32];
  double v[1];
  sum_slots<1>(part, nparts, nparts, v);
  block_reduce<1>(v, sm);
  if (threadIdx.x == 0) out[0] = v[0];
}
// beta_j = sqrt((w, w)); the next step's beta; m = j + 1; stop on beta_j == 0
__global__ void k_lz_beta(const double* __restrict__ part, int nparts, double* __restrict__ be_j,
                          double* __restrict__ beta, int* lz, int j) {
  if (lz[0]) return;
  __shared__ double sm[1][32];
  double v[1];
  sum_slots<1>(part, nparts, nparts, v);
  block_reduce<1>(v, sm);
  if (threadIdx.x == 0) {
    const double b = sqrt(v[0]);
    *be_j = b;
    *beta = b;
    lz[1] = j + 1;
    if (b == 0.0) lz[0] = 1;
  }
}

// w = s .* (A (s .* v)) - beta v_prev; partial (w, v)
__global__ void k_lz_matvec(CsrView A, const double* __restrict__ sd, const double* __restrict__ v,
                            const double* __restrict__ vprev, const double* __restrict__ beta,
                            double* __restrict__ w, double* part, const int* lz) {
  if (lz[0]) return;
  const double b = *beta;
  double a[1] = {0.0};
  GSTRIDE(i, A.n) {
    double acc = 0.0;
    for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      const int j = A.col[k];
      acc += A.val[k] * (sd[j] * v[j]);
    }
    const double wi = sd[i] * acc - b * vprev[i];
    w[i] = wi;
    a[0] += wi * v[i];
  }
  block_store<1>(a, part);
}

// the same on a coalesced layout: level 0 the handle's DIA / SELL rows (diagonal first, diag !=
// NULL), coarse levels their SELL-32 copy (diagonal inside the rows, CSR order: the same sums as
// k_lz_matvec)
template <class Fmt>
__global__ void k_lz_matvec_fmt(Fmt A, const double* __restrict__ diag, const double* __restrict__ sd,
                                const double* __restrict__ v, const double* __restrict__ vprev,
                                const double* __restrict__ beta, double* __restrict__ w, double* part,
                                const int* lz) {
  if (lz[0]) return;
  const double b = *beta;
  double a[1] = {0.0};
  GSTRIDE(i, A.n) {
    double acc = diag ? diag[i] * (sd[i] * v[i]) : 0.0;
    for_row_mv(A, (int)i, [&](int j, double aij) { acc += aij * (sd[j] * v[j]); });
    const double wi = sd[i] * acc - b * vprev[i];
    w[i] = wi;
    a[0] += wi * v[i];
  }
  block_store<1>(a, part);
}

// w -= alpha v; partial (w, w)
__global__ void k_lz_orth(int n, double* __restrict__ w, const double* __restrict__ v,
                          const double* __restrict__ alpha, double* part, const int* lz) {
  if (lz[0]) return;
  const double al = *alpha;
  double a[1] = {0.0};
  GSTRIDE(i, n) {
    const double wi = w[i] - al * v[i];
    w[i] = wi;
    a[0] += wi * wi;
  }
  block_store<1>(a, part);
}

// v_prev = v; v = w / beta
__global__ void k_lz_next(int n, double* __restrict__ vprev, double* __restrict__ v,
                          const double* __restrict__ w, const double* __restrict__ beta,
                          const int* lz) {
  if (lz[0]) return;
  const double b = *beta;
  GSTRIDE(i, n) {
    vprev[i] = v[i];
    v[i] = w[i] / b;
  }
}


// largest eigenvalue of the symmetric tridiagonal (alpha[0..m), beta[0..m-1)) by bisection on
// the Sturm count; then w = (4/3) / (1.05 lambda) (reading Z27)
__global__ void k_tridiag_max(const int* __restrict__ lz, const double* __restrict__ al,
                              const double* __restrict__ be, double* __restrict__ out) {
  if (threadIdx.x || blockIdx.x) return;
  const int m = lz[1];
  double lo = al[0], hi = al[0];
  for (int i = 0; i < m; ++i) {
    const double r = (i > 0 ? fabs(be[i - 1]) : 0.0) + (i + 1 < m ? fabs(be[i]) : 0.0);
    lo = fmin(lo, al[i] - r);
    hi = fmax(hi, al[i] + r);
  }
  // count(x) = number of eigenvalues < x
  auto count = [&](double x) {
    int c = 0;
    double d = al[0] - x;
    if (d < 0) ++c;
    for (int i = 1; i < m; ++i) {
      if (d == 0.0) d = 1e-300;
      d = al[i] - x - be[i - 1] * be[i - 1] / d;
      if (d < 0) ++c;
    }
    return c;
  };
  double a = lo, b = hi;  // invariant: count(a) < m, count(b) == m (largest eigenvalue in [a, b])
  b = hi + fabs(hi) * 1e-15 + 1e-300;
  for (int it = 0; it < 400; ++it) {
    const double mid = 0.5 * (a + b);
    if (mid <= a || mid >= b) break;
    if (count(mid) == m) b = mid;
    else a = mid;
  }
  const double lam = 0.5 * (a + b);
  out[0] = lam;
  out[1] = (4.0 / 3.0) / (1.05 * lam);
}

double lanczos_omega(const CsrMat& A, const double* diag, int steps, cudaStream_t s,
                     double* ritzOut, ldu_handle h0 = nullptr) {
  Scratch sc(s);
  const int n = A.nrows;
  const int G = nblk(n);
  double* v = sc.get<double>(n);
  double* vp = sc.get<double>(n);
  double* w = sc.get<double>(n);
  double* sd = sc.get<double>(n);
  double* part = sc.get<double>(G);
  const int ms = std::min(steps, n);
  double* al = sc.get<double>(ms + 1);
  double* be = sc.get<double>(ms + 1);
  double* scal = sc.get<double>(4);  // [0] |v|^2, [1] beta (current), [2..3] result
  k_lz_init<<<G, kSB, 0, s>>>(n, diag, v, sd, part);
  k_sum_parts<<<1, kSB, 0, s>>>(part, G, scal);
  k_lz_scale<<<G, kSB, 0, s>>>(n, v, scal);
  CUDA_CHECK(cudaMemsetAsync(vp, 0, sizeof(double) * n, s));
  CUDA_CHECK(cudaMemsetAsync(scal + 1, 0, sizeof(double), s));
  int* lz = sc.get<int>(2);
  CUDA_CHECK(cudaMemsetAsync(lz, 0, 2 * sizeof(int), s));
  for (int j = 0; j < ms; ++j) {  // enqueued without a host round trip (stop flag on the device)
    if (h0)  // level 0: the handle's layout instead of the assembled CSR (same operator)
      with_layout(h0, [&](auto L) {
        k_lz_matvec_fmt<<<G, kSB, 0, s>>>(L, diag, sd, v, vp, scal + 1, w, part, lz);
      });
    else if (A.useSell)
      k_lz_matvec_fmt<<<G, kSB, 0, s>>>(sell_view(A), (const double*)nullptr, sd, v, vp, scal + 1,
                                         w, part, lz);
    else
      k_lz_matvec<<<G, kSB, 0, s>>>(view(A), sd, v, vp, scal + 1, w, part, lz);
    k_lz_sum_ctl<<<1, kSB, 0, s>>>(part, G, al + j, lz);
    k_lz_orth<<<G, kSB, 0, s>>>(n, w, v, al + j, part, lz);
    k_lz_beta<<<1, kSB, 0, s>>>(part, G, be + j, scal + 1, lz, j);
    CUDA_CHECK(cudaGetLastError());
    if (j == ms - 1) break;
    k_lz_next<<<G, kSB, 0, s>>>(n, vp, v, w, be + j, lz);
  }
  k_tridiag_max<<<1, 1, 0, s>>>(lz, al, be, scal + 2);
  CUDA_CHECK(cudaGetLastError());
  double res[2];
  CUDA_CHECK(cudaMemcpyAsync(res, scal + 2, sizeof(res), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (ritzOut) *ritzOut = res[0];
  if (!(res[0] > 0.0) || !std::isfinite(res[1]))
    throw Error(LDU_ERR_STATE, "AMG: Lanczos estimate of rho(D^-1 A) is not positive");
  return res[1];
}

// ---------------------------------------------------------------------------------------------
// SELL-32 copy of a CSR for the V-cycle (coarse A_l): slice width = longest row of 32
// ---------------------------------------------------------------------------------------------
__global__ void k_sell_width(int n, const int* __restrict__ ptr, long long* __restrict__ np) {
  GSTRIDE(sl, (n + 31) / 32) {
    int w = 0;
    for (int r = (int)sl * 32; r < min(n, (int)sl * 32 + 32); ++r) w = max(w, ptr[r + 1] - ptr[r]);
    np[sl] = (w + 1) / 2;
  }
}
__global__ void k_l2i_n(long long n, const long long* __restrict__ a, int* __restrict__ b) {
  GSTRIDE(i, n) b[i] = (int)a[i];
}
__global__ void k_sell_fill(CsrView A, const long long* __restrict__ sp, const int* __restrict__ np,
                            int* __restrict__ col, double* __restrict__ val) {
  GSTRIDE(r, A.n) {
    const long long sl = r >> 5, lane = r & 31;
    const int b = A.ptr[r], e = A.ptr[r + 1];
    for (int jj = 0; jj < np[sl]; ++jj) {
      const long long slot = ((sp[sl] + jj) * 32 + lane) * 2;
      for (int h = 0; h < 2; ++h) {
        const int k = b + 2 * jj + h;
        // padding: coefficient 0 on a column the row already references (a valid index of the
        // operand even for rectangular P / R; no other row's value can leak in as 0 * NaN)
        col[slot + h] = k < e ? A.col[k] : (e > b ? A.col[b] : 0);
        val[slot + h] = k < e ? A.val[k] : 0.0;
      }
    }
  }
}

// Attach a SELL-32 copy when its padded slots stay within maxPad x the CSR entries.
void attach_sell(CsrMat& M, double maxPad, cudaStream_t s) {
  // one row per thread needs enough rows to fill the GPU; small levels stay CSR-vector
  if (M.nrows < 65536 || M.nnz <= 0) return;
  Scratch sc(s);
  const long long ns = (M.nrows + 31) / 32;
  long long* np = sc.get<long long>(ns + 1);
  long long* sp = dmalloc<long long>(ns + 1);
  k_sell_width<<<nblk(ns), kSB, 0, s>>>(M.nrows, M.ptr, np);
  exclusive_scan<long long>(np, sp, ns, s);
  const long long pairs = d2h(sp + ns, s);
  if ((double)pairs * 64.0 > maxPad * (double)M.nnz) {
    dfree(sp);
    return;
  }
  M.slicePtr = sp;
  M.npairs = dmalloc<int>(ns);
  k_l2i_n<<<nblk(ns), kSB, 0, s>>>(ns, np, M.npairs);
  M.sellSlots = pairs * 32;
  M.scol = dmalloc<int2>(M.sellSlots);
  M.sval = dmalloc<double2>(M.sellSlots);
  k_sell_fill<<<nblk(M.nrows), kSB, 0, s>>>(view(M), sp, M.npairs, (int*)M.scol, (double*)M.sval);
  CUDA_CHECK(cudaGetLastError());
  M.useSell = true;
}

// ---------------------------------------------------------------------------------------------
// prolongator, restriction, Galerkin product
// ---------------------------------------------------------------------------------------------
__global__ void k_diag_of(CsrView A, double* __restrict__ diag, double* __restrict__ rD,
                          int* __restrict__ bad) {
  GSTRIDE(i, A.n) {
    double d = 0.0;
    for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
      if (A.col[k] == i) d += A.val[k];
    diag[i] = d;
    rD[i] = 1.0 / d;
    if (!(d > 0.0) || !isfinite(d)) atomicAdd(bad, 1);
  }
}

// S = A T expansion (smoothed): row i, key (i, agg[j]) in A's column order
__global__ void k_count_row(CsrView A, long long* __restrict__ cnt) {
  GSTRIDE(i, A.n) cnt[i] = A.ptr[i + 1] - A.ptr[i];
}
__global__ void k_expand_AT(CsrView A, int nAgg, const int* __restrict__ agg, int r0, int r1,
                            const long long* __restrict__ off, unsigned long long* __restrict__ key,
                            double* __restrict__ val) {
  GSTRIDE(ii, r1 - r0) {
    const long long i = r0 + ii;
    const unsigned long long rk = (unsigned long long)ii * nAgg;
    long long o = off[i] - off[r0];
    for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      key[o] = rk + agg[A.col[k]];
      val[o++] = A.val[k];
    }
  }
}

__global__ void k_expand_T(int n, int nAgg, const int* __restrict__ agg,
                           unsigned long long* __restrict__ key, double* __restrict__ val) {
  GSTRIDE(i, n) {
    key[i] = (unsigned long long)i * nAgg + agg[i];
    val[i] = 1.0;
  }
}

// P_iJ = T_iJ - (w / a_ii) S_iJ   (oracle: T - diags(w / A.diagonal()) @ (A @ T))
__global__ void k_finish_P(CsrView S, const int* __restrict__ agg, const double* __restrict__ diag,
                           double omega, double* __restrict__ val, int* __restrict__ zeros) {
  GSTRIDE(i, S.n) {
    const double f = omega / diag[i];
    int z = 0;
    for (int k = S.ptr[i]; k < S.ptr[i + 1]; ++k) {
      const double t = (S.col[k] == agg[i]) ? 1.0 : 0.0;
      const double p = t - __dmul_rn(f, S.val[k]);  // two roundings, as T - (w/a_ii) S
      val[k] = p;
      z += (p == 0.0);
    }
    if (z) atomicAdd(zeros, z);
  }
}

// drop exact zeros of a CSR in place (rare; only called when some exist)
__global__ void k_nz_count(CsrView A, long long* __restrict__ cnt) {
  GSTRIDE(i, A.n) {
    long long c = 0;
    for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) c += (A.val[k] != 0.0);
    cnt[i] = c;
  }
}
__global__ void k_nz_copy(CsrView A, const long long* __restrict__ off, int* __restrict__ col,
                          double* __restrict__ val) {
  GSTRIDE(i, A.n) {
    long long o = off[i];
    for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
      if (A.val[k] != 0.0) {
        col[o] = A.col[k];
        val[o++] = A.val[k];
      }
  }
}

void drop_zeros(CsrMat& A, cudaStream_t s) {
  Scratch sc(s);
  long long* cnt = sc.get<long long>(A.nrows + 1);
  long long* off = sc.get<long long>(A.nrows + 1);
  k_nz_count<<<nblk(A.nrows), kSB, 0, s>>>(view(A), cnt);
  exclusive_scan<long long>(cnt, off, A.nrows, s);
  const long long nnz = d2h(off + A.nrows, s);
  int* col = dmalloc<int>(nnz);
  double* val = dmalloc<double>(nnz);
  k_nz_copy<<<nblk(A.nrows), kSB, 0, s>>>(view(A), off, col, val);
  int* ptr = dmalloc<int>(A.nrows + 1);
  k_l2i<<<nblk(A.nrows + 1), kSB, 0, s>>>(A.nrows + 1, off, ptr);
  CUDA_CHECK(cudaGetLastError());
  CUDA_CHECK(cudaStreamSynchronize(s));
  A.release();
  A.ptr = ptr;
  A.col = col;
  A.val = val;
  A.nnz = nnz;
  A.group = group_of(nnz, A.nrows);
}

// transpose expansion: P entry (i, J, p) -> key (J, i)
__global__ void k_expand_T_of(CsrView P, int nrowsT, unsigned long long* __restrict__ key,
                              double* __restrict__ val) {
  GSTRIDE(i, P.n) {
    for (int k = P.ptr[i]; k < P.ptr[i + 1]; ++k) {
      key[k] = (unsigned long long)P.col[k] * (unsigned long long)P.n + i;
      val[k] = P.val[k];
    }
  }
}

// expansion sizes of A P: row i -> sum over A's entries (i, j) of |P_j|
__global__ void k_count_AP(CsrView A, const int* __restrict__ Pptr, long long* __restrict__ cnt) {
  GSTRIDE(i, A.n) {
    long long c = 0;
    for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      const int j = A.col[k];
      c += Pptr[j + 1] - Pptr[j];
    }
    cnt[i] = c;
  }
}
__global__ void k_expand_AP(CsrView A, CsrView P, int ncols, int r0, int r1,
                            const long long* __restrict__ off, unsigned long long* __restrict__ key,
                            double* __restrict__ val) {
  GSTRIDE(ii, r1 - r0) {
    const long long i = r0 + ii;
    long long o = off[i] - off[r0];
    const unsigned long long rk = (unsigned long long)ii * ncols;
    for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      const int j = A.col[k];
      const double a = A.val[k];
      for (int t = P.ptr[j]; t < P.ptr[j + 1]; ++t) {
        key[o] = rk + P.col[t];
        val[o++] = a * P.val[t];
      }
    }
  }
}

// A_c = R (A P), row-wise over coarse rows I: (I, J) += R_Ii (AP)_iJ, i ascending then J.  For a
// given (I, J) the contributions come in ascending i -- the same order as expanding P^T (A P) by
// fine rows, so the sums are the same bitwise.
__global__ void k_count_RAP(CsrView R, const int* __restrict__ Qptr, long long* __restrict__ cnt) {
  GSTRIDE(I, R.n) {
    long long c = 0;
    for (int t = R.ptr[I]; t < R.ptr[I + 1]; ++t) {
      const int i = R.col[t];
      c += Qptr[i + 1] - Qptr[i];
    }
    cnt[I] = c;
  }
}
__global__ void k_expand_RAP(CsrView R, CsrView Q, int nc, int r0, int r1,
                             const long long* __restrict__ off, unsigned long long* __restrict__ key,
                             double* __restrict__ val) {
  GSTRIDE(II, r1 - r0) {
    const long long I = r0 + II;
    long long o = off[I] - off[r0];
    const unsigned long long rk = (unsigned long long)II * nc;
    for (int t = R.ptr[I]; t < R.ptr[I + 1]; ++t) {
      const int i = R.col[t];
      const double rv = R.val[t];
      for (int u = Q.ptr[i]; u < Q.ptr[i + 1]; ++u) {
        key[o] = rk + Q.col[u];
        val[o++] = rv * Q.val[u];
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Row-wise SpGEMM C = A B with a per-warp hash accumulator (one warp per output row).
// Row I of C is accumulated in the expansion order of the sort-based assembly (A's entries t
// ascending, then B_j's entries ascending): the warp walks A's row entry by entry; the lanes take
// the entries of B_j (distinct columns, so every accumulator slot gets at most one addend per
// step) and __syncwarp orders the steps -- each C_IJ is the same sequential sum, bit for bit, as
// assemble()'s stable radix sort + segmented sum, without expanding or sorting the products.
// A row with more than CAP distinct columns overflows: the caller retries with a larger CAP,
// then falls back to the sort path.
// ---------------------------------------------------------------------------------------------
struct PhaseTrace;
void sub_mark(const char* what);
constexpr int kGemmWarps = 4;   // warps per block (CAP = 512: 32 KB of shared memory)

struct BCsr {  // B as CSR
  CsrView m;
  __device__ __forceinline__ int begin(int j) const { return __ldg(m.ptr + j); }
  __device__ __forceinline__ int end(int j) const { return __ldg(m.ptr + j + 1); }
  __device__ __forceinline__ int col(int u, int) const { return __ldg(m.col + u); }
  __device__ __forceinline__ double val(int u) const { return __ldg(m.val + u); }
};
struct BAgg {  // B = T, the aggregate indicator: row j = {(agg[j], 1)}
  const int* __restrict__ agg;
  __device__ __forceinline__ int begin(int j) const { return j; }
  __device__ __forceinline__ int end(int j) const { return j + 1; }
  __device__ __forceinline__ int col(int u, int) const { return __ldg(agg + u); }
  __device__ __forceinline__ double val(int) const { return 1.0; }
};

// WRITE = false: cnt[I] = number of (non-zero, when drop) entries of row I; *overflow set when a
// row does not fit.  WRITE = true: the row's entries in ascending column order at ptr[I].
// G lanes per output row (32 / G rows per warp, each group with its own CAP-slot table).
template <class B, bool WRITE, int CAP, int G>
__global__ void __launch_bounds__(kGemmWarps * 32) k_spgemm_rows(CsrView A, B b, int drop,
                                                                 int* __restrict__ cnt,
                                                                 const int* __restrict__ ptr,
                                                                 int* __restrict__ ocol,
                                                                 double* __restrict__ oval,
                                                                 int* __restrict__ overflow) {
  static_assert((CAP & (CAP - 1)) == 0 && CAP >= G, "CAP: a power of two >= G");
  static_assert(G == 4 || G == 8 || G == 16 || G == 32, "G: 4, 8, 16 or 32 lanes per row");
  constexpr int LOG2 = CAP == 16 ? 4 : CAP == 32 ? 5 : CAP == 64 ? 6 : CAP == 128 ? 7 : CAP == 256 ? 8 : 9;
  constexpr int RPW = 32 / G;  // rows per warp
  __shared__ int keys[kGemmWarps * RPW][CAP];
  __shared__ double acc[kGemmWarps * RPW][CAP];
  __shared__ int lst[kGemmWarps * RPW][CAP];
  const int lane = threadIdx.x & 31, sub = lane % G, grp = (threadIdx.x >> 5) * RPW + lane / G;
  const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u) << ((lane / G) * G));
  int* K = keys[grp];
  double* V = acc[grp];
  int* L = lst[grp];
  const int rowsPerPass = gridDim.x * kGemmWarps * RPW;
  const int first = (blockIdx.x * kGemmWarps + (threadIdx.x >> 5)) * RPW + lane / G;
  const int trips = (A.n + rowsPerPass - 1) / rowsPerPass;  // group-uniform trip count
  for (int trip = 0; trip < trips; ++trip) {
    const int I = first + trip * rowsPerPass;
    const bool live = I < A.n;
    for (int q = sub; q < CAP; q += G) {
      K[q] = -1;
      V[q] = 0.0;
    }
    __syncwarp(gmask);
    bool full = false;
    const int t0 = live ? __ldg(A.ptr + I) : 0, t1 = live ? __ldg(A.ptr + I + 1) : 0;
    for (int tb = t0; tb < t1; tb += G) {  // A's entries G at a time: one load round trip
      const int tl = tb + sub;
      int jl = 0, bl = 0, el = 0;
      double al = 0.0;
      if (tl < t1) {
        jl = __ldg(A.col + tl);
        al = __ldg(A.val + tl);
        bl = b.begin(jl);
        el = b.end(jl);
      }
      const int tn = min(G, t1 - tb);
      for (int q = 0; q < tn; ++q) {  // group-uniform: A's entries in order
        const int j = __shfl_sync(gmask, jl, q, G);
        const double a = __shfl_sync(gmask, al, q, G);
        const int ub = __shfl_sync(gmask, bl, q, G), ue = __shfl_sync(gmask, el, q, G);
        for (int u = ub + sub; u < ue; u += G) {
          const int c = b.col(u, j);
          unsigned h = ((unsigned)c * 2654435761u) >> (32 - LOG2);
          int probes = 0;
          while (true) {
            const int prev = atomicCAS(&K[h], -1, c);
            if (prev == -1 || prev == c) break;
            h = (h + 1) & (CAP - 1);
            if (++probes == CAP) {
              full = true;
              break;
            }
          }
          if (full) break;
          V[h] += a * b.val(u);  // one addend per slot per step (B_j's columns are distinct)
        }
        __syncwarp(gmask);
      }
    }
    if (__any_sync(gmask, full)) {
      if (sub == 0) atomicExch(overflow, 1);
      if (!WRITE && sub == 0 && live) cnt[I] = 0;
      __syncwarp(gmask);
      continue;
    }
    // compact the kept entries (key set, value non-zero when dropping) into L
    int m = 0;
    for (int q0 = 0; q0 < CAP; q0 += G) {
      const int q = q0 + sub;
      const bool keep = K[q] >= 0 && !(drop && V[q] == 0.0);
      const unsigned bal = __ballot_sync(gmask, keep) >> ((lane / G) * G);
      if (keep) L[m + __popc(bal & ((1u << sub) - 1))] = q;
      m += __popc(bal);
    }
    __syncwarp(gmask);
    if (sub == 0 && live && cnt) cnt[I] = m;
    if (!WRITE) {
      __syncwarp(gmask);
      continue;
    }
    if (live) {
      const int base = __ldg(ptr + I);
      for (int e = sub; e < m; e += G) {  // rank by counting: ascending column order
        const int q = L[e], c = K[q];
        int rank = 0;
        for (int f = 0; f < m; ++f) rank += K[L[f]] < c;
        ocol[base + rank] = c;
        oval[base + rank] = V[q];
      }
    }
    __syncwarp(gmask);
  }
}

__global__ void k_i2l(long long n, const int* __restrict__ a, long long* __restrict__ b) {
  GSTRIDE(i, n) b[i] = a[i];
}

// per-row bound of C's row length: min(expansion size, CAP)
template <class B>
__global__ void k_expansion_bound(CsrView A, B b, int cap, long long* __restrict__ ub) {
  GSTRIDE(I, A.n) {
    long long e = 0;
    for (int t = A.ptr[I]; t < A.ptr[I + 1]; ++t) {
      const int j = A.col[t];
      e += b.end(j) - b.begin(j);
    }
    ub[I] = e < cap ? e : cap;
  }
}

// copy row I's cnt[I] entries from the bound-spaced scratch to the packed CSR (a warp per row)
__global__ void k_compact_rows(int rows, const long long* __restrict__ toff, const int* __restrict__ tcol,
                               const double* __restrict__ tval, const int* __restrict__ ptr,
                               int* __restrict__ col, double* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = warp; r < rows; r += nwarps) {
    const long long src = toff[r];
    const int dst = ptr[r], m = ptr[r + 1] - dst;
    for (int e = lane; e < m; e += 32) {
      col[dst + e] = tcol[src + e];
      val[dst + e] = tval[src + e];
    }
  }
}

// C = A B (nrows = A.n, ncols) by k_spgemm_rows in ONE pass: every row's sorted entries go to a
// scratch spaced by the row bound min(expansion, CAP), then are packed; returns false (C
// untouched) when a row overflows CAP
template <class B, int CAP, int G>
bool spgemm_rows_cap(const CsrMat& A, B b, int ncols, bool drop, CsrMat& C, cudaStream_t s) {
  Scratch sc(s);
  const int n = A.nrows;
  // one pass into bound-spaced scratch, then packed.  Narrow rows (A T, A P) were cheaper counted
  // then written in place while the scratch came from the stream-ordered pool (its growth cost
  // dominated); with the cudaMalloc block cache one pass wins for them too (256^3 setup 109-114
  // -> 100-103 ms).  LDU_AMG_GEMM_1PASS_NARROW=0 restores the two passes for narrow rows,
  // LDU_AMG_GEMM_2PASS=1 for all.
  static const bool twoPass = std::getenv("LDU_AMG_GEMM_2PASS") && std::atoi(std::getenv("LDU_AMG_GEMM_2PASS")) != 0;
  static const bool narrow1 = !std::getenv("LDU_AMG_GEMM_1PASS_NARROW") || std::atoi(std::getenv("LDU_AMG_GEMM_1PASS_NARROW")) != 0;
  bool onePass = (G == 32 || narrow1) && !twoPass;
  long long* toff = nullptr;
  int* toff32 = nullptr;
  int* tcol = nullptr;
  double* tval = nullptr;
  if (onePass) {
    long long* ub = sc.get<long long>(n + 1);
    toff = sc.get<long long>(n + 1);
    k_expansion_bound<<<nblk(n), kSB, 0, s>>>(view(A), b, CAP, ub);
    exclusive_scan<long long>(ub, toff, n, s);
    const long long tot = d2h(toff + n, s);
    onePass = tot < (1LL << 31) - 1;  // the kernel writes at int offsets
    if (onePass) {
      tcol = sc.get<int>(std::max(1LL, tot));
      tval = sc.get<double>(std::max(1LL, tot));
      toff32 = sc.get<int>(n + 1);
      k_l2i<<<nblk(n + 1), kSB, 0, s>>>(n + 1, toff, toff32);
    }
  }
  int* cnt = sc.get<int>(n + 1);
  int* ovf = sc.get<int>(1);
  CUDA_CHECK(cudaMemsetAsync(ovf, 0, sizeof(int), s));
  constexpr int rpb = kGemmWarps * (32 / G);
  const int grid = (int)std::max(1LL, std::min<long long>((n + rpb - 1) / rpb, 148LL * 16));
  if (onePass)
    k_spgemm_rows<B, true, CAP, G><<<grid, kGemmWarps * 32, 0, s>>>(view(A), b, drop ? 1 : 0, cnt,
                                                                    toff32, tcol, tval, ovf);
  else
    k_spgemm_rows<B, false, CAP, G><<<grid, kGemmWarps * 32, 0, s>>>(view(A), b, drop ? 1 : 0, cnt,
                                                                     nullptr, nullptr, nullptr, ovf);
  CUDA_CHECK(cudaGetLastError());
  sub_mark("gemm rows");
  if (d2h(ovf, s)) return false;
  long long* cl = sc.get<long long>(n + 1);
  long long* off64 = sc.get<long long>(n + 1);
  k_i2l<<<nblk(n), kSB, 0, s>>>(n, cnt, cl);
  exclusive_scan<long long>(cl, off64, n, s);
  const long long nnz = d2h(off64 + n, s);
  if (nnz >= (1LL << 31) - 1) throw Error(LDU_ERR_OOM, "AMG level exceeds 2^31 stored entries");
  C = CsrMat();
  C.nrows = n;
  C.ncols = ncols;
  C.nnz = nnz;
  C.ptr = dmalloc<int>(n + 1);
  C.col = dmalloc<int>(nnz);
  C.val = dmalloc<double>(nnz);
  k_l2i<<<nblk(n + 1), kSB, 0, s>>>(n + 1, off64, C.ptr);
  if (onePass) {
    const int g2 = (int)std::max(1LL, std::min<long long>(((long long)n * 32 + kSB - 1) / kSB, 148LL * 64));
    k_compact_rows<<<g2, kSB, 0, s>>>(n, toff, tcol, tval, C.ptr, C.col, C.val);
  } else {
    k_spgemm_rows<B, true, CAP, G><<<grid, kGemmWarps * 32, 0, s>>>(view(A), b, drop ? 1 : 0,
                                                                    nullptr, C.ptr, C.col, C.val, ovf);
  }
  CUDA_CHECK(cudaGetLastError());
  sub_mark("gemm pack");
  C.group = group_of(C.nnz, n);
  return true;
}

// narrow B rows (the aggregate indicator, P): 4 / 8 lanes per row; wide (A P): a warp per row
template <class B>
bool spgemm_rows(const CsrMat& A, B b, int ncols, bool drop, bool narrow, CsrMat& C, cudaStream_t s) {
  static const bool off = std::getenv("LDU_AMG_SORT_GEMM") && std::atoi(std::getenv("LDU_AMG_SORT_GEMM")) != 0;
  if (off) return false;
  if (narrow)
    return spgemm_rows_cap<B, 32, 4>(A, b, ncols, drop, C, s) ||
           spgemm_rows_cap<B, 64, 8>(A, b, ncols, drop, C, s) ||
           spgemm_rows_cap<B, 256, 32>(A, b, ncols, drop, C, s) ||
           spgemm_rows_cap<B, 512, 32>(A, b, ncols, drop, C, s);
  return spgemm_rows_cap<B, 128, 32>(A, b, ncols, drop, C, s) ||
         spgemm_rows_cap<B, 512, 32>(A, b, ncols, drop, C, s);
}

CsrMat build_P(const CsrMat& A, const int* agg, int nAgg, const double* diag, double omega,
               bool smooth, cudaStream_t s) {
  Scratch sc(s);
  const int n = A.nrows;
  if (!smooth) {
    unsigned long long* key = sc.get<unsigned long long>(n);
    double* val = sc.get<double>(n);
    k_expand_T<<<nblk(n), kSB, 0, s>>>(n, nAgg, agg, key, val);
    return assemble(n, nAgg, n, key, val, false, s);
  }
  CsrMat P;  // S = A T
  if (!spgemm_rows(A, BAgg{agg}, nAgg, false, true, P, s))
    P = assemble_rows(
        n, nAgg, false, s, [&](long long* cnt) { k_count_row<<<nblk(n), kSB, 0, s>>>(view(A), cnt); },
        [&](int r0, int r1, const long long* off, unsigned long long* key, double* val) {
          k_expand_AT<<<nblk(r1 - r0), kSB, 0, s>>>(view(A), nAgg, agg, r0, r1, off, key, val);
        });
  int* zeros = sc.get<int>(1);
  CUDA_CHECK(cudaMemsetAsync(zeros, 0, sizeof(int), s));
  k_finish_P<<<nblk(n), kSB, 0, s>>>(view(P), agg, diag, omega, P.val, zeros);
  CUDA_CHECK(cudaGetLastError());
  if (d2h(zeros, s)) drop_zeros(P, s);
  sub_mark("finish P");
  return P;
}

// Transpose by counting: column counts, scan, scatter through per-column cursors (arbitrary
// order), then every row of the transpose sorted by its (distinct) column indices -- a warp per
// row, rank by counting: deterministic, and equal to the stable-sort transpose.
__global__ void k_col_count(CsrView P, int* __restrict__ cnt) {
  GSTRIDE(i, P.n) for (int k = P.ptr[i]; k < P.ptr[i + 1]; ++k) atomicAdd(cnt + P.col[k], 1);
}
__global__ void k_col_scatter(CsrView P, const int* __restrict__ Rptr, int* __restrict__ cur,
                              int* __restrict__ tcol, double* __restrict__ tval) {
  GSTRIDE(i, P.n) {
    for (int k = P.ptr[i]; k < P.ptr[i + 1]; ++k) {
      const int J = P.col[k];
      const int pos = Rptr[J] + atomicAdd(cur + J, 1);
      tcol[pos] = (int)i;
      tval[pos] = P.val[k];
    }
  }
}
__global__ void k_row_sort(int rows, const int* __restrict__ ptr, const int* __restrict__ tcol,
                           const double* __restrict__ tval, int* __restrict__ col,
                           double* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = warp; r < rows; r += nwarps) {
    const int b = ptr[r], e = ptr[r + 1];
    for (int k = b + lane; k < e; k += 32) {
      const int c = tcol[k];
      int rank = 0;
      for (int f = b; f < e; ++f) rank += tcol[f] < c;
      col[b + rank] = c;
      val[b + rank] = tval[k];
    }
  }
}

CsrMat transpose(const CsrMat& P, cudaStream_t s) {
  static const bool sortPath = std::getenv("LDU_AMG_SORT_GEMM") && std::atoi(std::getenv("LDU_AMG_SORT_GEMM")) != 0;
  if (!sortPath) {
    Scratch sc(s);
    const int nr = P.ncols;
    int* cnt = sc.get<int>(nr + 1);
    int* cur = sc.get<int>(nr + 1);
    CUDA_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int) * (nr + 1), s));
    CUDA_CHECK(cudaMemsetAsync(cur, 0, sizeof(int) * (nr + 1), s));
    k_col_count<<<nblk(P.nrows), kSB, 0, s>>>(view(P), cnt);
    CsrMat R;
    R.nrows = nr;
    R.ncols = P.nrows;
    R.nnz = P.nnz;
    R.ptr = dmalloc<int>(nr + 1);
    exclusive_scan<int>(cnt, R.ptr, nr, s);
    int* tcol = sc.get<int>(std::max(1LL, P.nnz));
    double* tval = sc.get<double>(std::max(1LL, P.nnz));
    k_col_scatter<<<nblk(P.nrows), kSB, 0, s>>>(view(P), R.ptr, cur, tcol, tval);
    R.col = dmalloc<int>(P.nnz);
    R.val = dmalloc<double>(P.nnz);
    const int grid = (int)std::max(1LL, std::min<long long>(((long long)nr * 32 + kSB - 1) / kSB, 148LL * 64));
    k_row_sort<<<grid, kSB, 0, s>>>(nr, R.ptr, tcol, tval, R.col, R.val);
    CUDA_CHECK(cudaGetLastError());
    R.group = group_of(R.nnz, nr);
    sub_mark("transpose");
    return R;
  }
  Scratch sc(s);
  unsigned long long* key = sc.get<unsigned long long>(P.nnz);
  double* val = sc.get<double>(P.nnz);
  k_expand_T_of<<<nblk(P.nrows), kSB, 0, s>>>(view(P), P.ncols, key, val);
  CsrMat R = assemble(P.ncols, P.nrows, P.nnz, key, val, false, s);
  sub_mark("transpose");
  return R;
}

CsrMat galerkin(const CsrMat& A, const CsrMat& P, const CsrMat& R, cudaStream_t s) {
  const int n = A.nrows, nc = P.ncols;
  CsrMat AP;
  if (!spgemm_rows(A, BCsr{view(P)}, nc, true, true, AP, s))
    AP = assemble_rows(
        n, nc, true, s, [&](long long* cnt) { k_count_AP<<<nblk(n), kSB, 0, s>>>(view(A), P.ptr, cnt); },
        [&](int r0, int r1, const long long* off, unsigned long long* key, double* val) {
          k_expand_AP<<<nblk(r1 - r0), kSB, 0, s>>>(view(A), view(P), nc, r0, r1, off, key, val);
        });
  try {
    CsrMat Ac;
    if (!spgemm_rows(R, BCsr{view(AP)}, nc, true, false, Ac, s))
      Ac = assemble_rows(
          nc, nc, true, s,
          [&](long long* cnt) { k_count_RAP<<<nblk(nc), kSB, 0, s>>>(view(R), AP.ptr, cnt); },
          [&](int r0, int r1, const long long* off, unsigned long long* key, double* val) {
            k_expand_RAP<<<nblk(r1 - r0), kSB, 0, s>>>(view(R), view(AP), nc, r0, r1, off, key, val);
          });
    AP.release();
    return Ac;
  } catch (...) {
    AP.release();
    throw;
  }
}

// ---------------------------------------------------------------------------------------------
// coarsest level: dense Gauss-Jordan inverse (SPD, no pivoting; reading Z31)
// ---------------------------------------------------------------------------------------------
__global__ void k_dense_of(CsrView A, double* __restrict__ D, double* __restrict__ I) {
  GSTRIDE(i, A.n) {
    for (int j = 0; j < A.n; ++j) {
      D[i * A.n + j] = 0.0;
      I[i * A.n + j] = (i == j) ? 1.0 : 0.0;
    }
    for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) D[i * A.n + A.col[k]] += A.val[k];
  }
}

__global__ void k_gj_pivot(int n, int k, double* __restrict__ D, double* __restrict__ I,
                           double* __restrict__ fac, int* __restrict__ bad) {
  const double piv = D[(long long)k * n + k];
  if (!(piv > 0.0) || !isfinite(piv)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(bad, 1);
  }
  GSTRIDE(t, n) {
    fac[t] = (t == k) ? 0.0 : D[t * n + k];
  }
  __syncthreads();
  // row k scaled (after every fac read of column k in this grid: separate launch not needed
  // because only row k is written and fac[k] is not read from D)
  GSTRIDE(j, n) {
    D[(long long)k * n + j] /= piv;
    I[(long long)k * n + j] /= piv;
  }
}

__global__ void k_gj_elim(int n, int k, double* __restrict__ D, double* __restrict__ I,
                          const double* __restrict__ fac) {
  GSTRIDE(t, (long long)n * n) {
    const long long i = t / n, j = t % n;
    if (i == k) continue;
    const double f = fac[i];
    D[t] -= f * D[(long long)k * n + j];
    I[t] -= f * I[(long long)k * n + j];
  }
}

double* dense_inverse(const CsrMat& A, cudaStream_t s) {
  Scratch sc(s);
  const int n = A.nrows;
  double* D = sc.get<double>((size_t)n * n);
  double* I = dmalloc<double>((size_t)n * n);
  double* fac = sc.get<double>(n);
  int* bad = sc.get<int>(1);
  CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), s));
  k_dense_of<<<nblk(n), kSB, 0, s>>>(view(A), D, I);
  for (int k = 0; k < n; ++k) {
    // single block: the column-k reads and the row-k writes are ordered by __syncthreads
    k_gj_pivot<<<1, 1024, 0, s>>>(n, k, D, I, fac, bad);
    k_gj_elim<<<nblk((long long)n * n), kSB, 0, s>>>(n, k, D, I, fac);
  }
  CUDA_CHECK(cudaGetLastError());
  if (d2h(bad, s)) {
    dfree(I);
    throw Error(LDU_ERR_STATE, "AMG: coarsest matrix is not positive definite");
  }
  return I;
}

// LDU_AMG_TRACE=1: per-phase host wall times of the setup on stderr (stream synchronised);
// LDU_AMG_TRACE=2 adds the sub-phases of the products (sub_mark)
struct PhaseTrace;
PhaseTrace* g_trace = nullptr;
struct PhaseTrace {
  bool on = false;
  cudaStream_t s = nullptr;
  double t0 = 0;
  static double now() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  PhaseTrace(cudaStream_t st) : s(st) {
    const char* e = std::getenv("LDU_AMG_TRACE");
    on = e && std::atoi(e) != 0;
    t0 = now();
  }
  void mark(const char* what, int level) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const double t = now();
    fprintf(stderr, "[ldu amg setup] level %d %-10s %8.2f ms (mis rounds %d)\n", level, what,
            t - t0, g_mis_rounds);
    t0 = t;
  }
};
void sub_mark(const char* what) {
  static const bool on = std::getenv("LDU_AMG_TRACE") && std::atoi(std::getenv("LDU_AMG_TRACE")) >= 2;
  if (on && g_trace) g_trace->mark(what, -1);
}

void free_level(AmgLevel& L) {
  L.A.release();
  L.P.release();
  L.R.release();
  if (L.ownsDiag) {
    dfree(L.diag);
    dfree(L.rD);
  }
  for (void* p : {(void*)L.agg, (void*)L.r, (void*)L.x, (void*)L.f, (void*)L.z}) dfree(p);
  L = AmgLevel{};
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// public-internal entry points
// ---------------------------------------------------------------------------------------------
void amg_release(ldu_handle h) {
  AmgHierarchy* H = h->amg;
  if (!H) return;
  cudaSetDevice(h->device);
  if (h->own_stream) cudaStreamSynchronize(h->own_stream);
  for (cudaGraphExec_t g : H->graph)
    if (g) cudaGraphExecDestroy(g);
  for (AmgLevel& L : H->lv) free_level(L);
  H->Ac.release();
  DicFactor& D = H->dic;
  for (void* p : {(void*)D.perm, (void*)D.loPtr, (void*)D.loCol, (void*)D.loVal, (void*)D.upPtr,
                  (void*)D.upCol, (void*)D.upVal, (void*)D.rD, (void*)D.flag, (void*)D.ctl,
                  (void*)D.eLoCol, (void*)D.eUpCol, (void*)D.eLoVal, (void*)D.eUpVal,
                  (void*)D.dLevPtr})
    dfree(p);
  for (void* p : {(void*)H->Ainv, (void*)H->fL, (void*)H->zL, (void*)H->u, (void*)H->m,
                  (void*)H->zk, (void*)H->qk})
    dfree(p);
  delete H;
  h->amg = nullptr;
}

void amg_setup(ldu_handle h, const ldu_amg_opts* opts) {
  ldu_amg_opts o{};
  if (opts) o = *opts;
  if (o.reserved[0] || o.reserved[1] || o.reserved[2]) fail_arg("ldu_amg_opts.reserved must be zero");
  if (o.coarsest < 0 || o.maxLevels < 0 || o.lanczosSteps < 0) fail_arg("negative AMG option");
  if (o.keyIndexOrder != 0 && o.keyIndexOrder != 1) fail_arg("keyIndexOrder must be 0 or 1");
  if (o.unsmoothed != 0 && o.unsmoothed != 1) fail_arg("unsmoothed must be 0 or 1");
  if (o.maxLevels > LDU_AMG_MAX_LEVELS) fail_arg("maxLevels > LDU_AMG_MAX_LEVELS");
  if (!o.coarsest) o.coarsest = 64;
  if (!o.maxLevels) o.maxLevels = LDU_AMG_MAX_LEVELS;
  if (!o.lanczosSteps) o.lanczosSteps = 20;
  if (!h->symmetric) fail_arg("AMG requires a symmetric matrix (lower == NULL or lower == upper)");
  // multi-rank: the hierarchy of the rank's local matrix (block-Jacobi, reading Z33)
  cudaStream_t s = h->own_stream;
  // the previous hierarchy's buffers go to the setup's block cache (reused in stream order
  // after one device synchronisation: solves on other streams may still read them)
  ScratchScope scratch(s);
  const bool had = h->amg != nullptr;
  amg_release(h);
  if (had) CUDA_CHECK(cudaDeviceSynchronize());
  cudaMemPool_t pool;
  CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, h->device));
  unsigned long long keep = ~0ULL;  // keep freed scratch mapped for reuse during the build
  CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  if (h->stream != h->own_stream) {
    CUDA_CHECK(cudaEventRecord(h->ev_fork, h->stream));
    CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_fork, 0));
  }
  CUDA_CHECK(cudaEventRecord(h->ev[0], s));
  AmgHierarchy* H = new AmgHierarchy();
  H->opts = o;
  h->amg = H;
  try {
    const int hashed = o.keyIndexOrder ? 0 : 1;
    PhaseTrace tr(s);
    g_trace = &tr;
    CsrMat A = level0_csr(h, s);
    tr.mark("csr0", 0);
    double* diag = h->diag;
    double* rD = h->rD;
    bool owns = false;
    while (A.nrows > o.coarsest && (int)H->lv.size() < o.maxLevels) {
      const int n = A.nrows;
      int* agg = dmalloc<int>(n);
      const int nAgg = mis2_aggregate(A, hashed, agg, s);
      tr.mark("mis2", (int)H->lv.size());
      if (nAgg >= n) {  // no coarsening possible (Z31)
        dfree(agg);
        break;
      }
      AmgLevel L;
      L.n = n;
      L.nc = nAgg;
      L.A = A;
      L.diag = diag;
      L.rD = rD;
      L.ownsDiag = owns;
      L.agg = agg;
      L.omega = lanczos_omega(A, diag, o.lanczosSteps, s, nullptr, H->lv.empty() ? h : nullptr);
      tr.mark("lanczos", (int)H->lv.size());
      L.P = build_P(A, agg, nAgg, diag, L.omega, !o.unsmoothed, s);
      L.R = transpose(L.P, s);
      tr.mark("P,R", (int)H->lv.size());
      CsrMat Ac = galerkin(A, L.P, L.R, s);
      tr.mark("galerkin", (int)H->lv.size());
      L.r = dmalloc<double>(n);
      L.x = dmalloc<double>(n);
      if (!H->lv.empty()) {
        L.f = dmalloc<double>(n);
        L.z = dmalloc<double>(n);
      }
      static const double pad = env_double("LDU_AMG_SELL_PAD", 1.25);
      attach_sell(L.R, pad, s);  // V-cycle copies where rows are near-uniform
      attach_sell(L.P, pad, s);
      attach_sell(Ac, pad, s);
      tr.mark("sell", (int)H->lv.size());
      H->lv.push_back(L);
      // next level's diagonal
      diag = dmalloc<double>(Ac.nrows);
      rD = dmalloc<double>(Ac.nrows);
      owns = true;
      {
        Scratch sc(s);
        int* bad = sc.get<int>(1);
        CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), s));
        k_diag_of<<<nblk(Ac.nrows), kSB, 0, s>>>(view(Ac), diag, rD, bad);
        CUDA_CHECK(cudaGetLastError());
        if (d2h(bad, s)) {
          dfree(diag);
          dfree(rD);
          Ac.release();
          throw Error(LDU_ERR_STATE, "AMG: coarse matrix with a non-positive diagonal");
        }
      }
      A = Ac;
    }
    H->L = (int)H->lv.size();
    H->nc = A.nrows;
    if (H->nc > 8192) {
      A.release();
      if (owns) {
        dfree(diag);
        dfree(rD);
      }
      fail_arg("AMG: coarsest level has " + std::to_string(H->nc) + " rows (> 8192 for the dense solve)");
    }
    H->Ainv = dense_inverse(A, s);
    tr.mark("inverse", H->L);
    H->Ac = A;  // level L (for L == 0 this is the level-0 CSR itself)
    if (owns) {
      dfree(diag);
      dfree(rD);
    }
    if (H->L > 0) {
      H->fL = dmalloc<double>(H->nc);
      H->zL = dmalloc<double>(H->nc);
    }
    CUDA_CHECK(cudaEventRecord(h->ev[1], s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
    H->setupMs = ms;
    CUDA_CHECK(cudaMemPoolTrimTo(pool, 0));  // scratch of the single-stage helpers, if any
  } catch (...) {
    cudaStreamSynchronize(s);
    cudaMemPoolTrimTo(pool, 0);
    amg_release(h);
    throw;
  }
}

void amg_info(ldu_handle h, ldu_amg_info* out) {
  AmgHierarchy* H = h->amg;
  if (!H || H->kind != PREC_AMG) throw Error(LDU_ERR_STATE, "no AMG hierarchy (call ldu_amg_setup)");
  std::memset(out, 0, sizeof(*out));
  out->nLevels = H->L;
  out->coarsestN = H->nc;
  long long bytes = 8LL * H->nc * H->nc, nnz0 = 0, tot = 0;
  for (int l = 0; l < H->L; ++l) {
    const AmgLevel& L = H->lv[l];
    out->n[l] = L.n;
    out->nnzA[l] = L.A.nnz;
    out->nnzP[l] = L.P.nnz;
    out->omega[l] = L.omega;
    tot += L.A.nnz;
    bytes += 12LL * (L.A.nnz + L.P.nnz + L.R.nnz) + 4LL * (2 * L.n + L.nc + 3) + 8LL * 2 * L.n +
             4LL * L.n + (l ? 8LL * 4 * L.n : 0) +
             12LL * (L.A.sellSlots + L.P.sellSlots + L.R.sellSlots);
  }
  out->n[H->L] = H->nc;
  out->nnzA[H->L] = H->Ac.nnz;
  tot += H->Ac.nnz;
  nnz0 = H->L ? H->lv[0].A.nnz : H->Ac.nnz;
  out->operatorComplexity = nnz0 ? (double)tot / nnz0 : 0.0;
  out->setupMs = H->setupMs;
  out->deviceBytes = bytes + 12LL * H->Ac.nnz;
}

void amg_export(ldu_handle h, int level, int which, int* ptr, int* col, double* val) {
  AmgHierarchy* H = h->amg;
  if (!H || H->kind != PREC_AMG) throw Error(LDU_ERR_STATE, "no AMG hierarchy (call ldu_amg_setup)");
  if (which < 0 || which > 2) fail_arg("which must be 0 (A), 1 (P) or 2 (R)");
  const int maxLevel = which == 0 ? H->L : H->L - 1;
  if (level < 0 || level > maxLevel) fail_arg("level out of range");
  const CsrMat& M = which == 0 ? (level == H->L ? H->Ac : H->lv[level].A)
                               : (which == 1 ? H->lv[level].P : H->lv[level].R);
  if (ptr) CUDA_CHECK(cudaMemcpy(ptr, M.ptr, sizeof(int) * (M.nrows + 1), cudaMemcpyDefault));
  if (col) CUDA_CHECK(cudaMemcpy(col, M.col, sizeof(int) * M.nnz, cudaMemcpyDefault));
  if (val) CUDA_CHECK(cudaMemcpy(val, M.val, sizeof(double) * M.nnz, cudaMemcpyDefault));
}

void amg_export_agg(ldu_handle h, int level, int* agg) {
  AmgHierarchy* H = h->amg;
  if (!H || H->kind != PREC_AMG) throw Error(LDU_ERR_STATE, "no AMG hierarchy (call ldu_amg_setup)");
  if (level < 0 || level >= H->L) fail_arg("level out of range");
  if (!agg) fail_arg("agg is NULL");
  CUDA_CHECK(cudaMemcpy(agg, H->lv[level].agg, sizeof(int) * H->lv[level].n, cudaMemcpyDefault));
}

// ---------------------------------------------------------------------------------------------
// DIC preconditioner (readings Z35, Z36)
// ---------------------------------------------------------------------------------------------
namespace {

// D_c = diag_c - sum_{lower l} a_cl^2 / D_l over one level (all lower neighbours are final)
__global__ void k_dic_rD(int beg, int end, const int* __restrict__ perm,
                         const int* __restrict__ ptr, const int* __restrict__ col,
                         const double* __restrict__ val, const double* __restrict__ diag,
                         double* rD, int* bad) {
  for (int k = beg + blockIdx.x * blockDim.x + threadIdx.x; k < end; k += gridDim.x * blockDim.x) {
    const int c = perm[k];
    if (c < 0) continue;
    double d = diag[c];
    for (int j = ptr[k]; j < ptr[k + 1]; ++j) {
      const double a = val[j];
      d -= a * a * rD[col[j]];
    }
    if (!(d > 0.0) || !isfinite(d)) *bad = 1;
    rD[c] = 1.0 / d;
  }
}

}  // namespace

// The level analysis runs once on the host (a single pass in cell order: every lower neighbour
// of a cell has a smaller index); the factor itself (D) is computed on the device level by level.
void dic_setup(ldu_handle h) {
  if (!h->symmetric) fail_arg("DIC requires a symmetric matrix (lower == NULL or lower == upper)");
  amg_release(h);
  cudaStream_t s = h->own_stream;
  if (h->stream != h->own_stream) {
    CUDA_CHECK(cudaEventRecord(h->ev_fork, h->stream));
    CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_fork, 0));
  }
  CUDA_CHECK(cudaEventRecord(h->ev[0], s));
  AmgHierarchy* H = new AmgHierarchy();
  H->kind = PREC_DIC;
  h->amg = H;
  try {
    const int n = h->n;
    CsrMat A = level0_csr(h, s);  // local rows: interfaces dropped (block-Jacobi, Z33 / Z35)
    std::vector<int> ptr(n + 1), col(A.nnz);
    std::vector<double> val(A.nnz);
    CUDA_CHECK(cudaMemcpyAsync(ptr.data(), A.ptr, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaMemcpyAsync(col.data(), A.col, sizeof(int) * A.nnz, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaMemcpyAsync(val.data(), A.val, sizeof(double) * A.nnz, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    A.release();
    // levels (a zero coefficient is not a dependency, Z36)
    std::vector<int> lev(n, 0);
    int nLev = 0;
    long long nnzL = 0, nnzU = 0;
    for (int r = 0; r < n; ++r) {
      int lv = 0;
      for (int j = ptr[r]; j < ptr[r + 1]; ++j)
        if (val[j] != 0.0) {
          if (col[j] < r) {
            lv = std::max(lv, lev[col[j]] + 1);
            ++nnzL;
          } else if (col[j] > r) {
            ++nnzU;
          }
        }
      lev[r] = lv;
      nLev = std::max(nLev, lv + 1);
    }
    DicFactor& D = H->dic;
    D.nLev = nLev;
    D.nnzL = nnzL;
    std::vector<int> cnt(nLev, 0);
    for (int r = 0; r < n; ++r) cnt[lev[r]]++;
    D.levPtr.assign(nLev + 1, 0);
    for (int l = 0; l < nLev; ++l) {
      D.maxLevel = std::max(D.maxLevel, cnt[l]);
      D.levPtr[l + 1] = D.levPtr[l] + (cnt[l] + 31) / 32 * 32;  // warp-aligned levels
    }
    const int nPad = D.levPtr[nLev];
    D.nPad = nPad;
    std::vector<int> perm(nPad, -1), pos(D.levPtr.begin(), D.levPtr.end() - 1);
    for (int r = 0; r < n; ++r) perm[pos[lev[r]]++] = r;  // ascending cell index within a level
    std::vector<int> lp(nPad + 1), lc(nnzL), up(nPad + 1), uc(nnzU);
    std::vector<double> lvv(nnzL), uvv(nnzU);
    long long ol = 0, ou = 0;
    for (int k = 0; k < nPad; ++k) {
      const int r = perm[k];
      lp[k] = (int)ol;
      up[k] = (int)ou;
      if (r < 0) continue;
      for (int j = ptr[r]; j < ptr[r + 1]; ++j) {
        if (val[j] == 0.0) continue;
        if (col[j] < r) {
          lc[ol] = col[j];
          lvv[ol++] = val[j];
        } else if (col[j] > r) {
          uc[ou] = col[j];
          uvv[ou++] = val[j];
        }
      }
    }
    lp[nPad] = (int)ol;
    up[nPad] = (int)ou;
    // ELL copies (position-major) when the rows are short
    // host staging of the ELL copies lives until the final stream synchronisation below (the
    // uploads are stream-ordered on s like every other upload of this setup)
    std::vector<int> ecLo, ecUp;
    std::vector<double> evLo, evUp;
    auto ell = [&](const std::vector<int>& P, const std::vector<int>& C, const std::vector<double>& V,
                   int& w, int*& dc, double*& dv, std::vector<int>& ec, std::vector<double>& ev) {
      int Wmax = 0;
      for (int k = 0; k < nPad; ++k) Wmax = std::max(Wmax, P[k + 1] - P[k]);
      const int W = dic_ell_width(Wmax);
      if (W == 0) {  // no rows, or rows wider than any ELL instantiation: CSR sweeps
        w = Wmax;
        return;
      }
      w = W;
      ec.assign((size_t)W * nPad, -1);
      ev.assign((size_t)W * nPad, 0.0);
      for (int k = 0; k < nPad; ++k)
        for (int j = P[k]; j < P[k + 1]; ++j) {
          ec[(size_t)(j - P[k]) * nPad + k] = C[j];
          ev[(size_t)(j - P[k]) * nPad + k] = V[j];
        }
      dc = dmalloc<int>((size_t)W * nPad);
      dv = dmalloc<double>((size_t)W * nPad);
      CUDA_CHECK(cudaMemcpyAsync(dc, ec.data(), sizeof(int) * ec.size(), cudaMemcpyHostToDevice, s));
      CUDA_CHECK(cudaMemcpyAsync(dv, ev.data(), sizeof(double) * ev.size(), cudaMemcpyHostToDevice, s));
    };
    D.dLevPtr = dmalloc<int>(nLev + 1);
    CUDA_CHECK(cudaMemcpyAsync(D.dLevPtr, D.levPtr.data(), sizeof(int) * (nLev + 1),
                               cudaMemcpyHostToDevice, s));
    ell(lp, lc, lvv, D.wLo, D.eLoCol, D.eLoVal, ecLo, evLo);
    ell(up, uc, uvv, D.wUp, D.eUpCol, D.eUpVal, ecUp, evUp);
    D.perm = dmalloc<int>(nPad);
    D.loPtr = dmalloc<int>(nPad + 1);
    D.loCol = dmalloc<int>(std::max(1LL, nnzL));
    D.loVal = dmalloc<double>(std::max(1LL, nnzL));
    D.upPtr = dmalloc<int>(nPad + 1);
    D.upCol = dmalloc<int>(std::max(1LL, nnzU));
    D.upVal = dmalloc<double>(std::max(1LL, nnzU));
    D.rD = dmalloc<double>(n);
    D.flag = dmalloc<unsigned>(n);
    D.ctl = dmalloc<unsigned>(3);
    CUDA_CHECK(cudaMemsetAsync(D.flag, 0, sizeof(unsigned) * n, s));
    {
      static const unsigned ctl0[3] = {1u, 0u, 0u};
      CUDA_CHECK(cudaMemcpyAsync(D.ctl, ctl0, sizeof(ctl0), cudaMemcpyHostToDevice, s));
    }
    auto up_h2d = [&](void* d, const void* hsrc, size_t bytes) {
      if (bytes) CUDA_CHECK(cudaMemcpyAsync(d, hsrc, bytes, cudaMemcpyHostToDevice, s));
    };
    up_h2d(D.perm, perm.data(), sizeof(int) * nPad);
    up_h2d(D.loPtr, lp.data(), sizeof(int) * (nPad + 1));
    up_h2d(D.loCol, lc.data(), sizeof(int) * nnzL);
    up_h2d(D.loVal, lvv.data(), sizeof(double) * nnzL);
    up_h2d(D.upPtr, up.data(), sizeof(int) * (nPad + 1));
    up_h2d(D.upCol, uc.data(), sizeof(int) * nnzU);
    up_h2d(D.upVal, uvv.data(), sizeof(double) * nnzU);
    {
      Scratch sc(s);
      int* bad = sc.get<int>(1);
      CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), s));
      for (int l = 0; l < nLev; ++l) {
        const int b = D.levPtr[l], e = D.levPtr[l + 1];
        k_dic_rD<<<nblk(e - b), kSB, 0, s>>>(b, e, D.perm, D.loPtr, D.loCol, D.loVal, h->diag,
                                             D.rD, bad);
      }
      CUDA_CHECK(cudaGetLastError());
      if (d2h(bad, s)) throw Error(LDU_ERR_STATE, "DIC: non-positive pivot");
    }
    CUDA_CHECK(cudaEventRecord(h->ev[1], s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
    H->setupMs = ms;
  } catch (...) {
    cudaStreamSynchronize(s);
    amg_release(h);
    throw;
  }
}

void dic_export(ldu_handle h, double* rD, ldu_dic_info* info) {
  AmgHierarchy* H = h->amg;
  if (!H || H->kind != PREC_DIC) throw Error(LDU_ERR_STATE, "no DIC factor (call ldu_dic_setup)");
  if (rD) CUDA_CHECK(cudaMemcpy(rD, H->dic.rD, sizeof(double) * h->n, cudaMemcpyDefault));
  if (info) {
    std::memset(info, 0, sizeof(*info));
    info->nLevels = H->dic.nLev;
    info->widestLevel = H->dic.maxLevel;
    info->lowerEntries = H->dic.nnzL;
    info->setupMs = H->setupMs;
    info->ellWidthLower = H->dic.eLoCol ? H->dic.wLo : 0;
    info->ellWidthUpper = H->dic.eUpCol ? H->dic.wUp : 0;
  }
}

}  // namespace ldu
