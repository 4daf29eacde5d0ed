// ldu_setup.cu -- one-time conversion of an OpenFOAM lduMatrix (face addressing) into a
// row-gathered, cell-ordered device layout (P:95 converted to CSR, P:206 blames
// lduMatrix's random access and asks for "small, contiguous cache-friendly blocks").
//
// Everything runs on the device: validation, symmetry test, banded (DIA) detection, and for the
// general case a degree histogram -> exclusive scan -> scatter -> per-row sort by (column, face)
// -> SELL-32 pack.  The per-row sort makes the layout independent of atomic arrival order, so
// the layout (and every SpMV) is deterministic.
#include <cub/cub.cuh>

#include <algorithm>
#include <mutex>
#include <unordered_map>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "ldu_impl.cuh"

namespace ldu {

namespace {
std::mutex g_alloc_mu;
std::unordered_map<void*, size_t> g_alloc_sizes;
}  // namespace
AllocHook*& alloc_hook() {
  static thread_local AllocHook* hk = nullptr;
  return hk;
}
void alloc_register(void* p, size_t bytes) {
  std::lock_guard<std::mutex> g(g_alloc_mu);
  g_alloc_sizes[p] = bytes;
}
size_t alloc_unregister(void* p) {
  std::lock_guard<std::mutex> g(g_alloc_mu);
  auto it = g_alloc_sizes.find(p);
  if (it == g_alloc_sizes.end()) return 0;
  const size_t b = it->second;
  g_alloc_sizes.erase(it);
  return b;
}
size_t alloc_size(void* p) {
  std::lock_guard<std::mutex> g(g_alloc_mu);
  auto it = g_alloc_sizes.find(p);
  return it == g_alloc_sizes.end() ? 0 : it->second;
}
void* dmalloc_raw(size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 1;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {  // stream-ordered pool memory may still be mapped: release it, retry once
    cudaGetLastError();
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      cudaDeviceSynchronize();
      cudaMemPoolTrimTo(pool, 0);
      e = cudaMalloc(&p, bytes);
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error(LDU_ERR_OOM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
    }
  }
  alloc_register(p, bytes);
  return p;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

namespace {

constexpr int kSetupBlock = 256;

inline int blocks_for(long long n) {
  long long b = (n + kSetupBlock - 1) / kSetupBlock;
  if (b < 1) b = 1;
  if (b > 65535LL * 32) b = 65535LL * 32;
  return static_cast<int>(b);
}

template <class T>
T* to_device(const T* src, size_t n, cudaStream_t s) {
  T* d = dmalloc<T>(n);
  if (n) CUDA_CHECK(cudaMemcpyAsync(d, src, n * sizeof(T), cudaMemcpyDefault, s));
  return d;
}

// err[0]: first face with an index outside [0,n); err[1]: first face with l == u;
// err[2]: first face with a non-finite coefficient; err[3]: first cell with diag <= 0 / non-finite
__global__ void k_validate(int n, int nf, const int* __restrict__ l, const int* __restrict__ u,
                           const double* __restrict__ up, const double* __restrict__ lo,
                           const double* __restrict__ d, int* err) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nf; i += stride) {
    int li = l[i], ui = u[i];
    if (li < 0 || li >= n || ui < 0 || ui >= n) atomicMin(&err[0], (int)i);
    else if (li == ui) atomicMin(&err[1], (int)i);
    if (!isfinite(up[i]) || (lo && !isfinite(lo[i]))) atomicMin(&err[2], (int)i);
  }
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += stride) {
    double v = d[c];
    if (!(v > 0.0) || !isfinite(v)) atomicMin(&err[3], (int)c);
  }
}

__global__ void k_bits_differ(int nf, const double* __restrict__ a, const double* __restrict__ b,
                              int* flag) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nf; i += stride)
    if (__double_as_longlong(a[i]) != __double_as_longlong(b[i])) *flag = 1;
}

// Collect the distinct |u - l| offsets (at most kMaxDiag).  Reads first, CAS only on a miss.
__global__ void k_offsets(int nf, const int* __restrict__ l, const int* __restrict__ u, int* slots,
                          int* overflow) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nf; i += stride) {
    int d = abs(u[i] - l[i]);
    bool found = false;
    for (int k = 0; k < kMaxDiag && !found; ++k) {
      int v = *((volatile int*)&slots[k]);
      if (v == d) { found = true; break; }
      if (v == 0) {
        int old = atomicCAS(&slots[k], 0, d);
        if (old == 0 || old == d) found = true;
      }
    }
    if (!found) *overflow = 1;
  }
}

// DIA scatter: U[k][min(l,u)] = upper[f]; claim[] detects duplicate faces on one (offset,row).
__global__ void k_dia_scatter(int n, int nf, int nd, const int* __restrict__ offs,
                              const int* __restrict__ l, const int* __restrict__ u,
                              const double* __restrict__ up, double* U, int* claim, int* dup) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nf; i += stride) {
    int a = l[i], b = u[i];
    int lo = min(a, b), d = abs(b - a);
    int k = 0;
    while (k < nd && offs[k] != d) ++k;
    long long idx = (long long)k * n + lo;
    if (atomicExch(&claim[idx], 1) != 0) *dup = 1;
    U[idx] = up[i];
  }
}

__global__ void k_degree(int nf, const int* __restrict__ l, const int* __restrict__ u, int* deg) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nf; i += stride) {
    atomicAdd(&deg[l[i]], 1);
    atomicAdd(&deg[u[i]], 1);
  }
}

// Row c's entries: (u[f], upper[f]) for faces with l[f] == c and (l[f], lower[f]) for faces with
// u[f] == c.  Slot order is arbitrary here; k_sort_rows fixes it.
__global__ void k_scatter(int nf, const int* __restrict__ l, const int* __restrict__ u,
                          const double* __restrict__ up, const double* __restrict__ lo,
                          const long long* __restrict__ rowStart, int* cursor, int* ccol,
                          double* cval, int* cfid) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nf; i += stride) {
    int a = l[i], b = u[i];
    long long s1 = rowStart[a] + atomicAdd(&cursor[a], 1);
    ccol[s1] = b;
    cval[s1] = up[i];
    cfid[s1] = (int)i;
    long long s2 = rowStart[b] + atomicAdd(&cursor[b], 1);
    ccol[s2] = a;
    cval[s2] = lo ? lo[i] : up[i];
    cfid[s2] = (int)i;
  }
}

// Insertion sort of each row by (column, face id): ascending column order = the face-loop order
// for upper-triangular faces (SURVEY App. B check 1), deterministic for duplicates.
__global__ void k_sort_rows(int n, const long long* __restrict__ rowStart, int* ccol, double* cval,
                            int* cfid) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += stride) {
    long long b = rowStart[c], e = rowStart[c + 1];
    for (long long i = b + 1; i < e; ++i) {
      int kc = ccol[i], kf = cfid[i];
      double kv = cval[i];
      long long j = i - 1;
      while (j >= b && (ccol[j] > kc || (ccol[j] == kc && cfid[j] > kf))) {
        ccol[j + 1] = ccol[j];
        cval[j + 1] = cval[j];
        cfid[j + 1] = cfid[j];
        --j;
      }
      ccol[j + 1] = kc;
      cval[j + 1] = kv;
      cfid[j + 1] = kf;
    }
  }
}

__global__ void k_slice_pairs(int n, int nslices, const int* __restrict__ deg, int* npairs) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < nslices; s += stride) {
    int w = 0;
    for (int r = 0; r < 32; ++r) {
      long long c = s * 32 + r;
      if (c < n) w = max(w, deg[c]);
    }
    npairs[s] = (w + 1) / 2;
  }
}

__global__ void k_sell_pack(int n, const long long* __restrict__ rowStart,
                            const int* __restrict__ ccol, const double* __restrict__ cval,
                            const long long* __restrict__ slicePtr, int* col, double* val) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += stride) {
    long long s = c >> 5;
    int lane = (int)(c & 31);
    long long b = rowStart[c], e = rowStart[c + 1];
    for (long long j = 0; j < e - b; ++j) {
      long long idx = ((slicePtr[s] + j / 2) * 32 + lane) * 2 + (j & 1);
      col[idx] = ccol[b + j];
      val[idx] = cval[b + j];
    }
  }
}

__global__ void k_widen(long long n, const int* __restrict__ in, long long* __restrict__ out) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = in[i];
}

__global__ void k_recip(int n, const double* __restrict__ d, double* rD) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += stride)
    rD[c] = 1.0 / d[c];
}

struct TmpFree {
  std::vector<void*> ptrs;
  ~TmpFree() {
    for (void* p : ptrs) dfree(p);
  }
  template <class T>
  T* add(T* p) {
    ptrs.push_back((void*)p);
    return p;
  }
};

}  // namespace

void build_layout(ldu_handle h, const int* l_in, const int* u_in, const double* diag_in,
                  const double* lower_in, const double* upper_in, const ldu_interfaces* ifs) {
  const int n = h->n, nf = h->nf;
  cudaStream_t s = h->own_stream;
  // device-pointer inputs may have been written on the caller's stream (legacy by default)
  CUDA_CHECK(cudaEventRecord(h->ev_fork, h->stream));
  CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_fork, 0));
  TmpFree tmp;

  int* l = nf ? tmp.add(to_device(l_in, nf, s)) : nullptr;
  int* u = nf ? tmp.add(to_device(u_in, nf, s)) : nullptr;
  double* up = nf ? tmp.add(to_device(upper_in, nf, s)) : nullptr;
  double* lo = (nf && lower_in) ? tmp.add(to_device(lower_in, nf, s)) : nullptr;
  h->diag = to_device(diag_in, n, s);
  h->matrixBytes = 16LL * n;

  // ---- validation -----------------------------------------------------------------------
  int* err = tmp.add(dmalloc<int>(4));
  int init_err[4] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MAX};
  CUDA_CHECK(cudaMemcpyAsync(err, init_err, sizeof(init_err), cudaMemcpyHostToDevice, s));
  k_validate<<<blocks_for(std::max(n, nf)), kSetupBlock, 0, s>>>(n, nf, l, u, up, lo, h->diag, err);
  CUDA_CHECK(cudaGetLastError());
  int herr[4];
  CUDA_CHECK(cudaMemcpyAsync(herr, err, sizeof(herr), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (herr[0] != INT32_MAX) fail_arg("face " + std::to_string(herr[0]) + ": lowerAddr/upperAddr outside [0, nCells)");
  if (herr[1] != INT32_MAX) fail_arg("face " + std::to_string(herr[1]) + ": lowerAddr == upperAddr");
  if (herr[2] != INT32_MAX) fail_arg("face " + std::to_string(herr[2]) + ": non-finite coefficient");
  if (herr[3] != INT32_MAX) fail_arg("cell " + std::to_string(herr[3]) + ": diag must be > 0 and finite (Jacobi, reading Z9)");

  // ---- symmetry: lower bitwise equal to upper => treat as symmetric -----------------------
  bool symmetric = (lo == nullptr);
  if (!symmetric) {
    int* flag = tmp.add(dmalloc<int>(1));
    CUDA_CHECK(cudaMemsetAsync(flag, 0, sizeof(int), s));
    k_bits_differ<<<blocks_for(nf), kSetupBlock, 0, s>>>(nf, up, lo, flag);
    int hf = 0;
    CUDA_CHECK(cudaMemcpyAsync(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    symmetric = (hf == 0);
    if (symmetric) lo = nullptr;
  }
  h->symmetric = symmetric;

  // ---- banded symmetric => DIA ------------------------------------------------------------
  bool dia = false;
  const char* force = std::getenv("LDU_LAYOUT");  // "sell": disable the DIA layout (experiments)
  const bool allow_dia = !(force && std::strcmp(force, "sell") == 0);
  if (symmetric && nf > 0 && allow_dia) {
    int* slots = tmp.add(dmalloc<int>(kMaxDiag + 1));
    CUDA_CHECK(cudaMemsetAsync(slots, 0, sizeof(int) * (kMaxDiag + 1), s));
    k_offsets<<<blocks_for(nf), kSetupBlock, 0, s>>>(nf, l, u, slots, slots + kMaxDiag);
    int hs[kMaxDiag + 1];
    CUDA_CHECK(cudaMemcpyAsync(hs, slots, sizeof(hs), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (!hs[kMaxDiag]) {
      std::vector<int> offs;
      for (int k = 0; k < kMaxDiag; ++k)
        if (hs[k]) offs.push_back(hs[k]);
      std::sort(offs.begin(), offs.end());
      long long cap = 0;
      for (int d : offs) cap += (long long)n - d;
      if (!offs.empty() && 2LL * nf >= cap) {  // >= 50% of the band slots are real faces
        int nd = (int)offs.size();
        double* U = dmalloc<double>((size_t)nd * n);
        int* claim = tmp.add(dmalloc<int>((size_t)nd * n + 1));
        int* doffs = tmp.add(dmalloc<int>(nd));
        CUDA_CHECK(cudaMemcpyAsync(doffs, offs.data(), sizeof(int) * nd, cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaMemsetAsync(U, 0, sizeof(double) * (size_t)nd * n, s));
        CUDA_CHECK(cudaMemsetAsync(claim, 0, sizeof(int) * ((size_t)nd * n + 1), s));
        int* dup = claim + (size_t)nd * n;
        k_dia_scatter<<<blocks_for(nf), kSetupBlock, 0, s>>>(n, nf, nd, doffs, l, u, up, U, claim, dup);
        CUDA_CHECK(cudaGetLastError());
        int hdup = 0;
        CUDA_CHECK(cudaMemcpyAsync(&hdup, dup, sizeof(int), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        if (hdup) {
          dfree(U);  // duplicate faces: fall back to the general layout (keeps determinism)
        } else {
          dia = true;
          h->layout = LDU_LAYOUT_DIA_SYM;
          h->nd = nd;
          for (int k = 0; k < nd; ++k) h->off[k] = offs[k];
          h->U = U;
          h->storedEntries = (long long)nd * n;
          h->matrixBytes += 8LL * nd * n;
        }
      }
    }
  }

  // ---- general => SELL-32 -----------------------------------------------------------------
  if (!dia) {
    h->layout = LDU_LAYOUT_SELL32;
    int nslices = (n + 31) / 32;
    int* deg = tmp.add(dmalloc<int>(n + 1));
    CUDA_CHECK(cudaMemsetAsync(deg, 0, sizeof(int) * (n + 1), s));
    if (nf) k_degree<<<blocks_for(nf), kSetupBlock, 0, s>>>(nf, l, u, deg);
    long long* rowStart = tmp.add(dmalloc<long long>(n + 1));
    {  // rowStart = exclusive scan of deg (deg[n] = 0), widened to 64 bit
      long long* it = tmp.add(dmalloc<long long>(n + 1));
      k_widen<<<blocks_for(n + 1), kSetupBlock, 0, s>>>(n + 1, deg, it);
      size_t bytes = 0;
      CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, rowStart, n + 1, s));
      void* ws = tmp.add(dmalloc<char>(bytes));
      CUDA_CHECK(cub::DeviceScan::ExclusiveSum(ws, bytes, it, rowStart, n + 1, s));
    }
    long long nent = 2LL * nf;
    int* ccol = tmp.add(dmalloc<int>(nent));
    double* cval = tmp.add(dmalloc<double>(nent));
    int* cfid = tmp.add(dmalloc<int>(nent));
    int* cursor = tmp.add(dmalloc<int>(n));
    CUDA_CHECK(cudaMemsetAsync(cursor, 0, sizeof(int) * n, s));
    if (nf) {
      k_scatter<<<blocks_for(nf), kSetupBlock, 0, s>>>(nf, l, u, up, lo, rowStart, cursor, ccol, cval, cfid);
      k_sort_rows<<<blocks_for(n), kSetupBlock, 0, s>>>(n, rowStart, ccol, cval, cfid);
    }
    h->npairs = dmalloc<int>(nslices);
    k_slice_pairs<<<blocks_for(nslices), kSetupBlock, 0, s>>>(n, nslices, deg, h->npairs);
    h->slicePtr = dmalloc<long long>(nslices + 1);
    {  // slicePtr = exclusive scan of npairs over nslices + 1 entries (last input 0)
      int* np1 = tmp.add(dmalloc<int>(nslices + 1));
      CUDA_CHECK(cudaMemsetAsync(np1, 0, sizeof(int) * (nslices + 1), s));
      CUDA_CHECK(cudaMemcpyAsync(np1, h->npairs, sizeof(int) * nslices, cudaMemcpyDeviceToDevice, s));
      long long* it = tmp.add(dmalloc<long long>(nslices + 1));
      k_widen<<<blocks_for(nslices + 1), kSetupBlock, 0, s>>>(nslices + 1, np1, it);
      size_t bytes = 0;
      CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, h->slicePtr, nslices + 1, s));
      void* ws = tmp.add(dmalloc<char>(bytes));
      CUDA_CHECK(cub::DeviceScan::ExclusiveSum(ws, bytes, it, h->slicePtr, nslices + 1, s));
    }
    long long totPairs = 0;
    CUDA_CHECK(cudaMemcpyAsync(&totPairs, h->slicePtr + nslices, sizeof(long long), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    h->nPairSlots = totPairs * 32;
    h->col = dmalloc<int2>(h->nPairSlots);
    h->val = dmalloc<double2>(h->nPairSlots);
    CUDA_CHECK(cudaMemsetAsync(h->col, 0xff, sizeof(int2) * h->nPairSlots, s));  // col = -1
    CUDA_CHECK(cudaMemsetAsync(h->val, 0, sizeof(double2) * h->nPairSlots, s));
    if (nf)
      k_sell_pack<<<blocks_for(n), kSetupBlock, 0, s>>>(n, rowStart, ccol, cval, h->slicePtr,
                                                         (int*)h->col, (double*)h->val);
    CUDA_CHECK(cudaGetLastError());
    h->storedEntries = 2 * h->nPairSlots;
    h->matrixBytes += 24LL * h->nPairSlots + 12LL * nslices;
  }

  h->rD = dmalloc<double>(n);
  k_recip<<<blocks_for(n), kSetupBlock, 0, s>>>(n, h->diag, h->rD);
  CUDA_CHECK(cudaGetLastError());

  // ---- processor interfaces (P:79 halo layer) --------------------------------------------
  if (ifs && ifs->nInterfaces > 0) {
    if (!ifs->list) fail_arg("interfaces->list is NULL");
    if (!ifs->comm) fail_arg("interfaces require a comm (ldu_comm_init)");
    h->comm = ifs->comm;
    h->nRanks = ifs->comm->nRanks;
    h->rank = ifs->comm->rank;
    std::vector<int> fc;
    std::vector<double> cf;
    for (int k = 0; k < ifs->nInterfaces; ++k) {
      const ldu_interface& it = ifs->list[k];
      if (it.neighbRank < 0 || it.neighbRank >= h->nRanks || it.neighbRank == h->rank)
        fail_arg("interface " + std::to_string(k) + ": bad neighbRank");
      if (it.nFaces < 0) fail_arg("interface " + std::to_string(k) + ": nFaces < 0");
      if (it.nFaces > 0 && (!it.faceCells || !it.coeffs))
        fail_arg("interface " + std::to_string(k) + ": NULL faceCells/coeffs");
      DevInterface di{it.neighbRank, it.nFaces, (int)fc.size()};
      h->ifaces.push_back(di);
      size_t off = fc.size();
      fc.resize(off + it.nFaces);
      cf.resize(off + it.nFaces);
      if (it.nFaces) {
        CUDA_CHECK(cudaMemcpy(fc.data() + off, it.faceCells, sizeof(int) * it.nFaces, cudaMemcpyDefault));
        CUDA_CHECK(cudaMemcpy(cf.data() + off, it.coeffs, sizeof(double) * it.nFaces, cudaMemcpyDefault));
      }
      for (int i = 0; i < it.nFaces; ++i) {
        if (fc[off + i] < 0 || fc[off + i] >= n)
          fail_arg("interface " + std::to_string(k) + " face " + std::to_string(i) + ": faceCell outside [0, nCells)");
        if (!std::isfinite(cf[off + i]))
          fail_arg("interface " + std::to_string(k) + " face " + std::to_string(i) + ": non-finite coeff");
      }
    }
    h->nIfFaces = (int)fc.size();
    // unique interface cells; contributions in (interface order, face order) = packed order
    std::vector<int> order(h->nIfFaces);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return fc[a] < fc[b]; });
    std::vector<int> cells, ptr;
    for (int i = 0; i < h->nIfFaces; ++i) {
      if (i == 0 || fc[order[i]] != fc[order[i - 1]]) {
        cells.push_back(fc[order[i]]);
        ptr.push_back(i);
      }
    }
    ptr.push_back(h->nIfFaces);
    h->nIfCells = (int)cells.size();
    h->ifFaceCells = to_device(fc.data(), fc.size(), s);
    h->ifCoeffs = to_device(cf.data(), cf.size(), s);
    h->ifCell = to_device(cells.data(), cells.size(), s);
    h->ifCellPtr = to_device(ptr.data(), ptr.size(), s);
    h->ifFaceIdx = to_device(order.data(), order.size(), s);
    h->sendbuf = dmalloc<double>(h->nIfFaces);
    h->recvbuf = dmalloc<double>(h->nIfFaces);
    h->matrixBytes += 12LL * h->nIfFaces;
    // rotation of the multi-rank fused pipelined pass: start right after the interface cell
    // that opens the largest (cyclic) run of interface-free rows, so the rows needing the halo
    // are visited last (z-slabs: the bulk of the slab first, then its two boundary planes)
    {
      const int m = (int)cells.size();
      long long bestLen = -1;
      int bestStart = 0;
      for (int j = 0; j < m; ++j) {
        const long long nxt = (j + 1 < m) ? cells[j + 1] : (long long)cells[0] + n;
        const long long len = nxt - cells[j] - 1;
        if (len > bestLen) {
          bestLen = len;
          bestStart = (cells[j] + 1) % n;
        }
      }
      h->mrGapStart = bestStart;
      h->mrGapLen = (int)std::min<long long>(bestLen, n - bestStart);  // the bulk never wraps
      const int tail = n - h->mrGapLen;
      std::vector<int> tailIf(std::max(1, tail), -1);
      for (int j = 0; j < m; ++j) {
        long long t = (long long)cells[j] - bestStart;
        if (t < 0) t += n;
        if (t < h->mrGapLen || t >= n) throw Error(LDU_ERR_STATE, "internal: interface cell inside the gap");
        tailIf[t - h->mrGapLen] = j;
      }
      h->mrTailIf = to_device(tailIf.data(), tailIf.size(), s);
    }
  } else if (ifs && ifs->comm) {
    h->comm = ifs->comm;
    h->nRanks = ifs->comm->nRanks;
    h->rank = ifs->comm->rank;
  }
  CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace ldu
