// ldu_api.cu -- the extern "C" boundary of libldu_b200 (include/ldu.h).  Every entry point
// catches all C++ exceptions and CUDA / NCCL failures and turns them into an ldu_status plus a
// thread-local message (ldu_last_error).
#include <cstdio>
#include <cstring>
#include <string>

#include "ldu_amg.cuh"
#include "ldu_impl.cuh"

namespace {
thread_local std::string g_last_error;

void set_error(const std::string& m) { g_last_error = m; }

template <class F>
ldu_status guard(const char* fn, F&& f) {
  try {
    g_last_error.clear();
    return f();
  } catch (const ldu::Error& e) {
    set_error(std::string(fn) + ": " + e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    set_error(std::string(fn) + ": host allocation failed");
    return LDU_ERR_OOM;
  } catch (const std::exception& e) {
    set_error(std::string(fn) + ": " + e.what());
    return LDU_ERR_CUDA;
  }
}

void destroy_handle(ldu_handle h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->own_stream) cudaStreamSynchronize(h->own_stream);
  ldu::amg_release(h);
  ldu::release_work(h);
  ldu::p2p_release(h);
  for (void* p : {(void*)h->U, (void*)h->slicePtr, (void*)h->npairs, (void*)h->col,
                  (void*)h->val, (void*)h->diag, (void*)h->rD, (void*)h->partials,
                  (void*)h->ticket, (void*)h->sums, (void*)h->gsums, (void*)h->st,
                  (void*)h->ifFaceCells, (void*)h->ifCoeffs, (void*)h->sendbuf,
                  (void*)h->recvbuf, (void*)h->ifCell, (void*)h->ifCellPtr, (void*)h->ifFaceIdx,
                  (void*)h->mrTailIf, (void*)h->mrTailMeta})
    ldu::dfree(p);
  if (h->st_host) cudaFreeHost(h->st_host);
  for (cudaEvent_t e : {h->ev[0], h->ev[1], h->ev[2], h->ev[3], h->ev_fork, h->ev_red,
                        h->ev_halo, h->ev_pack})
    if (e) cudaEventDestroy(e);
  for (cudaStream_t s : {h->own_stream, h->red_stream, h->halo_stream})
    if (s) cudaStreamDestroy(s);
  delete h;
}
}  // namespace

namespace ldu {
void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  const ldu_status st = (e == cudaErrorMemoryAllocation) ? LDU_ERR_OOM : LDU_ERR_CUDA;
  throw Error(st, std::string(cudaGetErrorString(e)) + " in " + what + " (" + file + ":" +
                      std::to_string(line) + ")");
}
void check_nccl(ncclResult_t e, const char* what, const char* file, int line) {
  if (e == ncclSuccess) return;
  throw Error(LDU_ERR_NCCL, std::string(ncclGetErrorString(e)) + " in " + what + " (" + file +
                                ":" + std::to_string(line) + ")");
}
}  // namespace ldu

extern "C" {

int ldu_abi_version(void) { return LDU_ABI_VERSION; }

const char* ldu_last_error(void) { return g_last_error.c_str(); }

ldu_status ldu_get_unique_id(void* id128) {
  return guard("ldu_get_unique_id", [&] {
    if (!id128) ldu::fail_arg("id128 is NULL");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    NCCL_CHECK(ncclGetUniqueId(&id));
    std::memcpy(id128, &id, sizeof(id));
    return LDU_OK;
  });
}

ldu_status ldu_comm_init(int rank, int nRanks, const void* id128, int cudaDevice, ldu_comm* out) {
  return guard("ldu_comm_init", [&] {
    if (!id128 || !out) ldu::fail_arg("NULL argument");
    if (nRanks < 1 || rank < 0 || rank >= nRanks) ldu::fail_arg("bad rank / nRanks");
    CUDA_CHECK(cudaSetDevice(cudaDevice));
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ldu_comm c = new ldu_comm_s();
    c->rank = rank;
    c->nRanks = nRanks;
    c->device = cudaDevice;
    ncclResult_t r = ncclCommInitRank(&c->red, nRanks, id, rank);
    if (r != ncclSuccess) {
      delete c;
      NCCL_CHECK(r);
    }
    r = ncclCommSplit(c->red, 0, rank, &c->halo, nullptr);
    if (r != ncclSuccess) {
      ncclCommDestroy(c->red);
      delete c;
      NCCL_CHECK(r);
    }
    *out = c;
    return LDU_OK;
  });
}

ldu_status ldu_comm_init_host(int rank, int nRanks, int cudaDevice, ldu_host_allgather_fn fn,
                              void* ctx, ldu_comm* out) {
  return guard("ldu_comm_init_host", [&] {
    if (!fn || !out) ldu::fail_arg("NULL argument");
    if (nRanks < 1 || rank < 0 || rank >= nRanks) ldu::fail_arg("bad rank / nRanks");
    if (nRanks > 64) ldu::fail_arg("the peer-memory path supports <= 64 ranks");
    CUDA_CHECK(cudaSetDevice(cudaDevice));
    ldu_comm c = new ldu_comm_s();
    c->rank = rank;
    c->nRanks = nRanks;
    c->device = cudaDevice;
    c->hostAllgather = fn;
    c->hostCtx = ctx;
    *out = c;
    return LDU_OK;
  });
}

ldu_status ldu_comm_destroy(ldu_comm c) {
  return guard("ldu_comm_destroy", [&] {
    if (!c) return LDU_OK;
    if (c->halo) ncclCommDestroy(c->halo);
    if (c->red) ncclCommDestroy(c->red);
    delete c;
    return LDU_OK;
  });
}

ldu_status ldu_setup(int nCells, int nFaces, const int* lowerAddr, const int* upperAddr,
                     const double* diag, const double* lower, const double* upper,
                     const ldu_interfaces* interfaces, ldu_handle* out) {
  return guard("ldu_setup", [&] {
    if (!out) ldu::fail_arg("out is NULL");
    *out = nullptr;
    if (nCells <= 0) ldu::fail_arg("nCells must be > 0");
    if (nFaces < 0) ldu::fail_arg("nFaces must be >= 0");
    if (2LL * nFaces >= (1LL << 31)) ldu::fail_arg("2*nFaces must be < 2^31");
    if (!diag) ldu::fail_arg("diag is NULL");
    if (nFaces > 0 && (!lowerAddr || !upperAddr || !upper))
      ldu::fail_arg("lowerAddr / upperAddr / upper is NULL");
    if (interfaces && interfaces->nInterfaces < 0) ldu::fail_arg("nInterfaces < 0");
    ldu_handle h = new ldu_handle_s();
    try {
      if (interfaces && interfaces->comm) {
        h->device = interfaces->comm->device;
        CUDA_CHECK(cudaSetDevice(h->device));
      } else {
        CUDA_CHECK(cudaGetDevice(&h->device));
      }
      h->n = nCells;
      h->nf = nFaces;
      CUDA_CHECK(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
      CUDA_CHECK(cudaStreamCreateWithFlags(&h->red_stream, cudaStreamNonBlocking));
      CUDA_CHECK(cudaStreamCreateWithFlags(&h->halo_stream, cudaStreamNonBlocking));
      // the caller's stream defaults to the legacy default stream (CUDA stream 0, where torch
      // and plain cudaMemcpy work by default): every call orders its work after it and the
      // caller's later work after the call, so device inputs written there are never raced
      h->stream = cudaStreamLegacy;
      for (auto* e : {&h->ev[0], &h->ev[1], &h->ev[2], &h->ev[3]})
        CUDA_CHECK(cudaEventCreate(e));
      for (auto* e : {&h->ev_fork, &h->ev_red, &h->ev_halo, &h->ev_pack})
        CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
      ldu::build_layout(h, lowerAddr, upperAddr, diag, lower, upper, interfaces);
      ldu::configure(h);
    } catch (...) {
      destroy_handle(h);
      throw;
    }
    *out = h;
    return LDU_OK;
  });
}

ldu_status ldu_set_stream(ldu_handle h, void* cudaStream) {
  return guard("ldu_set_stream", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    h->stream = cudaStream ? (cudaStream_t)cudaStream : cudaStreamLegacy;
    return LDU_OK;
  });
}

ldu_status ldu_amul(ldu_handle h, const double* x, double* y) {
  return guard("ldu_amul", [&] {
    if (!h || !x || !y) ldu::fail_arg("NULL argument");
    if ((const void*)x == (const void*)y) ldu::fail_arg("x and y must not alias");
    CUDA_CHECK(cudaSetDevice(h->device));
    ldu::amul(h, x, y);
    return LDU_OK;
  });
}

ldu_status pcg_solve(ldu_handle h, const double* b, double* x, double tol, int maxIter,
                     int* nIter, double* finalRes) {
  return guard("pcg_solve", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    return ldu::solve(h, false, b, x, tol, maxIter, nullptr, nIter, finalRes);
  });
}

ldu_status pipecg_solve(ldu_handle h, const double* b, double* x, double tol, int maxIter,
                        int* nIter, double* finalRes) {
  return guard("pipecg_solve", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    return ldu::solve(h, true, b, x, tol, maxIter, nullptr, nIter, finalRes);
  });
}

ldu_status pcg_solve_ex(ldu_handle h, const double* b, double* x, double tol, int maxIter,
                        const ldu_solve_opts* opts, int* nIter, double* finalRes) {
  return guard("pcg_solve_ex", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    return ldu::solve(h, false, b, x, tol, maxIter, opts, nIter, finalRes);
  });
}

ldu_status pipecg_solve_ex(ldu_handle h, const double* b, double* x, double tol, int maxIter,
                           const ldu_solve_opts* opts, int* nIter, double* finalRes) {
  return guard("pipecg_solve_ex", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    return ldu::solve(h, true, b, x, tol, maxIter, opts, nIter, finalRes);
  });
}

ldu_status ldu_get_residual_history(ldu_handle h, double* hostOut, int cap, int* n) {
  return guard("ldu_get_residual_history", [&] {
    if (!h || !n || (cap > 0 && !hostOut) || cap < 0) ldu::fail_arg("bad argument");
    if (h->histN < 0) throw ldu::Error(LDU_ERR_STATE, "last solve did not record history");
    const int m = std::min(cap, h->histN);
    if (m > 0) CUDA_CHECK(cudaMemcpy(hostOut, h->hist, sizeof(double) * m, cudaMemcpyDeviceToHost));
    *n = m;
    return LDU_OK;
  });
}

ldu_status ldu_get_solve_stats(ldu_handle h, ldu_solve_stats* out) {
  return guard("ldu_get_solve_stats", [&] {
    if (!h || !out) ldu::fail_arg("NULL argument");
    *out = h->stats;
    return LDU_OK;
  });
}

ldu_status ldu_get_info(ldu_handle h, ldu_info* out) {
  return guard("ldu_get_info", [&] {
    if (!h || !out) ldu::fail_arg("NULL argument");
    std::memset(out, 0, sizeof(*out));
    out->layout = h->layout;
    out->nDiagonals = h->nd;
    for (int k = 0; k < h->nd; ++k) out->offsets[k] = h->off[k];
    out->storedEntries = h->storedEntries;
    out->matrixBytes = h->matrixBytes;
    out->nCells = h->n;
    out->nFaces = h->nf;
    out->nInterfaceFaces = h->nIfFaces;
    out->nRanks = h->nRanks;
    out->rank = h->rank;
    out->gridBlocks = h->grid;
    out->blockThreads = h->block;
    out->variant = h->variant;
    out->pipeFused = (h->fusePipe && (!(h->comm && h->comm->nRanks > 1) || h->p2pOn)) ? 1 : 0;
    return LDU_OK;
  });
}

ldu_status ldu_stream_triad(int device, long long n, int reps, double* gbps) {
  return guard("ldu_stream_triad", [&] {
    if (!gbps || n < 2 || reps < 1) ldu::fail_arg("bad argument");
    *gbps = ldu::stream_triad(device, n, reps);
    return LDU_OK;
  });
}

ldu_status ldu_amg_setup(ldu_handle h, const ldu_amg_opts* opts) {
  return guard("ldu_amg_setup", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    ldu::amg_setup(h, opts);
    return LDU_OK;
  });
}

ldu_status ldu_amg_get_info(ldu_handle h, ldu_amg_info* out) {
  return guard("ldu_amg_get_info", [&] {
    if (!h || !out) ldu::fail_arg("NULL argument");
    ldu::amg_info(h, out);
    return LDU_OK;
  });
}

ldu_status ldu_amg_get_matrix(ldu_handle h, int level, int which, int* ptr, int* col, double* val) {
  return guard("ldu_amg_get_matrix", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    ldu::amg_export(h, level, which, ptr, col, val);
    return LDU_OK;
  });
}

ldu_status ldu_amg_get_aggregates(ldu_handle h, int level, int* agg) {
  return guard("ldu_amg_get_aggregates", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    ldu::amg_export_agg(h, level, agg);
    return LDU_OK;
  });
}

ldu_status ldu_amg_vcycle(ldu_handle h, const double* r, double* z) {
  return guard("ldu_amg_vcycle", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    ldu::amg_vcycle(h, r, z, ldu::PREC_AMG);
    return LDU_OK;
  });
}

ldu_status amg_pcg_solve(ldu_handle h, const double* b, double* x, double tol, int maxIter,
                         const ldu_solve_opts* opts, int* nIter, double* finalRes) {
  return guard("amg_pcg_solve", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    return ldu::amg_solve(h, ldu::PREC_AMG, false, b, x, tol, maxIter, opts, nIter, finalRes);
  });
}

ldu_status amg_pipecg_solve(ldu_handle h, const double* b, double* x, double tol, int maxIter,
                            const ldu_solve_opts* opts, int* nIter, double* finalRes) {
  return guard("amg_pipecg_solve", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    return ldu::amg_solve(h, ldu::PREC_AMG, true, b, x, tol, maxIter, opts, nIter, finalRes);
  });
}

ldu_status ldu_dic_setup(ldu_handle h) {
  return guard("ldu_dic_setup", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    ldu::dic_setup(h);
    return LDU_OK;
  });
}

ldu_status ldu_dic_get(ldu_handle h, double* rD, ldu_dic_info* info) {
  return guard("ldu_dic_get", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    ldu::dic_export(h, rD, info);
    return LDU_OK;
  });
}

ldu_status ldu_dic_apply(ldu_handle h, const double* r, double* z) {
  return guard("ldu_dic_apply", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    ldu::amg_vcycle(h, r, z, ldu::PREC_DIC);
    return LDU_OK;
  });
}

ldu_status dic_pcg_solve(ldu_handle h, const double* b, double* x, double tol, int maxIter,
                         const ldu_solve_opts* opts, int* nIter, double* finalRes) {
  return guard("dic_pcg_solve", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    return ldu::amg_solve(h, ldu::PREC_DIC, false, b, x, tol, maxIter, opts, nIter, finalRes);
  });
}

ldu_status dic_pipecg_solve(ldu_handle h, const double* b, double* x, double tol, int maxIter,
                            const ldu_solve_opts* opts, int* nIter, double* finalRes) {
  return guard("dic_pipecg_solve", [&] {
    if (!h) ldu::fail_arg("handle is NULL");
    CUDA_CHECK(cudaSetDevice(h->device));
    return ldu::amg_solve(h, ldu::PREC_DIC, true, b, x, tol, maxIter, opts, nIter, finalRes);
  });
}

ldu_status ldu_destroy(ldu_handle h) {
  return guard("ldu_destroy", [&] {
    destroy_handle(h);
    return LDU_OK;
  });
}

}  // extern "C"
