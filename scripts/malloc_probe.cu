// Probe: latency of cudaMalloc / cudaFree / cudaMallocAsync of GB-sized buffers on this box.
#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
static double now() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
__global__ void touch(char* p, size_t n) { for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 1; }
int main() {
  cudaFree(0);
  size_t sizes[] = {256u << 20, 1ull << 30, 3ull << 30};
  for (size_t sz : sizes) {
    for (int r = 0; r < 6; ++r) {
      double t0 = now(); void* p; cudaMalloc(&p, sz); double t1 = now();
      touch<<<148 * 8, 256>>>((char*)p, sz); cudaDeviceSynchronize(); double t2 = now();
      cudaFree(p); double t3 = now();
      printf("cudaMalloc %5zu MB: malloc %7.2f ms  first-touch %7.2f ms  free %7.2f ms\n", sz >> 20, t1 - t0, t2 - t1, t3 - t2);
    }
  }
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaMemPool_t pool; cudaDeviceGetDefaultMemPool(&pool, 0);
  unsigned long long keep = ~0ULL; cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  for (size_t sz : sizes) {
    for (int r = 0; r < 6; ++r) {
      double t0 = now(); void* p; cudaMallocAsync(&p, sz, s); cudaStreamSynchronize(s); double t1 = now();
      touch<<<148 * 8, 256, 0, s>>>((char*)p, sz); cudaStreamSynchronize(s); double t2 = now();
      cudaFreeAsync(p, s); cudaStreamSynchronize(s); double t3 = now();
      cudaMemPoolTrimTo(pool, 0); double t4 = now();
      printf("pool       %5zu MB: malloc %7.2f ms  first-touch %7.2f ms  free %7.2f ms trim %7.2f ms\n", sz >> 20, t1 - t0, t2 - t1, t3 - t2, t4 - t3);
    }
  }
  return 0;
}
