// hmm_probe.cu — can a kernel read a page-cache-backed mmap of a file directly
// (HMM / pageable memory access), and how fast? One DRAM pass if so.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/build/hmm_probe tools/hmm_probe.cu
//   tools/build/hmm_probe FILE [MB]
#include <cuda_runtime.h>
#include <fcntl.h>
#include <stdio.h>
#include <stdlib.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <chrono>

__global__ void pull(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main(int argc, char** argv) {
  int pma = 0, pmahost = 0, hmm = 0;
  cudaDeviceGetAttribute(&pma, cudaDevAttrPageableMemoryAccess, 0);
  cudaDeviceGetAttribute(&pmahost, cudaDevAttrPageableMemoryAccessUsesHostPageTables, 0);
  cudaDeviceGetAttribute(&hmm, cudaDevAttrConcurrentManagedAccess, 0);
  printf("{\"pageableMemoryAccess\": %d, \"usesHostPageTables\": %d, \"concurrentManagedAccess\": %d}\n", pma, pmahost, hmm);
  if (argc < 2 || !pma) return 0;
  int fd = open(argv[1], O_RDONLY);
  struct stat st;
  fstat(fd, &st);
  size_t bytes = argc > 2 ? (size_t)atol(argv[2]) << 20 : (size_t)st.st_size;
  if (bytes > (size_t)st.st_size) bytes = st.st_size;
  bytes &= ~(size_t)15;
  void* m = mmap(nullptr, bytes, PROT_READ, MAP_SHARED, fd, 0);
  uint4* d;
  cudaMalloc(&d, bytes);
  for (int it = 0; it < 3; ++it) {
    auto t0 = std::chrono::steady_clock::now();
    pull<<<148 * 8, 512>>>((const uint4*)m, d, bytes / 16);
    cudaError_t e = cudaDeviceSynchronize();
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("{\"iter\": %d, \"bytes\": %zu, \"seconds\": %.4f, \"GBps\": %.2f, \"err\": \"%s\"}\n", it, bytes, s,
           bytes / s / 1e9, cudaGetErrorString(e));
    if (e != cudaSuccess) break;
  }
  return 0;
}
