// pinned_probe.cu — what does pinning the engine's host ring cost in a fresh
// process (the first load a model server pays)? 144 MiB = 36 x 4 MiB slots.
//   nvcc -O2 -o /tmp/pinned_probe tools/pinned_probe.cu -lpthread && /tmp/pinned_probe
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>

#include <chrono>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const size_t slot = 4u << 20, n = 36, total = slot * n;
  cudaFree(0);  // context up front
  std::vector<void*> p(n);
  double t = now();
  for (size_t i = 0; i < n; ++i) cudaHostAlloc(&p[i], slot, cudaHostAllocPortable);
  printf("{\"probe\": \"36 x cudaHostAlloc 4MiB, one thread\", \"ms\": %.1f}\n", (now() - t) * 1e3);
  for (auto q : p) cudaFreeHost(q);

  t = now();
  {
    std::vector<std::thread> th;
    for (int w = 0; w < 12; ++w)
      th.emplace_back([&, w] {
        for (int k = 0; k < 3; ++k) cudaHostAlloc(&p[w * 3 + k], slot, cudaHostAllocPortable);
      });
    for (auto& x : th) x.join();
  }
  printf("{\"probe\": \"36 x cudaHostAlloc 4MiB, 12 threads\", \"ms\": %.1f}\n", (now() - t) * 1e3);
  for (auto q : p) cudaFreeHost(q);

  void* big = nullptr;
  t = now();
  cudaHostAlloc(&big, total, cudaHostAllocPortable);
  printf("{\"probe\": \"1 x cudaHostAlloc 144MiB\", \"ms\": %.1f}\n", (now() - t) * 1e3);
  cudaFreeHost(big);

  for (int huge = 0; huge < 2; ++huge) {
    t = now();
    void* m = nullptr;
    if (posix_memalign(&m, 2u << 20, total)) return 1;
    if (huge) madvise(m, total, MADV_HUGEPAGE);
    memset(m, 0, total);
    const double t_touch = now() - t;
    cudaError_t e = cudaHostRegister(m, total, cudaHostRegisterPortable);
    printf("{\"probe\": \"memalign 144MiB%s + touch + cudaHostRegister\", \"ms\": %.1f, \"touch_ms\": %.1f, \"ok\": %d}\n",
           huge ? " + MADV_HUGEPAGE" : "", (now() - t) * 1e3, t_touch * 1e3, e == cudaSuccess);
    cudaHostUnregister(m);
    free(m);
  }
  // registration of a huge-page region in 4 MiB pieces from 12 threads
  {
    void* m = nullptr;
    if (posix_memalign(&m, 2u << 20, total)) return 1;
    madvise(m, total, MADV_HUGEPAGE);
    t = now();
    memset(m, 0, total);
    std::vector<std::thread> th;
    for (int w = 0; w < 12; ++w)
      th.emplace_back([&, w] {
        for (int k = 0; k < 3; ++k) cudaHostRegister((char*)m + (w * 3 + k) * slot, slot, cudaHostRegisterPortable);
      });
    for (auto& x : th) x.join();
    printf("{\"probe\": \"hugepage region, 36 x cudaHostRegister 4MiB from 12 threads\", \"ms\": %.1f}\n",
           (now() - t) * 1e3);
    for (size_t i = 0; i < n; ++i) cudaHostUnregister((char*)m + i * slot);
    free(m);
  }
  FILE* f = fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
  char buf[128] = {0};
  if (f) {
    if (!fgets(buf, sizeof buf, f)) buf[0] = 0;
    fclose(f);
  }
  printf("{\"thp\": \"%s\"}\n", strtok(buf, "\n"));
  return 0;
}
