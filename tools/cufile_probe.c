/* cufile_probe.c — does cuFile (compat mode, no nvidia-fs) work on this box?
 * Times cuFileDriverOpen / HandleRegister / cuFileRead of N MiB into HBM.
 *   gcc -O2 -I/usr/local/cuda/include tools/cufile_probe.c -o /tmp/cufile_probe \
 *       -L/usr/local/cuda/lib64 -lcufile -lcudart && /tmp/cufile_probe FILE MiB */
#define _GNU_SOURCE
#include <cuda_runtime.h>
#include <cufile.h>
#include <fcntl.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>
#include <unistd.h>

static double now(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + t.tv_nsec * 1e-9;
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  size_t n = (size_t)atoi(argv[2]) << 20;
  cudaFree(0);
  double t = now();
  CUfileError_t e = cuFileDriverOpen();
  printf("driver_open err=%d cu=%d %.3f s\n", e.err, e.cu_err, now() - t);
  fflush(stdout);
  int fd = open(argv[1], O_RDONLY | O_DIRECT);
  if (fd < 0) fd = open(argv[1], O_RDONLY);
  CUfileDescr_t d = {0};
  d.handle.fd = fd;
  d.type = CU_FILE_HANDLE_TYPE_OPAQUE_FD;
  CUfileHandle_t h;
  t = now();
  e = cuFileHandleRegister(&h, &d);
  printf("handle_register err=%d %.3f s\n", e.err, now() - t);
  fflush(stdout);
  void* dev;
  cudaMalloc(&dev, n);
  for (int bufreg = 0; bufreg < 2; ++bufreg) {
    if (bufreg) {
      e = cuFileBufRegister(dev, n, 0);
      printf("buf_register err=%d\n", e.err);
    }
    t = now();
    ssize_t r = cuFileRead(h, dev, n, 0, 0);
    double dt = now() - t;
    printf("read%s %zd bytes %.3f s %.2f GB/s\n", bufreg ? " (registered buf)" : "", r, dt, r / dt / 1e9);
    fflush(stdout);
  }
  cuFileHandleDeregister(h);
  cuFileDriverClose();
  return 0;
}
