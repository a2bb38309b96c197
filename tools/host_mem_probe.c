/* host_mem_probe.c — host DRAM copy bandwidth (the warm path's third bound:
 * page cache -> pinned slot is a CPU copy, then the DMA reads the slot).
 *   gcc -O2 -pthread tools/host_mem_probe.c -o /tmp/host_mem_probe && /tmp/host_mem_probe */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define PER (256ul << 20)
static char *src[64], *dst[64];
static int reps = 4;

static double now(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + t.tv_nsec * 1e-9;
}
static void* run(void* a) {
  long i = (long)a;
  for (int r = 0; r < reps; ++r) memcpy(dst[i], src[i], PER);
  return NULL;
}
int main(void) {
  int counts[] = {1, 4, 8, 12, 16};
  for (int i = 0; i < 16; ++i) {
    src[i] = aligned_alloc(4096, PER);
    dst[i] = aligned_alloc(4096, PER);
    memset(src[i], i, PER);
    memset(dst[i], 0, PER);
  }
  for (unsigned c = 0; c < sizeof counts / sizeof *counts; ++c) {
    int t = counts[c];
    pthread_t th[64];
    double t0 = now();
    for (long i = 0; i < t; ++i) pthread_create(&th[i], NULL, run, (void*)i);
    for (int i = 0; i < t; ++i) pthread_join(th[i], NULL);
    double dt = now() - t0;
    double copied = (double)t * reps * PER;
    printf("{\"threads\": %d, \"memcpy_GBps\": %.1f, \"dram_traffic_GBps\": %.1f}\n", t, copied / dt / 1e9,
           2 * copied / dt / 1e9);
  }
  return 0;
}
