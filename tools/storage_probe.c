// storage_probe.c — how fast can this box's storage deliver a cold file?
// O_DIRECT reads, (a) T threads of synchronous pread, (b) io_uring rings (one per
// thread) at queue depth Q (raw syscalls, no liburing). Prints one JSON line per config.
//   gcc -O2 -pthread -o /tmp/storage_probe tools/storage_probe.c
//   /tmp/storage_probe FILE... [quick|best]  (reads all FILEs as one job, dropped from the page
//                                             cache before each run; quick: two configs only;
//                                             best: the three configs that usually lead)
#define _GNU_SOURCE
#include <fcntl.h>
#include <linux/io_uring.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <time.h>
#include <unistd.h>

#define MAXF 64
static const char* g_paths[MAXF];
static uint64_t g_sizes[MAXF], g_starts[MAXF];
static int g_nfiles;
static uint64_t g_size, g_chunk;  // g_size: sum of the files' 4 KiB-rounded-down sizes
static atomic_uint_fast64_t g_cursor;

// global offset -> (file, offset); a chunk never crosses a file end (callers clip)
static int locate(uint64_t off, uint64_t* local) {
  int f = 0;
  while (f + 1 < g_nfiles && off >= g_starts[f + 1]) ++f;
  *local = off - g_starts[f];
  return f;
}

static double now(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + t.tv_nsec * 1e-9;
}

static void drop(void) {
  for (int i = 0; i < g_nfiles; ++i) {
    int fd = open(g_paths[i], O_RDONLY);
    fdatasync(fd);
    posix_fadvise(fd, 0, 0, POSIX_FADV_DONTNEED);
    close(fd);
  }
}

// 2 MiB-aligned, transparent-huge-page backed, pre-touched: the engine's ring is
// allocated this way, and O_DIRECT into 4 KiB pages spends its time pinning pages
static void* big_buffer(size_t bytes) {
  void* p = NULL;
  const size_t a = 2u << 20;
  if (posix_memalign(&p, a, (bytes + a - 1) / a * a)) return NULL;
  madvise(p, (bytes + a - 1) / a * a, MADV_HUGEPAGE);
  memset(p, 0, bytes);
  return p;
}

static void* worker(void* arg) {
  (void)arg;
  int fds[MAXF];
  for (int i = 0; i < g_nfiles; ++i) fds[i] = open(g_paths[i], O_RDONLY | O_DIRECT);
  void* buf = big_buffer(g_chunk);
  if (!buf) return NULL;
  for (;;) {
    uint64_t off = atomic_fetch_add(&g_cursor, g_chunk);
    if (off >= g_size) break;
    uint64_t local;
    const int f = locate(off, &local);
    uint64_t n = g_sizes[f] - local < g_chunk ? g_sizes[f] - local : g_chunk;
    if (pread(fds[f], buf, n, local) < 0) break;
  }
  free(buf);
  for (int i = 0; i < g_nfiles; ++i) close(fds[i]);
  return NULL;
}

static void threads(int t, uint64_t chunk) {
  drop();
  g_chunk = chunk;
  atomic_store(&g_cursor, 0);
  pthread_t th[256];
  double t0 = now();
  for (int i = 0; i < t; ++i) pthread_create(&th[i], NULL, worker, NULL);
  for (int i = 0; i < t; ++i) pthread_join(th[i], NULL);
  double dt = now() - t0;
  printf("{\"probe\": \"pread_threads\", \"threads\": %d, \"chunk_mb\": %.2f, \"GBps\": %.3f}\n", t,
         chunk / 1048576.0, g_size / dt / 1e9);
  fflush(stdout);
}

static int uring_setup(unsigned entries, struct io_uring_params* p) {
  return (int)syscall(__NR_io_uring_setup, entries, p);
}
static int uring_enter(int fd, unsigned submit, unsigned wait, unsigned flags) {
  return (int)syscall(__NR_io_uring_enter, fd, submit, wait, flags, NULL, 0);
}

static unsigned g_qd;

// one io_uring ring at depth g_qd; chunks claimed from the shared cursor (several
// threads = several rings, as the engine's cold reader runs)
static void* uring_worker(void* arg) {
  int* failed = (int*)arg;
  struct io_uring_params p;
  memset(&p, 0, sizeof p);
  const unsigned qd = g_qd;
  int rfd = uring_setup(qd, &p);
  if (rfd < 0) {
    *failed = 1;
    return NULL;
  }
  size_t sq_sz = p.sq_off.array + p.sq_entries * sizeof(unsigned);
  size_t cq_sz = p.cq_off.cqes + p.cq_entries * sizeof(struct io_uring_cqe);
  uint8_t* sq = mmap(NULL, sq_sz, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, rfd, IORING_OFF_SQ_RING);
  uint8_t* cq = mmap(NULL, cq_sz, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, rfd, IORING_OFF_CQ_RING);
  struct io_uring_sqe* sqes = mmap(NULL, p.sq_entries * sizeof(struct io_uring_sqe), PROT_READ | PROT_WRITE,
                                   MAP_SHARED | MAP_POPULATE, rfd, IORING_OFF_SQES);
  unsigned* sq_tail = (unsigned*)(sq + p.sq_off.tail);
  unsigned* sq_mask = (unsigned*)(sq + p.sq_off.ring_mask);
  unsigned* sq_array = (unsigned*)(sq + p.sq_off.array);
  unsigned* cq_head = (unsigned*)(cq + p.cq_off.head);
  unsigned* cq_tail = (unsigned*)(cq + p.cq_off.tail);
  unsigned* cq_mask = (unsigned*)(cq + p.cq_off.ring_mask);
  struct io_uring_cqe* cqes = (struct io_uring_cqe*)(cq + p.cq_off.cqes);
  int fds[MAXF];
  for (int i = 0; i < g_nfiles; ++i) fds[i] = open(g_paths[i], O_RDONLY | O_DIRECT);
  uint8_t* bufs = (uint8_t*)big_buffer((size_t)qd * g_chunk);
  if (!bufs) {
    *failed = 1;
    return NULL;
  }
  unsigned free_slots[1024];
  unsigned nfree = qd, inflight = 0;
  int claiming = 1;
  for (unsigned i = 0; i < qd; ++i) free_slots[i] = i;
  while (claiming || inflight) {
    unsigned queued = 0;
    while (claiming && nfree) {
      uint64_t off = atomic_fetch_add(&g_cursor, g_chunk);
      if (off >= g_size) {
        claiming = 0;
        break;
      }
      uint64_t local;
      const int f = locate(off, &local);
      uint64_t n = g_sizes[f] - local < g_chunk ? g_sizes[f] - local : g_chunk;
      unsigned slot = free_slots[--nfree];
      unsigned tail = *sq_tail;
      unsigned idx = tail & *sq_mask;
      struct io_uring_sqe* e = &sqes[idx];
      memset(e, 0, sizeof *e);
      e->opcode = IORING_OP_READ;
      e->fd = fds[f];
      e->addr = (uint64_t)(uintptr_t)(bufs + (size_t)slot * g_chunk);
      e->len = (uint32_t)n;
      e->off = local;
      e->user_data = slot;
      sq_array[idx] = idx;
      __atomic_store_n(sq_tail, tail + 1, __ATOMIC_RELEASE);
      ++queued;
      ++inflight;
    }
    if (!inflight) break;
    if (uring_enter(rfd, queued, 1, IORING_ENTER_GETEVENTS) < 0) {
      *failed = 1;
      break;
    }
    unsigned head = *cq_head;
    while (head != __atomic_load_n(cq_tail, __ATOMIC_ACQUIRE)) {
      struct io_uring_cqe* c = &cqes[head & *cq_mask];
      if (c->res < 0) *failed = 1;
      free_slots[nfree++] = (unsigned)c->user_data;
      --inflight;
      ++head;
    }
    __atomic_store_n(cq_head, head, __ATOMIC_RELEASE);
  }
  for (int i = 0; i < g_nfiles; ++i) close(fds[i]);
  close(rfd);
  free(bufs);
  return NULL;
}

static void uring_threads(int t, unsigned qd, uint64_t chunk) {
  drop();
  g_chunk = chunk;
  g_qd = qd;
  atomic_store(&g_cursor, 0);
  pthread_t th[64];
  int failed[64] = {0};
  double t0 = now();
  for (int i = 0; i < t; ++i) pthread_create(&th[i], NULL, uring_worker, &failed[i]);
  for (int i = 0; i < t; ++i) pthread_join(th[i], NULL);
  double dt = now() - t0;
  int bad = 0;
  for (int i = 0; i < t; ++i) bad |= failed[i];
  if (bad) {
    printf("{\"probe\": \"io_uring\", \"threads\": %d, \"qd\": %u, \"error\": \"io_uring setup or read failed\"}\n", t, qd);
  } else {
    printf("{\"probe\": \"io_uring\", \"threads\": %d, \"qd\": %u, \"chunk_mb\": %.2f, \"GBps\": %.3f}\n", t, qd,
           chunk / 1048576.0, g_size / dt / 1e9);
  }
  fflush(stdout);
}

static void uring(unsigned qd, uint64_t chunk) { uring_threads(1, qd, chunk); }

int main(int argc, char** argv) {
  int quick = 0, best = 0;
  for (int i = 1; i < argc && g_nfiles < MAXF; ++i) {
    if (strcmp(argv[i], "quick") == 0) {
      quick = 1;
      continue;
    }
    if (strcmp(argv[i], "best") == 0) {
      best = 1;
      continue;
    }
    struct stat st;
    if (stat(argv[i], &st)) return 2;
    g_paths[g_nfiles] = argv[i];
    g_sizes[g_nfiles] = (uint64_t)st.st_size & ~4095ull;
    g_starts[g_nfiles] = g_size;
    g_size += g_sizes[g_nfiles++];
  }
  if (!g_nfiles) return 2;
  if (quick) {
    threads(64, 4 << 20);
    uring(64, 1 << 20);
    return 0;
  }
  if (best) {  // the configs that led the full sweep on these boxes, again (bench.py: after the cold leg)
    uring(32, 1 << 20);
    uring_threads(2, 16, 1 << 20);
    threads(64, 1 << 20);
    return 0;
  }
  threads(16, 16 << 20);
  threads(32, 4 << 20);
  threads(48, 4 << 20);
  threads(32, 8 << 20);
  threads(64, 1 << 20);
  threads(64, 4 << 20);
  uring(32, 1 << 20);
  uring(64, 1 << 20);
  uring(64, 2 << 20);
  uring(128, 1 << 20);
  uring(128, 512 << 10);
  uring(64, 4 << 20);
  uring_threads(2, 16, 1 << 20);  // the engine's cold reader: 2 rings x 16 x 1 MiB
  uring_threads(4, 8, 1 << 20);
  return 0;
}
