// hl_io.cpp — bulk file -> HBM engine (the B200 replacement for the
// reference's execute_plan / transfer_from_file, ref transfer.py:305-389 and
// device.py:238-288).
//
// Data path per chunk (the caller's slot size, 4 MiB from the loader; 2 MiB
// chunks for plans under 2 GiB, 1 MiB for cold plans; 4 KiB aligned):
//
//   storage --pread (O_DIRECT, or buffered when the file is page-cache
//   resident)--> pinned slot (worker-private ring, NUMA-local) --cudaMemcpyAsync
//   on the worker's own stream--> HBM
//
// Every worker owns `slots_per_worker` pinned slots and one CUDA stream, so
// reads of chunk i+1 overlap the DMA of chunk i and several copy streams keep
// the PCIe link full. Chunks are claimed dynamically from one atomic cursor,
// so one large file is read by all workers in parallel (the reference's rule
// of one thread per file leaves a 2-file Llama-7B load with two readers,
// ref transfer.py:197-201). With HL_IO_CUFILE the chunk goes storage -> HBM
// directly through cuFileRead (GPUDirect Storage when nvidia-fs is loaded;
// cuFile's own compat mode otherwise), loaded with dlopen so the library
// has no hard dependency on libcufile.
//
// The ring is one pinned region per context (huge-page backed, first-touched
// on the GPU's NUMA node, see ensure_ring_memory), allocated before the first
// plan's workers start and reused by every later plan; its cost is reported in
// hl_plan_stats.ring_setup_seconds. A plan that is mostly cold (O_DIRECT) is
// read by io_uring threads keeping many O_DIRECT reads in flight over the
// team's slots (uring_loop), or, without io_uring, by a larger team of
// blocking readers (cold_workers) whose extra slots get a second region.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdlib.h>
#include <errno.h>
#include <fcntl.h>
#include <linux/io_uring.h>
#include <pthread.h>
#include <sched.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <sys/sysmacros.h>
#include <sys/uio.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "hl_internal.h"

namespace hl {

static constexpr uint64_t kAlign = 4096;
static inline uint64_t round_down(uint64_t x, uint64_t a) { return x / a * a; }
static inline uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ------------------------------------------------------------------ cuFile (dlopen)
// Minimal mirror of the cufile.h types we use; layouts follow cufile.h 1.14.
struct CUfileError { int err; int cu_err; };
struct CUfileDescr {
  int type;  // CU_FILE_HANDLE_TYPE_OPAQUE_FD = 1
  union { int fd; void* handle; } handle;
  const void* fs_ops;
};
struct CuFileApi {
  bool tried = false, ok = false;
  CUfileError (*driver_open)(void) = nullptr;
  CUfileError (*handle_register)(void**, CUfileDescr*) = nullptr;
  void (*handle_deregister)(void*) = nullptr;
  ssize_t (*read)(void*, void*, size_t, off_t, off_t) = nullptr;
};
static CuFileApi g_cufile;
static std::mutex g_cufile_mu;

static bool cufile_load(std::string* why) {
  std::lock_guard<std::mutex> g(g_cufile_mu);
  if (g_cufile.tried) {
    if (!g_cufile.ok && why) *why = "libcufile unavailable or cuFileDriverOpen failed";
    return g_cufile.ok;
  }
  g_cufile.tried = true;
  void* h = dlopen("libcufile.so.0", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libcufile.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    if (why) *why = std::string("dlopen libcufile: ") + dlerror();
    return false;
  }
  g_cufile.driver_open = (CUfileError(*)(void))dlsym(h, "cuFileDriverOpen");
  g_cufile.handle_register = (CUfileError(*)(void**, CUfileDescr*))dlsym(h, "cuFileHandleRegister");
  g_cufile.handle_deregister = (void (*)(void*))dlsym(h, "cuFileHandleDeregister");
  g_cufile.read = (ssize_t(*)(void*, void*, size_t, off_t, off_t))dlsym(h, "cuFileRead");
  if (!g_cufile.driver_open || !g_cufile.handle_register || !g_cufile.read) {
    if (why) *why = "libcufile lacks the expected symbols";
    return false;
  }
  CUfileError e = g_cufile.driver_open();
  if (e.err != 0) {
    if (why) *why = "cuFileDriverOpen failed (code " + std::to_string(e.err) + ")";
    return false;
  }
  g_cufile.ok = true;
  return true;
}

// ------------------------------------------------------------------ topology
// sysfs is read under $HL_SYSFS_ROOT when set (tests build a fake multi-node
// tree there); the NUMA node of the engine is, in order: the caller's
// hl_config.numa_node, $HL_NUMA_NODE, the GPU's PCI node.
static std::string sysfs_path(const char* rel) {
  const char* root = getenv("HL_SYSFS_ROOT");
  return std::string(root ? root : "") + rel;
}

static int pci_numa_node(const char* bus_id) {
  std::string bus(bus_id ? bus_id : "");
  for (auto& ch : bus) ch = (char)tolower(ch);
  char rel[160];
  snprintf(rel, sizeof rel, "/sys/bus/pci/devices/%s/numa_node", bus.c_str());
  FILE* f = fopen(sysfs_path(rel).c_str(), "r");
  if (!f) return -1;
  int node = -1;
  if (fscanf(f, "%d", &node) != 1) node = -1;
  fclose(f);
  return node;
}

// The node's CPUs (sysfs cpulist) that this process may run on; empty = no pinning.
static std::vector<int> node_cpus(int node) {
  std::vector<int> cpus;
  if (node < 0) return cpus;
  char rel[128];
  snprintf(rel, sizeof rel, "/sys/devices/system/node/node%d/cpulist", node);
  FILE* f = fopen(sysfs_path(rel).c_str(), "r");
  if (!f) return cpus;
  char buf[4096];
  if (fgets(buf, sizeof buf, f)) {
    char* save = nullptr;
    for (char* tok = strtok_r(buf, ",\n", &save); tok; tok = strtok_r(nullptr, ",\n", &save)) {
      int a, b;
      if (sscanf(tok, "%d-%d", &a, &b) == 2) {
        for (int c = a; c <= b; ++c) cpus.push_back(c);
      } else if (sscanf(tok, "%d", &a) == 1) {
        cpus.push_back(a);
      }
    }
  }
  fclose(f);
  cpu_set_t allowed;
  CPU_ZERO(&allowed);
  if (sched_getaffinity(0, sizeof allowed, &allowed) == 0) {
    std::vector<int> ok;
    for (int c : cpus)
      if (c >= 0 && c < CPU_SETSIZE && CPU_ISSET(c, &allowed)) ok.push_back(c);
    cpus.swap(ok);
  }
  return cpus;
}

static int resolve_node(const char* bus_id, int requested) {
  if (requested >= 0) return requested;
  if (const char* e = getenv("HL_NUMA_NODE")) {
    char* end = nullptr;
    long v = strtol(e, &end, 10);
    if (end != e && v >= 0) return (int)v;
  }
  return pci_numa_node(bus_id);
}

// NUMA node of the storage device holding `path`: /sys/dev/block/MAJ:MIN resolves
// into the device tree; the nearest ancestor with a numa_node file (the NVMe /
// virtio / HBA PCI function) names it. -1 when unknown (tmpfs, overlay, no sysfs).
static int storage_numa_node(const char* path) {
  struct stat st;
  if (!path || stat(path, &st) != 0) return -1;
  char rel[64];
  snprintf(rel, sizeof rel, "/sys/dev/block/%u:%u", major(st.st_dev), minor(st.st_dev));
  char real[4096];
  if (!realpath(sysfs_path(rel).c_str(), real)) return -1;
  const char* root = getenv("HL_SYSFS_ROOT");
  char rroot[4096] = "";
  if (root && !realpath(root, rroot)) return -1;
  const size_t stop = strlen(rroot) + strlen("/sys/devices");
  std::string d(real);
  while (d.size() > stop) {
    FILE* f = fopen((d + "/numa_node").c_str(), "r");
    if (f) {
      int node = -1;
      const bool ok = fscanf(f, "%d", &node) == 1;
      fclose(f);
      if (ok) return node;
    }
    const size_t cut = d.find_last_of('/');
    if (cut == std::string::npos || cut == 0) break;
    d.resize(cut);
  }
  return -1;
}

static void pin_to(const std::vector<int>& cpus) {
  if (cpus.empty()) return;
  cpu_set_t set;
  CPU_ZERO(&set);
  for (int c : cpus) CPU_SET(c, &set);
  sched_setaffinity(0, sizeof set, &set);
}

}  // namespace hl

using namespace hl;

struct Slot {
  uint8_t* host = nullptr;
  cudaEvent_t ev = nullptr;
  bool busy = false;
  void* reg = nullptr;  // HL_IO_MMAP: page-cache range pinned for the in-flight DMA
};
struct WorkerRing {
  std::vector<Slot> slots;
  cudaStream_t stream = nullptr;
  cudaEvent_t tail = nullptr;  // hl_execute_plan_async: this worker's last copy of the plan
  size_t next = 0;
};

struct hl_ctx {
  hl_config cfg{};
  std::vector<int> cpus;
  std::vector<WorkerRing> rings;
  bool ring_ready = false;
  uint64_t slot_bytes = 0;
  // Pinned slot memory: region i serves workers [w0, w1) (the warm team first,
  // the extra cold readers in a second region allocated by the first cold plan).
  struct RingRegion {
    uint8_t* mem;
    uint64_t bytes;
    bool registered;  // cudaHostRegister'ed malloc (else cudaHostAlloc)
    uint32_t w0, w1;
  };
  std::vector<RingRegion> regions;
  uint32_t ring_workers = 0;  // workers whose slots have memory
  uint32_t cold_workers = 0;  // team size for plans that are mostly O_DIRECT reads
  std::mutex mu;  // one plan at a time per context
  cudaEvent_t order_ev = nullptr;  // hl_execute_plan_after: the caller's stream position
  // Persistent worker team (threads live as long as the context): a plan is a
  // new generation; every team thread takes part (or sits it out) and checks in.
  std::vector<std::thread> team;
  std::mutex team_mu;
  std::condition_variable team_cv, team_done;
  uint64_t team_gen = 0;
  struct PlanRun* team_run = nullptr;
  uint32_t team_active = 0, team_left = 0;
  bool team_stop = false;
};

struct Chunk {
  uint32_t file;
  uint64_t off, len, dst;
};

struct FileState {
  int bfd = -1, dfd = -1;  // buffered / O_DIRECT descriptors
  int mode = HL_IO_BUFFERED;
  void* cufh = nullptr;
  uint8_t* map = nullptr;    // HL_IO_MMAP: read-only shared mapping of the file
  uint8_t* probe = nullptr;  // HL_IO_AUTO: mapping used only for mincore residency probes
  uint64_t size = 0;
  bool resident = false;     // HL_IO_AUTO: every sampled page was in the page cache at plan start
};

struct PlanRun {
  hl_ctx* ctx;
  cudaEvent_t order_ev = nullptr;  // every H2D waits for it (caller's stream position)
  bool async_tail = false;         // hand the copies' completion to `after` instead of draining
  uint32_t uring = 0;              // >0: cold plan read by this many io_uring threads (uring_loop)
  uint32_t uring_depth = 16;       // O_DIRECT reads in flight per io_uring thread
  uint32_t uring_rings = 0;        // io_uring threads share the slots of rings [0, uring_rings)
  cudaStream_t after = nullptr;
  const std::vector<Chunk>* chunks;
  std::vector<FileState>* files;
  std::atomic<size_t> cursor{0};
  std::atomic<bool> failed{false};
  std::mutex err_mu;
  int err_code = HL_OK;
  std::string err_msg;
  std::atomic<uint64_t> direct_bytes{0}, buffered_bytes{0}, cufile_bytes{0}, mmap_bytes{0}, uring_bytes{0};
  double ring_setup = 0;
  std::mutex setup_mu;
  std::atomic<uint64_t> read_ns{0}, wait_ns{0}, submit_ns{0};
  double t0 = 0;                                   // plan start (now_s clock)
  std::atomic<uint64_t> first_h2d_ns{~0ull}, last_h2d_ns{0};  // since t0

  void note_h2d() {
    const uint64_t t = (uint64_t)((now_s() - t0) * 1e9);
    uint64_t f = first_h2d_ns.load(std::memory_order_relaxed);
    while (t < f && !first_h2d_ns.compare_exchange_weak(f, t)) {
    }
    uint64_t l = last_h2d_ns.load(std::memory_order_relaxed);
    while (t > l && !last_h2d_ns.compare_exchange_weak(l, t)) {
    }
  }

  void fail(int code, const std::string& msg) {
    std::lock_guard<std::mutex> g(err_mu);
    if (err_code == HL_OK) {
      err_code = code;
      err_msg = msg;
    }
    failed.store(true);
  }
};

namespace {

bool pread_full(int fd, uint8_t* buf, uint64_t len, uint64_t off, uint64_t* got, int* err) {
  uint64_t done = 0;
  while (done < len) {
    ssize_t n = pread(fd, buf + done, len - done, (off_t)(off + done));
    if (n < 0) {
      if (errno == EINTR) continue;
      *err = errno;
      *got = done;
      return false;
    }
    if (n == 0) break;  // EOF
    done += (uint64_t)n;
  }
  *got = done;
  *err = 0;
  return true;
}

// The pinned memory of every worker's slots is ONE region, allocated before
// the first plan's workers start: 2 MiB-aligned, transparent-huge-page backed,
// first-touched by a thread on the GPU's NUMA node, then registered with
// cudaHostRegister. Measured on the B200 box (tools/pinned_probe.cu): 21 ms for
// 144 MiB, vs 74 ms for 36 separate cudaHostAlloc calls — and slot-by-slot
// allocation during the first load stalled behind the in-flight copies (first
// load 0.73 s vs 0.27 s steady; profiles/r01_first_load.jsonl).
int ensure_ring_memory(hl_ctx* ctx, uint32_t nworkers, double* seconds) {
  if (ctx->ring_workers >= nworkers) return HL_OK;
  const double t0 = now_s();
  const uint32_t w0 = ctx->ring_workers;
  const uint64_t bytes =
      round_up((uint64_t)(nworkers - w0) * ctx->cfg.slots_per_worker * ctx->slot_bytes, 2ull << 20);
  void* m = nullptr;
  bool registered = false;
  if (posix_memalign(&m, 2ull << 20, bytes) == 0) {
    madvise(m, bytes, MADV_HUGEPAGE);
    // first touch on the GPU's NUMA node, in parallel (page faults + zeroing dominate)
    const uint64_t nt = std::max<uint64_t>(1, std::min<uint64_t>(ctx->cfg.workers, bytes >> 21));
    const uint64_t piece = round_up((bytes + nt - 1) / nt, 2ull << 20);
    std::vector<std::thread> touchers;
    for (uint64_t i = 0; i < nt; ++i) {
      touchers.emplace_back([&, i] {
        pin_to(ctx->cpus);
        const uint64_t b = i * piece, e = std::min(bytes, b + piece);
        if (b < e) memset((uint8_t*)m + b, 0, e - b);
      });
    }
    for (auto& t : touchers) t.join();
    if (cudaHostRegister(m, bytes, cudaHostRegisterPortable) == cudaSuccess) {
      registered = true;
    } else {
      cudaGetLastError();
      free(m);
      m = nullptr;
    }
  }
  if (!m) {
    cudaError_t e = cudaHostAlloc(&m, bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) {
      return set_error(HL_ENOMEM, "pinned ring of %llu bytes: %s", (unsigned long long)bytes, cudaGetErrorString(e));
    }
  }
  ctx->regions.push_back({(uint8_t*)m, bytes, registered, w0, nworkers});
  ctx->ring_workers = nworkers;
  *seconds = now_s() - t0;
  return HL_OK;
}

// Stream + event per slot; slot memory comes from the context's pinned region.
int ensure_ring(hl_ctx* ctx, WorkerRing& r) {
  if (!r.slots.empty()) return HL_OK;
  cudaError_t e = cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return set_error(HL_ECUDA, "stream create: %s", cudaGetErrorString(e));
  e = cudaEventCreateWithFlags(&r.tail, cudaEventDisableTiming);
  if (e != cudaSuccess) return set_error(HL_ECUDA, "event create: %s", cudaGetErrorString(e));
  r.slots.resize(ctx->cfg.slots_per_worker);
  for (auto& s : r.slots) {
    e = cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return set_error(HL_ECUDA, "event create: %s", cudaGetErrorString(e));
  }
  return HL_OK;
}

int ensure_slot(hl_ctx* ctx, uint32_t w, uint32_t k, Slot& s) {
  if (s.host) return HL_OK;
  for (const auto& r : ctx->regions) {
    if (w >= r.w0 && w < r.w1) {
      s.host = r.mem + ((uint64_t)(w - r.w0) * ctx->cfg.slots_per_worker + k) * ctx->slot_bytes;
      return HL_OK;
    }
  }
  return set_error(HL_ENOMEM, "pinned ring not allocated for worker %u", w);
}

static void worker_loop(PlanRun* run, uint32_t w, WorkerRing& ring);
static void uring_loop(PlanRun* run, uint32_t u, WorkerRing& home);

// The slots a thread of `run` uses: its own ring's, or with io_uring every
// ring w = u, u + U, u + 2U, ... of the cold team (one read in flight per slot).
template <class F>
static void for_each_slot(PlanRun* run, uint32_t w, F&& fn) {
  hl_ctx* ctx = run->ctx;
  const uint32_t end = run->uring ? run->uring_rings : ctx->cold_workers;
  const uint32_t step = run->uring ? run->uring : end + 1;
  for (uint32_t r = w; r < end; r += step)
    for (auto& s : ctx->rings[r].slots) fn(s);
}

void worker_main(PlanRun* run, uint32_t w) {
  hl_ctx* ctx = run->ctx;
  WorkerRing& ring = ctx->rings[w];
  if (ring.slots.empty()) {
    const double t0 = now_s();
    int rc = ensure_ring(ctx, ring);
    {
      std::lock_guard<std::mutex> g(run->setup_mu);
      run->ring_setup = std::max(run->ring_setup, now_s() - t0);
    }
    if (rc) {
      run->fail(rc, hl_last_error());
      return;
    }
  }
  if (run->order_ev) {
    // Write-after-read guard: the destination buffers come from the caller's
    // allocator, which may hand out memory that kernels still queued on the
    // caller's stream are about to read. No H2D of this plan starts before
    // that stream position.
    cudaError_t e = cudaStreamWaitEvent(ring.stream, run->order_ev, 0);
    if (e != cudaSuccess) {
      run->fail(HL_ECUDA, std::string("stream ordering: ") + cudaGetErrorString(e));
      return;
    }
  }
  if (run->uring) {
    uring_loop(run, w, ring);
  } else {
    worker_loop(run, w, ring);
  }
  bool pinned = false;  // page-cache ranges pinned for in-flight copies are unpinned only after them
  for_each_slot(run, w, [&](Slot& s) { pinned |= s.reg != nullptr; });
  if (run->async_tail && !pinned && !run->failed.load()) {
    // Completion goes to the caller's stream: it waits for this worker's last
    // copy, so every kernel enqueued there afterwards sees the bytes, and the
    // caller's stream-ordered frees cannot recycle a destination under a copy.
    // The slots stay busy; their next user waits on their events.
    cudaError_t e = cudaEventRecord(ring.tail, ring.stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(run->after, ring.tail, 0);
    if (e == cudaSuccess) return;
    run->fail(HL_ECUDA, std::string("completion handoff: ") + cudaGetErrorString(e));
  }
  // Drain on every other exit, failed or not: the caller frees (or reuses) the
  // destination buffers as soon as hl_execute_plan returns, so no DMA of this
  // worker may still be in flight, and no page-cache range may stay pinned.
  cudaError_t e = cudaStreamSynchronize(ring.stream);
  for_each_slot(run, w, [&](Slot& s) {
    s.busy = false;
    if (s.reg) {
      cudaHostUnregister(s.reg);
      s.reg = nullptr;
    }
  });
  if (e != cudaSuccess) run->fail(HL_ECUDA, std::string("H2D stream: ") + cudaGetErrorString(e));
}

// One worker's share of a plan: claim chunks, read, submit their H2D copies.
// Returns on the first error (recorded in `run`); worker_main drains.
static void worker_loop(PlanRun* run, uint32_t w, WorkerRing& ring) {
  hl_ctx* ctx = run->ctx;
  const auto& chunks = *run->chunks;
  auto& files = *run->files;
  std::vector<unsigned char> vec;  // mincore scratch
  while (!run->failed.load(std::memory_order_relaxed)) {
    const size_t i = run->cursor.fetch_add(1);
    if (i >= chunks.size()) break;
    const Chunk& c = chunks[i];
    FileState& f = files[c.file];
    if (f.mode == HL_IO_CUFILE) {
      ssize_t n = g_cufile.read(f.cufh, (void*)c.dst, c.len, (off_t)c.off, 0);
      if (n < 0 || (uint64_t)n != c.len) {
        run->fail(HL_EIO, "cuFileRead of " + std::to_string(c.len) + " bytes at " + std::to_string(c.off) +
                              " returned " + std::to_string(n));
        return;
      }
      run->cufile_bytes += c.len;
      continue;
    }
    Slot& s = ring.slots[ring.next];
    ring.next = (ring.next + 1) % ring.slots.size();
    if (s.busy) {
      const double tw = now_s();
      cudaError_t e = cudaEventSynchronize(s.ev);
      run->wait_ns += (uint64_t)((now_s() - tw) * 1e9);
      if (e != cudaSuccess) {
        run->fail(HL_ECUDA, std::string("H2D completion: ") + cudaGetErrorString(e));
        return;
      }
      s.busy = false;
      if (s.reg) {
        cudaHostUnregister(s.reg);
        s.reg = nullptr;
      }
    }
    bool pin = f.mode == HL_IO_MMAP;
    if (f.mode == HL_IO_AUTO && f.probe && (ctx->cfg.flags & HL_CFG_AUTO_PIN_CACHE)) {
      // a fully resident chunk is DMA'd from the page cache in place (one DRAM pass)
      const uint64_t p0 = c.off / kAlign, p1 = (c.off + c.len + kAlign - 1) / kAlign;
      if (vec.size() < p1 - p0) vec.resize(p1 - p0);
      pin = mincore(f.probe + p0 * kAlign, (p1 - p0) * kAlign, vec.data()) == 0;
      for (uint64_t q = 0; pin && q < p1 - p0; ++q) pin = vec[q] & 1;
    }
    if (pin) {
      // pin the page-cache pages of this chunk in place and DMA them: no CPU copy
      uint8_t* p = (f.map ? f.map : f.probe) + c.off;
      uint8_t* a = (uint8_t*)round_down((uint64_t)(uintptr_t)p, kAlign);
      const uint64_t alen = round_up((uint64_t)(p - a) + c.len, kAlign);
      const double tp = now_s();
      cudaError_t e = cudaHostRegister(a, alen, cudaHostRegisterPortable | cudaHostRegisterReadOnly);
      run->read_ns += (uint64_t)((now_s() - tp) * 1e9);
      if (e == cudaSuccess) {
        e = cudaMemcpyAsync((void*)c.dst, p, c.len, cudaMemcpyHostToDevice, ring.stream);
        if (e == cudaSuccess) e = cudaEventRecord(s.ev, ring.stream);
        if (e != cudaSuccess) {
          run->fail(HL_ECUDA, std::string("H2D copy (mmap): ") + cudaGetErrorString(e));
          return;
        }
        s.reg = a;
        s.busy = true;
        run->mmap_bytes += c.len;
        run->note_h2d();
        continue;
      }
      cudaGetLastError();  // registration refused (overlap, limits): copy through the ring
      if (getenv("HL_IO_DEBUG"))
        fprintf(stderr, "hl_io: cudaHostRegister(%p, %llu) refused: %s\n", (void*)a, (unsigned long long)alen,
                cudaGetErrorString(e));
    } else if (getenv("HL_IO_DEBUG") && f.mode == HL_IO_AUTO) {
      fprintf(stderr, "hl_io: chunk at %llu not pinned (flags %u, probe %p)\n", (unsigned long long)c.off,
              ctx->cfg.flags, (void*)f.probe);
    }
    if (!s.host) {
      int rc = ensure_slot(ctx, w, (uint32_t)(&s - ring.slots.data()), s);
      if (rc) {
        run->fail(rc, hl_last_error());
        return;
      }
    }
    const double tr = now_s();
    // Slot layout: the chunk's bytes start at `head` = off % 4 KiB, so the
    // O_DIRECT part of any read lands 4 KiB-aligned in the slot.
    const uint64_t head = c.off % kAlign;
    uint64_t cached = 0;  // leading bytes served from the page cache
    // (an AUTO file sampled fully resident at plan start is read like a buffered one)
    if (f.mode == HL_IO_BUFFERED || (f.mode == HL_IO_DIRECT && f.dfd < 0) || (f.mode == HL_IO_AUTO && f.resident)) {
      uint64_t got = 0;
      int err = 0;
      if (!pread_full(f.bfd, s.host + head, c.len, c.off, &got, &err)) {
        run->fail(HL_EIO, std::string("read failed at offset ") + std::to_string(c.off) + ": " + strerror(err));
        return;
      }
      if (got < c.len) {
        run->fail(HL_EIO, "unexpected EOF at file offset " + std::to_string(c.off + got) + " (" +
                              std::to_string(c.len - got) + " bytes short)");
        return;
      }
      cached = c.len;
    } else {
      if (f.mode == HL_IO_AUTO && f.probe) {
        // hybrid: the page-cache-resident prefix of the chunk (mincore: no I/O is
        // triggered, unlike a RWF_NOWAIT probe whose readahead would race the
        // O_DIRECT reads) is copied from the cache, the rest read with O_DIRECT
        const uint64_t p0 = c.off / kAlign, p1 = (c.off + c.len + kAlign - 1) / kAlign;
        if (vec.size() < p1 - p0) vec.resize(p1 - p0);
        uint64_t res = 0;
        if (mincore(f.probe + p0 * kAlign, (p1 - p0) * kAlign, vec.data()) == 0) {
          while (res < p1 - p0 && (vec[res] & 1)) ++res;
        }
        const uint64_t upto = std::min<uint64_t>(c.off + c.len, (p0 + res) * kAlign);
        if (upto > c.off) {
          uint64_t got = 0;
          int err = 0;
          if (pread_full(f.bfd, s.host + head, upto - c.off, c.off, &got, &err)) cached = got;
        }
      }
      if (cached < c.len) {
        const uint64_t from = c.off + cached;
        const uint64_t aoff = round_down(from, kAlign);
        const uint64_t alen = round_up(c.off + c.len, kAlign) - aoff;
        uint8_t* dst = s.host + (aoff - (c.off - head));  // 4 KiB aligned: aoff >= c.off - head
        uint64_t got = 0;
        int err = 0;
        bool ok = f.dfd >= 0 && pread_full(f.dfd, dst, alen, aoff, &got, &err);
        if (ok && aoff + got < c.off + c.len) {
          run->fail(HL_EIO, "unexpected EOF at file offset " + std::to_string(aoff + got));
          return;
        }
        if (!ok && (f.dfd < 0 || err == EINVAL)) {  // no O_DIRECT on this file system: buffered
          ok = pread_full(f.bfd, s.host + head + cached, c.len - cached, from, &got, &err);
          if (ok && got < c.len - cached) {
            run->fail(HL_EIO, "unexpected EOF at file offset " + std::to_string(from + got));
            return;
          }
        }
        if (!ok) {
          run->fail(HL_EIO, std::string("read failed at offset ") + std::to_string(from) + ": " + strerror(err));
          return;
        }
        // an O_DIRECT read of the partial first page rewrote bytes before `from`
        // with identical file contents: harmless
        run->direct_bytes += c.len - cached;
      }
    }
    run->buffered_bytes += cached;
    run->read_ns += (uint64_t)((now_s() - tr) * 1e9);
    const double ts = now_s();
    cudaError_t e = cudaMemcpyAsync((void*)c.dst, s.host + head, c.len, cudaMemcpyHostToDevice, ring.stream);
    if (e == cudaSuccess) e = cudaEventRecord(s.ev, ring.stream);
    run->submit_ns += (uint64_t)((now_s() - ts) * 1e9);
    if (e != cudaSuccess) {
      run->fail(HL_ECUDA, std::string("H2D copy: ") + cudaGetErrorString(e));
      return;
    }
    s.busy = true;
    run->note_h2d();
  }
}

// ------------------------------------------------------------------ io_uring cold reader
// A cold plan is storage-latency bound: its rate follows the O_DIRECT requests
// in flight. Instead of 32 threads each blocked in one pread, a few threads each
// keep `uring_depth` reads in flight on an io_uring (raw syscalls, no liburing)
// and hand every completed read to the H2D stream. Same chunks, same slots,
// same bytes as worker_loop; io_uring unavailable (kernel, seccomp) or any
// setup failure falls back to worker_loop.
struct Uring {
  int fd = -1;
  uint8_t *sq = nullptr, *cq = nullptr;
  size_t sq_sz = 0, cq_sz = 0, sqe_sz = 0;
  io_uring_sqe* sqes = nullptr;
  io_uring_cqe* cqes = nullptr;
  unsigned *sq_head = nullptr, *sq_tail = nullptr, *sq_mask = nullptr, *sq_array = nullptr;
  unsigned *cq_head = nullptr, *cq_tail = nullptr, *cq_mask = nullptr;

  bool open(unsigned entries) {
    io_uring_params p;
    memset(&p, 0, sizeof p);
    fd = (int)syscall(__NR_io_uring_setup, entries, &p);
    if (fd < 0) return false;
    sq_sz = p.sq_off.array + p.sq_entries * sizeof(unsigned);
    cq_sz = p.cq_off.cqes + p.cq_entries * sizeof(io_uring_cqe);
    sqe_sz = p.sq_entries * sizeof(io_uring_sqe);
    void* a = mmap(nullptr, sq_sz, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd, IORING_OFF_SQ_RING);
    void* b = mmap(nullptr, cq_sz, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd, IORING_OFF_CQ_RING);
    void* c = mmap(nullptr, sqe_sz, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd, IORING_OFF_SQES);
    sq = a == MAP_FAILED ? nullptr : (uint8_t*)a;
    cq = b == MAP_FAILED ? nullptr : (uint8_t*)b;
    sqes = c == MAP_FAILED ? nullptr : (io_uring_sqe*)c;
    if (!sq || !cq || !sqes) return false;
    sq_head = (unsigned*)(sq + p.sq_off.head);
    sq_tail = (unsigned*)(sq + p.sq_off.tail);
    sq_mask = (unsigned*)(sq + p.sq_off.ring_mask);
    sq_array = (unsigned*)(sq + p.sq_off.array);
    cq_head = (unsigned*)(cq + p.cq_off.head);
    cq_tail = (unsigned*)(cq + p.cq_off.tail);
    cq_mask = (unsigned*)(cq + p.cq_off.ring_mask);
    cqes = (io_uring_cqe*)(cq + p.cq_off.cqes);
    return true;
  }
  ~Uring() {
    if (sqes) munmap(sqes, sqe_sz);
    if (cq) munmap(cq, cq_sz);
    if (sq) munmap(sq, sq_sz);
    if (fd >= 0) ::close(fd);
  }
  void read(int file, void* buf, uint32_t len, uint64_t off, uint64_t tag) {
    const unsigned tail = *sq_tail;
    const unsigned idx = tail & *sq_mask;
    io_uring_sqe* e = &sqes[idx];
    memset(e, 0, sizeof *e);
    e->opcode = IORING_OP_READ;
    e->fd = file;
    e->addr = (uint64_t)(uintptr_t)buf;
    e->len = len;
    e->off = off;
    e->user_data = tag;
    sq_array[idx] = idx;
    __atomic_store_n(sq_tail, tail + 1, __ATOMIC_RELEASE);
  }
  // submit every queued read the kernel has not consumed yet (a partial submit
  // leaves the rest for the next call), wait for at least `wait` completions
  int enter(unsigned wait) {
    for (;;) {
      const unsigned n = *sq_tail - __atomic_load_n(sq_head, __ATOMIC_ACQUIRE);
      int r = (int)syscall(__NR_io_uring_enter, fd, n, wait, wait ? IORING_ENTER_GETEVENTS : 0, nullptr, 0);
      if (r >= 0 || errno != EINTR) return r < 0 ? -errno : r;
    }
  }
  template <class F>
  void reap(F&& fn) {
    unsigned head = *cq_head;
    while (head != __atomic_load_n(cq_tail, __ATOMIC_ACQUIRE)) {
      const io_uring_cqe& c = cqes[head & *cq_mask];
      fn(c.user_data, c.res);
      ++head;
    }
    __atomic_store_n(cq_head, head, __ATOMIC_RELEASE);
  }
};

// io_uring usable in this process (kernel support, not disabled by sysctl or a
// seccomp filter): probed once. Without it cold plans keep the blocking readers
// of the whole cold team instead of 2 threads falling back to one read each.
static bool uring_available() {
  static const bool ok = [] {
    Uring r;
    return r.open(2);
  }();
  return ok;
}

static void uring_loop(PlanRun* run, uint32_t u, WorkerRing& home) {
  hl_ctx* ctx = run->ctx;
  const auto& chunks = *run->chunks;
  auto& files = *run->files;
  // this thread's slots: every slot of rings u, u + U, ... (streams/events made on first use)
  std::vector<Slot*> slots;
  for (uint32_t r = u; r < run->uring_rings; r += run->uring) {
    WorkerRing& wr = ctx->rings[r];
    int rc = ensure_ring(ctx, wr);
    for (uint32_t k = 0; rc == HL_OK && k < wr.slots.size(); ++k) {
      rc = ensure_slot(ctx, r, k, wr.slots[k]);
      slots.push_back(&wr.slots[k]);
    }
    if (rc) {
      run->fail(rc, hl_last_error());
      return;
    }
  }
  const uint32_t depth = (uint32_t)std::min<size_t>(run->uring_depth, slots.size());
  Uring ring;
  if (depth == 0 || !ring.open(depth)) {
    worker_loop(run, u, home);  // no io_uring here: the same chunks with blocking reads
    return;
  }
  struct Req {
    const Chunk* c = nullptr;
    uint64_t aoff = 0, alen = 0;
    bool reading = false;
  };
  std::vector<Req> req(slots.size());
  std::vector<unsigned char> vec;  // mincore scratch
  size_t hint = 0;
  uint32_t inflight = 0;
  bool claiming = true;
  auto h2d = [&](Slot& s, const Chunk& c, uint64_t head) -> bool {
    const double ts = now_s();
    cudaError_t e = cudaMemcpyAsync((void*)c.dst, s.host + head, c.len, cudaMemcpyHostToDevice, home.stream);
    if (e == cudaSuccess) e = cudaEventRecord(s.ev, home.stream);
    run->submit_ns += (uint64_t)((now_s() - ts) * 1e9);
    if (e != cudaSuccess) {
      run->fail(HL_ECUDA, std::string("H2D copy: ") + cudaGetErrorString(e));
      return false;
    }
    s.busy = true;
    run->note_h2d();
    return true;
  };
  // a slot with no read in flight whose previous DMA (if any) is done; -1 if none
  auto free_slot = [&](bool block) -> long {
    for (size_t n = 0; n < slots.size(); ++n) {
      const size_t i = (hint + n) % slots.size();
      Slot& s = *slots[i];
      if (req[i].reading) continue;
      if (s.busy) {
        if (cudaEventQuery(s.ev) != cudaSuccess) continue;
        s.busy = false;
      }
      hint = i + 1;
      return (long)i;
    }
    if (!block) return -1;
    for (size_t n = 0; n < slots.size(); ++n) {  // every slot is DMA-busy: wait for the next in order
      const size_t i = (hint + n) % slots.size();
      if (req[i].reading) continue;
      const double tw = now_s();
      cudaError_t e = cudaEventSynchronize(slots[i]->ev);
      run->wait_ns += (uint64_t)((now_s() - tw) * 1e9);
      if (e != cudaSuccess) {
        run->fail(HL_ECUDA, std::string("H2D completion: ") + cudaGetErrorString(e));
        return -1;
      }
      slots[i]->busy = false;
      hint = i + 1;
      return (long)i;
    }
    return -1;
  };
  // Every exit goes through the drain at the end: reads in flight target our
  // pinned slots, so none may still be running when the slots are handed on.
  for (;;) {
    while (claiming && inflight < depth && !run->failed.load(std::memory_order_relaxed)) {
      const long si = free_slot(inflight == 0);
      if (si < 0) break;  // wait for completions first (or a failed DMA wait)
      const size_t i = run->cursor.fetch_add(1);
      if (i >= chunks.size()) {
        claiming = false;
        break;
      }
      const Chunk& c = chunks[i];
      FileState& f = files[c.file];
      Slot& s = *slots[si];
      const uint64_t head = c.off % kAlign;
      bool direct = f.dfd >= 0 && (f.mode == HL_IO_AUTO || f.mode == HL_IO_DIRECT);
      if (direct && f.mode == HL_IO_AUTO && f.resident) {
        direct = false;  // sampled fully resident at plan start
      } else if (direct && f.mode == HL_IO_AUTO && f.probe) {
        // a chunk already in the page cache is copied from it (no storage read)
        const uint64_t p0 = c.off / kAlign, p1 = (c.off + c.len + kAlign - 1) / kAlign;
        if (vec.size() < p1 - p0) vec.resize(p1 - p0);
        bool resident = mincore(f.probe + p0 * kAlign, (p1 - p0) * kAlign, vec.data()) == 0;
        for (uint64_t q = 0; resident && q < p1 - p0; ++q) resident = vec[q] & 1;
        direct = !resident;
      }
      if (!direct) {
        uint64_t got = 0;
        int err = 0;
        const double tr = now_s();
        if (!pread_full(f.bfd, s.host + head, c.len, c.off, &got, &err) || got < c.len) {
          run->fail(HL_EIO, err ? std::string("read failed at offset ") + std::to_string(c.off) + ": " + strerror(err)
                                : "unexpected EOF at file offset " + std::to_string(c.off + got));
          break;
        }
        run->read_ns += (uint64_t)((now_s() - tr) * 1e9);
        run->buffered_bytes += c.len;
        if (!h2d(s, c, head)) break;
        continue;
      }
      Req& q = req[si];
      q.c = &c;
      q.aoff = round_down(c.off, kAlign);
      q.alen = round_up(c.off + c.len, kAlign) - q.aoff;
      q.reading = true;
      ring.read(f.dfd, s.host, (uint32_t)q.alen, q.aoff, (uint64_t)si);
      ++inflight;
    }
    if (run->failed.load(std::memory_order_relaxed)) claiming = false;  // stop claiming, reap what is in flight
    if (!claiming && inflight == 0) break;
    const double tr = now_s();
    const int r = ring.enter(inflight ? 1 : 0);  // always submits what was queued
    run->read_ns += (uint64_t)((now_s() - tr) * 1e9);
    if (r < 0) {
      run->fail(HL_EIO, std::string("io_uring_enter: ") + strerror(-r));
      break;
    }
    ring.reap([&](uint64_t tag, int res) {
      Req& q = req[tag];
      Slot& s = *slots[tag];
      const Chunk& c = *q.c;
      FileState& f = files[c.file];
      q.reading = false;
      --inflight;
      if (run->failed.load(std::memory_order_relaxed)) return;  // draining after a failure
      const uint64_t head = c.off % kAlign;
      const uint64_t need = c.off + c.len - q.aoff;  // bytes the chunk needs from the aligned start
      uint64_t got = res > 0 ? (uint64_t)res : 0;
      int err = res < 0 ? -res : 0;
      if (res == -EINVAL) {  // no O_DIRECT on this file system: buffered
        err = 0;
        uint64_t n = 0;
        if (!pread_full(f.bfd, s.host + head, c.len, c.off, &n, &err) || n < c.len) {
          run->fail(HL_EIO, "read failed at offset " + std::to_string(c.off));
          return;
        }
        run->buffered_bytes += c.len;
        h2d(s, c, head);
        return;
      }
      if (!err && got < need && got % kAlign == 0) {  // short read: finish it synchronously
        uint64_t n = 0;
        if (pread_full(f.dfd, s.host + got, q.alen - got, q.aoff + got, &n, &err)) got += n;
      }
      if (err || got < need) {
        run->fail(HL_EIO, err ? std::string("read failed at offset ") + std::to_string(c.off) + ": " + strerror(err)
                              : "unexpected EOF at file offset " + std::to_string(q.aoff + got));
        return;
      }
      run->direct_bytes += c.len;
      run->uring_bytes += c.len;
      h2d(s, c, head);
    });
  }
  // reads still in flight after a failure land in our slots before they are handed on
  while (inflight > 0 && ring.enter(1) >= 0) ring.reap([&](uint64_t tag, int) {
      req[tag].reading = false;
      --inflight;
    });
}

void team_thread(hl_ctx* ctx, uint32_t w) {
  cudaSetDevice(ctx->cfg.device);
  pin_to(ctx->cpus);
  char name[16];
  snprintf(name, sizeof name, "hl-io-%d-%u", ctx->cfg.device, w);
  pthread_setname_np(pthread_self(), name);
  uint64_t seen = 0;
  for (;;) {
    PlanRun* run = nullptr;
    bool active = false;
    {
      std::unique_lock<std::mutex> lk(ctx->team_mu);
      ctx->team_cv.wait(lk, [&] { return ctx->team_stop || ctx->team_gen != seen; });
      if (ctx->team_stop) return;
      seen = ctx->team_gen;
      run = ctx->team_run;
      active = w < ctx->team_active;
    }
    if (active) worker_main(run, w);
    std::lock_guard<std::mutex> g(ctx->team_mu);
    if (--ctx->team_left == 0) ctx->team_done.notify_all();
  }
}

// Run `run` on the first `n` team threads (spawned once per context) and wait.
void team_run(hl_ctx* ctx, PlanRun* run, uint32_t n) {
  while (ctx->team.size() < n) {
    const uint32_t w = (uint32_t)ctx->team.size();
    ctx->team.emplace_back(team_thread, ctx, w);
  }
  std::unique_lock<std::mutex> lk(ctx->team_mu);
  ctx->team_run = run;
  ctx->team_active = n;
  ctx->team_left = (uint32_t)ctx->team.size();
  ++ctx->team_gen;
  ctx->team_cv.notify_all();
  ctx->team_done.wait(lk, [&] { return ctx->team_left == 0; });
  ctx->team_run = nullptr;
}

double residency(int fd, uint64_t size) {
  if (size == 0) return 1.0;
  void* m = mmap(nullptr, size, PROT_READ, MAP_SHARED, fd, 0);
  if (m == MAP_FAILED) return 0.0;
  const long pg = sysconf(_SC_PAGESIZE);
  const size_t pages = (size + pg - 1) / pg;
  std::vector<unsigned char> vec(pages);
  double frac = 0.0;
  if (mincore(m, size, vec.data()) == 0) {
    size_t res = 0;
    for (unsigned char v : vec) res += v & 1;
    frac = (double)res / (double)pages;
  }
  munmap(m, size);
  return frac;
}

}  // namespace

extern "C" int hl_ctx_create(const hl_config* cfg, hl_ctx** out) {
  clear_error();
  if (!out) return set_error(HL_EINVAL, "null output pointer");
  hl_ctx* ctx = new hl_ctx();
  if (cfg) ctx->cfg = *cfg;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    delete ctx;
    return set_error(HL_ECUDA, "no CUDA device visible: %s", cudaGetErrorString(e));
  }
  if (ctx->cfg.device < 0 || ctx->cfg.device >= ndev) {
    int d = ctx->cfg.device;
    delete ctx;
    return set_error(HL_EINVAL, "device %d out of range (%d visible)", d, ndev);
  }
  if (ctx->cfg.io_mode > HL_IO_MMAP) {
    delete ctx;
    return set_error(HL_EINVAL, "unknown io_mode %u", cfg->io_mode);
  }
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, ctx->cfg.device) != cudaSuccess) bus[0] = 0;
  const int node = resolve_node(bus, ctx->cfg.numa_node);
  ctx->cfg.numa_node = node;
  ctx->cpus = node_cpus(node);
  if (ctx->cfg.workers == 0) {
    long n = ctx->cpus.empty() ? sysconf(_SC_NPROCESSORS_ONLN) : (long)ctx->cpus.size();
    long w = (long)(0.8 * (double)n);
    ctx->cfg.workers = (uint32_t)std::max(1L, std::min(w, 16L));
  }
  if (ctx->cfg.chunk_bytes == 0) ctx->cfg.chunk_bytes = 16ull << 20;
  ctx->cfg.chunk_bytes = round_up(ctx->cfg.chunk_bytes, kAlign);
  if (ctx->cfg.slots_per_worker == 0) {
    ctx->cfg.slots_per_worker = 3;
    if (const char* e = getenv("HL_ENGINE_SLOTS")) ctx->cfg.slots_per_worker = (uint32_t)std::max(1L, std::min(strtol(e, nullptr, 10), 16L));
  }
  ctx->slot_bytes = ctx->cfg.chunk_bytes + 2 * kAlign;  // O_DIRECT head/tail slack
  // Cold reads are storage-latency bound, not CPU bound: more requests in flight
  // raise the rate (O_DIRECT 4 MiB preads on the box: 16 threads 3.8 GB/s, 32
  // threads 4.8; profiles/r02_bench_n1_v4.json storage_probe). Plans whose bytes
  // are mostly not in the page cache run on this larger team ($HL_COLD_WORKERS).
  uint32_t cold = 32;
  if (const char* e = getenv("HL_COLD_WORKERS")) cold = (uint32_t)std::max(1L, std::min(strtol(e, nullptr, 10), 64L));
  ctx->cold_workers = std::max(ctx->cfg.workers, cold);
  ctx->rings.resize(ctx->cold_workers);
  *out = ctx;
  return HL_OK;
}

extern "C" int hl_ctx_config(const hl_ctx* ctx, hl_config* out) {
  if (!ctx || !out) return set_error(HL_EINVAL, "null argument");
  *out = ctx->cfg;
  return HL_OK;
}

extern "C" int hl_ctx_destroy(hl_ctx* ctx) {
  clear_error();
  if (!ctx) return HL_OK;
  {
    std::lock_guard<std::mutex> g(ctx->team_mu);
    ctx->team_stop = true;
    ctx->team_cv.notify_all();
  }
  for (auto& t : ctx->team) t.join();
  cudaSetDevice(ctx->cfg.device);
  if (ctx->order_ev) cudaEventDestroy(ctx->order_ev);
  for (auto& r : ctx->rings) {
    if (r.stream) cudaStreamSynchronize(r.stream);
    if (r.tail) cudaEventDestroy(r.tail);
    for (auto& s : r.slots) {
      if (s.ev) cudaEventDestroy(s.ev);
    }
    if (r.stream) cudaStreamDestroy(r.stream);
  }
  for (const auto& r : ctx->regions) {
    if (r.registered) {
      cudaHostUnregister(r.mem);
      free(r.mem);
    } else {
      cudaFreeHost(r.mem);
    }
  }
  delete ctx;
  return HL_OK;
}

static int execute(hl_ctx* ctx, const char* const* paths, uint32_t n_files, const hl_block* blocks,
                   uint32_t n_blocks, bool ordered, cudaStream_t after, hl_plan_stats* stats,
                   bool async_tail = false) {
  clear_error();
  if (!ctx) return set_error(HL_EINVAL, "null context");
  if (n_blocks && (!blocks || !paths)) return set_error(HL_EINVAL, "null blocks or paths");
  std::lock_guard<std::mutex> guard(ctx->mu);
  const double t0 = now_s();
  cudaSetDevice(ctx->cfg.device);

  // Merge blocks that continue each other (same file, contiguous in the file
  // and on the device), then cut chunks at absolute multiples of chunk_bytes in
  // file-offset space: chunk boundaries are page aligned, so O_DIRECT heads and
  // mmap-pinned page ranges of neighbouring chunks never overlap.
  std::vector<Chunk> chunks;
  std::vector<char> used(n_files, 0);
  uint64_t total = 0;
  std::vector<Chunk> ranges;
  for (uint32_t b = 0; b < n_blocks; ++b) {
    const hl_block& bl = blocks[b];
    if (bl.file >= n_files) return set_error(HL_EINVAL, "block %u names file %u of %u", b, bl.file, n_files);
    if (bl.len && !bl.dev_dst) return set_error(HL_EINVAL, "block %u has a null destination", b);
    used[bl.file] = 1;
    total += bl.len;
    if (!bl.len) continue;
    if (!ranges.empty()) {
      Chunk& r = ranges.back();
      if (r.file == bl.file && r.off + r.len == bl.file_off && r.dst + r.len == bl.dev_dst) {
        r.len += bl.len;
        continue;
      }
    }
    ranges.push_back({bl.file, bl.file_off, bl.len, bl.dev_dst});
  }
  // open files, pick the read mode per file
  std::vector<FileState> files(n_files);
  auto close_all = [&]() {
    for (auto& f : files) {
      if (f.map) munmap(f.map, f.size);
      if (f.probe) munmap(f.probe, f.size);
      if (f.cufh && g_cufile.handle_deregister) g_cufile.handle_deregister(f.cufh);
      if (f.bfd >= 0) close(f.bfd);
      if (f.dfd >= 0) close(f.dfd);
    }
  };
  uint32_t mode_mask = 0;
  for (uint32_t i = 0; i < n_files; ++i) {
    if (!used[i]) continue;
    FileState& f = files[i];
    f.bfd = open(paths[i], O_RDONLY | O_CLOEXEC);
    if (f.bfd < 0) {
      int err = errno;
      close_all();
      return set_error(HL_EIO, "cannot open %s: %s", paths[i], strerror(err));
    }
    struct stat st;
    fstat(f.bfd, &st);
    f.size = (uint64_t)st.st_size;
    uint32_t mode = ctx->cfg.io_mode;
    // cuFile only where it is real GPUDirect Storage (nvidia-fs loaded); without
    // it cuFile's compat mode is a slower POSIX bounce path than our own ring,
    // so the GDS-shaped backend reads through the ring instead: O_DIRECT for
    // what is on storage, the page cache for what is already resident (AUTO's
    // per-chunk probe; a warm file would otherwise be re-read from the disk).
    // HL_FORCE_CUFILE=1 keeps cuFile for experiments.
    if (mode == HL_IO_CUFILE && !hl_gds_available() && !getenv("HL_FORCE_CUFILE")) mode = HL_IO_AUTO;
    if (mode == HL_IO_AUTO && f.size) {
      void* m = mmap(nullptr, f.size, PROT_READ, MAP_SHARED, f.bfd, 0);
      if (m != MAP_FAILED) f.probe = (uint8_t*)m;
      // AUTO copies only pages mincore found resident: no (synchronous) readahead
      // on that descriptor, it would pull cold chunks in ahead of their probes
      posix_fadvise(f.bfd, 0, 0, POSIX_FADV_RANDOM);
    }
    if (mode == HL_IO_MMAP) {
      void* m = f.size ? mmap(nullptr, f.size, PROT_READ, MAP_SHARED, f.bfd, 0) : MAP_FAILED;
      if (m == MAP_FAILED) {
        mode = HL_IO_BUFFERED;
      } else {
        f.map = (uint8_t*)m;
      }
    }
    if (mode == HL_IO_AUTO || mode == HL_IO_DIRECT || mode == HL_IO_CUFILE) {
      f.dfd = open(paths[i], O_RDONLY | O_DIRECT | O_CLOEXEC);
      if (f.dfd < 0 && mode == HL_IO_DIRECT) mode = HL_IO_BUFFERED;  // e.g. tmpfs: EINVAL
    }
    if (mode == HL_IO_CUFILE) {
      std::string why;
      if (!cufile_load(&why)) {
        close_all();
        return set_error(HL_EIO, "cuFile path requested but unavailable: %s", why.c_str());
      }
      CUfileDescr d{};
      d.type = 1;
      d.handle.fd = f.dfd >= 0 ? f.dfd : f.bfd;
      CUfileError e = g_cufile.handle_register(&f.cufh, &d);
      if (e.err != 0) {
        close_all();
        return set_error(HL_EIO, "cuFileHandleRegister(%s) failed (code %d)", paths[i], e.err);
      }
    }
    f.mode = (int)mode;
    mode_mask |= 1u << mode;
  }
  for (const Chunk& c : ranges) {
    if (c.off + c.len > files[c.file].size) {
      close_all();
      return set_error(HL_EIO, "range [%llu, %llu) past end of %s (%llu bytes)", (unsigned long long)c.off,
                       (unsigned long long)(c.off + c.len), paths[c.file], (unsigned long long)files[c.file].size);
    }
  }

  PlanRun run;
  run.t0 = t0;
  run.ctx = ctx;
  run.chunks = &chunks;
  run.files = &files;
  if (ordered && !ranges.empty()) {
    cudaError_t e = ctx->order_ev ? cudaSuccess : cudaEventCreateWithFlags(&ctx->order_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->order_ev, after);
    // cuFile writes HBM from the host thread, outside any stream: wait here
    if (e == cudaSuccess && (mode_mask & (1u << HL_IO_CUFILE))) e = cudaEventSynchronize(ctx->order_ev);
    if (e != cudaSuccess) {
      close_all();
      return set_error(HL_ECUDA, "ordering after the caller's stream: %s", cudaGetErrorString(e));
    }
    run.order_ev = ctx->order_ev;
    run.async_tail = async_tail;
    run.after = after;
  }
  // Team size: the warm team, or the cold readers when most of the plan's bytes
  // will be read with O_DIRECT (direct mode; auto mode with < half resident).
  uint32_t team = ctx->cfg.workers;
  if (ctx->cold_workers > team && total > 0) {
    // estimate from 64 sampled pages per file (mincore of one page each: cheap)
    std::vector<uint64_t> plan_bytes(n_files, 0);
    for (const Chunk& c : ranges) plan_bytes[c.file] += c.len;
    double cold_bytes = 0;
    for (uint32_t i = 0; i < n_files; ++i) {
      const FileState& f = files[i];
      if (!plan_bytes[i]) continue;
      if (f.mode == HL_IO_DIRECT && f.dfd >= 0) {
        cold_bytes += (double)plan_bytes[i];
      } else if (f.mode == HL_IO_AUTO && f.probe && f.size >= kAlign) {
        const uint64_t pages = f.size / kAlign;
        const uint64_t n = std::min<uint64_t>(64, pages);
        uint64_t res = 0;
        for (uint64_t q = 0; q < n; ++q) {
          unsigned char v = 0;
          const uint64_t pg = (2 * q + 1) * pages / (2 * n);
          if (mincore(f.probe + pg * kAlign, kAlign, &v) == 0) res += v & 1;
        }
        cold_bytes += (double)plan_bytes[i] * (double)(n - res) / (double)n;
        // every sample resident: the workers skip the per-chunk mincore for this file
        // (~25 us per 2 MiB chunk of page lookups; a page evicted since is still read
        // correctly, by the buffered pread)
        files[i].resident = res == n;
      }
    }
    if (cold_bytes * 2 > (double)total) team = ctx->cold_workers;
  }
  const bool cold_plan = team > ctx->cfg.workers;
  // Small warm plans (< 2 GiB) on a large team (>= 8) run on half of it: their copy engine,
  // not the page-cache copies, is the bound, and fewer concurrent copies leave it more
  // host-memory bandwidth (GPT-2's 0.5 GB from a warm cache: 6 workers 12.2-12.4 ms to ready,
  // 12 workers 13.3-13.5, 16 workers 14.1; profiles/r02_c1_timeline.txt, r02_ring_sweep.jsonl).
  // Small teams (an explicit worker cap) are kept. $HL_SMALL_TEAM overrides.
  if (!cold_plan && total < (2ull << 30)) {
    const char* e = getenv("HL_SMALL_TEAM");
    const long v = e ? strtol(e, nullptr, 10) : (team >= 8 ? (long)(team + 1) / 2 : (long)team);
    team = (uint32_t)std::max(1L, std::min(v, (long)team));
  }
  // Chunk size. Plans under 2 GiB are cut into 2 MiB chunks: the pipeline fill
  // (first reads before any DMA) and drain are a visible part of a sub-second
  // load (GPT-2's 0.5 GB: 10.6 vs 11.3 ms engine at 4 MiB;
  // profiles/r02_c1_sweep.jsonl); large warm plans keep the slot size (4 MiB
  // measured best for them). Cold plans read 1 MiB O_DIRECT requests: the
  // storage rate follows the requests in flight, not their size (32 readers:
  // 1 MiB 5.87 GB/s, 2 MiB 5.27, 4 MiB 5.12 cold e2e on the same box, whose best
  // storage probe was io_uring depth 32 x 1 MiB; profiles/r02_cold_sweep.jsonl).
  // $HL_PLAN_CHUNK / $HL_COLD_CHUNK (bytes, <= the ring's slot size) override.
  uint64_t cb = ctx->cfg.chunk_bytes;
  if (total < (2ull << 30) && cb > (2ull << 20)) cb = 2ull << 20;
  if (cold_plan && cb > (1ull << 20)) cb = 1ull << 20;
  if (const char* e = getenv(cold_plan ? "HL_COLD_CHUNK" : "HL_PLAN_CHUNK")) {
    const uint64_t v = round_up(strtoull(e, nullptr, 10), kAlign);
    if (v >= kAlign && v <= ctx->cfg.chunk_bytes) cb = v;
  }
  for (const Chunk& r : ranges) {
    uint64_t o = r.off;
    const uint64_t end = r.off + r.len;
    while (o < end) {
      const uint64_t n = std::min<uint64_t>(round_down(o, cb) + cb, end) - o;
      chunks.push_back({r.file, o, n, r.dst + (o - r.off)});
      o += n;
    }
  }
  uint32_t nw = (uint32_t)std::min<size_t>(team, std::max<size_t>(chunks.size(), 1));
  uint32_t ring_workers = nw;
  // Cold plans on io_uring (default; $HL_COLD_URING=0 keeps the blocking readers):
  // $HL_URING_THREADS threads x $HL_URING_DEPTH reads in flight, using the slots
  // of the whole cold team. cuFile / mmap plans keep their own paths.
  const char* ue = getenv("HL_COLD_URING");
  if (cold_plan && !(ue && ue[0] == '0') && !(mode_mask & ((1u << HL_IO_CUFILE) | (1u << HL_IO_MMAP))) &&
      uring_available()) {
    auto env_u32 = [](const char* name, long dflt, long lo, long hi) {
      const char* v = getenv(name);
      return (uint32_t)std::max(lo, std::min(v ? strtol(v, nullptr, 10) : dflt, hi));
    };
    run.uring = std::min(env_u32("HL_URING_THREADS", 2, 1, 16), ctx->cold_workers);
    run.uring_depth = env_u32("HL_URING_DEPTH", 16, 1, 256);
    nw = (uint32_t)std::min<size_t>(run.uring, std::max<size_t>(chunks.size(), 1));
    run.uring = nw;
    // enough slots for every read in flight plus a few DMAs behind them: the warm team's
    // rings, grown if need be (not the whole 32-worker cold team's 384 MiB)
    const uint32_t spw = ctx->cfg.slots_per_worker;
    const uint32_t want = (nw * (run.uring_depth + 4) + spw - 1) / spw;
    ring_workers = std::min(ctx->cold_workers, std::max(std::max(ctx->cfg.workers, want), nw));
    run.uring_rings = ring_workers;
  }
  {
    double secs = 0;
    int rc = ensure_ring_memory(ctx, ring_workers, &secs);
    if (rc) {
      close_all();
      return rc;
    }
    run.ring_setup += secs;
  }
  const double t_dispatch = now_s();
  team_run(ctx, &run, nw);
  close_all();
  if (stats) {
    memset(stats, 0, sizeof *stats);
    stats->bytes = run.err_code == HL_OK ? total : 0;
    stats->seconds = now_s() - t0;
    stats->workers = nw;
    stats->blocks = n_blocks;
    stats->direct_bytes = run.direct_bytes.load();
    stats->buffered_bytes = run.buffered_bytes.load();
    stats->cufile_bytes = run.cufile_bytes.load();
    stats->mmap_bytes = run.mmap_bytes.load();
    stats->ring_setup_seconds = run.ring_setup;
    stats->io_mode_used = (run.buffered_bytes.load() ? 1u << HL_IO_BUFFERED : 0u) |
                          (run.direct_bytes.load() ? 1u << HL_IO_DIRECT : 0u) |
                          (run.cufile_bytes.load() ? 1u << HL_IO_CUFILE : 0u) |
                          (run.mmap_bytes.load() ? 1u << HL_IO_MMAP : 0u) |
                          (run.uring_bytes.load() ? HL_IO_USED_URING : 0u);
    stats->numa_node = ctx->cfg.numa_node;
    stats->read_seconds = run.read_ns.load() * 1e-9;
    stats->wait_seconds = run.wait_ns.load() * 1e-9;
    stats->submit_seconds = run.submit_ns.load() * 1e-9;
    stats->setup_seconds = t_dispatch - t0;
    stats->first_h2d_seconds = run.first_h2d_ns.load() == ~0ull ? 0.0 : run.first_h2d_ns.load() * 1e-9;
    stats->last_h2d_seconds = run.last_h2d_ns.load() * 1e-9;
  }
  if (run.err_code != HL_OK) return set_error(run.err_code, "%s", run.err_msg.c_str());
  return HL_OK;
}

extern "C" int hl_execute_plan(hl_ctx* ctx, const char* const* paths, uint32_t n_files, const hl_block* blocks,
                               uint32_t n_blocks, hl_plan_stats* stats) {
  return execute(ctx, paths, n_files, blocks, n_blocks, false, nullptr, stats);
}

extern "C" int hl_execute_plan_after(hl_ctx* ctx, const char* const* paths, uint32_t n_files,
                                     const hl_block* blocks, uint32_t n_blocks, void* stream,
                                     hl_plan_stats* stats) {
  return execute(ctx, paths, n_files, blocks, n_blocks, true, (cudaStream_t)stream, stats);
}

extern "C" int hl_execute_plan_async(hl_ctx* ctx, const char* const* paths, uint32_t n_files,
                                     const hl_block* blocks, uint32_t n_blocks, void* stream,
                                     hl_plan_stats* stats) {
  return execute(ctx, paths, n_files, blocks, n_blocks, true, (cudaStream_t)stream, stats, true);
}

extern "C" int hl_transfer_from_file(hl_ctx* ctx, const char* path, uint64_t file_off, uint64_t len, void* dev_dst) {
  hl_block b{0, 0, file_off, len, (uint64_t)(uintptr_t)dev_dst};
  if (len == 0) return HL_OK;
  return hl_execute_plan(ctx, &path, 1, &b, 1, nullptr);
}

extern "C" int hl_ctx_cpus(const hl_ctx* ctx, int32_t* cpus, uint32_t cap, uint32_t* n_cpus) {
  clear_error();
  if (!ctx || !n_cpus) return set_error(HL_EINVAL, "null argument");
  *n_cpus = (uint32_t)ctx->cpus.size();
  for (uint32_t i = 0; cpus && i < cap && i < ctx->cpus.size(); ++i) cpus[i] = ctx->cpus[i];
  return HL_OK;
}

extern "C" int hl_topology_resolve(const char* pci_bus_id, int32_t requested_node, int32_t* node, int32_t* cpus,
                                   uint32_t cap, uint32_t* n_cpus) {
  clear_error();
  if (!node || !n_cpus) return set_error(HL_EINVAL, "null argument");
  *node = resolve_node(pci_bus_id, requested_node);
  const std::vector<int> c = node_cpus(*node);
  *n_cpus = (uint32_t)c.size();
  for (uint32_t i = 0; cpus && i < cap && i < c.size(); ++i) cpus[i] = c[i];
  return HL_OK;
}

extern "C" int hl_storage_numa_node(const char* path, int32_t* node) {
  clear_error();
  if (!path || !node) return set_error(HL_EINVAL, "null argument");
  *node = storage_numa_node(path);
  return HL_OK;
}

extern "C" int hl_file_residency(const char* path, double* frac) {
  clear_error();
  if (!path || !frac) return set_error(HL_EINVAL, "null argument");
  int fd = open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) return set_error(HL_EIO, "cannot open %s: %s", path, strerror(errno));
  struct stat st;
  fstat(fd, &st);
  *frac = residency(fd, (uint64_t)st.st_size);
  close(fd);
  return HL_OK;
}

extern "C" int hl_drop_cache(const char* path) {
  clear_error();
  if (!path) return set_error(HL_EINVAL, "null path");
  int fd = open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) return set_error(HL_EIO, "cannot open %s: %s", path, strerror(errno));
  fdatasync(fd);
  int rc = posix_fadvise(fd, 0, 0, POSIX_FADV_DONTNEED);
  close(fd);
  if (rc) return set_error(HL_EIO, "posix_fadvise(%s): %s", path, strerror(rc));
  return HL_OK;
}

extern "C" int hl_gds_available(void) {
  return access("/proc/driver/nvidia-fs/stats", R_OK) == 0 ? 1 : 0;
}
