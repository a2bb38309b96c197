/*
 * hbmload.h — C ABI of the B200 load path (libhbmload.so).
 *
 * This is the drop-in boundary underneath the loader API
 * (SafeTensorsFileLoader.add_filenames / copy_files_to_device / get_tensor /
 * get_sharded / close). The host side (paper_2505_23072_b200/, Python, like the
 * reference) keeps the reference's semantics and calls these entry points for
 * everything that touches bytes:
 *
 *   bulk file -> HBM I/O         hl_ctx_create / hl_execute_plan(_after/_async) /
 *                                hl_transfer_from_file (pinned ring + per-worker H2D streams;
 *                                cold plans on io_uring O_DIRECT reads)
 *   realign / shard / cast       hl_gather (one batched sm_100a entry point, descriptor table;
 *                                TMA bulk-copy / TMA-staged kernels for contiguous tensors,
 *                                2-D tensor-map TMA tiles for column shards, LDG/STG warp
 *                                kernels for the rest and for peer pulls)
 *   peer memory                  hl_ipc_export / hl_ipc_import / hl_enable_peer_access
 *   placement                    hl_topology_resolve / hl_ctx_cpus / hl_storage_numa_node
 *   page-cache control           hl_file_residency / hl_drop_cache
 *   measurement                  hl_kernel_launches / hl_gather_timing(s)
 *
 * Conventions
 *   - Plain C types only: pointers, sizes, integers. No torch types. Device
 *     memory is always owned by the caller (the torch caching allocator on the
 *     Python side); the library never frees caller memory. The library owns
 *     only its pinned host ring, file descriptors and CUDA streams/events.
 *   - Every entry point returns an int status: 0 = HL_OK, negative = error.
 *     hl_last_error() returns a thread-local, human-readable message for the
 *     last failing call on the calling thread. Codes map 1:1 onto the
 *     reference's typed errors (pkg/src/aggload/errors.py:57-102).
 *   - Streams are passed as void* (a cudaStream_t / CUstream; NULL = legacy
 *     default stream).
 *
 * Reference interfaces replaced (pkg/src/aggload/...):
 *   hl_execute_plan(_after) transfer.py:305-389 execute_plan(plan, pools)
 *   hl_topology_resolve    transfer.py:51-121, 274-293  Topology / worker NUMA affinity
 *   hl_transfer_from_file  device.py:238-288    transfer_from_file(buf, dev_off, file, file_off, length, staging)
 *   hl_gather              device.py:466-534    align_and_convert(buf, landing, bounce, conversions)
 *                          device.py:551-586    convert_dtype(buf, view_meta, target, bounce)
 *                          collective.py:313-330 _clone_full / _clone_slice (owner-side shard pack)
 *                          loader.py:490-499    FilesBufferOnDevice._clone_of (auto-release copy)
 *   hl_conversion_supported device.py:293-298   _CONVERSIONS
 *   hl_file_residency / hl_drop_cache  cli.py:177-186 (fadvise-cold bench pass)
 */
#ifndef HBMLOAD_H_
#define HBMLOAD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HL_ABI_VERSION 2  /* 2: hl_execute_plan_after/_async, hl_ctx_cpus, hl_topology_resolve, stats.numa_node */

/* ---- status codes (errors.py class in brackets) ---------------------------- */
enum hl_status {
  HL_OK = 0,
  HL_EIO = -1,      /* [IoError]                  read/open failure, short read   */
  HL_EALIGN = -2,   /* [MisalignedDirectTransfer] alignment contract violated     */
  HL_ENOMEM = -3,   /* [OutOfMemory]              pinned/host allocation failure  */
  HL_EBOUNCE = -4,  /* [BounceTooSmall]           staging slot cannot hold a chunk */
  HL_ECONV = -5,    /* [UnsupportedConversion]    dtype pair not supported        */
  HL_EBOUNDS = -6,  /* [OutOfBoundsView]          range outside a buffer          */
  HL_ECUDA = -7,    /* [DeviceError]              CUDA runtime failure            */
  HL_EINVAL = -8    /* [ValueError]               bad argument                    */
};

/* ---- dtype codes: the order of format.DType (ref format.py:48-63) ----------- */
enum hl_dtype {
  HL_DT_BOOL = 0, HL_DT_U8 = 1, HL_DT_I8 = 2, HL_DT_I16 = 3, HL_DT_U16 = 4,
  HL_DT_I32 = 5, HL_DT_U32 = 6, HL_DT_I64 = 7, HL_DT_U64 = 8, HL_DT_F16 = 9,
  HL_DT_BF16 = 10, HL_DT_F32 = 11, HL_DT_F64 = 12
};

/* ---- I/O modes ----------------------------------------------------------------- */
enum hl_io_mode {
  HL_IO_AUTO = 0,      /* per chunk: the page-cache-resident prefix (mincore) buffered,
                          the rest O_DIRECT                                             */
  HL_IO_BUFFERED = 1,  /* pread through the page cache into the pinned ring            */
  HL_IO_DIRECT = 2,    /* O_DIRECT pread (4 KiB aligned) into the pinned ring            */
  HL_IO_CUFILE = 3,    /* cuFileRead straight into HBM (GPUDirect Storage, nvidia-fs)    */
  HL_IO_MMAP = 4       /* page-cache pages pinned in place (mmap + cudaHostRegister) and
                          DMA'd straight to HBM: no CPU copy                                */
};

const char* hl_version(void);
const char* hl_last_error(void);
int hl_abi_version(void);

/* ---- bulk file -> HBM engine ------------------------------------------------------ */
typedef struct hl_ctx hl_ctx;

typedef struct hl_config {
  int32_t device;            /* CUDA ordinal the engine copies into                       */
  uint32_t workers;          /* I/O threads (0 = library default: 0.8 x node CPUs, cap 16) */
  uint64_t chunk_bytes;      /* bytes per pread + H2D hop (0 = 16 MiB; rounded to 4 KiB)   */
  uint32_t slots_per_worker; /* pinned ring depth per worker (0 = 3)                       */
  uint32_t io_mode;          /* enum hl_io_mode                                            */
  int32_t numa_node;         /* pin workers + ring to this node; -1 = the GPU's node       */
  uint32_t flags;            /* HL_CFG_* bits                                              */
} hl_config;

/* HL_IO_AUTO: a chunk whose pages are all in the page cache is DMA'd straight
 * from those pages (pinned in place with cudaHostRegister, like HL_IO_MMAP)
 * instead of being copied into the pinned ring first: each delivered byte
 * crosses host DRAM once instead of three times (page cache read + ring write
 * + DMA read), which is what lets 8 GPUs of one host load warm files at once. */
#define HL_CFG_AUTO_PIN_CACHE 1u

/* One transfer block: file bytes [file_off, file_off+len) -> device address dev_dst.
 * Mirrors transfer.TransferBlock (ref transfer.py:135-142). */
typedef struct hl_block {
  uint32_t file;      /* index into the paths[] array of hl_execute_plan */
  uint32_t worker;    /* planner's worker hint (blocks are claimed dynamically) */
  uint64_t file_off;
  uint64_t len;
  uint64_t dev_dst;
} hl_block;

/* io_mode_used bit: some O_DIRECT reads were issued through io_uring (cold plans). */
#define HL_IO_USED_URING (1u << 5)

/* Mirrors transfer.PlanStats (ref transfer.py:167-188) plus the I/O mode actually used. */
typedef struct hl_plan_stats {
  uint64_t bytes;           /* file bytes moved to HBM                        */
  double seconds;           /* wall time of the whole plan                    */
  uint32_t workers;
  uint32_t blocks;
  uint64_t direct_bytes;    /* bytes read with O_DIRECT                       */
  uint64_t buffered_bytes;  /* bytes read through the page cache              */
  uint64_t cufile_bytes;    /* bytes read by cuFile                           */
  uint64_t mmap_bytes;      /* bytes DMA'd from pinned page-cache pages        */
  double ring_setup_seconds;/* pinned ring allocation charged to this call    */
  uint32_t io_mode_used;    /* bitmask of 1<<hl_io_mode actually used, | HL_IO_USED_URING */
  int32_t numa_node;        /* node the workers and the ring are pinned to (-1: none) */
  double read_seconds;      /* sum over workers: time inside pread / cuFileRead / pinning */
  double wait_seconds;      /* sum over workers: time waiting for a ring slot's DMA      */
  double submit_seconds;    /* sum over workers: time inside cudaMemcpyAsync/EventRecord */
  double setup_seconds;     /* plan start -> worker team dispatched (files opened, chunks cut) */
  double first_h2d_seconds; /* plan start -> first H2D copy submitted                        */
  double last_h2d_seconds;  /* plan start -> last H2D copy submitted (then the drain)        */
} hl_plan_stats;

int hl_ctx_create(const hl_config* cfg, hl_ctx** out);
int hl_ctx_destroy(hl_ctx* ctx);
/* Effective configuration (defaults resolved). */
int hl_ctx_config(const hl_ctx* ctx, hl_config* out);

/* Run every block; blocks until all bytes are resident in HBM (all H2D
 * copies complete). On failure no partial success is reported: the caller
 * discards the destination buffers (ref transfer.py:375-378).
 * The engine writes HBM from its own streams: hl_execute_plan does NOT order
 * those writes after work the caller queued earlier. Use it only for
 * destinations no queued kernel may still read. */
int hl_execute_plan(hl_ctx* ctx, const char* const* paths, uint32_t n_files,
                    const hl_block* blocks, uint32_t n_blocks, hl_plan_stats* stats);

/* hl_execute_plan whose writes are ordered after everything enqueued on
 * `stream` before the call (an event recorded there is waited on by every
 * engine stream; the cuFile path waits on the host). This is what a caller
 * with a stream-ordered allocator needs: memory recycled from a buffer that
 * kernels queued on `stream` still read is not overwritten before they ran.
 * NULL = the legacy default stream. The loader always uses this entry. */
int hl_execute_plan_after(hl_ctx* ctx, const char* const* paths, uint32_t n_files,
                          const hl_block* blocks, uint32_t n_blocks, void* stream,
                          hl_plan_stats* stats);

/* hl_execute_plan_after that returns once every byte has been read from
 * storage and its H2D copy submitted, instead of draining the copies: `stream`
 * is made to wait for all of them (cudaStreamWaitEvent), so work enqueued on
 * it afterwards — kernels, stream-ordered frees, a D2H read — sees the bytes,
 * while the host goes on (the drain of the last copies overlaps the caller's
 * next steps). Host access to the destinations needs a sync of `stream`.
 * Read errors are reported here as before. */
int hl_execute_plan_async(hl_ctx* ctx, const char* const* paths, uint32_t n_files,
                          const hl_block* blocks, uint32_t n_blocks, void* stream,
                          hl_plan_stats* stats);

/* Single range, synchronous (ref device.py:238). */
int hl_transfer_from_file(hl_ctx* ctx, const char* path, uint64_t file_off,
                          uint64_t len, void* dev_dst);

/* The CPUs the context's worker team and pinned ring are bound to (the
 * node's sysfs cpulist intersected with the process affinity). *n_cpus gets
 * the full count; at most `cap` are written. */
int hl_ctx_cpus(const hl_ctx* ctx, int32_t* cpus, uint32_t cap, uint32_t* n_cpus);
/* The placement rule without a GPU: node = requested_node if >= 0, else
 * $HL_NUMA_NODE, else the PCI device's sysfs numa_node; CPUs as hl_ctx_cpus.
 * sysfs is read under $HL_SYSFS_ROOT when that is set (ref transfer.py:51-121
 * Topology / 274-293 worker affinity). */
int hl_topology_resolve(const char* pci_bus_id, int32_t requested_node, int32_t* node, int32_t* cpus,
                        uint32_t cap, uint32_t* n_cpus);
/* NUMA node of the storage device holding `path` (the NVMe / virtio / HBA PCI
 * function that /sys/dev/block/MAJ:MIN resolves to; honours $HL_SYSFS_ROOT),
 * -1 when unknown (tmpfs, overlay). Reported beside the engine's node: the ring
 * stays on the GPU's node (H2D reads it every byte), so a different storage node
 * means O_DIRECT DMA crosses the socket link once (ref transfer.py:51-121). */
int hl_storage_numa_node(const char* path, int32_t* node);

/* Fraction of the file's pages resident in the page cache (mincore). */
int hl_file_residency(const char* path, double* frac);
/* posix_fadvise(DONTNEED) over the whole file: the reference's cold pass. */
int hl_drop_cache(const char* path);
/* Is GPUDirect Storage (nvidia-fs) usable on this host? 1 yes, 0 no. */
int hl_gds_available(void);

/* ---- peer memory: the multi-GPU data plane without a collective library ---------------
 * A rank exports the HBM buffer holding its landed files once; every other rank
 * imports it and its own hl_gather launch then reads the slice it needs straight
 * out of the owner's HBM over NVLink (peer loads), slicing and casting on the
 * way: the transfer and the shard/cast are one kernel (replaces the reference's
 * broadcast/scatter data movement, collective.py:175-255). Within one process,
 * hl_enable_peer_access gives the same for device pointers of other GPUs. */
typedef struct hl_ipc_handle {
  uint8_t handle[64];  /* cudaIpcMemHandle_t of the allocation containing the pointer */
  uint64_t offset;     /* byte offset of the pointer inside that allocation           */
} hl_ipc_handle;

int hl_ipc_export(const void* dev_ptr, hl_ipc_handle* out);
/* Open (reference counted per allocation) and return base + offset in this process. */
int hl_ipc_import(const hl_ipc_handle* h, int device, void** out_ptr);
/* Drop one reference taken by hl_ipc_import (by the pointer it returned). */
int hl_ipc_release(void* ptr);
int hl_enable_peer_access(int device, int peer);

/* ---- batched gather / realign / shard / cast ----------------------------------------
 * One descriptor = one strided 2-D copy with optional dtype conversion:
 *   for r in [0, rows): for c in [0, row_elems):
 *     dst[(r*row_elems + c) * size(dst_dtype)] = convert(src[r*src_pitch + c*size(src_dtype)])
 * src may sit at ANY byte address (misaligned landings are realigned here);
 * dst must be aligned to the destination element size (16 B for the vector path).
 * Shards: a rank's slice [lo,hi) along dim d of a row-major tensor of shape S is
 *   rows = prod(S[:d]), row_elems = (hi-lo)*prod(S[d+1:]),
 *   src = base + lo*prod(S[d+1:])*esize, src_pitch = S[d]*prod(S[d+1:])*esize.
 * Conversions are bit-exact with the reference (numpy) semantics:
 *   BF16->F16, F32->F16 (RNE, overflow -> inf, NaN payload = mant>>13 forced
 *   non-zero, no quieting), F16->F32 (exact, payload kept), BF16->F32 (bits<<16).
 */
typedef struct hl_desc {
  uint64_t src;        /* device byte address of element (0,0)           */
  uint64_t dst;        /* device byte address of the contiguous output   */
  uint64_t rows;
  uint64_t row_elems;
  uint64_t src_pitch;  /* bytes between consecutive source rows          */
  uint32_t src_dtype;  /* enum hl_dtype */
  uint32_t dst_dtype;  /* enum hl_dtype */
} hl_desc;

/* 1 if src->dst is supported (identity for every dtype, plus the four casts). */
int hl_conversion_supported(uint32_t src_dtype, uint32_t dst_dtype);

/* Enqueue the whole batch on `stream` (kernel launches only: no host sync, no
 * allocation; the descriptor table travels in the launch's parameter buffer,
 * up to hl_gather_max_batch() descriptors per launch; one launch per kernel
 * variant present: TMA bulk copy, TMA-staged cast/realign, row, element). */
int hl_gather(const hl_desc* descs, uint32_t n, void* stream);

/* hl_gather with flags. HL_GATHER_NO_TMA keeps every descriptor on the LDG/STG
 * warp kernels: the loader sets it when sources are another GPU's memory (peer
 * pulls over NVLink), whose rate is set by the link, not by the copy engine of
 * the SM. hl_gather(d, n, s) == hl_gather_ex(d, n, s, 0). */
#define HL_GATHER_NO_TMA 1u
int hl_gather_ex(const hl_desc* descs, uint32_t n, void* stream, uint32_t flags);
uint32_t hl_gather_max_batch(void);

/* Number of kernel launches hl_gather issued by this process so far. */
uint64_t hl_kernel_launches(void);
/* Launch timing for measurements (bench.py roofline): while enabled, every
 * hl_gather call records a CUDA event pair on its stream around its kernel
 * launches (after the host-side descriptor translation). hl_gather_timings
 * waits for the recorded pairs, writes their elapsed milliseconds in call
 * order (up to cap; *n = how many were recorded) and forgets them.
 * hl_gather_timing(0/1) switches it and drops pending pairs. */
int hl_gather_timing(int enable);
int hl_gather_timings(float* ms, uint32_t cap, uint32_t* n);

/* Load every hl_gather kernel variant for `device` ahead of use (CUDA loads
 * kernels lazily): call once per process, e.g. on a side thread while the first
 * transfer runs. Idempotent; no launches. */
int hl_gather_prepare(int device);

#ifdef __cplusplus
}
#endif
#endif /* HBMLOAD_H_ */
