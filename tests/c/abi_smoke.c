/* abi_smoke.c — the C ABI used from plain C, no Python and no torch: the
 * boundary a non-Python host (the reference's cgo / JNI / N-API binding, see
 * INTEGRATION.md) would call.
 *
 *   abi_smoke FILE OUT
 *
 * 1. hl_execute_plan_after: the whole FILE -> one cudaMalloc'd device buffer A
 * 2. hl_gather, one launch per kind:
 *      B = A[3 : 3 + nb]               (U8 copy from a misaligned source: realign)
 *      C = bf16 -> f16 of A[16 : 16 + 2*nc]
 *      D = rank 1 of 3 of a [rows, cols] bf16 tensor at A[64:] sliced along dim 1
 * 3. B || C || D -> OUT (host), checked by tests/test_abi.py against the oracle.
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/stat.h>

#include "hbmload.h"

#define CHECK(x)                                                             \
  do {                                                                       \
    int rc_ = (x);                                                           \
    if (rc_) {                                                               \
      fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, hl_last_error());     \
      return 1;                                                              \
    }                                                                        \
  } while (0)

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  struct stat st;
  if (stat(argv[1], &st)) return 2;
  const uint64_t size = (uint64_t)st.st_size;
  const uint64_t nb = 100003, nc = 65536, rows = 37, cols = 300, lo = 100, hi = 200;
  if (size < 64 + rows * cols * 2 || size < 16 + 2 * nc || size < 3 + nb) return 2;
  printf("abi %d version %s gds %d\n", hl_abi_version(), hl_version(), hl_gds_available());

  hl_config cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.device = 0;
  cfg.workers = 2;
  cfg.chunk_bytes = 1 << 20;
  cfg.io_mode = HL_IO_AUTO;
  cfg.numa_node = -1;
  hl_ctx* ctx = NULL;
  CHECK(hl_ctx_create(&cfg, &ctx));

  uint8_t *a = NULL, *out = NULL;
  const uint64_t ob = (nb + 15) / 16 * 16, oc = nc * 2, od = rows * (hi - lo) * 2;
  if (cudaMalloc((void**)&a, size + 16) || cudaMalloc((void**)&out, ob + oc + od)) return 3;
  const char* paths[1] = {argv[1]};
  hl_block blk = {0, 0, 0, size, (uint64_t)(uintptr_t)a};
  hl_plan_stats stats;
  CHECK(hl_execute_plan_after(ctx, paths, 1, &blk, 1, NULL, &stats));
  printf("landed %llu bytes in %.4f s\n", (unsigned long long)stats.bytes, stats.seconds);

  hl_desc d[3];
  memset(d, 0, sizeof d);
  d[0] = (hl_desc){(uint64_t)(uintptr_t)(a + 3), (uint64_t)(uintptr_t)out, 1, nb, nb, HL_DT_U8, HL_DT_U8};
  d[1] = (hl_desc){(uint64_t)(uintptr_t)(a + 16), (uint64_t)(uintptr_t)(out + ob), 1, nc, 2 * nc, HL_DT_BF16,
                   HL_DT_F16};
  d[2] = (hl_desc){(uint64_t)(uintptr_t)(a + 64 + lo * 2), (uint64_t)(uintptr_t)(out + ob + oc), rows, hi - lo,
                   cols * 2, HL_DT_BF16, HL_DT_BF16};
  if (!hl_conversion_supported(HL_DT_BF16, HL_DT_F16) || hl_conversion_supported(HL_DT_F64, HL_DT_F16)) return 4;
  const uint64_t before = hl_kernel_launches();
  CHECK(hl_gather(d, 3, NULL));
  if (cudaDeviceSynchronize()) return 3;
  printf("launches %llu\n", (unsigned long long)(hl_kernel_launches() - before));

  uint8_t* host = (uint8_t*)malloc(ob + oc + od);
  if (cudaMemcpy(host, out, ob + oc + od, cudaMemcpyDeviceToHost)) return 3;
  FILE* f = fopen(argv[2], "wb");
  fwrite(host, 1, nb, f);
  fwrite(host + ob, 1, oc, f);
  fwrite(host + ob + oc, 1, od, f);
  fclose(f);
  free(host);
  cudaFree(a);
  cudaFree(out);
  CHECK(hl_ctx_destroy(ctx));
  /* a typed error through the ABI: unsupported conversion */
  d[0].src_dtype = HL_DT_F64;
  d[0].dst_dtype = HL_DT_F16;
  if (hl_gather(d, 1, NULL) != HL_ECONV) return 5;
  printf("error path ok: %s\n", hl_last_error());
  return 0;
}
