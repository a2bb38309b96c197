// tile_probe.cu — minimal 2-D TMA box copy (one box per CTA) to validate
// tensor-map parameters on the box: src matrix rows x pitch (elements of
// `eb` bytes), segment [c0, c0+cols) -> dense dst. Variant 0: maps as two
// separate __grid_constant__ params; 1: maps inside a struct param (as
// hl_gather's tile kernels).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/build/tile_probe tools/tile_probe.cu
//   tools/build/tile_probe EB C0 ROWS COLS PITCH_ELEMS BX BY VARIANT
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <vector>

struct alignas(64) Two { CUtensorMap s, d; int nbx, bx, by, c0; unsigned bytes; };

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ void box(const CUtensorMap* s, const CUtensorMap* d, int nbx, int bx, int by, int c0, unsigned bytes) {
  extern __shared__ __align__(128) unsigned char st[];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x) return;
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int x = (blockIdx.x % nbx) * bx, y = (blockIdx.x / nbx) * by;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               :: "r"(su(st)), "l"(s), "r"(c0 + x), "r"(y), "r"(su(&bar)) : "memory");
  asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" :: "r"(su(&bar)) : "memory");
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];"
               :: "l"(d), "r"(x), "r"(y), "r"(su(st)) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__global__ void k0(const __grid_constant__ CUtensorMap s, const __grid_constant__ CUtensorMap d, int nbx, int bx, int by,
                   int c0, unsigned bytes) { box(&s, &d, nbx, bx, by, c0, bytes); }
__global__ void k1(const __grid_constant__ Two t) { box(&t.s, &t.d, t.nbx, t.bx, t.by, t.c0, t.bytes); }

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  if (argc < 9) return 2;
  const int eb = atoi(argv[1]), c0 = atoi(argv[2]), rows = atoi(argv[3]), cols = atoi(argv[4]), pitch = atoi(argv[5]);
  const int bx = atoi(argv[6]), by = atoi(argv[7]), variant = atoi(argv[8]);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = (Enc)fp;
  const size_t sbytes = (size_t)rows * pitch * eb, dbytes = (size_t)rows * cols * eb;
  std::vector<unsigned char> h(sbytes);
  for (size_t i = 0; i < sbytes; ++i) h[i] = (unsigned char)(i * 131 + 7);
  unsigned char *s, *d;
  cudaMalloc(&s, sbytes);
  cudaMalloc(&d, dbytes);
  cudaMemcpy(s, h.data(), sbytes, cudaMemcpyHostToDevice);
  cudaMemset(d, 0xA5, dbytes);
  CUtensorMapDataType ty = eb == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : eb == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                         : eb == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64;
  Two t;
  memset(&t, 0, sizeof t);
  cuuint64_t sd[2] = {(cuuint64_t)(c0 + cols), (cuuint64_t)rows}, ss[1] = {(cuuint64_t)pitch * eb};
  cuuint64_t dd[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, ds[1] = {(cuuint64_t)cols * eb};
  cuuint32_t b[2] = {(cuuint32_t)bx, (cuuint32_t)by}, e[2] = {1, 1};
  CUresult r1 = enc(&t.s, ty, 2, s, sd, ss, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&t.d, ty, 2, d, dd, ds, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  t.nbx = (cols + bx - 1) / bx;
  t.bx = bx;
  t.by = by;
  t.c0 = c0;
  t.bytes = (unsigned)(bx * by * eb);
  const int grid = t.nbx * ((rows + by - 1) / by);
  const size_t smem = (size_t)bx * by * eb;
  cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (variant == 0) k0<<<grid, 32, smem>>>(t.s, t.d, t.nbx, bx, by, c0, t.bytes);
  else k1<<<grid, 32, smem>>>(t);
  cudaError_t err = cudaDeviceSynchronize();
  std::vector<unsigned char> o(dbytes);
  cudaMemcpy(o.data(), d, dbytes, cudaMemcpyDeviceToHost);
  size_t bad = 0;
  for (int y = 0; y < rows; ++y)
    for (size_t x = 0; x < (size_t)cols * eb; ++x)
      bad += o[(size_t)y * cols * eb + x] != h[(size_t)y * pitch * eb + (size_t)c0 * eb + x];
  printf("{\"eb\": %d, \"c0\": %d, \"rows\": %d, \"cols\": %d, \"pitch\": %d, \"box\": [%d, %d], \"variant\": %d, "
         "\"encode\": [%d, %d], \"err\": \"%s\", \"bad_bytes\": %zu}\n",
         eb, c0, rows, cols, pitch, bx, by, variant, (int)r1, (int)r2, cudaGetErrorString(err), bad);
  return err != cudaSuccess || bad;
}
