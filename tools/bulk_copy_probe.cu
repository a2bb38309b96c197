// bulk_copy_probe.cu — does a TMA bulk-copy pipeline (cp.async.bulk global ->
// shared -> global, one elected thread per CTA, mbarrier-completed loads,
// bulk_group stores) move HBM bytes faster than hl_gather's copy path
// (16-byte ld.global.nc / st.global.cs, 8 vectors in flight per lane,
// persistent grid)? Same buffer, same bytes, CUDA events, best of N.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/bulk_copy_probe tools/bulk_copy_probe.cu
//   /tmp/bulk_copy_probe [GiB=6.75] [reps=10]     (one JSON line per variant)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

// ------------------------------------------------------------ LDG/STG baseline (hl_gather's copy path)
__global__ void __launch_bounds__(256) ldg_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, uint64_t nvec) {
  const uint64_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * 8ull) + (threadIdx.x >> 5);
  const uint64_t nwarps = gridDim.x * 8ull;
  constexpr int U = 8;
  for (uint64_t base = warp * 32 * U; base < nvec; base += nwarps * 32 * U) {
    uint4 v[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint64_t j = base + i * 32 + lane;
      if (j < nvec) asm("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[i].x), "=r"(v[i].y), "=r"(v[i].z), "=r"(v[i].w) : "l"(src + j));
    }
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint64_t j = base + i * 32 + lane;
      if (j < nvec) asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dst + j), "r"(v[i].x), "r"(v[i].y), "r"(v[i].z), "r"(v[i].w) : "memory");
    }
  }
}

// ------------------------------------------------------------ TMA bulk pipeline
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" :: "r"(smem_addr(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               :: "r"(smem_addr(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_addr(bar)), "l"(policy) : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
               :: "l"(gdst), "r"(smem_addr(ssrc)), "r"(bytes), "l"(policy) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// One warp per CTA, lane 0 issues. Chunk c of the buffer goes to stage c % S.
// Loads run S - LAG chunks ahead of the stores; a stage is reloaded once the
// store that read it has finished reading (wait_group.read LAG).
template <int S, int LAG>
__global__ void __launch_bounds__(32) bulk_copy(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                uint64_t bytes, uint32_t chunk) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[S];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint64_t policy = evict_first_policy();
  const uint64_t nchunks = (bytes + chunk - 1) / chunk;
  // this CTA's chunks: blockIdx.x, blockIdx.x + grid, ...
  const uint64_t mine = blockIdx.x < nchunks ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto chunk_of = [&](uint64_t k) { return blockIdx.x + k * gridDim.x; };
  auto len_of = [&](uint64_t c) { return (uint32_t)(c == nchunks - 1 ? bytes - c * chunk : chunk); };
  const uint64_t ahead = S - LAG;
  for (uint64_t k = 0; k < mine && k < ahead; ++k) {
    const uint64_t c = chunk_of(k);
    const int s = (int)(k % S);
    mbar_expect_tx(&bars[s], len_of(c));
    bulk_load(smem + (size_t)s * chunk, src + c * chunk, len_of(c), &bars[s], policy);
  }
  for (uint64_t k = 0; k < mine; ++k) {
    const uint64_t c = chunk_of(k);
    const int s = (int)(k % S);
    mbar_wait(&bars[s], (uint32_t)((k / S) & 1));
    bulk_store(dst + c * chunk, smem + (size_t)s * chunk, len_of(c), policy);
    bulk_commit();
    const uint64_t kn = k + ahead;  // next load goes to stage kn % S, last read by store kn - S = k - LAG
    if (kn < mine) {
      bulk_wait_read<LAG>();
      const uint64_t cn = chunk_of(kn);
      const int sn = (int)(kn % S);
      mbar_expect_tx(&bars[sn], len_of(cn));
      bulk_load(smem + (size_t)sn * chunk, src + cn * chunk, len_of(cn), &bars[sn], policy);
    }
  }
  bulk_wait_all();
}

template <class F>
static float best_ms(F launch, int reps, uint8_t* flush, size_t flush_bytes) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int r = 0; r < reps + 2; ++r) {
    CK(cudaMemsetAsync(flush, r, flush_bytes));  // L2 flush between reps
    CK(cudaEventRecord(a));
    launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (r >= 2 && ms < best) best = ms;
  }
  return best;
}

template <int S, int LAG>
static void run_bulk(const uint8_t* s, uint8_t* d, uint64_t bytes, uint32_t chunk, int ctas_per_sm, int sms, int reps,
                     uint8_t* flush, size_t fb, const uint8_t* ref_src) {
  const size_t smem = (size_t)S * chunk;
  auto k = bulk_copy<S, LAG>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 32, smem));
  if (occ < ctas_per_sm) return;
  const unsigned grid = (unsigned)(sms * ctas_per_sm);
  CK(cudaMemset(d, 0, bytes));
  float ms = best_ms([&] { k<<<grid, 32, smem>>>(s, d, bytes, chunk); }, reps, flush, fb);
  // verify a few spots
  uint8_t h1[64], h2[64];
  for (uint64_t off : {(uint64_t)0, bytes / 3, bytes - 64}) {
    CK(cudaMemcpy(h1, ref_src + off, 64, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2, d + off, 64, cudaMemcpyDeviceToHost));
    for (int i = 0; i < 64; ++i) if (h1[i] != h2[i]) { printf("{\"error\": \"mismatch\"}\n"); exit(2); }
  }
  printf("{\"variant\": \"tma_bulk\", \"stages\": %d, \"lag\": %d, \"chunk_kb\": %u, \"ctas_per_sm\": %d, "
         "\"smem_kb\": %zu, \"ms\": %.3f, \"GBps\": %.1f}\n",
         S, LAG, chunk >> 10, ctas_per_sm, smem >> 10, ms, 2.0 * bytes / ms / 1e6);
  fflush(stdout);
}

int main(int argc, char** argv) {
  const double gib = argc > 1 ? atof(argv[1]) : 6.75;
  const int reps = argc > 2 ? atoi(argv[2]) : 10;
  const uint64_t bytes = (uint64_t)(gib * (1ull << 30)) & ~(uint64_t)4095;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint8_t *s, *d, *flush;
  const size_t fb = 256ull << 20;
  CK(cudaMalloc(&s, bytes));
  CK(cudaMalloc(&d, bytes));
  CK(cudaMalloc(&flush, fb));
  CK(cudaMemset(s, 0x5a, bytes));
  CK(cudaMemset(s + bytes / 3, 0x17, 4096));
  // baseline: LDG/STG, 4 blocks of 256 per SM (hl_gather's resident grid)
  for (int bps : {4, 8}) {
    float ms = best_ms([&] { ldg_copy<<<sms * bps, 256>>>((const uint4*)s, (uint4*)d, bytes / 16); }, reps, flush, fb);
    printf("{\"variant\": \"ldg_stg_v4\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"GBps\": %.1f}\n", bps, ms, 2.0 * bytes / ms / 1e6);
  }
  {
    float ms = best_ms([&] { CK(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice)); }, reps, flush, fb);
    printf("{\"variant\": \"cudaMemcpy_d2d\", \"ms\": %.3f, \"GBps\": %.1f}\n", ms, 2.0 * bytes / ms / 1e6);
  }
  fflush(stdout);
  for (uint32_t chunk : {16u << 10, 32u << 10}) {
    for (int cps : {1, 2, 3}) {
      run_bulk<4, 1>(s, d, bytes, chunk, cps, sms, reps, flush, fb, s);
      run_bulk<6, 2>(s, d, bytes, chunk, cps, sms, reps, flush, fb, s);
      run_bulk<8, 2>(s, d, bytes, chunk, cps, sms, reps, flush, fb, s);
      run_bulk<12, 3>(s, d, bytes, chunk, cps, sms, reps, flush, fb, s);
    }
  }
  return 0;
}
