// hl_gather.cu — the batched gather / realign / shard / cast kernel (sm_100a).
//
// One launch processes a whole table of descriptors (include/hbmload.h,
// hl_desc). Each descriptor is a strided 2-D copy with an optional dtype
// conversion; together they express every byte-moving step of the loader:
//   * realign   — a tensor that landed at a misaligned device offset (odd
//                 header, GDS-style aligned landing) is copied to an aligned
//                 slot (ref device.py:466-534 align_and_convert, in place there,
//                 out of place here),
//   * clone     — auto_release copy of a tensor out of its file buffer
//                 (ref loader.py:490-499 _clone_of),
//   * shard     — a rank's slice along dim d (ref collective.py:318-330
//                 _clone_slice; rows = prod(shape[:d])),
//   * cast      — BF16/F32 -> F16 and F16/BF16 -> F32, bit-exact with the
//                 reference's numpy conversions (ref device.py:303-320).
//
// Work decomposition (no tensor cores: this is HBM-bound byte movement):
//   * The table travels in the kernel parameter buffer (__grid_constant__,
//     up to kMaxDescs entries, ~32 KB), i.e. it is device-resident constant
//     data with no host->device copy and no allocation per launch.
//   * The output of every descriptor is cut into warp units of 4 KiB (256
//     16-byte output vectors). Units of all descriptors form one global range;
//     each warp of a persistent grid (SM count x resident blocks) strides over
//     it and finds its descriptor by a warp-uniform search of the prefix
//     table ("warp-level descriptor dispatch").
//   * Vector path: every lane produces whole 16-byte output vectors. The source
//     span of a vector (8, 16 or 32 bytes depending on the conversion) may start
//     at any byte; it is assembled from aligned 16-byte loads with a funnel
//     shift, so every global access is a 16-byte aligned, coalesced
//     transaction. Stores are 16-byte aligned streaming stores.
//   * Element path: rows whose output length is not a multiple of 16 bytes
//     (odd shard widths, tiny tensors, tails) fall back to per-element moves.
//     Correct for every case the reference accepts; never hot for LLM shapes.
//   * Contiguous descriptors skip the warp units: aligned raw copies go to
//     bulk_kernel (TMA cp.async.bulk HBM -> smem -> HBM, one issuing thread per
//     SM), casts and misaligned sources to staged_kernel (TMA loads into smem
//     stages, consumer warps shift/convert into smem output stages, TMA bulk
//     stores). Both stride 8-16 KiB units per CTA. Multi-row (column shard)
//     descriptors stay on the warp kernels above.
#include <cuda.h>  // CUtensorMap (encoded through cudaGetDriverEntryPoint: no -lcuda)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include <atomic>
#include <mutex>
#include <vector>

#include "hl_internal.h"

namespace hl {

enum Kind : uint8_t {
  K_COPY1 = 0,  // identity, any dtype (raw bytes)
  K_BF16_F16 = 1,
  K_F32_F16 = 2,
  K_F16_F32 = 3,
  K_BF16_F32 = 4,
};

// M_ROWS   every row's output is a whole number of 16-byte vectors (or the
//          descriptor is one contiguous row); warp units never cross a row, so
//          the source of a unit is one contiguous byte range with one alignment.
// M_PACKED rows of fewer than kMinRowVecs vectors: units span several rows.
// M_ELEM   anything else (odd row widths, misaligned dst): per element.
enum Mode : uint8_t { M_ROWS = 0, M_PACKED = 1, M_ELEM = 2 };

struct KDesc {
  uint64_t src;        // byte address of element (0,0)
  uint64_t dst;        // byte address of the contiguous output
  uint64_t src_pitch;  // bytes between source rows
  uint64_t unit_begin; // first global unit of this descriptor
  uint64_t nvec;       // M_ROWS/M_PACKED: full 16 B output vectors; M_ELEM: elements
  uint64_t row_len;    // M_ROWS/M_PACKED: vectors per row; M_ELEM: elements per row
  uint32_t upr;        // M_ROWS: warp units per row
  uint32_t tail;       // single-row descriptors: trailing elements after the last vector
  uint8_t kind, mode, ss, ds;  // conversion kind, mode, src/dst element size
  uint32_t which;              // kernel: 0 generic, 1 + RowClass for M_ROWS
};
static_assert(sizeof(KDesc) == 64, "KDesc layout");

constexpr int kMaxDescs = 500;  // 500*64 + 16 = 32016 B < 32764 B param limit
constexpr uint64_t kMinRowVecs = 64;
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kUnroll = 8;
constexpr uint64_t kUnitVecs = 32 * kUnroll;   // 4 KiB of output per warp unit
// Row units of the bf16 -> f32 widening (8-byte source spans, a shift per
// element) are twice as long and run with twice the unroll, so a lane keeps
// as many source bytes in flight as the copy kernel (16 x 8 B, not 8 x 8 B).
// (f16 -> f32 keeps 8: its NaN-preserving conversion would need ~100 registers.)
__host__ __device__ constexpr uint64_t row_unit_vecs(int kind) { return kind == 4 ? 2 * kUnitVecs : kUnitVecs; }
constexpr uint64_t kUnitElems = 32 * kUnroll;  // elements per unit on the element path

constexpr int kSmallDescs = 4;  // single-key calls launch with a 240-byte parameter block

template <int N>
struct ParamsN {
  uint32_t n;
  uint32_t pad;
  uint64_t total_units;
  KDesc d[N];
};
using Params = ParamsN<kMaxDescs>;
using SmallParams = ParamsN<kSmallDescs>;

// ---------------------------------------------------------------- conversions
// numpy float32 -> float16 (npy_floatbits_to_halfbits): RNE, overflow -> inf,
// NaN keeps sign and mant>>13 (forced non-zero), no quieting.
__device__ __forceinline__ uint32_t np_f32_to_f16(uint32_t f) {
  const uint32_t sgn = (f >> 16) & 0x8000u;
  const uint32_t fexp = f & 0x7f800000u;
  const uint32_t fsig = f & 0x007fffffu;
  if (fexp >= 0x47800000u) {
    if (fexp == 0x7f800000u && fsig) {
      uint32_t r = 0x7c00u + (fsig >> 13);
      r += (r == 0x7c00u);
      return sgn + r;
    }
    return sgn + 0x7c00u;
  }
  if (fexp <= 0x38000000u) {
    if (fexp < 0x33000000u) return sgn;
    const uint32_t e = fexp >> 23;
    uint32_t sig = (0x00800000u + fsig) >> (113 - e);
    if (((sig & 0x3fffu) != 0x1000u) || (f & 0x7ffu)) sig += 0x1000u;
    return sgn + (sig >> 13);
  }
  uint32_t sig = fsig;
  if ((sig & 0x3fffu) != 0x1000u) sig += 0x1000u;
  return sgn + ((sig >> 13) + ((fexp - 0x38000000u) >> 13));
}

// numpy float16 -> float32 (npy_halfbits_to_floatbits): exact, NaN payload kept.
__device__ __forceinline__ uint32_t np_f16_to_f32(uint32_t h) {
  const uint32_t sgn = (h & 0x8000u) << 16;
  const uint32_t hexp = h & 0x7c00u;
  const uint32_t hsig = h & 0x03ffu;
  if (hexp == 0x7c00u) return sgn | 0x7f800000u | (hsig << 13);
  if (hexp == 0) {
    if (hsig == 0) return sgn;
    // subnormal: normalise; value = hsig * 2^-24
    const int lz = __clz(hsig) - 21;  // leading zeros within the 10-bit field (1..10)
    const uint32_t m = (hsig << lz) & 0x3ffu;
    const uint32_t e = 113u - (uint32_t)lz;  // f32 exponent of hsig * 2^-24
    return sgn | (e << 23) | (m << 13);
  }
  return sgn | ((((h & 0x7fffu) + 0x1c000u)) << 13);
}

// Vectorised narrowing: two f32 bit patterns -> packed f16x2 (lo in bits 0..15).
// The hardware RNE conversion equals numpy's for every non-NaN input (overflow
// to inf, subnormal rounding); NaNs are patched to numpy's payload rule. (Two
// alternatives measured slower on the 7B batch, profiles/r01_kernel_bench*:
// one Inf/NaN screen per vector with the slow path inline, 57% of HBM peak,
// and out of line, 78%; this per-pair form: 87%.)
__device__ __forceinline__ uint32_t f32x2_to_f16x2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(__uint_as_float(b)), "f"(__uint_as_float(a)));
  if (((a & 0x7fffffffu) > 0x7f800000u) | ((b & 0x7fffffffu) > 0x7f800000u)) {
    const uint32_t lo = np_f32_to_f16(a), hi = np_f32_to_f16(b);
    r = lo | (hi << 16);
  }
  return r;
}

// Two bf16 (one 32-bit word) -> packed f16x2: the same hardware conversion,
// with the NaN test done on the packed bf16 halves in two ops
// (bit 15 / 31 of ((w & 0x7fff7fff) + 0x007f007f) is set iff that half is a NaN).
__device__ __forceinline__ uint32_t bf16x2_to_f16x2(uint32_t w) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(__uint_as_float(w & 0xffff0000u)), "f"(__uint_as_float(w << 16)));
  if (((w & 0x7fff7fffu) + 0x007f007fu) & 0x80008000u) {
    r = np_f32_to_f16(w << 16) | (np_f32_to_f16(w & 0xffff0000u) << 16);
  }
  return r;
}

// Widening: f16 bits -> f32 bits, hardware exact path with NaN payload patch.
__device__ __forceinline__ uint32_t f16_to_f32_bits(uint32_t h) {
  if ((h & 0x7c00u) == 0x7c00u && (h & 0x3ffu)) return ((h & 0x8000u) << 16) | 0x7f800000u | ((h & 0x3ffu) << 13);
  float f;
  asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"((unsigned short)h));
  return __float_as_uint(f);
}

// scalar conversion on raw element bits (element path)
__device__ __forceinline__ uint64_t convert_scalar(uint64_t x, uint8_t kind) {
  switch (kind) {
    case K_BF16_F16: return np_f32_to_f16((uint32_t)x << 16);
    case K_F32_F16: return np_f32_to_f16((uint32_t)x);
    case K_F16_F32: return np_f16_to_f32((uint32_t)x & 0xffffu);
    case K_BF16_F32: return (uint64_t)((uint32_t)x << 16);
    default: return x;
  }
}

// ---------------------------------------------------------------- memory ops
__device__ __forceinline__ uint4 ldg16(const void* p) {
  uint4 r;
  asm("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint64_t ldg8(const void* p) {
  uint64_t r;
  asm("ld.global.nc.u64 %0, [%1];" : "=l"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg16(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// bytes [s, s+16) of the 32-byte concatenation a||b (s in 0..15), branch-free.
__device__ __forceinline__ uint4 extract16(uint4 a, uint4 b, uint32_t s) {
  uint32_t x0 = a.x, x1 = a.y, x2 = a.z, x3 = a.w, x4 = b.x, x5 = b.y, x6 = b.z, x7 = b.w;
  const bool q2 = s & 8, q1 = s & 4;
  // shift by two words
  uint32_t y0 = q2 ? x2 : x0, y1 = q2 ? x3 : x1, y2 = q2 ? x4 : x2, y3 = q2 ? x5 : x3,
           y4 = q2 ? x6 : x4, y5 = q2 ? x7 : x5;
  // shift by one word
  uint32_t z0 = q1 ? y1 : y0, z1 = q1 ? y2 : y1, z2 = q1 ? y3 : y2, z3 = q1 ? y4 : y3,
           z4 = q1 ? y5 : y4;
  const uint32_t r = (s & 3) * 8;
  uint4 o;
  o.x = __funnelshift_r(z0, z1, r);
  o.y = __funnelshift_r(z1, z2, r);
  o.z = __funnelshift_r(z2, z3, r);
  o.w = __funnelshift_r(z3, z4, r);
  return o;
}

// Source span of one output vector: NB bytes (16 for copies and bf16->f16, 32
// for f32->f16, 8 for the widening casts) starting at any byte.
template <int NB>
struct Span {
  uint4 v[NB >= 16 ? NB / 16 : 1];
};

// Generic span load (M_PACKED rows): aligned granules + funnel shift.
template <int NB>
__device__ __forceinline__ void load_span(const uint8_t* p, Span<NB>& out) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if constexpr (NB == 8) {
    const uint32_t s = a & 7;
    const uint64_t* b = reinterpret_cast<const uint64_t*>(a - s);
    uint64_t lo = ldg8(b);
    if (s) {
      const uint64_t hi = ldg8(b + 1);
      lo = (lo >> (8 * s)) | (hi << (64 - 8 * s));
    }
    out.v[0] = make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), 0, 0);
  } else {
    const uint32_t s = a & 15;
    const uint4* b = reinterpret_cast<const uint4*>(a - s);
    if (s == 0) {
#pragma unroll
      for (int i = 0; i < NB / 16; ++i) out.v[i] = ldg16(b + i);
    } else {
      uint4 c0 = ldg16(b);
#pragma unroll
      for (int i = 0; i < NB / 16; ++i) {
        const uint4 c1 = ldg16(b + i + 1);
        out.v[i] = extract16(c0, c1, s);
        c0 = c1;
      }
    }
  }
}

__device__ __forceinline__ uint4 shfl_down16(uint4 v) {
  return make_uint4(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1),
                    __shfl_down_sync(0xffffffffu, v.z, 1), __shfl_down_sync(0xffffffffu, v.w, 1));
}
__device__ __forceinline__ uint64_t shfl_down8(uint64_t v) {
  const uint32_t lo = __shfl_down_sync(0xffffffffu, (uint32_t)v, 1);
  const uint32_t hi = __shfl_down_sync(0xffffffffu, (uint32_t)(v >> 32), 1);
  return ((uint64_t)hi << 32) | lo;
}

template <int K>
struct KindTraits;
template <> struct KindTraits<K_COPY1> { static constexpr int NB = 16; };
template <> struct KindTraits<K_BF16_F16> { static constexpr int NB = 16; };
template <> struct KindTraits<K_F32_F16> { static constexpr int NB = 32; };
template <> struct KindTraits<K_F16_F32> { static constexpr int NB = 8; };
template <> struct KindTraits<K_BF16_F32> { static constexpr int NB = 8; };

template <int K>
__device__ __forceinline__ uint4 convert_vec(const Span<KindTraits<K>::NB>& s) {
  if constexpr (K == K_COPY1) {
    return s.v[0];
  } else if constexpr (K == K_BF16_F16) {
    const uint4 v = s.v[0];
    return make_uint4(bf16x2_to_f16x2(v.x), bf16x2_to_f16x2(v.y), bf16x2_to_f16x2(v.z), bf16x2_to_f16x2(v.w));
  } else if constexpr (K == K_F32_F16) {
    uint4 o;
    o.x = f32x2_to_f16x2(s.v[0].x, s.v[0].y);
    o.y = f32x2_to_f16x2(s.v[0].z, s.v[0].w);
    o.z = f32x2_to_f16x2(s.v[1].x, s.v[1].y);
    o.w = f32x2_to_f16x2(s.v[1].z, s.v[1].w);
    return o;
  } else if constexpr (K == K_F16_F32) {
    const uint32_t a = s.v[0].x, b = s.v[0].y;
    return make_uint4(f16_to_f32_bits(a & 0xffffu), f16_to_f32_bits(a >> 16),
                      f16_to_f32_bits(b & 0xffffu), f16_to_f32_bits(b >> 16));
  } else {  // K_BF16_F32
    const uint32_t a = s.v[0].x, b = s.v[0].y;
    return make_uint4(a << 16, a & 0xffff0000u, b << 16, b & 0xffff0000u);
  }
}

// ---------------------------------------------------------------- element path
__device__ __forceinline__ uint64_t load_elem(const uint8_t* p, uint32_t sz) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if ((a & (sz - 1)) == 0) {
    switch (sz) {
      case 1: return *p;
      case 2: return *reinterpret_cast<const uint16_t*>(p);
      case 4: return *reinterpret_cast<const uint32_t*>(p);
      default: return *reinterpret_cast<const uint64_t*>(p);
    }
  }
  uint64_t x = 0;
  for (uint32_t i = 0; i < sz; ++i) x |= (uint64_t)p[i] << (8 * i);
  return x;
}
__device__ __forceinline__ void store_elem(uint8_t* p, uint32_t sz, uint64_t x) {
  switch (sz) {  // dst is aligned to its element size (checked on the host)
    case 1: *p = (uint8_t)x; break;
    case 2: *reinterpret_cast<uint16_t*>(p) = (uint16_t)x; break;
    case 4: *reinterpret_cast<uint32_t*>(p) = (uint32_t)x; break;
    default: *reinterpret_cast<uint64_t*>(p) = x; break;
  }
}

__device__ __forceinline__ void elem_move(const KDesc& d, uint64_t e) {
  const uint64_t row = e / d.row_len, col = e - row * d.row_len;
  const uint8_t* s = reinterpret_cast<const uint8_t*>(d.src) + row * d.src_pitch + col * d.ss;
  uint8_t* o = reinterpret_cast<uint8_t*>(d.dst) + e * d.ds;
  store_elem(o, d.ds, convert_scalar(load_elem(s, d.ss), d.kind));
}

// Element path unit (cold: odd row widths, misaligned destinations).
__device__ __noinline__ void elem_unit(const KDesc& d, uint64_t lu, uint32_t lane) {
  const uint64_t e0 = lu * kUnitElems;
  for (uint32_t k = 0; k < kUnroll; ++k) {
    const uint64_t e = e0 + k * 32 + lane;
    if (e < d.nvec) elem_move(d, e);
  }
}

// ---------------------------------------------------------------- row units
// One warp makes vectors [0, n) of one row ready: `rsrc` is the source span of
// vector 0, `rdst` its 16-byte aligned destination. The source is one
// contiguous range, so its alignment is uniform across the warp.
//
// Aligned source: each lane loads its span with G-byte aligned loads (G = 16,
// or 8 for the 8-byte spans of widening casts), U vectors in flight per lane.
//
// Shifted source (realign): lane i loads the W aligned granules that START its
// span's window, and takes the one granule past it from lane i+1 with a warp
// shuffle; lane 31 only serves as that neighbour, so an iteration makes 31
// vectors ready from 32 coalesced granule loads. Every global load is aligned
// and used once: no L1 re-reads, half the load instructions of a two-load
// realign, and the same memory-level parallelism as the aligned path.
// The shifted (realign) loop for 16-byte granules.
template <int K, int US>
__device__ __forceinline__ void shifted_rows(const uint8_t* gb, uint8_t* rdst, uint32_t n, uint32_t lane,
                                             uint32_t sh) {
  constexpr int NB = KindTraits<K>::NB;
  constexpr int W = NB / 16;
  for (uint32_t base = 0; base < n; base += 31 * US) {
    const uint8_t* pg = gb + (size_t)(base + lane) * NB;
    uint8_t* pd = rdst + (size_t)(base + lane) * 16;
    const int32_t left = (int32_t)(n - base) - (int32_t)lane;  // lane's vector k in range iff k*31 < left
    uint4 g[US][W];
#pragma unroll
    for (int k = 0; k < US; ++k) {
      if (k * 31 < left) {
#pragma unroll
        for (int w = 0; w < W; ++w) g[k][w] = ldg16(pg + k * 31 * NB + w * 16);
      } else if (k * 31 == left) {
        g[k][0] = ldg16(pg + k * 31 * NB);  // the last span's tail granule
      }
    }
#pragma unroll
    for (int k = 0; k < US; ++k) {
      const uint4 nb = shfl_down16(g[k][0]);
      if (lane < 31 && k * 31 < left) {
        Span<NB> sp;
        if constexpr (W == 1) {
          sp.v[0] = extract16(g[k][0], nb, sh);
        } else {
          sp.v[0] = extract16(g[k][0], g[k][1], sh);
          sp.v[1] = extract16(g[k][1], nb, sh);
        }
        stg16(pd + k * 31 * 16, convert_vec<K>(sp));
      }
    }
  }
}

// Alignment class of a row-kernel launch (decided on the host per descriptor):
// every row aligned, every row shifted, or rows that differ (pitch not a
// multiple of the granule). Separate instantiations keep each hot loop's
// register budget at 64 (4 resident blocks per SM).
enum RowClass : int { R_MIXED = 0, R_ALIGNED = 1, R_SHIFTED = 2 };

template <int K, int RC>
__device__ __forceinline__ void row_unit(const uint8_t* rsrc, uint8_t* rdst, uint32_t n,
                                         uint32_t lane) {
  constexpr int NB = KindTraits<K>::NB;
  constexpr int G = NB >= 16 ? 16 : 8;  // granule
  constexpr int W = NB / G;             // granules per span (1 or 2)
  constexpr int U = (W == 2) ? kUnroll / 2 : (K == K_BF16_F32 ? 2 * kUnroll : kUnroll);
  const uintptr_t a = reinterpret_cast<uintptr_t>(rsrc);
  const uint32_t sh = a & (G - 1);
  if (RC == R_ALIGNED || (RC == R_MIXED && sh == 0)) {
    for (uint32_t base = 0; base < n; base += 32 * U) {
      // one base pointer per lane; the U vectors sit at constant offsets from it
      const uint8_t* ps = rsrc + (size_t)(base + lane) * NB;
      uint8_t* pd = rdst + (size_t)(base + lane) * 16;
      const int32_t left = (int32_t)(n - base) - (int32_t)lane;  // vector k in range iff k*32 < left
      Span<NB> sp[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        if (k * 32 < left) {
          if constexpr (G == 8) {
            const uint64_t x = ldg8(ps + k * 32 * NB);
            sp[k].v[0] = make_uint4((uint32_t)x, (uint32_t)(x >> 32), 0, 0);
          } else {
#pragma unroll
            for (int w = 0; w < W; ++w) sp[k].v[w] = ldg16(ps + k * 32 * NB + w * 16);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        if (k * 32 < left) stg16(pd + k * 32 * 16, convert_vec<K>(sp[k]));
      }
    }
    return;
  }
  const uint8_t* gb = rsrc - sh;  // aligned start of vector 0's window
  // in-flight vectors on the shifted path: the mixed kernel carries both loops
  // and the casts need registers for conversion temporaries
  constexpr int US = (RC == R_SHIFTED && K == K_COPY1) ? U : U / 2;
  if constexpr (G == 8) {
    for (uint32_t base = 0; base < n; base += 31 * US) {
      const uint8_t* pg = gb + (size_t)(base + lane) * NB;
      uint8_t* pd = rdst + (size_t)(base + lane) * 16;
      const int32_t left = (int32_t)(n - base) - (int32_t)lane;  // lane's vector k in range iff k*31 < left
      uint64_t g[US];
#pragma unroll
      for (int k = 0; k < US; ++k) g[k] = (k * 31 <= left) ? ldg8(pg + k * 31 * 8) : 0;  // == : tail granule
#pragma unroll
      for (int k = 0; k < US; ++k) {
        const uint64_t nb = shfl_down8(g[k]);
        if (lane < 31 && k * 31 < left) {
          const uint64_t x = (g[k] >> (8 * sh)) | (nb << (64 - 8 * sh));
          Span<NB> sp;
          sp.v[0] = make_uint4((uint32_t)x, (uint32_t)(x >> 32), 0, 0);
          stg16(pd + k * 31 * 16, convert_vec<K>(sp));
        }
      }
    }
  } else {
    shifted_rows<K, US>(gb, rdst, n, lane, sh);
  }
}

// Rows shorter than kMinRowVecs vectors: a unit spans several rows; each
// vector finds its row (M_PACKED, rare for model weights).
template <int K>
__device__ __noinline__ void packed_unit(const KDesc& d, uint64_t lu, uint32_t lane) {
  constexpr int NB = KindTraits<K>::NB;
  constexpr int U = 2;  // cold path: keep its registers below the hot loop's
  const uint8_t* src = reinterpret_cast<const uint8_t*>(d.src);
  uint8_t* dst = reinterpret_cast<uint8_t*>(d.dst);
  const uint64_t vbeg = lu * kUnitVecs;
  const uint64_t vend = min(vbeg + kUnitVecs, d.nvec);
  const uint64_t vpr = d.row_len;
  for (uint64_t base = vbeg; base < vend; base += 32 * U) {
    Span<NB> sp[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint64_t v = base + k * 32 + lane;
      if (v < vend) {
        const uint64_t row = v / vpr;
        load_span<NB>(src + row * d.src_pitch + (v - row * vpr) * NB, sp[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint64_t v = base + k * 32 + lane;
      if (v < vend) stg16(dst + v * 16, convert_vec<K>(sp[k]));
    }
  }
}

template <class P>
__device__ __forceinline__ uint32_t find_desc(const P& p, uint64_t u, uint32_t hint) {
  // descriptors are visited in increasing unit order by each warp: gallop from the hint
  uint32_t lo = hint, hi = p.n;  // invariant: d[lo].unit_begin <= u
  if (p.d[lo].unit_begin > u) lo = 0;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (p.d[mid].unit_begin <= u) lo = mid; else hi = mid;
  }
  return lo;
}

// Two kernels per conversion kind, so the hot one carries no cold code (and no
// call ABI) in its register budget:
//   row_kernel      M_ROWS descriptors — every model weight, clone, realign, pack;
//   generic_kernel  M_PACKED rows and M_ELEM elements (odd widths, tails).
template <int K, class P, int RC>
__global__ void __launch_bounds__(kThreads) row_kernel(const __grid_constant__ P p) {
  constexpr int NB = KindTraits<K>::NB;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  uint32_t di = 0;
  for (uint64_t u = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); u < p.total_units; u += nwarps) {
    di = find_desc(p, u, di);
    const KDesc& d = p.d[di];
    const uint32_t lu = (uint32_t)(u - d.unit_begin);  // < 2^32 units (16 TiB) per descriptor
    const uint32_t row = lu / d.upr;
    constexpr uint64_t UV = row_unit_vecs(K);
    const uint64_t v0 = (uint64_t)(lu - row * d.upr) * UV;
    const uint64_t v1 = min(v0 + UV, d.row_len);
    const uint8_t* rsrc = reinterpret_cast<const uint8_t*>(d.src) + (uint64_t)row * d.src_pitch + v0 * NB;
    uint8_t* rdst = reinterpret_cast<uint8_t*>(d.dst) + ((uint64_t)row * d.row_len + v0) * 16;
    row_unit<K, RC>(rsrc, rdst, (uint32_t)(v1 - v0), lane);
  }
}

template <int K, class P>
__global__ void __launch_bounds__(kThreads) generic_kernel(const __grid_constant__ P p) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  uint32_t di = 0;
  for (uint64_t u = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); u < p.total_units; u += nwarps) {
    di = find_desc(p, u, di);
    const KDesc& d = p.d[di];
    const uint64_t lu = u - d.unit_begin;
    if (d.mode == M_PACKED) packed_unit<K>(d, lu, lane);
    else elem_unit(d, lu, lane);
  }
}

// ---------------------------------------------------------------- TMA bulk copy
// Aligned raw copies (clones, dim-0 shards, aligned rows of column shards: the
// value leg's whole workload) need no register work at all, so they bypass the
// SM's load/store pipes: one elected thread per CTA streams 16 KiB row chunks
// HBM -> shared memory with cp.async.bulk (TMA, completion counted on an
// mbarrier) and shared -> HBM with bulk_group stores, kBulkStages chunks in
// flight. Measured on a flat 7.25 GB copy (tools/bulk_copy_probe.cu,
// profiles/r01_bulk_copy_probe.jsonl): 6.51 TB/s vs 6.25 TB/s for the 16-byte
// LDG/STG loop at this kernel's 4 resident blocks per SM.
constexpr uint32_t kBulkChunk = 16u << 10;
constexpr uint64_t kBulkVecs = kBulkChunk / 16;
constexpr int kBulkStages = 4;
constexpr int kBulkLag = 1;  // stores allowed to be still reading shared memory when a stage is refilled
constexpr size_t kBulkSmem = (size_t)kBulkStages * kBulkChunk;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Unit u of a bulk launch: descriptors are single contiguous rows, so unit lu of
// descriptor d is bytes [lu * kBulkChunk, ...) of it. Each stream of units
// (loads, stores) visits increasing u, so its descriptor index only walks forward.
template <class P>
__device__ __forceinline__ void bulk_unit(const P& p, uint64_t u, uint32_t& di, const uint8_t*& src, uint8_t*& dst,
                                          uint32_t& bytes) {
  while (di + 1 < p.n && p.d[di + 1].unit_begin <= u) ++di;
  const KDesc& d = p.d[di];
  const uint64_t off = (u - d.unit_begin) * kBulkChunk;
  const uint64_t total = d.row_len * 16;
  src = reinterpret_cast<const uint8_t*>(d.src) + off;
  dst = reinterpret_cast<uint8_t*>(d.dst) + off;
  bytes = (uint32_t)min((uint64_t)kBulkChunk, total - off);
}

template <class P>
__global__ void __launch_bounds__(32) bulk_kernel(const __grid_constant__ P p) {
  extern __shared__ __align__(128) uint8_t stage[];
  __shared__ __align__(8) uint64_t bar[kBulkStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kBulkStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t policy;  // streaming: neither side is re-read by this launch
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  const uint64_t first = blockIdx.x, step = gridDim.x;
  const uint64_t mine = first < p.total_units ? (p.total_units - first + step - 1) / step : 0;
  uint32_t load_hint = 0, store_hint = 0;
  auto load = [&](uint64_t k) {
    const uint8_t* src;
    uint8_t* dst;
    uint32_t bytes;
    bulk_unit(p, first + k * step, load_hint, src, dst, bytes);
    const int s = (int)(k % kBulkStages);
    const uint32_t b = smem_u32(&bar[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        :: "r"(smem_u32(stage + (size_t)s * kBulkChunk)), "l"(src), "r"(bytes), "r"(b), "l"(policy) : "memory");
  };
  constexpr uint64_t ahead = kBulkStages - kBulkLag;
  for (uint64_t k = 0; k < mine && k < ahead; ++k) load(k);
  for (uint64_t k = 0; k < mine; ++k) {
    const uint8_t* src;
    uint8_t* dst;
    uint32_t bytes;
    bulk_unit(p, first + k * step, store_hint, src, dst, bytes);
    const int s = (int)(k % kBulkStages);
    asm volatile(
        "{\n .reg .pred ready;\n"
        "WAIT: mbarrier.try_wait.parity.shared::cta.b64 ready, [%0], %1;\n"
        " @!ready bra WAIT;\n}\n" :: "r"(smem_u32(&bar[s])), "r"((uint32_t)((k / kBulkStages) & 1)) : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                 :: "l"(dst), "r"(smem_u32(stage + (size_t)s * kBulkChunk)), "r"(bytes), "l"(policy) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (k + ahead < mine) {
      // the refilled stage was last read by store k - kBulkLag
      asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(kBulkLag) : "memory");
      load(k + ahead);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------- TMA-staged realign / cast
// Contiguous tensors whose bytes must change on the way (a cast, or a source
// that is not 16-byte aligned): a producer thread streams each unit's aligned
// source window HBM -> shared memory with cp.async.bulk (mbarrier "full"),
// kConsumerWarps warps read the window out of shared memory at the tensor's
// byte shift, convert, and write the unit's output into a shared-memory output
// stage, then release the stage (mbarrier "empty"); the producer bulk-stores the
// output stage to HBM (cp.async.bulk bulk_group) and refills the input stage once
// that store has read it. Widening casts (output twice the input) use half-size
// source units so the output stage stays 16 KiB. Neither loads nor stores depend on how many
// vectors the registers of the SM keep in flight — the limit of the LDG/STG row
// kernel. Used for every contiguous cast and every misaligned contiguous source
// (bf16/f32 -> f16: 6.47 / 6.79 TB/s vs 6.07 / 6.16 on the row kernel).
// (the HL_STAGED_* macros exist for tuning sweeps: tools/staged_sweep.sh)
#ifndef HL_STAGED_IN_KB
#define HL_STAGED_IN_KB 16
#endif
#ifndef HL_STAGED_STAGES
#define HL_STAGED_STAGES 6
#endif
#ifndef HL_STAGED_WARPS
#define HL_STAGED_WARPS 16
#endif
#ifndef HL_STAGED_CTAS
#define HL_STAGED_CTAS 2
#endif
#ifndef HL_STAGED_STAGES_TS
#define HL_STAGED_STAGES_TS 3
#endif
#ifndef HL_STAGED_ALIGNED
#define HL_STAGED_ALIGNED 1
#endif
constexpr uint32_t kStageIn = HL_STAGED_IN_KB << 10;  // source bytes per unit (half for widening casts)
constexpr int kStagedStagesMax = HL_STAGED_STAGES > HL_STAGED_STAGES_TS ? HL_STAGED_STAGES : HL_STAGED_STAGES_TS;
constexpr int kConsumerWarps = HL_STAGED_WARPS;
constexpr int kStagedCtasPerSm = HL_STAGED_CTAS;  // 2 x (1 + 16) warps and 2 x <= 113 KiB of stages per SM
constexpr int kStagedThreads = 32 * (1 + kConsumerWarps);
#ifndef HL_STAGED_TMA_STORE
#define HL_STAGED_TMA_STORE 1
#endif
#ifndef HL_STAGED_WIDEN_TS
#define HL_STAGED_WIDEN_TS 1
#endif
__host__ __device__ constexpr uint32_t span_bytes(int kind) { return kind == 2 ? 32 : (kind >= 3 ? 8 : 16); }
// output staging: consumers write the unit to shared memory and the producer
// bulk-stores it; widening casts (output = 2 x input) then use half-size units
__host__ __device__ constexpr bool staged_tma_store(int kind) {
  return HL_STAGED_TMA_STORE && (span_bytes(kind) >= 16 || HL_STAGED_WIDEN_TS);
}
__host__ __device__ constexpr uint32_t stage_in(int kind) {
  return (span_bytes(kind) == 8 && staged_tma_store(kind)) ? kStageIn / 2 : kStageIn;
}
__host__ __device__ constexpr uint32_t stage_bytes(int kind) { return stage_in(kind) + 32; }  // + shift, tail granule
__host__ __device__ constexpr uint64_t staged_unit_vecs(int kind) { return stage_in(kind) / span_bytes(kind); }
__host__ __device__ constexpr uint32_t staged_out_bytes(int kind) {
  return staged_tma_store(kind) ? (uint32_t)(staged_unit_vecs(kind) * 16) : 0;
}
// stages in flight: input + output stages share the 2 x ~113 KiB per SM when the output is staged
__host__ __device__ constexpr int staged_stages(int kind) {
  return staged_tma_store(kind) ? HL_STAGED_STAGES_TS : HL_STAGED_STAGES;
}
__host__ __device__ constexpr size_t staged_smem(int kind) {
  return (size_t)staged_stages(kind) * (stage_bytes(kind) + staged_out_bytes(kind));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred ready;\n"
      "WAIT: mbarrier.try_wait.parity.shared::cta.b64 ready, [%0], %1;\n"
      " @!ready bra WAIT;\n}\n" :: "r"(bar), "r"(parity) : "memory");
}

struct StagedUnit {
  const uint8_t* win;  // 16-byte aligned source window
  uint8_t* dst;
  uint32_t wbytes;     // window bytes (multiple of 16)
  uint32_t sh;         // byte shift of the first span inside the window
  uint32_t nv;         // output vectors
};

template <int K, class P>
__device__ __forceinline__ StagedUnit staged_unit(const P& p, uint64_t u, uint32_t& di) {
  constexpr uint32_t NB = KindTraits<K>::NB;
  constexpr uint64_t UV = staged_unit_vecs(K);
  while (di + 1 < p.n && p.d[di + 1].unit_begin <= u) ++di;
  const KDesc& d = p.d[di];
  const uint64_t v0 = (u - d.unit_begin) * UV;
  StagedUnit x;
  x.nv = (uint32_t)min(UV, d.row_len - v0);
  const uint64_t s0 = d.src + v0 * NB;
  const uint64_t a0 = s0 & ~(uint64_t)15;
  x.win = reinterpret_cast<const uint8_t*>(a0);
  x.sh = (uint32_t)(s0 - a0);
  x.wbytes = (uint32_t)(((s0 + (uint64_t)x.nv * NB + 15) & ~(uint64_t)15) - a0);
  x.dst = reinterpret_cast<uint8_t*>(d.dst) + v0 * 16;
  return x;
}

__device__ __forceinline__ uint4 lds16(const uint8_t* p) { return *reinterpret_cast<const uint4*>(p); }

template <int K, class P>
__global__ void __launch_bounds__(kStagedThreads) staged_kernel(const __grid_constant__ P p) {
  constexpr uint32_t NB = KindTraits<K>::NB;
  constexpr bool TS = staged_tma_store(K);
  constexpr uint32_t OUTB = staged_out_bytes(K);
  constexpr int kStagedStages = staged_stages(K);
  constexpr uint32_t kStageBytes = stage_bytes(K);
  extern __shared__ __align__(128) uint8_t stage[];
  uint8_t* const outs = stage + (size_t)kStagedStages * kStageBytes;  // TS: output stage s at outs + s * OUTB
  __shared__ __align__(8) uint64_t full[kStagedStagesMax], empty[kStagedStagesMax];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagedStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&empty[s])), "r"(32 * kConsumerWarps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t first = blockIdx.x, step = gridDim.x;
  const uint64_t mine = first < p.total_units ? (p.total_units - first + step - 1) / step : 0;
  uint32_t di = 0;
  if (warp == 0) {  // producer
    if (lane != 0) return;
    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    auto load = [&](uint64_t k) {
      const int s = (int)(k % kStagedStages);
      const StagedUnit x = staged_unit<K>(p, first + k * step, di);
      const uint32_t b = smem_u32(&full[s]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(x.wbytes) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
          :: "r"(smem_u32(stage + (size_t)s * kStageBytes)), "l"(x.win), "r"(x.wbytes), "r"(b), "l"(policy)
          : "memory");
    };
    if constexpr (!TS) {
      for (uint64_t k = 0; k < mine; ++k) {
        if (k >= (uint64_t)kStagedStages)
          mbar_wait(smem_u32(&empty[k % kStagedStages]), (uint32_t)((k / kStagedStages - 1) & 1));
        load(k);
      }
    } else {
      uint32_t sdi = 0;
      for (uint64_t k = 0; k < mine && k < (uint64_t)kStagedStages; ++k) load(k);
      for (uint64_t k = 0; k < mine; ++k) {
        const int s = (int)(k % kStagedStages);
        mbar_wait(smem_u32(&empty[s]), (uint32_t)((k / kStagedStages) & 1));  // unit k converted
        const StagedUnit x = staged_unit<K>(p, first + k * step, sdi);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                     :: "l"(x.dst), "r"(smem_u32(outs + (size_t)s * OUTB)), "r"(x.nv * 16u), "l"(policy)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (k + kStagedStages < mine) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // output stage s read out
          load(k + kStagedStages);
        }
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    return;
  }
  const uint32_t ct = threadIdx.x - 32;  // consumer thread
  for (uint64_t k = 0; k < mine; ++k) {
    const int s = (int)(k % kStagedStages);
    const StagedUnit x = staged_unit<K>(p, first + k * step, di);
    mbar_wait(smem_u32(&full[s]), (uint32_t)((k / kStagedStages) & 1));
    const uint8_t* w = stage + (size_t)s * kStageBytes;
    // every consumer thread owns CU vectors of the unit: all their shared-memory
    // reads are issued before the first conversion (ILP across the vectors)
    constexpr uint32_t CT = 32 * kConsumerWarps;
    constexpr uint32_t CU = (uint32_t)((staged_unit_vecs(K) + CT - 1) / CT);
    Span<NB> sp[CU];
#pragma unroll
    for (uint32_t i = 0; i < CU; ++i) {
      const uint32_t v = ct + i * CT;
      if (v >= x.nv) break;
      const uint32_t o = x.sh + v * NB;
      if constexpr (NB == 8) {
        const uint64_t* q = reinterpret_cast<const uint64_t*>(w + (o & ~7u));
        const uint32_t r = o & 7;
        uint64_t lo = q[0];
        if (r) lo = (lo >> (8 * r)) | (q[1] << (64 - 8 * r));
        sp[i].v[0] = make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), 0, 0);
      } else {
        const uint8_t* g = w + (o & ~15u);
        const uint32_t r = o & 15;
        if (r == 0) {
#pragma unroll
          for (int j = 0; j < (int)(NB / 16); ++j) sp[i].v[j] = lds16(g + 16 * j);
        } else {
          uint4 c0 = lds16(g);
#pragma unroll
          for (int j = 0; j < (int)(NB / 16); ++j) {
            const uint4 c1 = lds16(g + 16 * (j + 1));
            sp[i].v[j] = extract16(c0, c1, r);
            c0 = c1;
          }
        }
      }
    }
#pragma unroll
    for (uint32_t i = 0; i < CU; ++i) {
      const uint32_t v = ct + i * CT;
      if (v >= x.nv) break;
      if constexpr (TS) {
        *reinterpret_cast<uint4*>(outs + (size_t)s * OUTB + (size_t)v * 16) = convert_vec<K>(sp[i]);
      } else {
        stg16(x.dst + (size_t)v * 16, convert_vec<K>(sp[i]));
      }
    }
    // generic-proxy smem writes must be visible to the async proxy (the bulk store); every
    // consumer thread releases its own reads and writes of the stage on the empty barrier
    if constexpr (TS) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&empty[s])) : "memory");
  }
}

// ---------------------------------------------------------------- TMA tensor tiles (column shards)
// Multi-row descriptors (a rank's column shard: `rows` row segments of a few
// KiB at a fixed source pitch, ref collective.py:318-330 _clone_slice along
// dim >= 1) move as 2-D boxes of a tensor map: the source is described as a
// rows x cols matrix at the tensor's pitch, the destination as the dense
// rows x seg matrix, and a box is BY rows x BX columns (<= 16 KiB). One
// elected thread per CTA streams boxes HBM -> shared memory with
// cp.async.bulk.tensor.2d (UTMALDG: the TMA unit walks the strided rows, no
// per-row address arithmetic in any warp) and writes them back with
// cp.async.bulk.tensor.2d stores (UTMASTG, clipped to the shard's edges by the
// destination map). Casts add consumer warps that convert each staged box in
// shared memory into an output box first (staged_kernel's scheme). Raw copies
// use the widest element (8/4/2/1 B) the shard's offsets allow, so a box row
// is up to 2 KiB of contiguous source bytes.
constexpr uint32_t kTileBox = 16u << 10;  // bytes of one box (input and output)
#ifndef HL_TILE_STAGES
#define HL_TILE_STAGES 6
#endif
#ifndef HL_TILE_CAST_STAGES
#define HL_TILE_CAST_STAGES 3
#endif
constexpr int kTileStages = HL_TILE_STAGES;          // raw copies: 1 thread, 1 CTA per SM
constexpr int kTileCastStages = HL_TILE_CAST_STAGES;  // casts: in + out stage each, 2 CTAs per SM
#ifndef HL_TILE_WARPS
#define HL_TILE_WARPS 8
#endif
#ifndef HL_TILE_CAST_CTAS
#define HL_TILE_CAST_CTAS 2
#endif
constexpr int kTileConsumerWarps = HL_TILE_WARPS;
constexpr int kTileCastThreads = 32 * (1 + kTileConsumerWarps);
constexpr int kMaxTiles = 96;  // 64 + 96 * 320 = 30784 B of kernel parameters

struct alignas(64) TileDesc {
  CUtensorMap src;      // {cols, rows} at the source pitch; element = the copy unit or the src dtype
  CUtensorMap dst;      // {seg cols, rows} dense
  uint64_t unit_begin;  // first unit (box) of this descriptor in the launch
  uint32_t nbx;         // boxes across the segment
  int32_t c0;           // first source column of the segment (tensor-map elements)
  uint32_t bx, by;      // box dims (elements, rows)
  uint32_t in_bytes;    // bytes of one source box (mbarrier transaction count)
  uint16_t grp;         // descriptors in this one's interleave group (>= 1, see tile_unit)
  uint16_t gi;          // index in the group
};
static_assert(sizeof(TileDesc) == 320, "TileDesc layout");

struct TileParams {
  uint32_t n;
  uint32_t pad;
  uint64_t total_units;
  TileDesc d[kMaxTiles];
};

struct TileUnit {
  const TileDesc* d;
  int32_t sx, sy, dx;  // source box origin (col, row), destination col (row = sy)
};

// Descriptors come in interleave groups: `grp` consecutive descriptors with the
// same unit count share one unit range, unit u of the group being unit u / grp
// of member u % grp. The W shards of one tensor form a group, so the boxes the
// grid streams at any moment are the same rows of every shard — whole source
// rows — instead of one narrow column band at the source pitch (which leaves
// HBM channels idle). `di` always names a group's first member.
__device__ __forceinline__ TileUnit tile_unit(const TileParams& p, uint64_t u, uint32_t& di) {
  for (;;) {
    const uint32_t nx = di + p.d[di].grp;
    if (nx < p.n && p.d[nx].unit_begin <= u) di = nx;
    else break;
  }
  const uint64_t lg = u - p.d[di].unit_begin;
  const uint32_t g = p.d[di].grp;
  const TileDesc& d = p.d[di + (uint32_t)(lg % g)];
  const uint64_t lu = lg / g;
  const uint32_t by = (uint32_t)(lu / d.nbx), bx = (uint32_t)(lu % d.nbx);
  TileUnit t;
  t.d = &d;
  t.dx = (int32_t)(bx * d.bx);
  t.sx = d.c0 + t.dx;
  t.sy = (int32_t)(by * d.by);
  return t;
}

__device__ __forceinline__ void tile_load(const TileUnit& t, uint32_t smem, uint32_t bar, uint64_t policy) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(t.d->in_bytes) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;"
      :: "r"(smem), "l"(&t.d->src), "r"(t.sx), "r"(t.sy), "r"(bar), "l"(policy) : "memory");
}

__device__ __forceinline__ void tile_store(const TileUnit& t, uint32_t smem, uint64_t policy) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;"
               :: "l"(&t.d->dst), "r"(t.dx), "r"(t.sy), "r"(smem), "l"(policy) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Raw column shards: load box -> store the same shared-memory box.
__global__ void __launch_bounds__(32) tile_copy_kernel(const __grid_constant__ TileParams p) {
  extern __shared__ __align__(128) uint8_t stage[];
  __shared__ __align__(8) uint64_t bar[kTileStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kTileStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t policy;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  const uint64_t first = blockIdx.x, step = gridDim.x;
  const uint64_t mine = first < p.total_units ? (p.total_units - first + step - 1) / step : 0;
  uint32_t ldi = 0, sdi = 0;
  constexpr uint64_t ahead = kTileStages - 1;  // one store may still be reading its stage
  for (uint64_t k = 0; k < mine && k < ahead; ++k) {
    const int s = (int)(k % kTileStages);
    tile_load(tile_unit(p, first + k * step, ldi), smem_u32(stage + (size_t)s * kTileBox), smem_u32(&bar[s]), policy);
  }
  for (uint64_t k = 0; k < mine; ++k) {
    const int s = (int)(k % kTileStages);
    const TileUnit t = tile_unit(p, first + k * step, sdi);
    mbar_wait(smem_u32(&bar[s]), (uint32_t)((k / kTileStages) & 1));
    tile_store(t, smem_u32(stage + (size_t)s * kTileBox), policy);
    if (k + ahead < mine) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // store k-1 has read its stage
      const uint64_t j = k + ahead;
      const int sj = (int)(j % kTileStages);
      tile_load(tile_unit(p, first + j * step, ldi), smem_u32(stage + (size_t)sj * kTileBox), smem_u32(&bar[sj]),
                policy);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Cast column shards: producer lane loads boxes, consumer warps convert box s
// (flat element order: the in and out boxes have the same rows x cols) into
// output stage s, the producer stores it.
template <int K>
__global__ void __launch_bounds__(kTileCastThreads) tile_cast_kernel(const __grid_constant__ TileParams p) {
  constexpr uint32_t NB = KindTraits<K>::NB;  // source bytes per 16-byte output vector
  extern __shared__ __align__(128) uint8_t stage[];
  uint8_t* const outs = stage + (size_t)kTileCastStages * kTileBox;
  __shared__ __align__(8) uint64_t full[kTileCastStages], empty[kTileCastStages];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTileCastStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&empty[s])), "r"(kTileConsumerWarps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t first = blockIdx.x, step = gridDim.x;
  const uint64_t mine = first < p.total_units ? (p.total_units - first + step - 1) / step : 0;
  if (warp == 0) {
    if (lane != 0) return;
    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    uint32_t ldi = 0, sdi = 0;
    for (uint64_t k = 0; k < mine && k < (uint64_t)kTileCastStages; ++k) {
      const int s = (int)(k % kTileCastStages);
      tile_load(tile_unit(p, first + k * step, ldi), smem_u32(stage + (size_t)s * kTileBox), smem_u32(&full[s]),
                policy);
    }
    for (uint64_t k = 0; k < mine; ++k) {
      const int s = (int)(k % kTileCastStages);
      const TileUnit t = tile_unit(p, first + k * step, sdi);
      mbar_wait(smem_u32(&empty[s]), (uint32_t)((k / kTileCastStages) & 1));  // box k converted
      tile_store(t, smem_u32(outs + (size_t)s * kTileBox), policy);
      if (k + kTileCastStages < mine) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // output stage s read out
        const uint64_t j = k + kTileCastStages;
        tile_load(tile_unit(p, first + j * step, ldi), smem_u32(stage + (size_t)s * kTileBox), smem_u32(&full[s]),
                  policy);
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    return;
  }
  const uint32_t ct = threadIdx.x - 32;
  constexpr uint32_t CT = 32 * kTileConsumerWarps;
  uint32_t di = 0;
  for (uint64_t k = 0; k < mine; ++k) {
    const int s = (int)(k % kTileCastStages);
    const TileUnit t = tile_unit(p, first + k * step, di);
    const uint32_t nv = t.d->in_bytes / NB;  // output vectors of the box
    mbar_wait(smem_u32(&full[s]), (uint32_t)((k / kTileCastStages) & 1));
    const uint8_t* in = stage + (size_t)s * kTileBox;
    uint8_t* out = outs + (size_t)s * kTileBox;
    for (uint32_t v = ct; v < nv; v += CT) {
      Span<NB> sp;
      if constexpr (NB == 8) {
        const uint64_t x = *reinterpret_cast<const uint64_t*>(in + (size_t)v * 8);
        sp.v[0] = make_uint4((uint32_t)x, (uint32_t)(x >> 32), 0, 0);
      } else {
#pragma unroll
        for (int j = 0; j < (int)(NB / 16); ++j) sp.v[j] = lds16(in + (size_t)v * NB + 16 * j);
      }
      *reinterpret_cast<uint4*>(out + (size_t)v * 16) = convert_vec<K>(sp);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&empty[s])) : "memory");
  }
}

// ---------------------------------------------------------------- host side
static const uint32_t kSize[13] = {1, 1, 1, 2, 2, 4, 4, 8, 8, 2, 2, 4, 8};

static int conversion_kind(uint32_t s, uint32_t d) {
  if (s > 12 || d > 12) return -1;
  if (s == d) return K_COPY1;
  if (s == HL_DT_BF16 && d == HL_DT_F16) return K_BF16_F16;
  if (s == HL_DT_F32 && d == HL_DT_F16) return K_F32_F16;
  if (s == HL_DT_F16 && d == HL_DT_F32) return K_F16_F32;
  if (s == HL_DT_BF16 && d == HL_DT_F32) return K_BF16_F32;
  return -1;
}

static std::atomic<uint64_t> g_launches{0};

// Optional launch timing (hl_gather_timing): a CUDA event pair per hl_gather
// call, recorded on its stream right before the first kernel launch and after
// the last one — the host-side descriptor translation stays outside, so a
// short launch is timed as the kernels, not as the host path in front of them.
static std::mutex g_timing_mu;
static std::atomic<bool> g_timing_on{false};
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_timing_events;

struct LaunchTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  explicit LaunchTimer(cudaStream_t st) : s(st) {
    if (!g_timing_on.load(std::memory_order_relaxed)) return;  // the hot path: one relaxed load
    if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess ||
        cudaEventRecord(a, s) != cudaSuccess) {
      cudaGetLastError();
      release();
    }
  }
  void done() {
    if (!a) return;
    if (cudaEventRecord(b, s) != cudaSuccess) {
      cudaGetLastError();
      release();
      return;
    }
    std::lock_guard<std::mutex> g(g_timing_mu);
    g_timing_events.emplace_back(a, b);
    a = b = nullptr;
  }
  void release() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    a = b = nullptr;
  }
  ~LaunchTimer() { release(); }
};

// which: 0 = generic, 1 + RowClass = row kernel of that class
template <class P, int K>
static auto kernel_for(int which) -> void (*)(P) {
  switch (which) {
    case 0: return generic_kernel<K, P>;
    case 1 + R_ALIGNED: return row_kernel<K, P, R_ALIGNED>;
    case 1 + R_SHIFTED: return row_kernel<K, P, R_SHIFTED>;
    default: return row_kernel<K, P, R_MIXED>;
  }
}
// Contiguous aligned raw copies (whole tensors, dim-0 shards) run on the TMA
// bulk kernel (32 threads, kBulkSmem of dynamic shared memory). Multi-row
// descriptors (column shards: rows of 2-14 KiB) stay on the LDG/STG row kernel,
// where 32 lanes share the per-row address work.
constexpr int kBulkWhich = 4;
static bool is_bulk(int kind, int which) { return kind == K_COPY1 && which == kBulkWhich; }
// Contiguous casts and realigns run on the TMA-staged kernel.
constexpr int kStagedWhich = 5;
static bool is_staged(int which) { return which == kStagedWhich; }
template <class P>
static auto staged_of(int kind) -> void (*)(P) {
  switch (kind) {
    case K_COPY1: return staged_kernel<K_COPY1, P>;
    case K_BF16_F16: return staged_kernel<K_BF16_F16, P>;
    case K_F32_F16: return staged_kernel<K_F32_F16, P>;
    case K_F16_F32: return staged_kernel<K_F16_F32, P>;
    default: return staged_kernel<K_BF16_F32, P>;
  }
}

template <class P>
static auto kernel_of(int kind, int which) -> void (*)(P) {
  if (is_bulk(kind, which)) return bulk_kernel<P>;
  if (is_staged(which)) return staged_of<P>(kind);
  switch (kind) {
    case K_COPY1: return kernel_for<P, K_COPY1>(which);
    case K_BF16_F16: return kernel_for<P, K_BF16_F16>(which);
    case K_F32_F16: return kernel_for<P, K_F32_F16>(which);
    case K_F16_F32: return kernel_for<P, K_F16_F32>(which);
    default: return kernel_for<P, K_BF16_F32>(which);
  }
}
constexpr int kWhich = 6;  // generic, 3 row classes, bulk, staged

struct DevInfo {
  int sms = 0;
  int blocks_per_sm[5][kWhich] = {};
};

// Resident-grid cap of one kernel variant on the current device: SM count x
// blocks per SM, queried the first time that variant launches (querying all
// 20 variants up front would load every kernel of the module in a fresh
// process — lazy module loading makes that a first-load cost).
static uint64_t grid_cap(int kind, int which) {
  static std::mutex mu;
  static DevInfo cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  DevInfo& di = cache[dev & 63];
  if (di.sms == 0) cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev);
  if (di.blocks_per_sm[kind][which] == 0) {
    int b = 0;
    if (is_bulk(kind, which) || is_staged(which)) {
      // bulk: one CTA per SM keeps its stages in flight (more CTAs measured slower);
      // staged: two, so 32 consumer warps per SM hide the conversion latency
      const int smem = (int)(is_bulk(kind, which) ? kBulkSmem : staged_smem(kind));
      cudaFuncSetAttribute(kernel_of<Params>(kind, which), cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(kernel_of<SmallParams>(kind, which), cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      b = is_bulk(kind, which) ? 1 : kStagedCtasPerSm;
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel_of<Params>(kind, which), kThreads, 0);
    }
    di.blocks_per_sm[kind][which] = b > 0 ? b : 1;
  }
  return (uint64_t)di.sms * di.blocks_per_sm[kind][which];
}

// Translate one ABI descriptor into kernel descriptors: the main one, plus an
// element-path descriptor for the < 16-byte tail of a single-row copy.
// Returns the number produced (0 = empty descriptor).
static int make_kdesc(const hl_desc& h, uint32_t i, KDesc out[2], uint64_t units[2], int* count, bool tma) {
  *count = 0;
  const int kind = conversion_kind(h.src_dtype, h.dst_dtype);
  if (kind < 0) return set_error(HL_ECONV, "unsupported conversion %u -> %u (descriptor %u)", h.src_dtype, h.dst_dtype, i);
  const uint32_t ss = kSize[h.src_dtype], ds = kSize[h.dst_dtype];
  if (h.rows == 0 || h.row_elems == 0) return HL_OK;
  if (!h.src || !h.dst) return set_error(HL_EINVAL, "descriptor %u: null pointer", i);
  if (h.dst % ds) return set_error(HL_EALIGN, "descriptor %u: dst 0x%llx not aligned to %u", i, (unsigned long long)h.dst, ds);
  KDesc k{};
  k.src = h.src;
  k.dst = h.dst;
  k.kind = (uint8_t)kind;
  k.ss = (uint8_t)ss;
  k.ds = (uint8_t)ds;
  uint64_t rows = h.rows, relems = h.row_elems;
  const uint64_t pitch = h.src_pitch;
  if (rows > 1 && pitch == relems * ss) {  // contiguous rows collapse into one
    relems *= rows;
    rows = 1;
  }
  k.src_pitch = pitch;
  const uint64_t out_row = relems * ds;
  auto elem = [&](KDesc e, uint64_t nrows, uint64_t n_per_row) {
    e.mode = M_ELEM;
    e.which = 0;
    e.nvec = nrows * n_per_row;
    e.row_len = n_per_row;
    out[*count] = e;
    units[*count] = (e.nvec + kUnitElems - 1) / kUnitElems;
    ++*count;
  };
  if (h.dst % 16 == 0 && (rows == 1 || out_row % 16 == 0)) {
    const uint64_t vpr = out_row / 16;
    if (vpr) {
      k.row_len = vpr;
      k.nvec = rows * vpr;
      if (rows == 1 || vpr >= kMinRowVecs) {
        k.mode = M_ROWS;
        const uint64_t g = (kind == K_F16_F32 || kind == K_BF16_F32) ? 8 : 16;  // load granule
        const bool uniform = rows == 1 || pitch % g == 0;
        k.which = 1 + (uniform ? (h.src % g == 0 ? R_ALIGNED : R_SHIFTED) : R_MIXED);
        // contiguous: aligned raw copies -> TMA bulk; misaligned sources -> TMA-staged
        // (aligned casts measured faster on the LDG/STG row kernel: 6.05 vs 5.72 TB/s bf16->f16)
        if (tma && rows == 1 && kind == K_COPY1 && k.which == 1 + R_ALIGNED) k.which = kBulkWhich;
        if (tma && rows == 1 && (k.which == 1 + R_SHIFTED ||
                          (HL_STAGED_ALIGNED && k.which == 1 + R_ALIGNED && staged_tma_store(kind))))
          k.which = kStagedWhich;
        const uint64_t uv = is_bulk(kind, k.which) ? kBulkVecs
                            : is_staged(k.which) ? staged_unit_vecs(kind) : row_unit_vecs(kind);
        k.upr = (uint32_t)((vpr + uv - 1) / uv);
        units[*count] = rows * k.upr;
      } else {
        k.mode = M_PACKED;
        units[*count] = (k.nvec + kUnitVecs - 1) / kUnitVecs;
      }
      out[(*count)++] = k;
    }
    const uint64_t tail = rows == 1 ? (out_row % 16) / ds : 0;
    if (tail) {
      KDesc t = k;
      const uint64_t done = vpr * (16 / ds);  // elements covered by the vectors
      t.src = h.src + done * ss;
      t.dst = h.dst + done * ds;
      t.upr = 0;
      elem(t, 1, tail);
    }
  } else {
    elem(k, rows, relems);
  }
  return HL_OK;
}

// ---- TMA tensor tiles (host): tensor maps for column-shard descriptors
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
static EncodeTiled encode_tiled() {
  static EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      p = nullptr;
    }
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

// Largest interleave group (tile_unit); $HL_TILE_GROUP=1 keeps descriptor-major order.
static size_t tile_group() {
  static const size_t g = [] {
    const char* e = getenv("HL_TILE_GROUP");
    const long v = e ? strtol(e, nullptr, 10) : 16;
    return (size_t)std::max(1L, std::min(v, 64L));
  }();
  return g;
}

static bool tiles_enabled() {
  static const bool on = [] {
    const char* e = getenv("HL_GATHER_TILES");
    return !(e && e[0] == '0');
  }();
  return on && encode_tiled() != nullptr;
}

static CUtensorMapDataType tmap_type(uint32_t bytes) {
  switch (bytes) {
    case 1: return CU_TENSOR_MAP_DATA_TYPE_UINT8;
    case 2: return CU_TENSOR_MAP_DATA_TYPE_UINT16;
    case 4: return CU_TENSOR_MAP_DATA_TYPE_UINT32;
    default: return CU_TENSOR_MAP_DATA_TYPE_UINT64;
  }
}

// A column shard the tile kernels take: several rows, a source pitch larger
// than the row, 16-byte aligned destination rows of at least 64 bytes.
// Fills `t` (all but unit_begin) and its unit (box) count; false = not a tile.
static bool make_tile(const hl_desc& h, int kind, TileDesc& t, uint64_t& units) {
  const uint32_t ss = kSize[h.src_dtype], ds = kSize[h.dst_dtype];
  if (h.rows < 2 || h.row_elems == 0) return false;
  const uint64_t in_row = h.row_elems * ss, out_row = h.row_elems * ds;
  if (h.src_pitch == in_row) return false;  // contiguous rows: bulk / staged kernels
  // A box whose first byte is not 16-byte aligned faults the TMA unit (illegal
  // instruction; tools/tile_probe.cu, profiles/r02_tile_probe.jsonl), so the
  // segment must start 16-byte aligned: every TP=2/4/8 shard of an LLM weight
  // does; others (TP=3 of 4096 columns, realigned odd landings) stay on the
  // LDG/STG row kernel.
  if (h.dst % 16 || h.src % 16 || out_row % 16 || out_row < 64 || h.src_pitch % 16) return false;
  if (h.src_pitch >= (1ull << 40) || h.rows >= (1ull << 31)) return false;
  const uint64_t base = h.src;
  const uint32_t lead = 0;
  uint32_t ui = ss, uo = ds;  // tensor-map element bytes
  if (kind == K_COPY1) {      // raw bytes: the widest unit the row allows
    uint32_t u = 8;
    while (u > 1 && in_row % u) u >>= 1;
    ui = uo = u;
  }
  const uint64_t cols = in_row / ui;  // = out_row / uo
  const uint32_t wide = std::max(ui, uo), g = 16 / std::min(ui, uo);
  const uint64_t bx_max = std::min<uint64_t>(256, 2048 / wide);
  const uint32_t bx = (uint32_t)std::min<uint64_t>(bx_max, (cols + g - 1) / g * g);
  const uint32_t by = (uint32_t)std::min<uint64_t>({256, kTileBox / ((uint64_t)bx * wide), h.rows});
  t.c0 = (int32_t)(lead / ui);
  t.bx = bx;
  t.by = by;
  t.nbx = (uint32_t)((cols + bx - 1) / bx);
  t.in_bytes = bx * by * ui;
  units = (uint64_t)t.nbx * ((h.rows + by - 1) / by);
  const cuuint32_t box[2] = {bx, by}, estr[2] = {1, 1};
  const cuuint64_t sdim[2] = {t.c0 + cols, h.rows}, sstr[1] = {h.src_pitch};
  const cuuint64_t ddim[2] = {cols, h.rows}, dstr[1] = {out_row};
  EncodeTiled enc = encode_tiled();
  if (enc(&t.src, tmap_type(ui), 2, reinterpret_cast<void*>(base), sdim, sstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (enc(&t.dst, tmap_type(uo), 2, reinterpret_cast<void*>(h.dst), ddim, dstr, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  return true;
}

static auto tile_kernel_of(int kind) -> void (*)(TileParams) {
  switch (kind) {
    case K_COPY1: return tile_copy_kernel;
    case K_BF16_F16: return tile_cast_kernel<K_BF16_F16>;
    case K_F32_F16: return tile_cast_kernel<K_F32_F16>;
    case K_F16_F32: return tile_cast_kernel<K_F16_F32>;
    default: return tile_cast_kernel<K_BF16_F32>;
  }
}
static size_t tile_smem(int kind) {
  return kind == K_COPY1 ? (size_t)kTileStages * kTileBox : (size_t)2 * kTileCastStages * kTileBox;
}

static int launch_tiles(int kind, TileParams& p, cudaStream_t stream) {
  if (p.total_units == 0) return HL_OK;
  static std::mutex mu;
  static bool attr_set[64][5] = {};
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  {
    std::lock_guard<std::mutex> g(mu);
    if (!attr_set[dev & 63][kind]) {
      cudaFuncSetAttribute(tile_kernel_of(kind), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile_smem(kind));
      attr_set[dev & 63][kind] = true;
    }
  }
  const uint64_t cap = (uint64_t)sms * (kind == K_COPY1 ? 1 : HL_TILE_CAST_CTAS);
  const unsigned grid = (unsigned)std::min<uint64_t>(p.total_units, cap);
  tile_kernel_of(kind)<<<grid, kind == K_COPY1 ? 32 : kTileCastThreads, tile_smem(kind), stream>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(HL_ECUDA, "tile launch failed: %s", cudaGetErrorString(e));
  g_launches.fetch_add(1);
  p.n = 0;
  p.total_units = 0;
  return HL_OK;
}

static int launch(int kind, int which, Params& p, cudaStream_t stream) {
  if (p.total_units == 0) return HL_OK;
  const bool bulk = is_bulk(kind, which), staged = is_staged(which);
  const uint64_t want = (bulk || staged) ? p.total_units : (p.total_units + kWarps - 1) / kWarps;
  const uint64_t cap = grid_cap(kind, which);
  const unsigned grid = (unsigned)(want < cap ? want : cap);
  const unsigned threads = bulk ? 32 : staged ? kStagedThreads : kThreads;
  const size_t smem = bulk ? kBulkSmem : staged ? staged_smem(kind) : 0;
  if (p.n <= (uint32_t)kSmallDescs) {
    SmallParams sp;
    sp.n = p.n;
    sp.pad = 0;
    sp.total_units = p.total_units;
    for (uint32_t i = 0; i < p.n; ++i) sp.d[i] = p.d[i];
    kernel_of<SmallParams>(kind, which)<<<grid, threads, smem, stream>>>(sp);
  } else {
    kernel_of<Params>(kind, which)<<<grid, threads, smem, stream>>>(p);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(HL_ECUDA, "gather launch failed: %s", cudaGetErrorString(e));
  g_launches.fetch_add(1);
  p.n = 0;
  p.total_units = 0;
  return HL_OK;
}

}  // namespace hl

using namespace hl;

extern "C" int hl_conversion_supported(uint32_t s, uint32_t d) { return conversion_kind(s, d) >= 0 ? 1 : 0; }

extern "C" uint32_t hl_gather_max_batch(void) { return kMaxDescs; }

extern "C" uint64_t hl_kernel_launches(void) { return g_launches.load(); }

extern "C" int hl_gather_timing(int enable) {
  clear_error();
  std::lock_guard<std::mutex> g(g_timing_mu);
  g_timing_on = enable != 0;
  for (auto& e : g_timing_events) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  g_timing_events.clear();
  return HL_OK;
}

extern "C" int hl_gather_timings(float* ms, uint32_t cap, uint32_t* n) {
  clear_error();
  if (!n) return set_error(HL_EINVAL, "null argument");
  std::lock_guard<std::mutex> g(g_timing_mu);
  *n = (uint32_t)g_timing_events.size();
  int rc = HL_OK;
  for (size_t i = 0; i < g_timing_events.size(); ++i) {
    auto& e = g_timing_events[i];
    float t = -1.0f;
    if (cudaEventSynchronize(e.second) != cudaSuccess || cudaEventElapsedTime(&t, e.first, e.second) != cudaSuccess) {
      rc = set_error(HL_ECUDA, "launch timing: %s", cudaGetErrorString(cudaGetLastError()));
    }
    if (ms && i < cap) ms[i] = t;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  g_timing_events.clear();
  return rc;
}

extern "C" int hl_gather_prepare(int device) {
  // Load every kernel variant and set its launch attributes ahead of the first
  // hl_gather (CUDA loads kernels lazily, on first use): the loader calls this
  // on a side thread while the first file transfer runs, so a fresh process's
  // first retrievals do not pay the module loading.
  clear_error();
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return set_error(HL_ECUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
  for (int kind = 0; kind < 5; ++kind) {
    for (int which = 0; which < kWhich; ++which) {
      if (which == kBulkWhich && kind != K_COPY1) continue;  // bulk copies only
      cudaFuncAttributes a;
      cudaFuncGetAttributes(&a, kernel_of<SmallParams>(kind, which));
      grid_cap(kind, which);  // the Params variant: occupancy / shared-memory attributes
    }
  }
  for (int kind = 0; kind < 5; ++kind) {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, tile_kernel_of(kind));
    cudaFuncSetAttribute(tile_kernel_of(kind), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile_smem(kind));
  }
  encode_tiled();
  cudaGetLastError();
  cudaSetDevice(prev);
  return HL_OK;
}

extern "C" int hl_gather(const hl_desc* descs, uint32_t n, void* stream) { return hl_gather_ex(descs, n, stream, 0); }

extern "C" int hl_gather_ex(const hl_desc* descs, uint32_t n, void* stream, uint32_t flags) {
  clear_error();
  const bool tma = !(flags & HL_GATHER_NO_TMA);
  if (n && !descs) return set_error(HL_EINVAL, "null descriptor table");
  // translate + validate everything once, before launching anything
  static thread_local std::vector<KDesc> kds;
  static thread_local std::vector<uint64_t> units;
  static thread_local std::vector<uint16_t> bucket;  // kind * kWhich + which
  kds.clear();
  units.clear();
  bucket.clear();
  KDesc kd[2];
  uint64_t ku[2];
  int cnt = 0;
  uint32_t present = 0;  // bitmask of non-empty buckets
  static thread_local std::vector<TileDesc> tiles[5];  // column shards per conversion kind
  static thread_local std::vector<uint64_t> tile_units[5];
  for (int k = 0; k < 5; ++k) {
    tiles[k].clear();
    tile_units[k].clear();
  }
  const bool use_tiles = tma && tiles_enabled();
  for (uint32_t i = 0; i < n; ++i) {
    if (use_tiles) {
      const int kind = conversion_kind(descs[i].src_dtype, descs[i].dst_dtype);
      TileDesc t;
      uint64_t tu = 0;
      if (kind >= 0 && descs[i].src && descs[i].dst && make_tile(descs[i], kind, t, tu)) {
        tiles[kind].push_back(t);
        tile_units[kind].push_back(tu);
        continue;
      }
    }
    int rc = make_kdesc(descs[i], i, kd, ku, &cnt, tma);
    if (rc) return rc;
    for (int j = 0; j < cnt; ++j) {
      const uint16_t b = (uint16_t)(kd[j].kind * kWhich + kd[j].which);
      kds.push_back(kd[j]);
      units.push_back(ku[j]);
      bucket.push_back(b);
      present |= 1u << b;
    }
  }
  LaunchTimer timer((cudaStream_t)stream);  // hl_gather_timing: events around the launches only
  static thread_local Params* p = nullptr;  // ~32 KB: keep it off the stack
  if (!p) p = new Params();
  // one launch per (conversion kind, kernel variant) present in the batch
  for (int b = 0; b < 5 * kWhich; ++b) {
    if (!(present & (1u << b))) continue;
    const int kind = b / kWhich, which = b % kWhich;
    p->n = 0;
    p->total_units = 0;
    for (size_t i = 0; i < kds.size(); ++i) {
      if (bucket[i] != b) continue;
      kds[i].unit_begin = p->total_units;
      p->d[p->n++] = kds[i];
      p->total_units += units[i];
      if (p->n == (uint32_t)kMaxDescs) {
        int rc = launch(kind, which, *p, (cudaStream_t)stream);
        if (rc) return rc;
      }
    }
    int rc = launch(kind, which, *p, (cudaStream_t)stream);
    if (rc) return rc;
  }
  static thread_local TileParams* tp = nullptr;  // ~30 KB
  for (int kind = 0; kind < 5; ++kind) {
    if (tiles[kind].empty()) continue;
    if (!tp) tp = new TileParams();
    tp->n = 0;
    tp->total_units = 0;
    const auto& tv = tiles[kind];
    const auto& uv = tile_units[kind];
    for (size_t i = 0; i < tv.size();) {
      // an interleave group: consecutive tiles with equal unit counts (a tensor's W shards)
      size_t j = i + 1;
      while (j < tv.size() && j - i < tile_group() && uv[j] == uv[i]) ++j;
      const uint32_t g = (uint32_t)(j - i);
      if (tp->n + g > (uint32_t)kMaxTiles) {
        int rc = launch_tiles(kind, *tp, (cudaStream_t)stream);
        if (rc) return rc;
      }
      for (uint32_t m = 0; m < g; ++m) {
        TileDesc& t = tp->d[tp->n++];
        t = tv[i + m];
        t.unit_begin = tp->total_units;
        t.grp = (uint16_t)g;
        t.gi = (uint16_t)m;
      }
      tp->total_units += (uint64_t)g * uv[i];
      i = j;
    }
    int rc = launch_tiles(kind, *tp, (cudaStream_t)stream);
    if (rc) return rc;
  }
  timer.done();
  return HL_OK;
}
