/*
 * oracle_c.c — CPU restatement of the reference's byte/float arithmetic for
 * the load path. TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg use it as the checker; the product path
 * never links or calls it.
 *
 * What it restates (reference = /root/reference/pkg/src/aggload):
 *   - device.py:303-320  _as_f32 / _convert_elements: BF16 widens by bits<<16;
 *     F16 widens exactly; narrowing to F16 is numpy's astype(np.float16).
 *     numpy (not vendored; pyproject.toml:10 "numpy>=1.24", 2.3.5 here) does
 *     that with npy_floatbits_to_halfbits / npy_halfbits_to_floatbits
 *     (numpy/_core/src/npymath/halffloat.cpp): round-to-nearest-even with a
 *     sticky check on the bits shifted out for subnormal results, overflow to
 *     +-inf, NaN -> sign | 0x7c00 | (mantissa >> 13) forced non-zero (no
 *     quieting), and F16 -> F32 NaN keeps its payload.
 *   - collective.py:318-330 _clone_slice / reference.py:56-66 load_shard_bytes:
 *     a rank's slice [lo, hi) along dim d of a row-major tensor, as
 *     rows = prod(shape[:d]) strided row copies.
 * Pinned against the reference itself: tests/golden/ holds vectors produced
 * by the reference's own functions (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <string.h>

/* dtype codes: the order of format.DType / include/hbmload.h hl_dtype */
enum { DT_BOOL, DT_U8, DT_I8, DT_I16, DT_U16, DT_I32, DT_U32, DT_I64, DT_U64, DT_F16, DT_BF16, DT_F32, DT_F64 };
static const int SIZES[13] = {1, 1, 1, 2, 2, 4, 4, 8, 8, 2, 2, 4, 8};

uint16_t oracle_f32_to_f16(uint32_t f) {
  uint32_t f_exp = f & 0x7f800000u, f_sig;
  uint16_t h_sgn = (uint16_t)((f & 0x80000000u) >> 16);
  if (f_exp >= 0x47800000u) {          /* overflow, inf or NaN */
    if (f_exp == 0x7f800000u) {
      f_sig = f & 0x007fffffu;
      if (f_sig != 0) {
        uint16_t r = (uint16_t)(0x7c00u + (f_sig >> 13));
        if (r == 0x7c00u) r++;         /* stay a NaN */
        return (uint16_t)(h_sgn + r);
      }
      return (uint16_t)(h_sgn + 0x7c00u);
    }
    return (uint16_t)(h_sgn + 0x7c00u);
  }
  if (f_exp <= 0x38000000u) {          /* subnormal half or signed zero */
    if (f_exp < 0x33000000u) return h_sgn;
    f_exp >>= 23;
    f_sig = 0x00800000u + (f & 0x007fffffu);
    f_sig >>= (113 - f_exp);
    /* ties-to-even: add the rounding bit unless exactly a tie onto an even
       value; bits lost by the shift above are checked in the original */
    if (((f_sig & 0x00003fffu) != 0x00001000u) || (f & 0x000007ffu)) f_sig += 0x00001000u;
    return (uint16_t)(h_sgn + (uint16_t)(f_sig >> 13));
  }
  uint16_t h_exp = (uint16_t)((f_exp - 0x38000000u) >> 13);
  f_sig = f & 0x007fffffu;
  if ((f_sig & 0x00003fffu) != 0x00001000u) f_sig += 0x00001000u;
  uint16_t h_sig = (uint16_t)(f_sig >> 13);
  h_sig = (uint16_t)(h_sig + h_exp);  /* a carry into the exponent is correct (may reach inf) */
  return (uint16_t)(h_sgn + h_sig);
}

uint32_t oracle_f16_to_f32(uint16_t h) {
  uint16_t h_exp = h & 0x7c00u, h_sig;
  uint32_t f_sgn = ((uint32_t)h & 0x8000u) << 16;
  switch (h_exp) {
    case 0x0000u:
      h_sig = h & 0x03ffu;
      if (h_sig == 0) return f_sgn;
      h_sig <<= 1;
      while ((h_sig & 0x0400u) == 0) {
        h_sig <<= 1;
        h_exp++;
      }
      return f_sgn + (((uint32_t)(127 - 15 - h_exp)) << 23) + (((uint32_t)(h_sig & 0x03ffu)) << 13);
    case 0x7c00u:
      return f_sgn + 0x7f800000u + (((uint32_t)(h & 0x03ffu)) << 13);
    default:
      return f_sgn + (((uint32_t)(h & 0x7fffu) + 0x1c000u) << 13);
  }
}

static uint64_t load(const uint8_t* p, int sz) {
  uint64_t x = 0;
  memcpy(&x, p, (size_t)sz); /* little endian host */
  return x;
}
static void store(uint8_t* p, int sz, uint64_t x) { memcpy(p, &x, (size_t)sz); }

/* 1 if supported (identity, BF16->F16, F32->F16, F16->F32, BF16->F32; ref device.py:293-298) */
int oracle_conversion_supported(int s, int d) {
  if (s < 0 || s > 12 || d < 0 || d > 12) return 0;
  if (s == d) return 1;
  return (s == DT_BF16 && d == DT_F16) || (s == DT_F32 && d == DT_F16) || (s == DT_F16 && d == DT_F32) ||
         (s == DT_BF16 && d == DT_F32);
}

static uint64_t convert1(uint64_t x, int s, int d) {
  if (s == d) return x;
  uint32_t f32;
  if (s == DT_BF16) f32 = (uint32_t)x << 16;
  else if (s == DT_F16) f32 = oracle_f16_to_f32((uint16_t)x);
  else f32 = (uint32_t)x;
  if (d == DT_F32) return f32;
  return oracle_f32_to_f16(f32);
}

/* Strided 2-D copy with conversion: the same contract as hl_desc. Returns 0,
   or -5 for an unsupported pair (HL_ECONV). */
int oracle_gather(const uint8_t* src, uint8_t* dst, uint64_t rows, uint64_t row_elems, uint64_t src_pitch,
                  int sdt, int ddt) {
  if (!oracle_conversion_supported(sdt, ddt)) return -5;
  const int ss = SIZES[sdt], ds = SIZES[ddt];
  for (uint64_t r = 0; r < rows; ++r) {
    const uint8_t* s = src + r * src_pitch;
    uint8_t* o = dst + r * row_elems * (uint64_t)ds;
    if (sdt == ddt) {
      memcpy(o, s, row_elems * (uint64_t)ss);
      continue;
    }
    for (uint64_t c = 0; c < row_elems; ++c) store(o + c * ds, ds, convert1(load(s + c * ss, ss), sdt, ddt));
  }
  return 0;
}
