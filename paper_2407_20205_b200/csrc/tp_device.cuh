// tp_device.cuh -- device-side primitives of the B200 Gray-code Ryser walk.
//
// Encoding.  The reference packs a trit vector as (mag, sgn) bit planes
// (src/core_f3.py:1-21).  On the device every running column
// vector is held as 32-bit words (z, g) with z = ~mag (bit set <=> trit is
// zero) and g = sgn.  The reference's sub_reps (src/core_f3.py:134-138)
//     d = mag & (sgn ^ s2);  mag' = d | (mag ^ m2);  sgn' = d ^ m2 ^ s2
// becomes, with mag = ~z,
//     d  = ~z & (g ^ s2)      lop3 lut 0x06 over (z, g, s2)
//     z' = ~d & (z ^ m2)      lop3 lut 0x06 over (d, z, m2)
//     g' = d ^ m2 ^ s2        lop3 lut 0x96 over (d, m2, s2)
// i.e. exactly three LOP3 per 32 columns (a brute-force search over all
// 2-bit encodings finds no 2-op sequence), and "every column nonzero"
// (src/core_f3.py:159-161) is z' == 0: ptxas folds that test into the
// predicate output of the LOP3 that produces z', so the full-magnitude test
// costs no ALU instruction.  ADD of a row is SUB of the negated row
// (m2, m2 ^ s2) (closure under alternate zeros, src/core_f3.py:9-12), so the
// walk only ever issues the sub sequence, with a pre-negated operand.
//
// Padding columns (bits >= n) carry a constant nonzero trit (z = 0, g = 0):
// rows are zero there, and sub of a zero column leaves (z, g) unchanged, so
// the full test needs no mask (the reference masks, src/_kernels.py:99,123).
#pragma once
#include <cstdint>

namespace tp {

#define TP_LOP3(d, a, b, c, lut) \
  asm("lop3.b32 %0, %1, %2, %3, " #lut ";" : "=r"(d) : "r"(a), "r"(b), "r"(c))

constexpr unsigned FULL = 0xffffffffu;

// One packed matrix row as the walk consumes it.  w = 32-column word
// (word 0 = reference plane bits 0..31, word 1 = bits 32..63).
// m = mag, s = sgn (SUB operand), a = m ^ s (ADD operand = negated row).
struct __align__(32) RowRec {
  uint32_t m[2];
  uint32_t s[2];
  uint32_t a[2];
  uint32_t pad[2];
};

__host__ __device__ constexpr int ctz_c(int j) {
  int t = 0;
  while (!(j & 1)) { j >>= 1; ++t; }
  return t;
}

// z-encoded SUB of one 32-column word (see header).
__device__ __forceinline__ void sub_word(uint32_t& z, uint32_t& g, uint32_t m, uint32_t s) {
  uint32_t d, zn, gn;
  TP_LOP3(d, z, g, s, 0x06);
  TP_LOP3(zn, d, z, m, 0x06);
  TP_LOP3(gn, d, m, s, 0x96);
  z = zn;
  g = gn;
}

// Reference add_reps formula (src/core_f3.py:123-131) on (mag, sgn), used by
// the self-test only: c = m2 & (mag ^ sgn ^ s2); mag' = c | (mag ^ m2); sgn' = c ^ sgn.
__device__ __forceinline__ void add_ref_word(uint32_t& mag, uint32_t& sgn, uint32_t m2, uint32_t s2) {
  uint32_t x, c, mn, sn;
  TP_LOP3(x, mag, sgn, s2, 0x96);
  TP_LOP3(c, m2, x, 0u, 0xC0);
  TP_LOP3(mn, c, mag, m2, 0xF6);
  TP_LOP3(sn, c, sgn, 0u, 0x3C);
  mag = mn;
  sgn = sn;
}

// Inverse 5-bit Gray code.
__device__ __forceinline__ uint32_t ginv5(uint32_t x) {
  x ^= x >> 1;
  x ^= x >> 2;
  x ^= x >> 4;
  return x & 31u;
}

// Event recording on the fast path.  The predicate p = (z == 0) comes for
// free from the LOP3 that produced z; both consumers are predicated IMADs
// (FMA pipe), so the ALU pipe only sees the three LOP3 of the step.
// `one` is a runtime 1 the compiler cannot fold (keeps these as IMAD).
__device__ __forceinline__ void record_slot(uint32_t z, uint32_t g, uint32_t& cnt, uint32_t& slot, uint32_t one) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.eq.u32 p, %2, 0;\n\t"
      "@p mad.lo.u32 %0, %4, %4, %0;\n\t"
      "@p mad.lo.u32 %1, %3, %4, 0;\n\t}"
      : "+r"(cnt), "+r"(slot)
      : "r"(z), "r"(g), "r"(one));
}

__device__ __forceinline__ void record_count(uint32_t z, uint32_t& cnt, uint32_t one) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.eq.u32 p, %1, 0;\n\t"
      "@p mad.lo.u32 %0, %2, %2, %0;\n\t}"
      : "+r"(cnt)
      : "r"(z), "r"(one));
}

template <int NW>
__device__ __forceinline__ bool is_full(const uint32_t (&z)[2]) {
  if (NW == 1) return z[0] == 0;
  return (z[0] | z[1]) == 0;
}

template <int NW>
__device__ __forceinline__ uint32_t sign_parity(const uint32_t (&g)[2]) {
  if (NW == 1) return __popc(g[0]) & 1u;
  return (__popc(g[0]) + __popc(g[1])) & 1u;
}

// Starting vector of lane `lane` at high step `a`: the subset
// (gray(a) << 5) | lane, i.e. rows 0..4 from the lane bits and rows >= 5 from
// gray(a) (random access seeding, src/graycode.py:41-45,
// src/_kernels.py:99-109).  Rows are ADDed (= SUB of the negated row).
template <int NW>
__device__ __forceinline__ void seed_state(const RowRec* R, int n, unsigned long long a, uint32_t lane,
                                           uint32_t z0i, uint32_t z1i, uint32_t (&z)[2], uint32_t (&g)[2]) {
  z[0] = z0i;
  z[1] = z1i;
  g[0] = 0;
  g[1] = 0;
  const unsigned long long hs = a ^ (a >> 1);
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    if (((lane >> r) & 1u) && r < n) {
#pragma unroll
      for (int w = 0; w < NW; ++w) sub_word(z[w], g[w], R[r].m[w], R[r].a[w]);
    }
  }
  for (int r = 5; r < n; ++r) {
    if ((hs >> (r - 5)) & 1ull) {
#pragma unroll
      for (int w = 0; w < NW; ++w) sub_word(z[w], g[w], R[r].m[w], R[r].a[w]);
    }
  }
}

// One runtime Gray step to high step a (a >= 1): flip row 5 + tz(a); the row
// leaves iff bit tz(a)+1 of a is set (graycode.advance, src/graycode.py:48-61;
// src/_kernels.py:112-122).
template <int NW>
__device__ __forceinline__ void runtime_step(const RowRec* R, unsigned long long a, uint32_t (&z)[2],
                                             uint32_t (&g)[2]) {
  const int t = __ffsll((long long)a) - 1;
  const bool leave = (a >> (t + 1)) & 1ull;
  const RowRec& row = R[5 + t];
#pragma unroll
  for (int w = 0; w < NW; ++w) sub_word(z[w], g[w], row.m[w], leave ? row.s[w] : row.a[w]);
}

}  // namespace tp
