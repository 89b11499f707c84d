// tp_walk_common.cuh -- device helpers shared by the walk kernels
// (tp_walk_lane.cu, tp_walk_wide.cu, tp_walk_pair.cu): replays, the work
// queue, row loading, per-warp flushes, compile-time loops and the pair-test
// primitives.
#pragma once
#include <utility>

#include "tp_device.cuh"
#include "tp_kernels.cuh"

namespace tp {

// ---------------------------------------------------------------------------
// Exact replay of one superblock from its saved entry state.  Used only when
// the fast path's event slots cannot represent the block exactly (two events
// of the same step parity in one lane, or -- for NW=2 -- any primary event).
// abase is even, so the parity of step abase+j is j&1.
// ---------------------------------------------------------------------------
// Returns ev | odd << 32.
template <int NW>
__device__ __noinline__ unsigned long long replay_block(const RowRec* R, uint32_t ze0, uint32_t ze1, uint32_t ge0,
                                                        uint32_t ge1, unsigned long long abase, int len,
                                                        uint32_t lanepar) {
  uint32_t z[2] = {ze0, ze1}, g[2] = {ge0, ge1};
  uint32_t ev = 0, odd = 0;
  for (int j = 0; j < len; ++j) {
    if (j > 0) runtime_step<NW>(R, abase + (unsigned long long)j, z, g);
    if (is_full<NW>(z)) {
      ev += 1;
      odd += (sign_parity<NW>(g) ^ (uint32_t)(j & 1) ^ lanepar) & 1u;
    }
  }
  return (unsigned long long)ev | ((unsigned long long)odd << 32);
}

__device__ __forceinline__ void warp_flush(unsigned long long* pm, uint32_t plus, uint32_t minus, uint32_t lane) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    plus += __shfl_xor_sync(FULL, plus, off);
    minus += __shfl_xor_sync(FULL, minus, off);
  }
  if (lane == 0) {
    if (plus) atomicAdd(pm, (unsigned long long)plus);
    if (minus) atomicAdd(pm + 1, (unsigned long long)minus);
  }
}

// ---------------------------------------------------------------------------
// Work distribution of the fast walks.  Items are L-aligned chunks of one
// matrix's fast region (L = nblk superblocks, a power of two), taken from a
// global atomic queue: B200's warp arbiter is not fair (highest warp id
// first), so a static split leaves the starved warps as a long tail, while a
// dynamic queue lets the favoured warps take more items.  Because every item
// starts at a multiple of L, the superblock loop below runs on a kernel
// parameter and the entry row of superblock kb is 5+V+tz(kb) -- the loop
// control, row indices and step directions are warp-uniform and live on the
// uniform datapath, so the vector ALU pipe only sees the LOP3s of the walk.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int tz64(unsigned long long a) {
  const uint32_t lo = (uint32_t)a;
  return lo ? __ffs(lo) - 1 : 31 + __ffs((uint32_t)(a >> 32));
}

// Copy rows 0..n-1 (two uint4 per 32-byte RowRec); rows >= n stay stale and
// are never read by the walks (row indices are < n).
__device__ __forceinline__ void load_rows(RowRec* R, const RowRec* src, uint32_t lane, int n) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(R);
  for (int q = lane; q < 2 * n; q += 32) d[q] = s[q];
}

// Broadcast through REDUX (__reduce_or_sync), whose result lands in a
// uniform register, so everything derived from the item stays uniform.
__device__ __forceinline__ unsigned long long next_item(const FastParams& p, uint32_t lane,
                                                        unsigned long long taken, uint32_t warp_global) {
  if (p.static_items) return taken ? ~0ull : (unsigned long long)warp_global;
  unsigned long long item = 0;
  if (lane == 0) item = atomicAdd(p.queue, 1ull);
  const uint32_t lo = __reduce_or_sync(FULL, (uint32_t)item);
  const uint32_t hi = __reduce_or_sync(FULL, (uint32_t)(item >> 32));
  return ((unsigned long long)hi << 32) | lo;
}

// Entry step of superblock kb (1 <= kb < nblk) of an item starting at
// superblock B0 (B0 = 0 mod nblk): a = (B0 + kb) << V flips row FIX + V + tz(kb);
// the row leaves iff bit tz(kb)+1 of B0 + kb is set.
__device__ __forceinline__ bool entry_leave(uint32_t kb, int t, const FastParams& p, unsigned long long B0) {
  return (t + 1 < p.lognblk) ? (((kb >> (t + 1)) & 1u) != 0) : (((B0 >> p.lognblk) & 1ull) != 0);
}

// Called by every warp after its last next_item: the last warp of the grid
// resets the queue for the next launch (all fetches are done by then).
__device__ __forceinline__ void queue_done(const FastParams& p, uint32_t lane) {
  if (p.static_items || lane != 0) return;
  const unsigned long long total = (unsigned long long)gridDim.x * (blockDim.x >> 5);
  if (atomicAdd(p.queue + 1, 1ull) == total - 1) {
    atomicExch(p.queue, 0ull);
    atomicExch(p.queue + 1, 0ull);
  }
}

__device__ __forceinline__ void trace_end(const FastParams& p, unsigned long long t_start, unsigned long long n_items,
                                          uint32_t warp_global, uint32_t lane) {
  if (p.trace && lane == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned long long* t = p.trace + 4ull * warp_global;
    t[0] = smid;
    t[1] = t_start;
    t[2] = clock64();
    t[3] = n_items;
  }
}

// ---------------------------------------------------------------------------
// Wide walk, 33 <= n <= 64: K subsets ("slots") per lane that differ in rows
// 5..5+log2(K)-1, walked in lockstep over high steps of 32*K reference steps.
// Only the primary word (columns 0..31) is walked: 3 LOP3 per subset for
// every n.  A primary hit (all 32 primary columns nonzero, probability
// (2/3)^32 on uniform inputs) is recorded with two predicated IMADs (count,
// (step, slot) id); at the end of the superblock a lane with one hit
// recomputes that subset's full n-column vector from scratch (O(n)) and
// evaluates the term exactly, and a lane with two or more hits replays the
// superblock exactly.  The secondary columns thus cost nothing per subset.
// Subset of (lane l, slot k, high step a): S = (gray(a) << (5+KB)) | (k << 5) | l.
// ---------------------------------------------------------------------------
template <int KB>
__device__ __forceinline__ void wide_subset_state(const RowRec* R, int n, unsigned long long a, uint32_t low,
                                                  uint32_t z0i, uint32_t z1i, uint32_t (&z)[2], uint32_t (&g)[2]) {
  constexpr int FIX = 5 + KB;
  z[0] = z0i;
  z[1] = z1i;
  g[0] = g[1] = 0;
  const unsigned long long hs = a ^ (a >> 1);
  for (int r = 0; r < n; ++r) {
    const bool in = r < FIX ? ((low >> r) & 1u) : ((hs >> (r - FIX)) & 1ull);
    if (in) {
      sub_word(z[0], g[0], R[r].m[0], R[r].a[0]);
      sub_word(z[1], g[1], R[r].m[1], R[r].a[1]);
    }
  }
}

template <int KB>
static __device__ __noinline__ unsigned long long replay_wide(const RowRec* R, int n, unsigned long long abase,
                                                              int len, uint32_t lane, uint32_t z0i, uint32_t z1i) {
  constexpr int FIX = 5 + KB;
  uint32_t ev = 0, odd = 0;
  for (int k = 0; k < (1 << KB); ++k) {
    uint32_t z[2], g[2];
    wide_subset_state<KB>(R, n, abase, ((uint32_t)k << 5) | lane, z0i, z1i, z, g);
    const uint32_t kp = (__popc(k) + __popc(lane)) & 1u;
    for (int j = 0; j < len; ++j) {
      if (j > 0) {
        const unsigned long long a = abase + (unsigned long long)j;
        const int t = tz64(a);
        const bool leave = (a >> (t + 1)) & 1ull;
        const RowRec& row = R[FIX + t];
        sub_word(z[0], g[0], row.m[0], leave ? row.s[0] : row.a[0]);
        sub_word(z[1], g[1], row.m[1], leave ? row.s[1] : row.a[1]);
      }
      if ((z[0] | z[1]) == 0) {
        ev += 1;
        odd += (__popc(g[0]) + __popc(g[1]) + (uint32_t)(j & 1) + kp) & 1u;
      }
    }
  }
  return (unsigned long long)ev | ((unsigned long long)odd << 32);
}

// cnt += 1 and rec = ID on a primary hit (predicated IMADs, FMA pipe).
template <uint32_t ID>
__device__ __forceinline__ void record_hit(uint32_t z, uint32_t& cnt, uint32_t& rec, uint32_t one, uint32_t zero) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.eq.u32 p, %2, 0;\n\t"
      "@p mad.lo.u32 %0, %3, %3, %0;\n\t"
      "@p mad.lo.u32 %1, %3, %5, %4;\n\t}"
      : "+r"(cnt), "+r"(rec)
      : "r"(z), "r"(one), "r"(zero), "n"(ID));
}

template <class F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}
__host__ __device__ constexpr int gray_c(int i) { return i ^ (i >> 1); }

// ---------------------------------------------------------------------------
// Pair walk (meet in the middle), any n >= 5+KB+V+1.  Split the rows into
// A = rows 0..h-1 (h = 5+KB: the lane bits and the K = 2^KB slot bits) and
// B = rows h..n-1.  Every subset is S = S1 u S2 with v_S = v1 + v2; a lane
// keeps its K A-side vectors v1 FIXED in registers and the warp walks only
// the B-side vector v2 in Gray order.  The term is nonzero iff v1 + v2 has
// no zero column, which is the first two LOP3 of the z-encoded sub of -v2:
//     u2 = ~(z2 ^ g2)                     (once per step, shared by all pairs)
//     d  = ~z1 & (g1 ^ u2)                lop3 0x06
//     z' = ~d & ~(z1 ^ z2)                lop3 0x09, predicate z' != 0 free
// and, only for a hit, the sign word is g' = d ^ g2.  So a subset costs 2
// LOP3 (the walk costs 3) plus one predicated IMAD that adds
// (id << 16) | 1 to a per-lane record: count in the low half, and the id of
// the (step, slot) of a single hit in the high half.
// n <= 32 (WIDE = false): the test is exact; the B-side states of the
// superblock are kept in shared memory so a single hit's sign is
// g' = d ^ g2(step) at the superblock end.  n > 32 (WIDE): the test covers
// the 32 primary columns only; a hit is re-evaluated from scratch over all
// n columns.  Two hits in one lane and superblock replay it exactly.
// Subset of (lane l, slot k, high step a): S = (gray(a) << h) | (k << 5) | l,
// the same indexing as the wide walk.
// ---------------------------------------------------------------------------
template <uint32_t IMM>
__device__ __forceinline__ void pair_test(uint32_t z1, uint32_t g1, uint32_t z2, uint32_t u2, uint32_t& rec,
                                          uint32_t one) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 d, zp;\n\t"
      "lop3.b32 d, %1, %2, %4, 0x06;\n\t"
      "lop3.b32 zp, d, %1, %3, 0x09;\n\t"
      "setp.eq.u32 p, zp, 0;\n\t"
      "@p mad.lo.u32 %0, %5, %6, %0;\n\t}"
      : "+r"(rec)
      : "r"(z1), "r"(g1), "r"(z2), "r"(u2), "r"(one), "n"(IMM));
}

// Packed pair test (tp_walk_packed.cu): two pairs per 32-bit word on 16
// columns each; sets BIT of m when either half has no zero column.
template <uint32_t BIT>
__device__ __forceinline__ void packed_test(uint32_t z1, uint32_t g1, uint32_t z2, uint32_t u2, uint32_t& m,
                                            uint32_t one, uint32_t cneg) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 d, zp, t, h;\n\t"
      "lop3.b32 d, %1, %2, %4, 0x06;\n\t"
      "lop3.b32 zp, d, %1, %3, 0x09;\n\t"
      "mad.lo.u32 t, zp, %5, %6;\n\t"
      "lop3.b32 h, t, 0x80008000, zp, 0x40;\n\t"
      "setp.ne.u32 p, h, 0;\n\t"
      "@p mad.lo.u32 %0, %5, %7, %0;\n\t}"
      : "+r"(m)
      : "r"(z1), "r"(g1), "r"(z2), "r"(u2), "r"(one), "r"(cneg), "n"(BIT));
}

// The same test for three (two) B states against one packed A word with ONE
// zero-field test: the halfword-wise minimum of the zp words (VIMNMX3.U16x2,
// ptxas fuses the two min.u16x2) has a zero field iff one of them has.  Sets
// BIT of m when any of the states passes on either half: per word and state
// 2 LOP3 + 1/3 (VIMNMX3 + LOP3) on the ALU pipe and 2/3 IMAD on the FMA pipe,
// against 3 LOP3 + 2 IMAD for packed_test.  The verify finds the state.
template <uint32_t BIT>
__device__ __forceinline__ void packed_test3(uint32_t z1, uint32_t g1, uint32_t za, uint32_t ua, uint32_t zb,
                                             uint32_t ub, uint32_t zc, uint32_t uc, uint32_t& m, uint32_t one,
                                             uint32_t cneg) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 da, zpa, db, zpb, dc, zpc, mn, t, h;\n\t"
      "lop3.b32 da, %1, %2, %4, 0x06;\n\t"
      "lop3.b32 zpa, da, %1, %3, 0x09;\n\t"
      "lop3.b32 db, %1, %2, %6, 0x06;\n\t"
      "lop3.b32 zpb, db, %1, %5, 0x09;\n\t"
      "lop3.b32 dc, %1, %2, %8, 0x06;\n\t"
      "lop3.b32 zpc, dc, %1, %7, 0x09;\n\t"
      "min.u16x2 mn, zpa, zpb;\n\t"
      "min.u16x2 mn, mn, zpc;\n\t"
      "mad.lo.u32 t, mn, %9, %10;\n\t"
      "lop3.b32 h, t, 0x80008000, mn, 0x40;\n\t"
      "setp.ne.u32 p, h, 0;\n\t"
      "@p mad.lo.u32 %0, %9, %11, %0;\n\t}"
      : "+r"(m)
      : "r"(z1), "r"(g1), "r"(za), "r"(ua), "r"(zb), "r"(ub), "r"(zc), "r"(uc), "r"(one), "r"(cneg), "n"(BIT));
}
template <uint32_t BIT>
__device__ __forceinline__ void packed_test2(uint32_t z1, uint32_t g1, uint32_t za, uint32_t ua, uint32_t zb,
                                             uint32_t ub, uint32_t& m, uint32_t one, uint32_t cneg) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 da, zpa, db, zpb, mn, t, h;\n\t"
      "lop3.b32 da, %1, %2, %4, 0x06;\n\t"
      "lop3.b32 zpa, da, %1, %3, 0x09;\n\t"
      "lop3.b32 db, %1, %2, %6, 0x06;\n\t"
      "lop3.b32 zpb, db, %1, %5, 0x09;\n\t"
      "min.u16x2 mn, zpa, zpb;\n\t"
      "mad.lo.u32 t, mn, %7, %8;\n\t"
      "lop3.b32 h, t, 0x80008000, mn, 0x40;\n\t"
      "setp.ne.u32 p, h, 0;\n\t"
      "@p mad.lo.u32 %0, %7, %9, %0;\n\t}"
      : "+r"(m)
      : "r"(z1), "r"(g1), "r"(za), "r"(ua), "r"(zb), "r"(ub), "r"(one), "r"(cneg), "n"(BIT));
}

__device__ __forceinline__ uint32_t pair_u2(uint32_t z2, uint32_t g2) {
  uint32_t u;
  TP_LOP3(u, z2, g2, 0u, 0xC3);
  return u;
}

// The B side is kept as (z2, u2) with u2 = ~(z2 ^ g2), the form the pair
// test consumes; the z-encoded sub of a row (m, s), with c = m ^ s, is then
//   d = ~z & ~(z ^ u ^ s)   (0x09);  z' = ~d & (z ^ m)   (0x06);
//   u' = ~(z' ^ d ^ c)      (0x69)   -- still 3 LOP3, and no separate u2 op.
__device__ __forceinline__ void sub_word_u(uint32_t& z, uint32_t& u, uint32_t m, uint32_t s, uint32_t c) {
  uint32_t d, zn, un;
  TP_LOP3(d, z, u, s, 0x09);
  TP_LOP3(zn, d, z, m, 0x06);
  TP_LOP3(un, zn, d, c, 0x69);
  z = zn;
  u = un;
}
// Exact fold of one pair (n <= 32): if v1 + v2 is full, n += 1 and
// a += parity(popc(sign word)).  4 LOP3 per pair on the ALU pipe; the
// popcount goes to the (quarter-rate) XU pipe and the two accumulations to the
// FMA pipe (a runtime `one` keeps ptxas from turning them into ALU adds).
__device__ __forceinline__ void exact_fold(uint32_t z1, uint32_t g1, uint32_t z2, uint32_t u2, uint32_t g2,
                                           uint32_t cm, uint32_t& n, uint32_t& a, uint32_t one) {
  uint32_t d, zp, x;
  TP_LOP3(d, z1, g1, u2, 0x06);
  TP_LOP3(zp, d, z1, z2, 0x09);
  TP_LOP3(x, d, g2, cm, 0x28);
  if (zp == 0) {
    uint32_t t;
    asm("and.b32 %0, %1, 1;" : "=r"(t) : "r"(__popc(x)));  // opaque to the front end: stays an IMAD below
    n = one * one + n;
    a = t * one + a;
  }
}

__device__ __forceinline__ uint32_t pair_g2(uint32_t z2, uint32_t u2) {  // g2 = ~(u2 ^ z2)
  uint32_t g;
  TP_LOP3(g, z2, u2, 0u, 0xC3);
  return g;
}

}  // namespace tp
