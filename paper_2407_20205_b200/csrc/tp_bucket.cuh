// tp_bucket.cuh -- the bucket tables shared by the bucketed pair walks
// (tp_walk_bucket.cu: k_bucket_group and k_walk_bucket; tp_walk_batch.cu:
// k_walk_batch): configurations, the per-matrix half tables, the run cursor
// that decodes a piece's slots, and the rare-path secondary-word lookups.
// DESIGN.md section 5c.
#pragma once
#include <type_traits>

#include "tp_walk_common.cuh"

//   TP_CHECKED         1: device-side bounds checks on every table, list and
//                      shared-memory index of the bucketed walk (__trap on a
//                      violation); the checked build stands in for
//                      compute-sanitizer, which this GPU pool does not allow
#ifndef TP_CHECKED
#define TP_CHECKED 0
#endif
#if TP_CHECKED
#define TP_CHECK(c)    \
  do {                 \
    if (!(c)) __trap(); \
  } while (0)
#else
#define TP_CHECK(c) \
  do {              \
  } while (0)
#endif


namespace tp {

namespace {

// Bucket configurations (bucket_cfg): A side = rows 0..FIX-1, sorted by the
// trits of KEYS key columns into 3^KEYS buckets; pieces per matrix:
// 2^(FIX-10) full ones plus one partial per bucket.
__host__ __device__ constexpr int nbuckets(int keys) { return keys <= 0 ? 1 : 3 * nbuckets(keys - 1); }

// Packed-filter widths per configuration: pieces with at most WB packed words
// of real slots run the filter on WB words, at most WA on WA, else all 16
// (each width is one copy of the filter loop; WA = WB = 16: a single copy).
// A bucket holds 2^FIX / 3^KEYS subsets on uniform inputs: its last piece is
// the remainder, e.g. ~594 slots (10 words) for 17 rows and 4 keys.
template <int FIX, int KEYS>
struct FilterWidths {
  static constexpr int WA = FIX == 13 && KEYS == 2 ? 15 : FIX == 14 && KEYS == 3 ? 11 : FIX == 14 && KEYS == 2 ? 14
                            : FIX == 17 && KEYS == 4 ? 11
                            : FIX == 17 && KEYS == 5 ? 10 : 16;
  static constexpr int WB = FIX == 13 && KEYS == 2 ? 12 : FIX == 14 && KEYS == 3 ? 10 : FIX == 14 && KEYS == 2 ? 13
                            : FIX == 17 && KEYS == 4 ? 10
                            : FIX == 17 && KEYS == 5 ? 9 : 16;
  __host__ __device__ static constexpr uint32_t width(uint32_t nwd) {
    return nwd > (uint32_t)WA ? 16u : nwd > (uint32_t)WB ? (uint32_t)WA : (uint32_t)WB;
  }
};
__host__ __device__ constexpr int pieces_of(int fix, int keys) { return (1 << (fix - 10)) + nbuckets(keys); }
__host__ __device__ constexpr int align16(int x) { return (x + 15) & ~15; }

// Key pattern arithmetic: a pattern is the base-3 number of the trits on the
// key columns (first key column most significant); the pattern of a sum is
// the digit-wise sum mod 3.
template <int KEYS>
__host__ __device__ __forceinline__ uint32_t pat_sub(uint32_t g, uint32_t a) {
  uint32_t r = 0, m = 1;
#pragma unroll
  for (int i = 0; i < KEYS; ++i) {
    r += ((g % 3u + 3u - a % 3u) % 3u) * m;
    g /= 3u;
    a /= 3u;
    m *= 3u;
  }
  return r;
}

// Per-matrix bucket table.  The A side (rows 0..FIX-1) splits into a low
// half (rows 0..TB-1) and a high half (rows TB..FIX-1); an A subset is a pair
// (low subset, high subset) and its vector the sum of the halves' vectors, so
// its key pattern is pat(low) + pat(high) digit-wise.  Bucket g is therefore
// the union over low patterns a of  low_a x high_(g - a),  and the table only
// holds each half sorted by pattern:
//   u16 off[2][NB + 1]     start of each pattern's run in the sorted half
//   u32 wt[N0 + N1]        the entries' weights: (subsets of even size) |
//                          (subsets of odd size) << 16 with this vector
//   vec[N0 + N1]           their vectors: low (z, g) words, high in row form
//                          (m, a = m ^ s), so slot = one 3-LOP3 add; WIDE
//                          tables carry both 32-column words (16 bytes)
// Duplicates.  Two subsets of a half have equal vectors iff the half's rows
// are linearly dependent over F3 (their difference is a nonzero F3
// combination of the rows).  Independent halves (every uniform or sparse
// C2/C3/C4/C5 input) keep all 2^TB entries, each of weight (1, 0) or (0, 1).
// A dependent half (all-ones rows: 3 distinct vectors; a zero row; repeated
// rows) keeps one entry per distinct vector with the parity counts of the
// subsets that share it, and the matrix is "weighted" (ptab bit 31): its
// items are evaluated exactly with the weights (bucket_exact_weighted).  An
// all-ones 32x32 matrix then has 9 slots instead of 2^17.
// Position p of bucket g is decoded by walking the runs a = 0, 1, ..: run a
// holds |low_a| * |high_(g-a)| subsets, low index fastest.  A piece of 1024
// slots is positions [1024 q, 1024 q + 1024) of its bucket (ptab).
// Replaces the materialised per-piece subset lists of round 1 (2 KB per
// piece, 35x the input bytes in HBM on C2): a C2 table is 1,968 bytes per
// matrix against 17 pieces x 2 KB.
template <int FIX, int KEYS, bool WIDE>
struct Tab {
  static constexpr int NB = nbuckets(KEYS);
  static constexpr int TB = (FIX + 1) / 2, HB = FIX - TB;
  static constexpr int N0 = 1 << TB, N1 = 1 << HB;
  static constexpr int VE = WIDE ? 16 : 8;  // bytes per vector entry
  static constexpr int kWt = align16(4 * (NB + 1));
  static constexpr int kVec = kWt + 4 * (N0 + N1);
  // n > 32 (WIDE) also: u32 rstart[NB][NB + 1], the start of run a in bucket
  // g, so the rare primary-hit path finds a slot's run by binary search
  static constexpr int kRun = kVec + VE * (N0 + N1);
  static constexpr int kBytes = align16(kRun + (WIDE ? 4 * NB * (NB + 1) : 0));
};

// F3 linear independence of rows r0..r0+cnt-1 (bit planes of all n columns):
// sequential elimination, each new row reduced by the earlier pivots (whose
// rows are zero at every earlier pivot column).  The reference's add_reps /
// sub_reps (src/core_f3.py:123-138) on 64-bit planes.  One thread.
__device__ __forceinline__ bool f3_rows_independent(const RowRec* R, int r0, int cnt) {
  uint64_t PM[9], PS[9];
  int pc[9];
  int rank = 0;
  for (int t = 0; t < cnt; ++t) {
    uint64_t m = (uint64_t)R[r0 + t].m[0] | ((uint64_t)R[r0 + t].m[1] << 32);
    uint64_t s = (uint64_t)R[r0 + t].s[0] | ((uint64_t)R[r0 + t].s[1] << 32);
    for (int q = 0; q < rank; ++q) {
      if (!((m >> pc[q]) & 1ull)) continue;
      const uint64_t m2 = PM[q], s2 = PS[q];
      if (((s ^ s2) >> pc[q]) & 1ull) {  // opposite trits: add the pivot row
        const uint64_t c = m2 & (m ^ s ^ s2);
        const uint64_t nm = c | (m ^ m2);
        s = c ^ s;
        m = nm;
      } else {  // equal trits: subtract it
        const uint64_t d = m & (s ^ s2);
        const uint64_t nm = d | (m ^ m2);
        s = d ^ m2 ^ s2;
        m = nm;
      }
      s &= m;
    }
    if (m == 0) return false;
    PM[rank] = m;
    PS[rank] = s;
    pc[rank] = __ffsll((long long)m) - 1;
    ++rank;
  }
  return true;
}

// Sequential decoder of bucket positions (monotone p): the current run a,
// its position range [start, end), the halves' run offsets and the low
// run's length c0.  Reads the table's offsets (L1-resident).
template <int KEYS>
struct RunCursor {
  const uint16_t* off;  // off[0..NB] low half, off[NB+1..2NB+1] high half
  uint32_t grp, a, start, end, o0, o1, c0;
  __device__ __forceinline__ void load() {
    constexpr uint32_t NB = nbuckets(KEYS);
    const uint32_t ga = pat_sub<KEYS>(grp, a);
    o0 = off[a];
    c0 = off[a + 1] - o0;
    o1 = off[NB + 1 + ga];
    end = start + c0 * (uint32_t)(off[NB + 2 + ga] - o1);
  }
  __device__ __forceinline__ void init(const uint16_t* o, uint32_t g) {
    off = o;
    grp = g;
    a = 0;
    start = 0;
    load();
  }
  // requires p < the bucket's size and p >= every earlier p
  __device__ __forceinline__ void seek(uint32_t p) {
    while (p >= end) {
      ++a;
      TP_CHECK(a < (uint32_t)nbuckets(KEYS));
      start = end;
      load();
    }
  }
  // table indices (low, high) of position p (after seek(p))
  __device__ __forceinline__ void index(uint32_t p, uint32_t& i0, uint32_t& i1) const {
    TP_CHECK(p >= start && p < end && c0 > 0);
    const uint32_t rel = p - start, j = rel / c0;
    i0 = o0 + (rel - j * c0);
    i1 = o1 + j;
    TP_CHECK(i0 < off[nbuckets(KEYS)] && i1 < off[2 * nbuckets(KEYS) + 1]);
  }
};


// Position of the k-th (0-based) set bit of m (rare paths only).
__device__ __forceinline__ uint32_t nth_set(uint32_t m, uint32_t k) {
  for (; k; --k) m &= m - 1;
  return __ffs(m) - 1;
}

// List row of physical slot k = w + 16 h (packed word w, half h): 2 w + h.
// The first 2W rows of a piece then fill packed words 0..W-1, so a piece
// with at most 64 W real slots runs the filter on W words only.
__device__ __forceinline__ uint32_t lrow(int k) { return 2u * (uint32_t)(k & 15) + ((uint32_t)k >> 4); }

// n > 32: the secondary word (columns 32..n-1) of the A subset at position
// p of bucket grp, from the table (random access: the runs are walked from
// the first; rare paths only).
template <int FIX, int KEYS>
__device__ __forceinline__ void a_word1(const uint8_t* Tm, uint32_t grp, uint32_t p, uint32_t& z, uint32_t& g) {
  using T = Tab<FIX, KEYS, true>;
  constexpr uint32_t NB = T::NB;
  // the run a of position p: the last run start <= p (binary search; empty
  // runs share their start with the next run, the search lands on a
  // non-empty one since p < the bucket's size)
  const uint32_t* rs = reinterpret_cast<const uint32_t*>(Tm + T::kRun) + grp * (NB + 1);
  uint32_t lo_a = 0, hi_a = NB;  // rs[lo_a] <= p < rs[hi_a]
  while (hi_a - lo_a > 1) {
    const uint32_t mid = (lo_a + hi_a) >> 1;
    if (rs[mid] <= p) lo_a = mid;
    else hi_a = mid;
  }
  const uint16_t* off = reinterpret_cast<const uint16_t*>(Tm);
  const uint32_t o0 = off[lo_a], c0 = off[lo_a + 1] - o0, o1 = off[NB + 1 + pat_sub<KEYS>(grp, lo_a)];
  TP_CHECK(c0 > 0 && p < rs[NB]);
  const uint32_t rel = p - rs[lo_a], j = rel / c0;
  const uint32_t i0 = o0 + (rel - j * c0), i1 = o1 + j;
  const uint4* v = reinterpret_cast<const uint4*>(Tm + T::kVec);
  const uint4 lo = v[i0], hi = v[T::N0 + i1];
  z = lo.z;
  g = lo.w;
  sub_word(z, g, hi.z, hi.w);
}

// n > 32, a pair whose 32 primary columns are all nonzero: 1 | parity of the
// secondary sign word << 1 if the secondary columns are nonzero too, else 0.
template <int FIX, int KEYS>
static __device__ __noinline__ uint32_t bucket_wide_term(const uint8_t* Tm, uint32_t grp, uint32_t p, uint2 h1,
                                                         uint32_t z1i) {
  uint32_t za, ga, d, zp;
  a_word1<FIX, KEYS>(Tm, grp, p, za, ga);
  TP_LOP3(d, za, ga, h1.y, 0x06);
  TP_LOP3(zp, d, za, h1.x, 0x09);
  if (zp != 0) return 0u;
  return 1u | ((__popc((d ^ pair_g2(h1.x, h1.y)) & z1i) & 1u) << 1);
}

// Cooperative decode table of bucket g's runs (k_walk_batch): one uint4 per
// run a = (start, o0 | c0 << 16, o1, 1/c0 as float) plus a sentinel whose
// start is the bucket size, built by the 32 lanes in parallel (the runs'
// sizes |low_a| |high_(g-a)| prefix-summed with a warp scan).  A lane then
// finds the run of each of its (increasing) positions with a linear walk
// over the starts and splits rel = p - start into rel / c0, rel % c0 with a
// float reciprocal: rel < 2^17 and c0 < 2^10, so (rel + 1/2) / c0 lies at
// least 1/(2 c0) from an integer and the product's 2^-23 relative error
// (< 2^-6 / c0 absolute) cannot move the truncation.  Replaces the per-lane
// RunCursor (a base-3 digit subtraction and a runtime division per slot).
template <int KEYS>
__device__ __forceinline__ void run_table(const uint16_t* off, uint32_t grp, uint4* RT, uint32_t lane) {
  constexpr uint32_t NB = nbuckets(KEYS);
  uint32_t carry = 0;
#pragma unroll 1
  for (uint32_t a0 = 0; a0 < NB; a0 += 32) {
    const uint32_t a = a0 + lane;
    uint32_t sz = 0, o0 = 0, c0 = 0, o1 = 0;
    if (a < NB) {
      const uint32_t ga = pat_sub<KEYS>(grp, a);
      o0 = off[a];
      c0 = off[a + 1] - o0;
      o1 = off[NB + 1 + ga];
      sz = c0 * (uint32_t)(off[NB + 2 + ga] - o1);
    }
    uint32_t incl = sz;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL, incl, d);
      if (lane >= d) incl += t;
    }
    if (a < NB) RT[a] = make_uint4(carry + incl - sz, o0 | (c0 << 16), o1, __float_as_uint(c0 ? __frcp_rn((float)c0) : 0.f));
    carry += __shfl_sync(FULL, incl, 31);
  }
  if (lane == 0) RT[NB] = make_uint4(carry, 0, 0, 0);
  __syncwarp();
}

// Table indices (low i0, high i1) of bucket position p in run record rec.
__device__ __forceinline__ void run_index(uint4 rec, uint32_t p, uint32_t& i0, uint32_t& i1) {
  const uint32_t rel = p - rec.x, c0 = rec.y >> 16;
  const float rc = __uint_as_float(rec.w);
  const uint32_t j = __float2uint_rz(__fmaf_rn((float)rel, rc, 0.5f * rc));
  TP_CHECK(c0 > 0 && j * c0 <= rel && rel - j * c0 < c0);
  i0 = (rec.y & 0xFFFFu) + rel - j * c0;
  i1 = rec.z + j;
}

// Exact fold of one pair with the A subset's parity bit sp: n += full,
// a += full & (parity(popc(sign word)) ^ sp).
__device__ __forceinline__ void exact_fold_par(uint32_t z1, uint32_t g1, uint32_t z2, uint32_t u2, uint32_t g2,
                                               uint32_t cm, uint32_t sp, uint32_t& n, uint32_t& a, uint32_t one) {
  uint32_t d, zp, x;
  TP_LOP3(d, z1, g1, u2, 0x06);
  TP_LOP3(zp, d, z1, z2, 0x09);
  TP_LOP3(x, d, g2, cm, 0x28);
  if (zp == 0) {
    uint32_t t;
    TP_LOP3(t, (uint32_t)__popc(x), 1u, sp, 0x6A);  // (popc & 1) ^ sp
    n = one * one + n;
    a = t * one + a;
  }
}

// Kernel argument: the 3-key kernels also carry their configuration.  The
// two parameter layouts are the ones measured fastest for each kernel: with
// the larger block ptxas schedules the filter loop differently, which costs
// the 2-key kernel 4 % on C2 and gains the 3-key kernels 3-5 % on C3-C5.
struct BucketParamsCfg {  // BucketParams' fields, then the configuration
  FastParams fp;
  const void* tab;
  const uint32_t* ptab;
  unsigned long long* tested;
  unsigned long long s_end;
  int fix, keys;
  unsigned int* chunk_ctr;  // (BucketParams' sticky-piece fields)
  unsigned long long npieces;
};
}  // namespace

}  // namespace tp
