// tp_walk_bucket.cu -- the pair walk with the A side bucketed by key columns:
// the default walk for 21 <= n <= 64 (full traversals and the superblock-
// aligned middle of step ranges).
//
// The pair walk (tp_walk_pair.cu) tests every (A vector, B state) pair.  A pair
// whose sum has a zero in ANY column is a zero term, so pairs can be skipped
// wholesale by looking at a few "key" columns first:
//
//   * the A side is rows 0..FIX-1 (FIX = 13 below n = 28, 17 from n = 28;
//     bucket_cfg).  k_bucket_group sorts its 2^FIX subsets by their trits on
//     KEYS key columns (n-1, n-2 and, for KEYS = 3, n-3; 31, 30, 29 for
//     n > 32) into 3^KEYS buckets and cuts each bucket into pieces of 1024
//     (= 32 lanes x 32 slots, the pair walk's A side per warp; the last piece
//     of a bucket is padded with dummy slots);
//   * a warp takes one piece, so all its A vectors share their key trits x,
//     and walks B-side superblocks (rows FIX..n-1) in Gray order as usual;
//   * a B state y is compatible with the piece iff y_k != -x_k on every key
//     column; otherwise every one of the warp's 1024 pairs with it has a zero
//     key column.  Compatibility is warp-uniform: the packed filter runs on
//     the compatible steps only.
//
// On uniform inputs 4/9 (KEYS = 2) or 8/27 (KEYS = 3) of the steps are
// compatible; with the padding of partly filled pieces 47 % / 31 % of all
// pairs are tested.  The sum is unchanged: only zero terms are skipped, so
// raw partials equal chunk_sum (src/_kernels.py:90-128) bit for bit.  Dummy
// slots carry a -1 in padding column 31 for n <= 31 (the B side has +1
// there), so their sums always have a zero column; for n >= 32 they are the
// zero vector and the verify and exact paths exclude them by a slot mask.
// For n > 32 the filter and verify cover the 32 primary columns, and a pair
// whose primary columns are all nonzero gets its secondary word tested.
#include <type_traits>

#include "tp_bucket.cuh"

// Build variants for A/B timing (tools/ab_build.sh ... EXTRA=-D...):
//   TP_BUCKET_MACC     1 / 2 pass-mask accumulators in the filter
//   TP_BUCKET_COMPACT  1: the compatible steps' packed states compacted, the
//                      filter loop on a counter; 0: popped from the mask (ffs)
//   TP_BUCKET_REDUX    1: piece word and dense flag through REDUX (uniform)
//   TP_BUCKET_ROLLED   1: the A-slot decode as a rolled loop; 0: unrolled
#ifndef TP_BUCKET_MACC
#define TP_BUCKET_MACC 1
#endif
#ifndef TP_BUCKET_COMPACT
#define TP_BUCKET_COMPACT 0
#endif
#ifndef TP_BUCKET_REDUX
#define TP_BUCKET_REDUX 0
#endif
#ifndef TP_BUCKET_ROLLED
#define TP_BUCKET_ROLLED 1
#endif
#if TP_BUCKET_REDUX
#define TP_ANY(x) (__reduce_or_sync(FULL, (x) ? 1u : 0u) != 0)
#else
#define TP_ANY(x) __any_sync(FULL, (x))
#endif

namespace tp {

namespace {

// ----------------------------------------------------------------- grouping
// One CTA per matrix: every half subset's vector and key pattern; for a half
// whose rows are F3-dependent, one representative per distinct vector (the
// lowest subset) carrying the parity counts of its duplicates; a
// deterministic counting sort of each half by pattern (rank = earlier
// representatives with the same half and pattern), the table, then the
// bucket sizes sum_a |low_a| |high_(g-a)| and the pieces (ptab).  DEDUP =
// false (the unpacked pair-test kernel) keeps every subset.
template <int FIX, int KEYS, bool WIDE, bool DEDUP>
__global__ void __launch_bounds__(256) k_bucket_group(const RowRec* rows, int n, uint8_t* tab, uint32_t* ptab) {
  using T = Tab<FIX, KEYS, WIDE>;
  constexpr int NB = T::NB, N0 = T::N0, NE = T::N0 + T::N1, NT = 256, NW = NT / 32;
  constexpr int EPT = (NE + NT - 1) / NT, NK = 2 * NB, P = pieces_of(FIX, KEYS);
  __shared__ RowRec R[FIX];
  __shared__ uint32_t wcnt[NW][NK];  // per-warp key counts of the current round
  __shared__ uint32_t kcnt[NK];      // key counts of the earlier rounds, then totals
  __shared__ uint32_t offs[2][NB + 1];
  __shared__ uint32_t bsize[NB];
  __shared__ uint4 vs[DEDUP ? NE : 1];      // dependent halves: every entry's vector
  __shared__ uint32_t wts[DEDUP ? NE : 1];  // representatives' weights (even | odd << 16)
  __shared__ int dep[2];                    // half h has F3-dependent rows
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  {
    const uint4* src = reinterpret_cast<const uint4*>(rows + (size_t)blockIdx.x * 64);
    if (tid < 2 * FIX) reinterpret_cast<uint4*>(R)[tid] = src[tid];
  }
  for (uint32_t k = tid; k < (uint32_t)NK; k += NT) kcnt[k] = 0;
  uint8_t* Tm = tab + (size_t)blockIdx.x * T::kBytes;
  const int k1 = (n < 32 ? n : 32) - 1;  // key columns k1, k1-1 (, k1-2): primary word for n > 32
  const uint32_t cm0 = n >= 32 ? 0xffffffffu : (1u << n) - 1u;
  const uint32_t cm1 = n <= 32 ? 0u : n >= 64 ? 0xffffffffu : (1u << (n - 32)) - 1u;
  uint32_t key[EPT], rank[EPT], wt[EPT];
  uint4 vec[EPT];
  // Forced rows (packed variants).  A column with a single nonzero entry, in
  // row r, is zero in every subset sum without row r, so only subsets
  // containing r give terms: A-side subsets without a forced row of their
  // half stay out of the table.  A column without any nonzero entry makes
  // every term zero: the table stays empty (all pieces count 0) and the
  // matrix's counters stay 0.  Only zero terms are dropped, so the raw
  // partials are unchanged.  (Permutation-like and very sparse matrices;
  // uniform inputs have no such columns.)
  __shared__ uint32_t forcedA;  // forced rows among 0..FIX-1
  __shared__ int deadm;         // a zero column
  if (warp == 0) {
    uint32_t fa = 0;
    int dd = 0;
    if (DEDUP) {
      const RowRec* rr = rows + (size_t)blockIdx.x * 64;
      uint32_t o0 = 0, m0 = 0, o1 = 0, m1 = 0;  // columns seen in a row / in more than one row
      uint32_t own0 = 0, own1 = 0;              // this lane's row r = lane
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int r = (int)lane + 32 * k;
        const uint32_t a0 = r < n ? rr[r].m[0] & cm0 : 0u, a1 = r < n ? rr[r].m[1] & cm1 : 0u;
        if (k == 0) {
          own0 = a0;
          own1 = a1;
        }
        m0 |= o0 & a0;
        o0 |= a0;
        m1 |= o1 & a1;
        o1 |= a1;
      }
#pragma unroll
      for (int sft = 16; sft; sft >>= 1) {
        const uint32_t po0 = __shfl_xor_sync(FULL, o0, sft), pm0 = __shfl_xor_sync(FULL, m0, sft);
        const uint32_t po1 = __shfl_xor_sync(FULL, o1, sft), pm1 = __shfl_xor_sync(FULL, m1, sft);
        m0 |= pm0 | (o0 & po0);
        o0 |= po0;
        m1 |= pm1 | (o1 & po1);
        o1 |= po1;
      }
      dd = ((~o0 & cm0) | (~o1 & cm1)) != 0u;
      fa = __ballot_sync(FULL, ((own0 & o0 & ~m0) | (own1 & o1 & ~m1)) != 0u) & ((1u << FIX) - 1u);
    }
    if (lane == 0) {
      forcedA = fa;
      deadm = dd;
    }
  }
  __syncthreads();
  if (tid < 2) dep[tid] = DEDUP && !f3_rows_independent(R, tid ? T::TB : 0, tid ? T::HB : T::TB);
#pragma unroll
  for (int q = 0; q < EPT; ++q) {  // vectors and patterns
    const uint32_t e = (uint32_t)q * NT + tid;
    const bool act = e < (uint32_t)NE;
    const uint32_t h = e >= (uint32_t)N0 ? 1u : 0u;
    const uint32_t sub = h ? e - N0 : e;
    uint32_t z0 = cm0, g0 = 0, z1 = cm1, g1 = 0;
    if (act) {
      for (uint32_t x = sub; x; x &= x - 1) {
        const int r = __ffs(x) - 1 + (h ? T::TB : 0);
        sub_word(z0, g0, R[r].m[0], R[r].a[0]);
        if (WIDE) sub_word(z1, g1, R[r].m[1], R[r].a[1]);
      }
    }
    auto trit = [&](int c) -> uint32_t { return ((z0 >> c) & 1u) ? 0u : ((g0 >> c) & 1u) ? 2u : 1u; };
    uint32_t pat = 0;  // first key column most significant
#pragma unroll
    for (int i = 0; i < KEYS; ++i) pat = 3u * pat + trit(k1 - i);
    const uint32_t fh = h ? forcedA >> T::TB : forcedA & ((1u << T::TB) - 1u);
    key[q] = act && !deadm && (sub & fh) == fh ? h * NB + pat : 0xFFFFu;
    wt[q] = (__popc(sub) & 1) ? 1u << 16 : 1u;
    // canonical sign bits (zero columns carry sgn 0) so equal vectors compare equal
    g0 &= ~z0;
    g1 &= ~z1;
    if (h) {  // high half in row form: the slot adds it with one sub_word
      const uint32_t m0 = ~z0 & cm0, m1 = ~z1 & cm1;
      vec[q] = make_uint4(m0, m0 ^ (g0 & m0), m1, m1 ^ (g1 & m1));
    } else {
      vec[q] = make_uint4(z0, g0, z1, g1);
    }
    if (DEDUP && act) {
      vs[e] = vec[q];
      wts[e] = 0;
    }
  }
  __syncthreads();
  if (DEDUP && (dep[0] || dep[1])) {
    // duplicates of a dependent half: each entry finds its representative
    // (the first equal vector of its half) and adds its parity count there
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
      const uint32_t e = (uint32_t)q * NT + tid;
      if (key[q] == 0xFFFFu) continue;
      const uint32_t h = e >= (uint32_t)N0 ? 1u : 0u;
      if (!dep[h]) continue;
      uint32_t rep = e;
      for (uint32_t f = h ? N0 : 0; f < e; ++f) {
        const uint4 o = vs[f];
        if (o.x == vec[q].x && o.y == vec[q].y && o.z == vec[q].z && o.w == vec[q].w) {
          rep = f;
          break;
        }
      }
      atomicAdd(&wts[rep], wt[q]);
      if (rep != e) key[q] = 0xFFFFu;  // not a representative: not in the table
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
      const uint32_t e = (uint32_t)q * NT + tid;
      if (key[q] != 0xFFFFu && dep[e >= (uint32_t)N0 ? 1 : 0]) wt[q] = wts[e];
    }
  }
#pragma unroll
  for (int q = 0; q < EPT; ++q) {  // deterministic ranks within (half, pattern)
    __syncthreads();  // the previous round's wcnt consumed
    for (uint32_t e = tid; e < (uint32_t)(NW * NK); e += NT) wcnt[e / NK][e % NK] = 0;
    const bool act = key[q] != 0xFFFFu;
    const uint32_t mm = __match_any_sync(FULL, key[q]);
    __syncthreads();  // wcnt cleared
    if (act && lane == (uint32_t)(__ffs(mm) - 1)) wcnt[warp][key[q]] = __popc(mm);
    __syncthreads();
    if (act) {
      uint32_t r = kcnt[key[q]] + __popc(mm & ((1u << lane) - 1u));
      for (uint32_t w = 0; w < warp; ++w) r += wcnt[w][key[q]];
      rank[q] = r;
    }
    __syncthreads();
    for (uint32_t k = tid; k < (uint32_t)NK; k += NT) {
      uint32_t c = 0;
      for (int w = 0; w < NW; ++w) c += wcnt[w][k];
      kcnt[k] += c;
    }
  }
  __syncthreads();
  if (tid < 2) {  // run offsets of each half
    uint32_t o = 0;
    for (int a = 0; a < NB; ++a) {
      offs[tid][a] = o;
      o += kcnt[tid * NB + a];
    }
    offs[tid][NB] = o;
  }
  __syncthreads();
  for (uint32_t k = tid; k < (uint32_t)(2 * (NB + 1)); k += NT)
    reinterpret_cast<uint16_t*>(Tm)[k] = (uint16_t)offs[k / (NB + 1)][k % (NB + 1)];
  for (uint32_t g = tid; g < (uint32_t)NB; g += NT) {
    uint32_t c = 0;
    if (WIDE) {  // run starts of bucket g (the partial sums, kept per run)
      uint32_t* rs = reinterpret_cast<uint32_t*>(Tm + T::kRun) + g * (NB + 1);
      for (uint32_t a = 0; a < (uint32_t)NB; ++a) {
        rs[a] = c;
        c += kcnt[a] * kcnt[NB + pat_sub<KEYS>(g, a)];
      }
      rs[NB] = c;
    } else {
      for (uint32_t a = 0; a < (uint32_t)NB; ++a) c += kcnt[a] * kcnt[NB + pat_sub<KEYS>(g, a)];
    }
    bsize[g] = c;
  }
  uint32_t* wout = reinterpret_cast<uint32_t*>(Tm + T::kWt);
#pragma unroll
  for (int q = 0; q < EPT; ++q) {
    if (key[q] == 0xFFFFu) continue;
    const uint32_t h = key[q] >= (uint32_t)NB ? 1u : 0u;
    const uint32_t idx = h * N0 + offs[h][key[q] - h * NB] + rank[q];
    TP_CHECK(idx < (uint32_t)(h ? NE : N0));
    wout[idx] = wt[q];
    if (WIDE) reinterpret_cast<uint4*>(Tm + T::kVec)[idx] = vec[q];
    else reinterpret_cast<uint2*>(Tm + T::kVec)[idx] = make_uint2(vec[q].x, vec[q].y);
  }
  __syncthreads();
  // Piece order (longest first, so the dynamic queue ends on the shortest
  // items): every full piece of 1024 slots, bucket by bucket, then the
  // partial pieces by decreasing slot count (ties by bucket).  Thread g
  // places bucket g's pieces.
  const uint32_t weighted = (dep[0] || dep[1]) ? 1u << 31 : 0u;
  uint32_t* Pt = ptab + (size_t)blockIdx.x * P;
  __shared__ uint32_t nfull;
  if (tid == 0) {  // full pieces before bucket g, in offs[0][g] (free now)
    uint32_t f = 0;
    for (uint32_t g = 0; g < (uint32_t)NB; ++g) {
      offs[0][g] = f;
      f += bsize[g] >> 10;
    }
    nfull = f;
  }
  __syncthreads();
  for (uint32_t g = tid; g < (uint32_t)NB; g += NT) {
    const uint32_t c = bsize[g], nf = c >> 10, part = c & 1023u;
    for (uint32_t q = 0; q < nf; ++q) {
      TP_CHECK(offs[0][g] + q < (uint32_t)P);
      Pt[offs[0][g] + q] = g | (1024u << 8) | (q << 20) | weighted;
    }
    if (part) {
      uint32_t rank = 0;
      for (uint32_t h = 0; h < (uint32_t)NB; ++h) {
        const uint32_t ph = bsize[h] & 1023u;
        rank += (ph > part || (ph == part && h < g)) ? 1u : 0u;
      }
      TP_CHECK(nfull + rank < (uint32_t)P);
      Pt[nfull + rank] = g | (part << 8) | (nf << 20) | weighted;
    }
  }
  if (tid == 0) {  // unused pieces: count 0
    uint32_t used = nfull;
    for (uint32_t g = 0; g < (uint32_t)NB; ++g) used += (bsize[g] & 1023u) ? 1u : 0u;
    for (uint32_t piece = used; piece < (uint32_t)P; ++piece) Pt[piece] = 0;
  }
}

// Exact evaluation of the steps in `mask` against this lane's 32 slots (the
// packed variant's dense mode and list-overflow path).  Out of line, so its
// registers do not constrain the filter loop.  Returns ev | odd << 32.
static __device__ __noinline__ unsigned long long bucket_exact_packed(const uint4 (*A2)[32], const uint2* H,
                                                                      uint32_t mask, uint32_t lane, uint32_t spm,
                                                                      uint32_t vmask, uint32_t colmask, int n,
                                                                      uint32_t one) {
  constexpr int K = 32;
  uint32_t bev = 0, bodd = 0;
#pragma unroll 1
  for (; mask; mask &= mask - 1) {
    const int j = __ffs(mask) - 1;
    const uint2 h = H[j];
    const uint32_t gh = pair_g2(h.x, h.y);
    uint32_t n0 = 0, a0 = 0;
    if (n <= 31) {
      // the subset parity rides in padding column 31 of the sign word
      const uint32_t cmp = colmask | 0x80000000u;
#pragma unroll
      for (int w = 0; w < K / 2; ++w) {
        const uint4 a = A2[w][lane];
        exact_fold(a.x, a.y, h.x, h.y, gh, cmp, n0, a0, one);
        exact_fold(a.z, a.w, h.x, h.y, gh, cmp, n0, a0, one);
      }
    } else {
      // n = 32: the slot's subset parity is a runtime bit, folded into the
      // sign parity with one LOP3 instead of a divergent branch
#pragma unroll
      for (int w = 0; w < K / 2; ++w) {
        const uint4 a = A2[w][lane];
        exact_fold_par(a.x, a.y, h.x, h.y, gh, colmask, (spm >> w) & 1u, n0, a0, one);
        exact_fold_par(a.z, a.w, h.x, h.y, gh, colmask, (spm >> (w + K / 2)) & 1u, n0, a0, one);
      }
      // padding slots hold the zero vector (no column to kill it): each
      // pairs fully with a full y, with subset parity 0; remove them
      if (h.x == 0u) {
        const uint32_t nd = (uint32_t)K - __popc(vmask);
        n0 -= nd;
        a0 -= nd * (__popc(gh) & 1u);
      }
    }
    // term is odd iff popc(sgn) + j + parity(A subset) is odd
    bev += n0;
    bodd += (j & 1) ? (n0 - a0) : a0;
  }
  return (unsigned long long)bev | ((unsigned long long)bodd << 32);
}


// n > 32: exact evaluation of the steps in `mask` against this lane's real
// slots, both words (dense mode, list overflow).  Slot-major in position
// order (one run cursor), so each slot's secondary word is built once.
// Returns ev | odd << 32.
template <int FIX, int KEYS>
static __device__ __noinline__ unsigned long long bucket_exact_wide(const uint4 (*A2)[32], const uint2* H,
                                                                    const uint2* H1, const uint8_t* Tm,
                                                                    uint32_t grp, uint32_t pbase, uint32_t cnt,
                                                                    uint32_t mask, uint32_t lane, uint32_t spm,
                                                                    uint32_t z1i) {
  using T = Tab<FIX, KEYS, true>;
  const uint4* vec = reinterpret_cast<const uint4*>(Tm + T::kVec);
  RunCursor<KEYS> cur;
  cur.init(reinterpret_cast<const uint16_t*>(Tm), grp);
  uint32_t ev = 0, odd = 0;
#pragma unroll 1
  for (uint32_t r = 0; 32u * r + lane < cnt; ++r) {  // this lane's real slots: rows r = lrow(k)
    const uint32_t k = (r >> 1) + ((r & 1u) << 4);
    const uint32_t p = pbase + 32u * r + lane;
    uint32_t i0, i1;
    cur.seek(p);
    cur.index(p, i0, i1);
    const uint4 lo = vec[i0], hi = vec[T::N0 + i1];
    uint32_t za1 = lo.z, ga1 = lo.w;
    sub_word(za1, ga1, hi.z, hi.w);
    const uint4 a4 = A2[k & 15][lane];
    const uint32_t za = k < 16 ? a4.x : a4.z, ga = k < 16 ? a4.y : a4.w;
    const uint32_t kp = (spm >> k) & 1u;
#pragma unroll 1
    for (uint32_t m = mask; m; m &= m - 1) {
      const uint32_t j = __ffs(m) - 1;
      const uint2 h = H[j];
      uint32_t d, zp;
      TP_LOP3(d, za, ga, h.y, 0x06);
      TP_LOP3(zp, d, za, h.x, 0x09);
      if (zp == 0) {
        const uint2 h1 = H1[j];
        uint32_t d1, zp1;
        TP_LOP3(d1, za1, ga1, h1.y, 0x06);
        TP_LOP3(zp1, d1, za1, h1.x, 0x09);
        if (zp1 == 0) {
          ev += 1;
          odd += (__popc(d ^ pair_g2(h.x, h.y)) + __popc((d1 ^ pair_g2(h1.x, h1.y)) & z1i) + j + kp) & 1u;
        }
      }
    }
  }
  return (unsigned long long)ev | ((unsigned long long)odd << 32);
}

// Weighted matrices (a deduplicated A side, Tab): exact evaluation of the
// steps in `mask` against this lane's real slots, each slot standing for
// `we` subsets of even and `wo` of odd size with the same vector.  A term of
// sign parity s (popcount of the sign word + step parity) counts we times
// with parity s and wo times with parity s + 1.  Both words for n > 32; the
// slot's vector is rebuilt from the table without the padding-column parity
// trick (column 31 is +1 + +1 = -1 for n <= 31, so the sign parity masks it
// out with colmask).  The superblock's counts (per lane <= 2^17 subsets x 32
// steps, per warp < 2^27) are flushed into pm[0..1] right away, so the
// weights' totals never ride in the walk's 32-bit per-lane counters.
template <int FIX, int KEYS, bool WIDE>
static __device__ __noinline__ void bucket_exact_weighted(const uint2* H, const uint2* H1, const uint8_t* Tm,
                                                          uint32_t grp, uint32_t pbase, uint32_t cnt, uint32_t mask,
                                                          uint32_t lane, uint32_t colmask, uint32_t z1i,
                                                          unsigned long long* pm) {
  using T = Tab<FIX, KEYS, WIDE>;
  const uint32_t* wts = reinterpret_cast<const uint32_t*>(Tm + T::kWt);
  RunCursor<KEYS> cur;
  cur.init(reinterpret_cast<const uint16_t*>(Tm), grp);
  uint32_t ev = 0, odd = 0;
#pragma unroll 1
  for (uint32_t r = 0; 32u * r + lane < cnt; ++r) {
    const uint32_t p = pbase + 32u * r + lane;
    uint32_t i0, i1;
    cur.seek(p);
    cur.index(p, i0, i1);
    const uint32_t w0 = wts[i0], w1 = wts[T::N0 + i1];
    const uint32_t e0 = w0 & 0xFFFFu, o0 = w0 >> 16, e1 = w1 & 0xFFFFu, o1 = w1 >> 16;
    const uint32_t we = e0 * e1 + o0 * o1, wo = e0 * o1 + o0 * e1;
    uint32_t za, ga, za1 = 0, ga1 = 0;
    if constexpr (WIDE) {
      const uint4 lo = reinterpret_cast<const uint4*>(Tm + T::kVec)[i0];
      const uint4 hi = reinterpret_cast<const uint4*>(Tm + T::kVec)[T::N0 + i1];
      za = lo.x;
      ga = lo.y;
      sub_word(za, ga, hi.x, hi.y);
      za1 = lo.z;
      ga1 = lo.w;
      sub_word(za1, ga1, hi.z, hi.w);
    } else {
      const uint2 lo = reinterpret_cast<const uint2*>(Tm + T::kVec)[i0];
      const uint2 hi = reinterpret_cast<const uint2*>(Tm + T::kVec)[T::N0 + i1];
      za = lo.x;
      ga = lo.y;
      sub_word(za, ga, hi.x, hi.y);
    }
#pragma unroll 1
    for (uint32_t m = mask; m; m &= m - 1) {
      const uint32_t j = __ffs(m) - 1;
      const uint2 h = H[j];
      uint32_t d, zp;
      TP_LOP3(d, za, ga, h.y, 0x06);
      TP_LOP3(zp, d, za, h.x, 0x09);
      if (zp != 0) continue;
      uint32_t sp = __popc((d ^ pair_g2(h.x, h.y)) & colmask) + j;
      if constexpr (WIDE) {
        const uint2 h1 = H1[j];
        uint32_t d1, zp1;
        TP_LOP3(d1, za1, ga1, h1.y, 0x06);
        TP_LOP3(zp1, d1, za1, h1.x, 0x09);
        if (zp1 != 0) continue;
        sp += __popc((d1 ^ pair_g2(h1.x, h1.y)) & z1i);
      }
      ev += we + wo;
      odd += (sp & 1u) ? we : wo;
    }
  }
  warp_flush(pm, ev - odd, odd, lane);
}

template <int KEYS>
struct BucketArg {
  using type = BucketParams;
};
template <>
struct BucketArg<3> {
  using type = BucketParamsCfg;
};
template <>
struct BucketArg<4> {
  using type = BucketParamsCfg;
};
template <>
struct BucketArg<5> {
  using type = BucketParamsCfg;
};

}  // namespace

template <int V, int WARPS, bool PACKED, bool WIDE, int FIX, int KEYS>
__global__ void __launch_bounds__(32 * WARPS, 4) k_walk_bucket(const typename BucketArg<KEYS>::type bp) {
  constexpr int KB = 5;
  constexpr int K = 1 << KB;
  constexpr int kBucketPieces = pieces_of(FIX, KEYS);
  using T = Tab<FIX, KEYS, WIDE>;
  constexpr int SB = 1 << V;
  const FastParams& p = bp.fp;
  static_assert(PACKED || !WIDE, "n > 32 needs the packed filter");
  __shared__ RowRec Rs[WARPS][WIDE ? 64 : 32];
  __shared__ uint2 Hs[WARPS][SB];  // the superblock's B states (z, u), by step
  // packed filter: the compatible steps' doubled low 16 columns (zz, uu),
  // compacted in step order (a pair of steps = one 16-byte load)
  __shared__ __align__(16) uint2 Hcs[WARPS][PACKED ? SB : 2];
  __shared__ uint2 H1s[WARPS][WIDE ? SB : 1];  // n > 32: secondary words (z, u) of the superblock's B states
  __shared__ uint2 As[WARPS][K][32];  // full A words; packed: [w][lane] pairs (slot w, slot w + 16) as uint4
  constexpr int ECAP = PACKED ? (WIDE ? 5 : 6) : 1;  // (48 KB of static shared memory)  // per-lane pass-list capacity (overflow: exact superblock)
  __shared__ uint2 Es[WARPS][ECAP][32];   // per-lane filter passes: (mask, steps)
  const uint32_t lane = threadIdx.x & 31u;
  uint2 (*E)[32] = Es[threadIdx.x >> 5];
  const uint32_t cneg = 0xfffeffffu * p.one;  // -0x00010001, runtime so ptxas keeps the IMAD
  RowRec* R = Rs[threadIdx.x >> 5];
  uint2* H = Hs[threadIdx.x >> 5];
  uint2* Hc = Hcs[threadIdx.x >> 5];
  uint2* H1 = H1s[threadIdx.x >> 5];
  uint2 (*A)[32] = As[threadIdx.x >> 5];
  uint4 (*A2)[32] = reinterpret_cast<uint4 (*)[32]>(As[threadIdx.x >> 5]);
  const uint32_t one = p.one;
  const uint32_t colmask = p.z0_init;  // real columns (n <= 31: bit 31 is padding)
  const uint32_t colmask1 = p.z1_init;  // n > 32: real columns of the secondary word
  const int k1 = (WIDE ? 32 : p.n) - 1;  // key columns k1, k1-1 (, k1-2)
  unsigned long long n_items = 0;

  for (;;) {
    const unsigned long long item = next_item(p, lane, n_items, blockIdx.x * WARPS + (threadIdx.x >> 5));
    if (item >= p.items) break;
    ++n_items;
    // item = (piece * chunks + chunk) * B + matrix: consecutive items go to
    // different matrices, so the slow items of event-dense matrices spread
    // over the whole launch instead of forming its tail (and the unused
    // high pieces come last)
    const unsigned long long nmat = p.items / ((unsigned long long)kBucketPieces * p.chunks);
    const unsigned long long rest = item / nmat;
    const unsigned long long b = item - rest * nmat;
    const uint32_t q = (uint32_t)(rest / p.chunks);
    const unsigned long long c = rest - (unsigned long long)q * p.chunks;
    // superblocks [sb0, sb0 + nsb) of the B side (global indices: the
    // region [F0, s_end) need not be aligned to the item length)
    const unsigned long long sb0 = p.F0 + c * p.nblk;
    const uint32_t nsb = (uint32_t)min((unsigned long long)p.nblk, bp.s_end - sb0);
    const unsigned long long A0 = sb0 << V;
    // (through REDUX: a uniform register, so every branch on the piece --
    // the filter width, the dummy-slot tests -- is a uniform branch and the
    // step loop below can live on the uniform datapath)
#if TP_BUCKET_REDUX
    const uint32_t pt = __reduce_or_sync(FULL, lane == 0 ? bp.ptab[b * kBucketPieces + q] : 0u);
#else
    TP_CHECK(q < (uint32_t)kBucketPieces && b < nmat);
    const uint32_t pt = bp.ptab[b * kBucketPieces + q];
#endif
    const uint32_t cnt = (pt >> 8) & 0xFFFu;  // real slots of the piece
    if (cnt == 0) continue;  // unused piece
    const uint32_t grp = pt & 0xFFu;
    const uint32_t pbase = ((pt >> 20) & 0x7FFu) << 10;  // the piece is positions [pbase, pbase + cnt) of its bucket
    const bool weighted = (pt >> 31) != 0;  // deduplicated A side (bucket_exact_weighted)
    TP_CHECK(((pt >> 8) & 0xFFFu) <= 1024u && (pt & 0xFFu) < (uint32_t)nbuckets(KEYS));
    const uint32_t nwd = (cnt + 63u) >> 6;  // packed words holding the piece's real slots
    __syncwarp();
    load_rows(R, p.rows + b * 64, lane, p.n);
    __syncwarp();

    // A side: slot k of this lane is position pbase + 32 lrow(k) + lane of
    // the bucket, decoded from the matrix's table (low-half vector + high-half
    // row: one 3-LOP3 add); full words in shared memory (verify, exact
    // fallback), registers: the unpacked walk keeps all 32 slots, the packed
    // one only the packed words (low 16 columns of slot w in the low half, of
    // slot w + 16 in the high).  Slots are built in position order, so one
    // run cursor serves them all.
    uint32_t z1[PACKED ? 1 : K], g1[PACKED ? 1 : K];
    uint32_t Zp[PACKED ? K / 2 : 1], Gp[PACKED ? K / 2 : 1];
    uint32_t spm = 0;  // bit k: parity of slot k's subset
    uint32_t vmask = 0;  // bit k: slot k holds a real A subset (not padding)
    const uint8_t* Tm = static_cast<const uint8_t*>(bp.tab) + b * T::kBytes;
    {
      const uint32_t* wts = reinterpret_cast<const uint32_t*>(Tm + T::kWt);
      RunCursor<KEYS> cur;
      cur.init(reinterpret_cast<const uint16_t*>(Tm), grp);
      auto slot = [&](int k, uint32_t& z, uint32_t& g) {
        const uint32_t r = 32u * lrow(k) + lane;
        if (r >= cnt) {  // dummy slot
          // n <= 31: -1 in padding column 31 (B side: +1), never a full sum;
          // n = 32 has no padding column: the verify and exact paths test vmask
          z = colmask;
          g = p.n <= 31 ? 0x80000000u : 0u;
        } else {
          uint32_t i0, i1;
          cur.seek(pbase + r);
          cur.index(pbase + r, i0, i1);
          const uint2 lo = *reinterpret_cast<const uint2*>(Tm + T::kVec + T::VE * i0);
          const uint2 hi = *reinterpret_cast<const uint2*>(Tm + T::kVec + T::VE * (T::N0 + i1));
          // subset parity (unweighted entries: weight (1, 0) or (0, 1))
          const uint32_t par = ((wts[i0] ^ wts[T::N0 + i1]) >> 16) & 1u;
          z = lo.x;
          g = lo.y;
          sub_word(z, g, hi.x, hi.y);
          vmask |= 1u << k;
          // n <= 31: padding column 31 carries the subset parity p as the trit
          // p (0 or +1; B side +1): the sum there is +1 or -1, so it never
          // zeroes a column and its sign bit is p (the exact fold counts it)
          if (p.n <= 31 && !par) z |= 0x80000000u;
          spm |= par << k;
        }
        if constexpr (!PACKED) A[k][lane] = make_uint2(z, g);
      };
#if !TP_BUCKET_ROLLED
      if constexpr (PACKED) {
#pragma unroll
        for (int w = 0; w < K / 2; ++w) {
          uint32_t za, ga, zb, gb;
          slot(w, za, ga);
          slot(w + K / 2, zb, gb);
          Zp[w] = __byte_perm(za, zb, 0x5410);
          Gp[w] = __byte_perm(ga, gb, 0x5410);
          A2[w][lane] = make_uint4(za, ga, zb, gb);
        }
      } else
#endif
      if constexpr (PACKED) {
        // a rolled loop in position order (one copy of the decode: the
        // unrolled 32 copies doubled the kernel's code and cost the 3-key
        // kernels 10 % in instruction fetch), full words to shared memory,
        // then the packed registers from there
#pragma unroll 1
        for (uint32_t r = 0; r < (uint32_t)K; ++r) {
          const int k = (int)((r >> 1) + ((r & 1u) << 4));
          uint32_t z, g;
          slot(k, z, g);
          reinterpret_cast<uint2*>(&A2[k & 15][lane])[k >> 4] = make_uint2(z, g);
        }
        __syncwarp();
#pragma unroll
        for (int w = 0; w < K / 2; ++w) {
          const uint4 a = A2[w][lane];
          Zp[w] = __byte_perm(a.x, a.z, 0x5410);
          Gp[w] = __byte_perm(a.y, a.w, 0x5410);
        }
      } else {
        // position order (row r = lrow(k)) for the run cursor
#pragma unroll
        for (int r = 0; r < K; ++r) slot((r >> 1) + ((r & 1) << 4), z1[(r >> 1) + ((r & 1) << 4)], g1[(r >> 1) + ((r & 1) << 4)]);
      }
    }
    // forbidden key trits of this piece: f = -x (mod 3)
    // (digit i of grp, weight 3^(KEYS-1-i), is the trit of column k1 - i)
    uint32_t F0 = 0, F1 = 0, F2 = 0;
    if constexpr (KEYS == 2) {  // (this form keeps the 2-key kernel's register allocation spill-free)
      const int k2 = k1 - 1;
      const uint32_t x1 = grp / 3, x2 = grp % 3;
      const uint32_t f1 = (3 - x1) % 3, f2 = (3 - x2) % 3;
      F0 = (f1 == 0 ? 1u << k1 : 0u) | (f2 == 0 ? 1u << k2 : 0u);
      F1 = (f1 == 1 ? 1u << k1 : 0u) | (f2 == 1 ? 1u << k2 : 0u);
      F2 = (f1 == 2 ? 1u << k1 : 0u) | (f2 == 2 ? 1u << k2 : 0u);
    } else {
      uint32_t rest = grp;
#pragma unroll
      for (int i = KEYS - 1; i >= 0; --i) {
        const uint32_t x = rest % 3u;
        rest /= 3u;
        const uint32_t f = (3u - x) % 3u, bit = 1u << (k1 - i);
        F0 |= f == 0 ? bit : 0u;
        F1 |= f == 1 ? bit : 0u;
        F2 |= f == 2 ? bit : 0u;
      }
    }
    // B side: v2 for S2 = gray(A0) on rows >= FIX (low bits empty)
    uint32_t z2, u2;
    uint32_t z2w = 0, u2w = 0;  // n > 32: secondary word of the entry state
    {
      uint32_t z = colmask, g = 0, zw = colmask1, gw = 0;
      const unsigned long long hs = A0 ^ (A0 >> 1);
      for (int r = FIX; r < p.n; ++r)
        if ((hs >> (r - FIX)) & 1ull) {
          sub_word(z, g, R[r].m[0], R[r].a[0]);
          if (WIDE) sub_word(zw, gw, R[r].m[1], R[r].a[1]);
        }
      z2 = z;
      u2 = pair_u2(z, g);
      z2w = zw;
      u2w = pair_u2(zw, gw);
    }
    uint32_t ev = 0, odd = 0;
    uint32_t tested_steps = 0;  // compatible steps of this item (x the slots the filter tests)
    // exact evaluation of every pair of the superblock from H (replays, dense mode)
    // (only the steps in `mask`: incompatible steps have no full term)
    auto exact_block = [&](uint32_t& bev, uint32_t& bodd, uint32_t mask) {
      if constexpr (WIDE) {
        const unsigned long long r =
            bucket_exact_wide<FIX, KEYS>(A2, H, H1, Tm, grp, pbase, cnt, mask, lane, spm, colmask1);
        bev = (uint32_t)r;
        bodd = (uint32_t)(r >> 32);
        return;
      } else if constexpr (PACKED) {
        const unsigned long long r = bucket_exact_packed(A2, H, mask, lane, spm, vmask, colmask, p.n, one);
        bev = (uint32_t)r;
        bodd = (uint32_t)(r >> 32);
        return;
      }
      bev = bodd = 0;
#pragma unroll 1
      for (; mask; mask &= mask - 1) {
        const int j = __ffs(mask) - 1;
        const uint2 h = H[j];
        const uint32_t gh = pair_g2(h.x, h.y);
        uint32_t n0 = 0, a0 = 0, n1 = 0, a1 = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if ((spm >> k) & 1u) exact_fold(z1[k], g1[k], h.x, h.y, gh, colmask, n1, a1, one);
          else exact_fold(z1[k], g1[k], h.x, h.y, gh, colmask, n0, a0, one);
        }
        // term is odd iff popc(sgn) + j + parity(A subset) is odd
        bev += n0 + n1;
        bodd += (j & 1) ? (n0 - a0) + a1 : a0 + (n1 - a1);
      }
    };
    bool dense = false;
    for (uint32_t kb = 0; kb < nsb; ++kb) {
      // the B states of the superblock, one per lane (step j = lane mod SB),
      // as in the pair walk; the top row's direction follows the parity of
      // the global superblock index
      const bool godd = ((sb0 + kb) & 1ull) != 0;
      uint32_t zj = z2, uj = u2;
      uint32_t zjw = z2w, ujw = u2w;
      {
        const uint32_t j = lane & (SB - 1), gj = j ^ (j >> 1);
#pragma unroll
        for (int r = 0; r < V; ++r) {
          if ((gj >> r) & 1u) {
            const bool lv = (r == V - 1) && godd;
            const RowRec& row = R[FIX + r];
            sub_word_u(zj, uj, row.m[0], lv ? row.s[0] : row.a[0], lv ? row.a[0] : row.s[0]);
            if (WIDE) sub_word_u(zjw, ujw, row.m[1], lv ? row.s[1] : row.a[1], lv ? row.a[1] : row.s[1]);
          }
        }
      }
      // compatible steps: no key column of y equals the forbidden trit
      // (y = 0 <=> z; y = 2 <=> ~z & ~u; y = 1 <=> ~z & u)
      const uint32_t match = (zj & F0) | (~zj & ~uj & F2) | (~zj & uj & F1);
      // (REDUX: a uniform register, so everything derived from it is uniform)
#if TP_BUCKET_REDUX
      const uint32_t cmask = __reduce_or_sync(FULL, (match == 0u && lane < (uint32_t)SB) ? 1u << lane : 0u);
#else
      const uint32_t cmask = __ballot_sync(FULL, match == 0u) & (SB == 32 ? 0xffffffffu : ((1u << SB) - 1u));
#endif
      const uint32_t ncomp = __popc(cmask);
      tested_steps += ncomp;
      if (PACKED && weighted) {
        // deduplicated A side: every compatible step exactly, with weights
        __syncwarp();
        if (lane < (uint32_t)SB) {
          H[lane] = make_uint2(zj, uj);
          if (WIDE) H1[lane] = make_uint2(zjw, ujw);
        }
        __syncwarp();
        bucket_exact_weighted<FIX, KEYS, WIDE>(H, H1, Tm, grp, pbase, cnt, cmask, lane, colmask, colmask1,
                                               p.pm + 2 * b);
      } else {
      __syncwarp();
      if (lane < (uint32_t)SB) {
        H[lane] = make_uint2(zj, uj);
        if (WIDE) H1[lane] = make_uint2(zjw, ujw);
        // compacted packed states: the filter loop walks positions 0..ncomp-1
        // with a plain counter (no per-step bit pops)
#if TP_BUCKET_COMPACT
        if (PACKED && ((cmask >> lane) & 1u))
          Hc[__popc(cmask & ((1u << lane) - 1u))] = make_uint2(__byte_perm(zj, zj, 0x1010), __byte_perm(uj, uj, 0x1010));
#else
        if (PACKED) Hc[lane] = make_uint2(__byte_perm(zj, zj, 0x1010), __byte_perm(uj, uj, 0x1010));
#endif
      }
      if (dense) {
        __syncwarp();
        uint32_t bev, bodd;
        exact_block(bev, bodd, cmask);
        ev += bev;
        odd += bodd;
        dense = TP_ANY(bev >= (uint32_t)K / 2);
      } else {
        // the compatible steps only: a rolled loop over the set bits of
        // cmask, the next step's B state loaded (uniform shared-memory
        // broadcast) before the current step's 32 tests
        __syncwarp();
        // hit records (slot of the last hit) << 16 | hit count, four of them
        // (slots k mod 4) so that the predicated IMADs do not form one chain
        uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
        if constexpr (PACKED) {
          // packed filter over the compatible steps, two per iteration: bit w
          // (step a) / 16 + w (step b) of M = a pass of word w; nonzero masks
          // go to this lane's list E for the exact verify after the loop
          uint32_t ne = 0;
          // W packed words hold every real slot of the piece (the rest are
          // padding): 15 for most 2-key pieces (<= 960 of 1024 slots)
          auto filter = [&](auto Wc) {
          constexpr int W = decltype(Wc)::value;
          // two compatible steps (compacted positions i, i + 1) per
          // iteration while two remain ...
#if TP_BUCKET_COMPACT
          uint32_t i = 0;
#pragma unroll 1
          for (; i + 2 <= ncomp; i += 2) {
            const uint4 hab = *reinterpret_cast<const uint4*>(Hc + i);
#else
          uint32_t cm = cmask;
          while (cm & (cm - 1)) {
            const uint32_t ja = __ffs(cm) - 1;
            cm &= cm - 1;
            const uint32_t jb = __ffs(cm) - 1;
            cm &= cm - 1;
            const uint2 ha2 = Hc[ja], hb2 = Hc[jb];
            const uint4 hab = make_uint4(ha2.x, ha2.y, hb2.x, hb2.y);
            const uint32_t i = ja | (jb << 8);  // (the pass entry records the steps)
#endif
#if TP_BUCKET_MACC == 2
            // two pass-mask accumulators (even / odd words): the predicated
            // IMADs form two dependency chains of 16 instead of one of 32
            uint32_t M = 0, M1 = 0;
            static_for<W>([&](auto wc) {
              constexpr int w = decltype(wc)::value;
              uint32_t& Mw = (w & 1) ? M1 : M;
              packed_test<(1u << w)>(Zp[w], Gp[w], hab.x, hab.y, Mw, one, cneg);
              packed_test<(1u << (16 + w))>(Zp[w], Gp[w], hab.z, hab.w, Mw, one, cneg);
            });
            M = M1 * one + M;
#else
            uint32_t M = 0;
            static_for<W>([&](auto wc) {
              constexpr int w = decltype(wc)::value;
              packed_test<(1u << w)>(Zp[w], Gp[w], hab.x, hab.y, M, one, cneg);
              packed_test<(1u << (16 + w))>(Zp[w], Gp[w], hab.z, hab.w, M, one, cneg);
            });
#endif
            if (M) {
              if (ne < (uint32_t)ECAP) E[ne][lane] = make_uint2(M, i);
              ++ne;
            }
          }
          // ... and an odd last step alone (half the tests)
#if TP_BUCKET_COMPACT
          if (i < ncomp) {
            const uint2 ha = Hc[i];
#else
          if (cm) {
            const uint32_t i = (__ffs(cm) - 1) | (0xFFu << 8);
            const uint2 ha = Hc[i & 0xFFu];
#endif
            uint32_t M = 0;
            static_for<W>([&](auto wc) {
              constexpr int w = decltype(wc)::value;
              packed_test<(1u << w)>(Zp[w], Gp[w], ha.x, ha.y, M, one, cneg);
            });
            if (M) {
              if (ne < (uint32_t)ECAP) E[ne][lane] = make_uint2(M, i);
              ++ne;
            }
          }
          };
          // (17 rows / 3 keys: one copy; its pieces are nearly all full, and
          // the extra loop copies cost more in schedule quality than the 4 %
          // of tests they would save)
          using FW = FilterWidths<FIX, KEYS>;
          if constexpr (FW::WA == 16) {
            filter(std::integral_constant<int, 16>{});
          } else {
            if (nwd > (uint32_t)FW::WA) filter(std::integral_constant<int, 16>{});
            else if (nwd > (uint32_t)FW::WB) filter(std::integral_constant<int, FW::WA>{});
            else filter(std::integral_constant<int, FW::WB>{});
          }
#if TP_BUCKET_VOTE1
          const uint32_t nemax = __reduce_max_sync(FULL, ne);  // one REDUX for both tests below
          if (nemax > (uint32_t)ECAP) {
#else
          if (__any_sync(FULL, ne > (uint32_t)ECAP)) {
#endif
            // a lane's pass list overflowed (event-dense matrix): evaluate the
            // superblock's compatible steps exactly instead
            __syncwarp();
            uint32_t bev, bodd;
            exact_block(bev, bodd, cmask);
            ev += bev;
            odd += bodd;
            dense = p.dense_ok != 0 && TP_ANY(bev >= (uint32_t)K / 2);
#if TP_BUCKET_VOTE1
          } else if (nemax != 0) {
#else
          } else if (__any_sync(FULL, ne != 0)) {
#endif
            uint32_t bev = 0, bodd = 0;
            for (uint32_t e = 0; e < ne; ++e) {
              const uint2 ent = E[e][lane];
              uint32_t M = ent.x;
              while (M) {
                const uint32_t bit = __ffs(M) - 1;
                M &= M - 1;
#if TP_BUCKET_COMPACT
                // compacted position -> step: the (pos)-th set bit of cmask
                const uint32_t j = nth_set(cmask, ent.y + (bit >> 4)), w = bit & 15u;
#else
                const uint32_t j = (bit < 16) ? (ent.y & 0xFFu) : (ent.y >> 8), w = bit & 15u;
#endif
                TP_CHECK(j < (uint32_t)SB && ((cmask >> j) & 1u));
                const uint2 h = H[j];
                const uint32_t gh = pair_g2(h.x, h.y);
  #pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                  const uint32_t k = w + 16 * hf;
                  const uint4 a4 = A2[w][lane];
                  const uint2 a = hf ? make_uint2(a4.z, a4.w) : make_uint2(a4.x, a4.y);
                  uint32_t d, zp;
                  TP_LOP3(d, a.x, a.y, h.y, 0x06);
                  TP_LOP3(zp, d, a.x, h.x, 0x09);
                  if (zp == 0 && ((vmask >> k) & 1u)) {
                    uint32_t par = 0;
                    if constexpr (WIDE) {
                      // the primary columns are nonzero: test the secondary ones
                      const uint32_t r =
                          bucket_wide_term<FIX, KEYS>(Tm, grp, pbase + 32u * lrow(k) + lane, H1[j], colmask1);
                      if (!r) continue;
                      par = r >> 1;
                    }
                    bev += 1;
                    bodd += (__popc((d ^ gh) & colmask) + par + j + ((spm >> k) & 1u)) & 1u;
                  }
                }
              }
            }
            ev += bev;
            odd += bodd;
            // event-dense (e.g. all-ones rows): exact mode for the next superblocks
            dense = p.dense_ok != 0 && TP_ANY(bev >= (uint32_t)K / 2);
          }
        } else {
          // two compatible steps per iteration (independent tests interleave);
          // the next two states are loaded before the current tests
          uint32_t cm = cmask;
          uint32_t ja = 0, jb = 0, hj = 0;
          uint2 ha = make_uint2(0, 0), hb = ha;
          auto pop2 = [&]() {
            ja = __ffs(cm) - 1;
            cm &= cm - 1;
            jb = __ffs(cm) - 1;
            cm &= cm - 1;
          };
          if (__popc(cm) >= 2) {
            pop2();
            ha = H[ja];
            hb = H[jb];
            for (;;) {
              const uint2 ca = ha, cb = hb;
              const uint32_t cja = ja, cjb = jb;
              const bool more = __popc(cm) >= 2;
              if (more) {
                pop2();
                ha = H[ja];
                hb = H[jb];
              }
              const uint32_t sa = r0 + r1, sb = r2 + r3;
              static_for<K>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                uint32_t& r = (k & 1) ? r1 : r0;
                uint32_t& rr = (k & 1) ? r3 : r2;
                pair_test<((uint32_t)k << 16) | 1u>(z1[k], g1[k], ca.x, ca.y, r, one);
                pair_test<((uint32_t)k << 16) | 1u>(z1[k], g1[k], cb.x, cb.y, rr, one);
              });
              // step of this lane's latest hit (the single-hit path needs it)
              if (r0 + r1 != sa) hj = cja;
              if (r2 + r3 != sb) hj = cjb;
              if (!more) break;
            }
          }
          if (cm) {
            const uint32_t jc = __ffs(cm) - 1;
            const uint2 hc = H[jc];
            const uint32_t sa = r0 + r1;
            static_for<K>([&](auto kc) {
              constexpr int k = decltype(kc)::value;
              uint32_t& r = (k & 1) ? r1 : r0;
              pair_test<((uint32_t)k << 16) | 1u>(z1[k], g1[k], hc.x, hc.y, r, one);
            });
            if (r0 + r1 != sa) hj = jc;
          }
          const uint32_t cnt = (r0 & 0xffffu) + (r1 & 0xffffu) + (r2 & 0xffffu) + (r3 & 0xffffu);
          const uint32_t rec = (r0 & 0xffffu) ? r0 : (r1 & 0xffffu) ? r1 : (r2 & 0xffffu) ? r2 : r3;
          if (__any_sync(FULL, cnt != 0)) {
            uint32_t bev = 0, bodd = 0;
            if (__any_sync(FULL, cnt > 1)) {
              exact_block(bev, bodd, cmask);
              dense = p.dense_ok != 0 && TP_ANY(bev >= (uint32_t)K / 2);
            } else if (cnt == 1) {
              // one hit: slot k from the record, step hj tracked in the loop
              const uint32_t k = rec >> 16;
              const uint2 a1 = A[k][lane];
              const uint2 hh = H[hj];
              uint32_t d;
              TP_LOP3(d, a1.x, a1.y, hh.y, 0x06);
              bev = 1;
              bodd = (__popc((d ^ pair_g2(hh.x, hh.y)) & colmask) + hj + ((spm >> k) & 1u)) & 1u;
            }
            ev += bev;
            odd += bodd;
          }
        }
      }
      }  // unweighted
      // (z2, u2) = step SB-1 of this superblock, then the entry step of kb + 1
      z2 = __shfl_sync(FULL, zj, SB - 1);
      u2 = __shfl_sync(FULL, uj, SB - 1);
      if (WIDE) {
        __syncwarp();
        const uint2 e = H1[SB - 1];
        z2w = e.x;
        u2w = e.y;
      }
      if (kb + 1 < nsb) {
        // entry of global superblock G flips row FIX + V + tz(G); it leaves
        // iff bit tz(G) + 1 of G is set
        const unsigned long long G = sb0 + kb + 1;
        const int t = tz64(G);
        const RowRec& row = R[FIX + V + t];
        const bool lv = ((G >> (t + 1)) & 1ull) != 0;
        sub_word_u(z2, u2, row.m[0], lv ? row.s[0] : row.a[0], lv ? row.a[0] : row.s[0]);
        if (WIDE) sub_word_u(z2w, u2w, row.m[1], lv ? row.s[1] : row.a[1], lv ? row.a[1] : row.s[1]);
      }
    }
    warp_flush(p.pm + 2 * b, ev - odd, odd, lane);
    if (bp.tested && lane == 0) {
      const uint32_t words = PACKED ? FilterWidths<FIX, KEYS>::width(nwd) : 16u;
      atomicAdd(bp.tested, 64ull * words * tested_steps);
    }
  }
  queue_done(p, lane);
}

int bucket_pieces(BucketCfg c) { return pieces_of(c.fix, c.keys); }
int bucket_v(bool packed) { return packed ? 5 : 4; }  // log2 superblock length
size_t bucket_tab_bytes(BucketCfg c, bool wide) {
  if (c.fix == 13 && c.keys == 2) return Tab<13, 2, false>::kBytes;
  if (c.fix == 14 && c.keys == 3) return Tab<14, 3, false>::kBytes;
  if (c.fix == 14 && c.keys == 2) return Tab<14, 2, false>::kBytes;
  if (c.fix == 17 && c.keys == 5) return wide ? Tab<17, 5, true>::kBytes : Tab<17, 5, false>::kBytes;
  return wide ? Tab<17, 4, true>::kBytes : Tab<17, 4, false>::kBytes;
}

// Configurations (A side rows FIX, KEYS key columns).
//  * Unpacked pair tests (TRITPERM_BUCKET=2): 14 rows, 2 keys.
//  * k_walk_batch (the default): n < 28 14 rows and 3 keys (27 buckets of
//    ~607 slots, 8/27 of the steps tested); 28 <= n <= 32 17 rows and 5
//    keys (243 buckets of ~539 slots, 32/243 tested); n > 32 17 rows and 4
//    keys (81 buckets, 16/81 tested: 5 keys would need 237 KB of run starts
//    per matrix for the primary-hit lookup).  Its batched filter loop keeps
//    the short pieces efficient; measured on B200 against 13
//    rows / 2 keys and 17 rows / 4 keys: C2 14.78 -> 13.78 ms, C3 313 -> 276
//    ms, C5 507 -> 477 ms with 5 keys (kept at 4 for the table size).
//  * k_walk_bucket (TRITPERM_BATCH=0): n < 28 13 rows and 2 keys, else 17
//    rows and 4 keys, its measured best: its per-superblock
//    filter set-up makes short pieces expensive.
BucketCfg bucket_cfg(int n, bool packed, bool batch, unsigned long long B) {
  if (!packed) return BucketCfg{14, 2};
  // n > 32: 5 keys while the run-start tables (237 KB per matrix) stay
  // under ~1 GB, i.e. single matrices and small batches (C4, C5, ranges)
  if (batch) return n < 28 ? BucketCfg{14, 3} : n <= 32 || B <= 4096 ? BucketCfg{17, 5} : BucketCfg{17, 4};
  return n < 28 ? BucketCfg{13, 2} : BucketCfg{17, 4};
}

cudaError_t launch_bucket_group(const RowRec* rows, long long B, int n, BucketCfg c, bool packed, void* tab,
                                uint32_t* ptab, cudaStream_t st) {
  const unsigned grid = (unsigned)B;
  uint8_t* t = static_cast<uint8_t*>(tab);
  if (!packed) k_bucket_group<14, 2, false, false><<<grid, 256, 0, st>>>(rows, n, t, ptab);
  else if (c.fix == 13 && c.keys == 2) k_bucket_group<13, 2, false, true><<<grid, 256, 0, st>>>(rows, n, t, ptab);
  else if (c.fix == 14 && c.keys == 3) k_bucket_group<14, 3, false, true><<<grid, 256, 0, st>>>(rows, n, t, ptab);
  else if (c.fix == 17 && c.keys == 5 && n <= 32) k_bucket_group<17, 5, false, true><<<grid, 256, 0, st>>>(rows, n, t, ptab);
  else if (c.fix == 17 && c.keys == 5) k_bucket_group<17, 5, true, true><<<grid, 256, 0, st>>>(rows, n, t, ptab);
  else if (c.fix == 17 && c.keys == 4 && n > 32) k_bucket_group<17, 4, true, true><<<grid, 256, 0, st>>>(rows, n, t, ptab);
  else if (c.fix == 17 && c.keys == 4) k_bucket_group<17, 4, false, true><<<grid, 256, 0, st>>>(rows, n, t, ptab);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_walk_bucket(int grid, const BucketParams& bp, bool packed, cudaStream_t st) {
  const BucketCfg c = bucket_cfg(bp.fp.n, packed, false);
  const BucketParamsCfg bc{bp.fp, bp.tab, bp.ptab, bp.tested, bp.s_end, c.fix, c.keys, nullptr, 0};
  if (bp.fp.n > 32) k_walk_bucket<5, 4, true, true, 17, 4><<<grid, 128, 0, st>>>(bc);
  else if (!packed) k_walk_bucket<4, 4, false, false, 14, 2><<<grid, 128, 0, st>>>(bp);
  else if (c.fix == 13) k_walk_bucket<5, 4, true, false, 13, 2><<<grid, 128, 0, st>>>(bp);
  else k_walk_bucket<5, 4, true, false, 17, 4><<<grid, 128, 0, st>>>(bc);
  return cudaGetLastError();
}

const void* walk_bucket_symbol(bool packed) {
  return packed ? reinterpret_cast<const void*>(&k_walk_bucket<5, 4, true, false, 13, 2>)
                : reinterpret_cast<const void*>(&k_walk_bucket<4, 4, false, false, 14, 2>);
}

}  // namespace tp
