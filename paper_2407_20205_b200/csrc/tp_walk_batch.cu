// tp_walk_batch.cu -- the bucketed pair walk with batched compatible steps:
// the default walk for 21 <= n <= 64 (full traversals and the superblock-
// aligned middle of step ranges).
//
// Same decomposition as k_walk_bucket (tp_walk_bucket.cu): a warp holds one
// piece of 1024 A subsets of one key bucket (decoded from the matrix's half
// tables, tp_bucket.cuh) and walks the B side in superblocks of 32 Gray
// steps, one B state per lane; a B state is compatible with the piece iff no
// key column of the sum is forced to zero.  The difference is where the
// compatible states go.  k_walk_bucket runs the packed filter once per
// superblock over the ~14 (2 keys) or ~6 (4 keys) compatible steps it finds,
// so the per-superblock fixed cost (loop set-up, pops of the step mask,
// pass-list votes, the verify dispatch) is paid for every 7 or 3 filter
// iterations.  Here each superblock's compatible states are compacted into a
// per-warp list in shared memory (ballot + prefix popcount), NBAT superblocks
// (4; 8 for n > 32) fill one list, and the filter then runs one long counted
// loop over it (lists of 8 superblocks in segments of 96 entries):
//
//   * list entry e: the doubled low 16 columns (Hc, what the filter reads,
//     two entries = one 16-byte load), the full state (Hf, z and u words;
//     n > 32: recomputed from the superblock's H and the lane's L when a
//     pass needs it) and the step within the batch (Hj, whose parity is the
//     B subset's size parity: batches start at even steps);
//   * the filter is the packed test of tp_walk_bucket.cu (two pairs per
//     32-bit word on 16 columns each) for three entries at a time with one
//     zero-field test on the halfword-wise minimum of their three result
//     words (packed_test3: 4/3 ALU ops per pair); a lane's passes (mask of
//     words, list index of the three entries) go to its pass list E; after
//     the loop the warp compacts the lists and verifies the passes exactly,
//     one record per lane and round;
//   * a pass list that overflows, and event-dense matrices, take the exact
//     evaluation of the segment or list; deduplicated (weighted) A sides
//     take the weighted exact walk, as in k_walk_bucket.
//
// Only zero terms are skipped, so the raw partials equal chunk_sum
// (src/_kernels.py:90-128) bit for bit.
#include "tp_bucket.cuh"

namespace tp {

namespace {

// Per-warp shared-memory layout (dynamic shared memory, 4 warps per block).
template <int NBAT, int ECAP, bool WIDE, int FIX>
struct BatchSmem {
  static constexpr int NR = (WIDE ? 64 : 32) - FIX;  // B-side rows FIX..n-1
  // the list keeps only what the filter reads; the entries' full states are
  // recomputed from the superblock's H and the lane's L (n > 32, and
  // batches of 8 superblocks, whose lists leave no room for them)
  static constexpr bool RECOMP = WIDE || NBAT > 4;
  static constexpr int NS = NBAT * 32;               // list capacity: steps per batch
  // B-side rows, row r at r - FIX: RowRec[NR] (32 bytes), n > 32 uint4 (m0, m1, s0, s1) with a = m ^ s
  // derived at use, which makes room for longer lists
  static constexpr int kRow = WIDE ? 16 : 32;
  static constexpr int oR = 0;
  static constexpr int oA = align16(oR + kRow * NR);    // uint4[16][32]: full A words (slot w | slot w + 16)
  static constexpr int oHc = oA + 16 * 32 * 16;         // uint2[NS]: doubled low 16 columns (zz, uu)
  static constexpr int oHs = oHc + 8 * NS;              // RECOMP: uint4[NBAT] H of each superblock (z, u, zw, uw)
  // stored states: uint2[NS] the entries' full states (z, u); RECOMP
  // recomputes them from Hs and the L tables (entry_state) and keeps the
  // room for a longer list
  static constexpr int oHf = oHs + (RECOMP ? 16 * NBAT : 0);
  static constexpr int oHj = oHf + (RECOMP ? 0 : 8 * NS);  // uint8[NS]: step within the batch (32 t + lane)
  static constexpr int oE = align16(oHj + NS);          // uint2[ECAP + 1][32]: passes (mask, list index)
  // per lane the low-row part of its B state in row form, for superblocks
  // of even / odd index: uint2 (m, s) [2][32], n > 32 uint4 (m0, s0, m1, s1)
  static constexpr int oL = oE + 8 * 32 * (ECAP + 1);
  static constexpr int kWarp = align16(oL + 2 * 32 * (WIDE ? 16 : 8));
  // RECOMP: the exact paths materialise the entries' full states (Hf, H1)
  // in the pass-list area, which they do not use, a chunk of at least 64
  // entries at a time
  __host__ __device__ static constexpr bool states_fit() { return !RECOMP || (WIDE ? 16 : 8) * 64 <= oL - oE; }
  // the A decode's run table (run_table) borrows [oHc, kWarp): the lists,
  // the pass list and the L tables are all written after the decode
  template <int KEYS>
  __host__ __device__ static constexpr bool run_table_fits() { return 16 * (nbuckets(KEYS) + 1) <= kWarp - oHc; }
  // ... and behind it a copy of the matrix's half table, when that fits too
  template <int KEYS, int TBYTES>
  __host__ __device__ static constexpr bool tab_fits() {
    return align16(16 * (nbuckets(KEYS) + 1)) + TBYTES <= kWarp - oHc;
  }
};

// Exact evaluation of list entries [0, L) against this lane's 32 slots, n <= 32
// (dense mode and pass-list overflow).  Returns ev | odd << 32.
// (One copy per A-side height: ptxas allocates a shared out-of-line callee
// against all its callers, which ties the kernels' register allocation
// together; a change in one kernel then moves the others' code.)
template <int FIX>
static __device__ __noinline__ unsigned long long batch_exact_packed(const uint4 (*A2)[32], const uint2* Hf,
                                                                     const uint8_t* Hj, uint32_t L, uint32_t lane,
                                                                     uint32_t spm, uint32_t vmask, uint32_t colmask,
                                                                     int n, uint32_t one) {
  constexpr int K = 32;
  uint32_t bev = 0, bodd = 0;
#pragma unroll 1
  for (uint32_t e = 0; e < L; ++e) {
    const uint2 h = Hf[e];
    const uint32_t jp = Hj[e] & 1u;
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
      // n = 32: the slot parity is a runtime bit folded into the sign parity
#pragma unroll
      for (int w = 0; w < K / 2; ++w) {
        const uint4 a = A2[w][lane];
        exact_fold_par(a.x, a.y, h.x, h.y, gh, colmask, (spm >> w) & 1u, n0, a0, one);
        exact_fold_par(a.z, a.w, h.x, h.y, gh, colmask, (spm >> (w + K / 2)) & 1u, n0, a0, one);
      }
      // padding slots hold the zero vector: each pairs fully with a full y
      // with subset parity 0; remove them
      if (h.x == 0u) {
        const uint32_t nd = (uint32_t)K - __popc(vmask);
        n0 -= nd;
        a0 -= nd * (__popc(gh) & 1u);
      }
    }
    bev += n0;
    bodd += jp ? (n0 - a0) : a0;
  }
  return (unsigned long long)bev | ((unsigned long long)bodd << 32);
}

// n > 32: exact evaluation of list entries [0, L) against this lane's real
// slots, both words; slot-major in position order (one run cursor).
template <int FIX, int KEYS>
static __device__ __noinline__ unsigned long long batch_exact_wide(const uint4 (*A2)[32], const uint2* Hf,
                                                                   const uint2* H1, const uint8_t* Hj, uint32_t L,
                                                                   const uint8_t* Tm, uint32_t grp, uint32_t pbase,
                                                                   uint32_t cnt, uint32_t lane, uint32_t spm,
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
    for (uint32_t e = 0; e < L; ++e) {
      const uint2 h = Hf[e];
      uint32_t d, zp;
      TP_LOP3(d, za, ga, h.y, 0x06);
      TP_LOP3(zp, d, za, h.x, 0x09);
      if (zp == 0) {
        const uint2 h1 = H1[e];
        uint32_t d1, zp1;
        TP_LOP3(d1, za1, ga1, h1.y, 0x06);
        TP_LOP3(zp1, d1, za1, h1.x, 0x09);
        if (zp1 == 0) {
          ev += 1;
          odd += (__popc(d ^ pair_g2(h.x, h.y)) + __popc((d1 ^ pair_g2(h1.x, h1.y)) & z1i) + Hj[e] + kp) & 1u;
        }
      }
    }
  }
  return (unsigned long long)ev | ((unsigned long long)odd << 32);
}

// Weighted matrices (deduplicated A side): exact evaluation of list entries
// [0, L) against this lane's real slots, each slot standing for `we` subsets
// of even and `wo` of odd size with the same vector (k_walk_bucket's
// bucket_exact_weighted over the list; the slots' table indices IX[r][lane]
// come from the item's A decode).  Flushed into pm right away: per
// lane <= 2^17 subsets x NS steps, per warp < 2^(22 + log2 NS) < 2^32.
template <int FIX, int KEYS, bool WIDE>
static __device__ __noinline__ void batch_exact_weighted(const uint2* Hf, const uint2* H1, const uint8_t* Hj,
                                                         uint32_t L, const uint8_t* Tm, const uint32_t* IX,
                                                         uint32_t cnt, uint32_t lane, uint32_t colmask, uint32_t z1i,
                                                         unsigned long long* pm) {
  using T = Tab<FIX, KEYS, WIDE>;
  const uint32_t* wts = reinterpret_cast<const uint32_t*>(Tm + T::kWt);
  uint32_t ev = 0, odd = 0;
#pragma unroll 1
  for (uint32_t r = 0; 32u * r + lane < cnt; ++r) {
    // the slot's half-table indices, decoded once per item (IX)
    const uint32_t i0 = IX[32u * r + lane] & 0xFFFFu, i1 = IX[32u * r + lane] >> 16;
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
    for (uint32_t e = 0; e < L; ++e) {
      const uint2 h = Hf[e];
      uint32_t d, zp;
      TP_LOP3(d, za, ga, h.y, 0x06);
      TP_LOP3(zp, d, za, h.x, 0x09);
      if (zp != 0) continue;
      uint32_t sp = __popc((d ^ pair_g2(h.x, h.y)) & colmask) + Hj[e];
      if constexpr (WIDE) {
        const uint2 h1 = H1[e];
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

}  // namespace

// TP_BATCH_SIX = W: pieces of at most W packed words filter six entries per
// iteration and pass record (0: three everywhere).  Measured on B200: C2
// -0.9 %, C4 -0.9 %, C5 -0.3 %, but C3 (n <= 32, 17 rows / 5 keys) +3.5 %, so
// that kernel keeps three.
#ifndef TP_BATCH_SIX
#define TP_BATCH_SIX 10
#endif

template <int NBAT, int ECAP, bool WIDE, int FIX, int KEYS>
__global__ void __launch_bounds__(128, 4) k_walk_batch(const BucketParamsCfg bp) {
  constexpr int V = 5, K = 32, SB = 32;
  constexpr int kBucketPieces = pieces_of(FIX, KEYS);
  using T = Tab<FIX, KEYS, WIDE>;
  using S = BatchSmem<NBAT, ECAP, WIDE, FIX>;
  static_assert(S::template run_table_fits<KEYS>(), "k_walk_batch: the run table must fit the list area");
  static_assert(S::states_fit(), "k_walk_batch: the exact paths need room for 64 entries' states in the pass-list area");
  const FastParams& p = bp.fp;
  extern __shared__ __align__(16) uint8_t batch_smem[];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint8_t* ws = batch_smem + warp * S::kWarp;
  // B-side row r at index r - FIX, as the walk consumes it (a = m ^ s: the add operand)
  struct BRow {
    uint32_t m0, s0, a0, m1, s1, a1;
  };
  auto brow = [&](int i) -> BRow {
    if constexpr (WIDE) {
      const uint4 v = reinterpret_cast<const uint4*>(ws + S::oR)[i];
      return BRow{v.x, v.z, v.x ^ v.z, v.y, v.w, v.y ^ v.w};
    } else {
      const RowRec& r = reinterpret_cast<const RowRec*>(ws + S::oR)[i];
      return BRow{r.m[0], r.s[0], r.a[0], 0u, 0u, 0u};
    }
  };
  uint4 (*A2)[32] = reinterpret_cast<uint4 (*)[32]>(ws + S::oA);
  uint32_t* IX = reinterpret_cast<uint32_t*>(ws + S::oA);  // weighted items: slot r's table indices [r][lane]
  uint2* Hc = reinterpret_cast<uint2*>(ws + S::oHc);
  uint4* Hs = reinterpret_cast<uint4*>(ws + S::oHs);
  // the entries' full states: stored (n <= 32) or materialised for the
  // exact paths in the pass-list area (n > 32)
  constexpr bool RECOMP = S::RECOMP;
  uint2* Hf = reinterpret_cast<uint2*>(ws + (RECOMP ? S::oE : S::oHf));
  // recompute mode: the exact paths materialise the states of kChunk entries at a time (Hf, then H1)
  constexpr uint32_t kChunk = RECOMP ? (uint32_t)(((S::oL - S::oE) / (WIDE ? 16 : 8)) & ~1) : (uint32_t)S::NS;
  uint2* H1 = reinterpret_cast<uint2*>(ws + S::oE) + kChunk;
  uint8_t* Hj = ws + S::oHj;
  uint2 (*E)[32] = reinterpret_cast<uint2 (*)[32]>(ws + S::oE);
  uint2* L2 = reinterpret_cast<uint2*>(ws + S::oL);  // [parity][lane] (m, s), n <= 32
  uint4* L4 = reinterpret_cast<uint4*>(ws + S::oL);  // [parity][lane] (m0, s0, m1, s1), n > 32
  const uint32_t cneg = 0xfffeffffu * p.one;  // -0x00010001, runtime so ptxas keeps the IMAD
  const uint32_t one = p.one;
  const uint32_t colmask = p.z0_init;   // real columns (n <= 31: bit 31 is padding)
  const uint32_t colmask1 = p.z1_init;  // n > 32: real columns of the secondary word
  const int k1 = (WIDE ? 32 : p.n) - 1;  // key columns k1, k1-1, ..
  const uint32_t lanemask_lt = (1u << lane) - 1u;
  unsigned long long n_items = 0;

  for (;;) {
    const unsigned long long item = next_item(p, lane, n_items, blockIdx.x * 4 + warp);
    if (item >= p.items) break;
    ++n_items;
    // item = (piece * chunks + chunk) * B + matrix (k_walk_bucket's order);
    // sticky pieces (n > 32): item = ticket, piece (t % npieces) = q * B + b,
    // the chunks come from the piece's counter
    const bool sticky = WIDE && bp.chunk_ctr != nullptr;
    unsigned long long b, c, pid = 0;
    uint32_t q;
    auto grab = [&]() -> unsigned long long {  // the piece's next chunk
      unsigned int v = 0;
      if (lane == 0) v = atomicAdd(bp.chunk_ctr + pid, 1u);
      return (unsigned long long)__shfl_sync(FULL, v, 0);
    };
    if (sticky) {
      const unsigned long long nmat = bp.npieces / kBucketPieces;
      pid = item % bp.npieces;
      q = (uint32_t)(pid / nmat);
      b = pid - (unsigned long long)q * nmat;
      TP_CHECK(q < (uint32_t)kBucketPieces && b < nmat);
    } else {
      const unsigned long long nmat = p.items / ((unsigned long long)kBucketPieces * p.chunks);
      const unsigned long long rest = item / nmat;
      b = item - rest * nmat;
      q = (uint32_t)(rest / p.chunks);
      c = rest - (unsigned long long)q * p.chunks;
      TP_CHECK(q < (uint32_t)kBucketPieces && b < nmat);
    }
    const uint32_t pt = bp.ptab[b * kBucketPieces + q];
    const uint32_t cnt = (pt >> 8) & 0xFFFu;  // real slots of the piece
    if (cnt == 0) continue;                   // unused piece
    if (sticky) {
      c = grab();
      if (c >= p.chunks) continue;  // the piece is done
    }
    const uint32_t grp = pt & 0xFFu;
    const uint32_t pbase = ((pt >> 20) & 0x7FFu) << 10;  // positions [pbase, pbase + cnt) of the bucket
    const bool weighted = (pt >> 31) != 0;
    TP_CHECK(cnt <= 1024u && grp < (uint32_t)nbuckets(KEYS));
    const uint32_t nwd = (cnt + 63u) >> 6;  // packed words holding the piece's real slots
    __syncwarp();
    {  // B-side rows FIX..n-1
      const uint4* s = reinterpret_cast<const uint4*>(p.rows + b * 64 + FIX);
      uint4* d = reinterpret_cast<uint4*>(ws + S::oR);
      TP_CHECK(p.n - FIX <= S::NR);
      if constexpr (WIDE) {  // (m0, m1, s0, s1): the first half of each RowRec
        for (int x = (int)lane; x < p.n - FIX; x += 32) d[x] = s[2 * x];
      } else {
        for (int x = (int)lane; x < 2 * (p.n - FIX); x += 32) d[x] = s[x];
      }
    }

    // A side: slot k of this lane is position pbase + 32 lrow(k) + lane of
    // the bucket (tp_bucket.cuh); full words to shared memory, the packed
    // words (low 16 columns of slots w and w + 16) to registers.
    uint32_t Zp[K / 2], Gp[K / 2];
    uint32_t spm = 0;    // bit k: parity of slot k's subset
    uint32_t vmask = 0;  // bit k: slot k holds a real A subset
    const uint8_t* Tm = static_cast<const uint8_t*>(bp.tab) + b * T::kBytes;
    {
      // the bucket's run table in the (still unused) list / pass-list area,
      // and (short items, n < 28) a copy of the half table behind it: one
      // coalesced read instead of a dependent L2 round trip per slot
      uint4* RT = reinterpret_cast<uint4*>(ws + S::oHc);
      const uint8_t* Td = Tm;
      if constexpr (S::template tab_fits<KEYS, T::kBytes>()) {
        uint4* dst = reinterpret_cast<uint4*>(ws + S::oHc + align16(16 * (nbuckets(KEYS) + 1)));
        const uint4* src = reinterpret_cast<const uint4*>(Tm);
#pragma unroll
        for (int x = 0; x < T::kBytes / 16; x += 32)
          if (x + (int)lane < T::kBytes / 16) dst[x + lane] = src[x + lane];
        __syncwarp();
        Td = reinterpret_cast<const uint8_t*>(dst);
      }
      const uint32_t* wts = reinterpret_cast<const uint32_t*>(Td + T::kWt);
      run_table<KEYS>(reinterpret_cast<const uint16_t*>(Td), grp, RT, lane);
      uint32_t ra = 0;  // this lane's current run
      if (weighted) {
        // the weighted walk rebuilds its slots from their table indices:
        // IX[r][lane] (in the A2 area, which weighted items do not use)
#pragma unroll 1
        for (uint32_t r = 0; 32u * r + lane < cnt; ++r) {
          const uint32_t pp = pbase + 32u * r + lane;
          while (RT[ra + 1].x <= pp) ++ra;
          TP_CHECK(ra < (uint32_t)nbuckets(KEYS));
          uint32_t i0, i1;
          run_index(RT[ra], pp, i0, i1);
          IX[32u * r + lane] = i0 | (i1 << 16);
        }
      } else
#pragma unroll 1
      for (uint32_t r = 0; r < (uint32_t)K; ++r) {
        const int k = (int)((r >> 1) + ((r & 1u) << 4));
        const uint32_t rr = 32u * r + lane;
        uint32_t z, g;
        if (rr >= cnt) {  // dummy slot: n <= 31 -1 in padding column 31; n = 32: vmask
          z = colmask;
          g = p.n <= 31 ? 0x80000000u : 0u;
        } else {
          const uint32_t pp = pbase + rr;
          while (RT[ra + 1].x <= pp) ++ra;
          TP_CHECK(ra < (uint32_t)nbuckets(KEYS));
          uint32_t i0, i1;
          run_index(RT[ra], pp, i0, i1);
          const uint2 lo = *reinterpret_cast<const uint2*>(Td + T::kVec + T::VE * i0);
          const uint2 hi = *reinterpret_cast<const uint2*>(Td + T::kVec + T::VE * (T::N0 + i1));
          const uint32_t par = ((wts[i0] ^ wts[T::N0 + i1]) >> 16) & 1u;
          z = lo.x;
          g = lo.y;
          sub_word(z, g, hi.x, hi.y);
          vmask |= 1u << k;
          // n <= 31: padding column 31 carries the subset parity as the trit p
          if (p.n <= 31 && !par) z |= 0x80000000u;
          spm |= par << k;
        }
        reinterpret_cast<uint2*>(&A2[k & 15][lane])[k >> 4] = make_uint2(z, g);
      }
      __syncwarp();
#pragma unroll
      for (int w = 0; w < K / 2; ++w) {
        const uint4 a = A2[w][lane];
        Zp[w] = __byte_perm(a.x, a.z, 0x5410);
        Gp[w] = __byte_perm(a.y, a.w, 0x5410);
      }
    }
    // forbidden key trits of this piece: f = -x (mod 3)
    uint32_t F0 = 0, F1 = 0, F2 = 0;
    {
      uint32_t rest_g = grp;
#pragma unroll
      for (int i = KEYS - 1; i >= 0; --i) {
        const uint32_t x = rest_g % 3u;
        rest_g /= 3u;
        const uint32_t f = (3u - x) % 3u, bit = 1u << (k1 - i);
        F0 |= f == 0 ? bit : 0u;
        F1 |= f == 1 ? bit : 0u;
        F2 |= f == 2 ? bit : 0u;
      }
    }
    // B side.  Step j of superblock G is the subset gray(32 G + j) of rows
    // FIX.. : rows FIX+5.. from gray(G) (the "high" state H, the same for
    // every lane) and rows FIX..FIX+4 from gray(j) ^ (G odd ? 16 : 0) (this
    // lane's low part, two vectors per item, L[G & 1][lane]).  So a lane's
    // state is one add, H + L, and H changes by one row per superblock.
    {
#pragma unroll
      for (uint32_t par = 0; par < 2; ++par) {
        const uint32_t gl = (lane ^ (lane >> 1)) ^ (par << 4);
        uint32_t zl = colmask, gll = 0, zlw = colmask1, glw = 0;
#pragma unroll
        for (int r = 0; r < V; ++r)
          if ((gl >> r) & 1u) {
            const BRow rw = brow(r);
            sub_word(zl, gll, rw.m0, rw.a0);
            if (WIDE) sub_word(zlw, glw, rw.m1, rw.a1);
          }
        // row form on the real columns (padding columns stay H's +1)
        const uint32_t m0 = ~zl & colmask, m1 = ~zlw & colmask1;
        if (WIDE) L4[32 * par + lane] = make_uint4(m0, gll & m0, m1, glw & m1);
        else L2[32 * par + lane] = make_uint2(m0, gll & m0);
      }
    }
    for (;;) {  // the item's chunk; sticky pieces: every chunk this warp can take
    const unsigned long long sb0 = p.F0 + c * p.nblk;
    const uint32_t nsb = (uint32_t)min((unsigned long long)p.nblk, bp.s_end - sb0);
    uint32_t zh, uh, zhw = 0, uhw = 0;
    {
      uint32_t z = colmask, g = 0, zw = colmask1, gw = 0;
      const unsigned long long hs = sb0 ^ (sb0 >> 1);
      for (int r = FIX + V; r < p.n; ++r)
        if ((hs >> (r - FIX - V)) & 1ull) {
          const BRow rw = brow(r - FIX);
          sub_word(z, g, rw.m0, rw.a0);
          if (WIDE) sub_word(zw, gw, rw.m1, rw.a1);
        }
      zh = z;
      uh = pair_u2(z, g);
      zhw = zw;
      uhw = pair_u2(zw, gw);
    }
    uint32_t ev = 0, odd = 0;
    uint32_t tested_steps = 0;
    bool dense = false;
    for (uint32_t kb0 = 0; kb0 < nsb; kb0 += NBAT) {
      const uint32_t nbt = min((uint32_t)NBAT, nsb - kb0);
      uint32_t L = 0;  // list length
      __syncwarp();    // the previous batch's list is consumed
      // superblock kb0 + t of the batch: this lane's B state H + L[G & 1][lane]
      // (L in row form: add = sub of the negated row, sign m ^ s), its
      // compatibility, and the compacted list entry
      auto superblock = [&](uint32_t t, uint32_t gp) {
        if (RECOMP && lane == 0) Hs[t] = make_uint4(zh, uh, zhw, uhw);
        uint32_t zj = zh, uj = uh, zjw = zhw, ujw = uhw;
        if constexpr (WIDE) {
          const uint4 l = L4[32 * gp + lane];
          sub_word_u(zj, uj, l.x, l.x ^ l.y, l.y);
          sub_word_u(zjw, ujw, l.z, l.z ^ l.w, l.w);
        } else {
          const uint2 l = L2[32 * gp + lane];
          sub_word_u(zj, uj, l.x, l.x ^ l.y, l.y);
        }
        // compatible: no key column of y equals the forbidden trit
        const uint32_t match = (zj & F0) | (~zj & ~uj & F2) | (~zj & uj & F1);
        const uint32_t cmask = __ballot_sync(FULL, match == 0u);
        if (match == 0u) {
          const uint32_t pos = L + __popc(cmask & lanemask_lt);
          TP_CHECK(pos < (uint32_t)S::NS);
          Hc[pos] = make_uint2(__byte_perm(zj, zj, 0x1010), __byte_perm(uj, uj, 0x1010));
          if (!RECOMP) Hf[pos] = make_uint2(zj, uj);
          Hj[pos] = (uint8_t)(32u * t + lane);
        }
        L += __popc(cmask);
      };
      // H of global superblock G flips row FIX + V + tz(G); it leaves iff
      // bit tz(G) + 1 of G is set
      auto h_flip = [&](const BRow& row, bool lv) {
        sub_word_u(zh, uh, row.m0, lv ? row.s0 : row.a0, lv ? row.a0 : row.s0);
        if (WIDE) sub_word_u(zhw, uhw, row.m1, lv ? row.s1 : row.a1, lv ? row.a1 : row.s1);
      };
      const unsigned long long G0 = sb0 + kb0;
      if (nbt == (uint32_t)NBAT && (G0 & (unsigned long long)(NBAT - 1)) == 0) {
        // an aligned full batch: G = G0 + t has parity t & 1 and, inside the
        // batch, flips row FIX + V + tz(t) (compile-time); only the next
        // batch's entry needs the runtime tz of G0 + NBAT
        constexpr int LNB = NBAT == 2 ? 1 : NBAT == 4 ? 2 : 3;
        static_assert(NBAT == (1 << LNB), "NBAT: a power of two <= 8");
        static_for<NBAT>([&](auto tc) {
          constexpr uint32_t t = decltype(tc)::value;
          superblock(t, t & 1u);
          if constexpr (t + 1 < (uint32_t)NBAT) {
            constexpr int tzt = __builtin_ctz(t + 1);
            // bit tz + 1 of G0 + t + 1: inside the batch offset unless it is bit LNB (of G0)
            const bool lv = tzt + 1 < LNB ? (((t + 1) >> (tzt + 1)) & 1u) != 0 : ((G0 >> LNB) & 1ull) != 0;
            h_flip(brow(V + tzt), lv);
          }
        });
        if (kb0 + NBAT < nsb) {
          const unsigned long long G = G0 + NBAT;
          const int tzg = tz64(G);
          h_flip(brow(V + tzg), ((G >> (tzg + 1)) & 1ull) != 0);
        }
      } else {
#pragma unroll 1
        for (uint32_t t = 0; t < nbt; ++t) {
          const uint32_t kb = kb0 + t;
          superblock(t, (uint32_t)((sb0 + kb) & 1ull));
          if (kb + 1 < nsb) {
            const unsigned long long G = sb0 + kb + 1;
            const int tzg = tz64(G);
            h_flip(brow(V + tzg), ((G >> (tzg + 1)) & 1ull) != 0);
          }
        }
      }
      tested_steps += L;
      __syncwarp();
      if (L == 0) continue;
      // the full state of list entry j (step 32 t + l of the batch): H of
      // superblock t plus L[parity][l], as in the compaction
      auto entry_state = [&](uint32_t j, uint32_t& z, uint32_t& u, uint32_t& zw, uint32_t& uw) {
        if constexpr (!RECOMP) {
          const uint2 h = Hf[j];
          z = h.x;
          u = h.y;
          return;
        }
        const uint32_t hj = Hj[j], t = hj >> 5;
        const uint4 h = Hs[t];
        const uint32_t gp = (uint32_t)((G0 + t) & 1ull);
        z = h.x;
        u = h.y;
        if constexpr (WIDE) {
          const uint4 l = L4[32 * gp + (hj & 31u)];
          sub_word_u(z, u, l.x, l.x ^ l.y, l.y);
          zw = h.z;
          uw = h.w;
          sub_word_u(zw, uw, l.z, l.z ^ l.w, l.w);
        } else {
          const uint2 l = L2[32 * gp + (hj & 31u)];
          sub_word_u(z, u, l.x, l.x ^ l.y, l.y);
        }
      };
      // the exact paths read their entries' states: stored (Hf), or
      // materialised kChunk entries at a time in the pass-list area
      auto materialise = [&](uint32_t e0, uint32_t cn) {
        __syncwarp();
        for (uint32_t e = lane; e < cn; e += 32) {
          uint32_t z, u, zw = 0, uw = 0;
          entry_state(e0 + e, z, u, zw, uw);
          Hf[e] = make_uint2(z, u);
          if (WIDE) H1[e] = make_uint2(zw, uw);
        }
        __syncwarp();
      };
      if (weighted) {  // deduplicated A side: every listed step exactly, with weights
        if constexpr (!RECOMP) {
          batch_exact_weighted<FIX, KEYS, WIDE>(Hf, H1, Hj, L, Tm, IX, cnt, lane, colmask, colmask1, p.pm + 2 * b);
        } else {
          for (uint32_t c0 = 0; c0 < L; c0 += kChunk) {
            const uint32_t cc = min(kChunk, L - c0);
            materialise(c0, cc);
            batch_exact_weighted<FIX, KEYS, WIDE>(Hf, H1, Hj + c0, cc, Tm, IX, cnt, lane, colmask, colmask1,
                                                  p.pm + 2 * b);
          }
        }
        continue;
      }
      // list entries [ib, ib + cn) exactly
      auto exact_range = [&](uint32_t ib, uint32_t cn, uint32_t& bev, uint32_t& bodd) {
        if constexpr (!RECOMP) {  // stored states: one call
          const unsigned long long r = batch_exact_packed<FIX>(A2, Hf + ib, Hj + ib, cn, lane, spm, vmask, colmask, p.n, one);
          bev = (uint32_t)r;
          bodd = (uint32_t)(r >> 32);
          return;
        }
        bev = bodd = 0;
        for (uint32_t c0 = ib; c0 < ib + cn; c0 += kChunk) {
          const uint32_t cc = min(kChunk, ib + cn - c0);
          materialise(c0, cc);
          unsigned long long r;
          if constexpr (WIDE)
            r = batch_exact_wide<FIX, KEYS>(A2, Hf, H1, Hj + c0, cc, Tm, grp, pbase, cnt, lane, spm, colmask1);
          else
            r = batch_exact_packed<FIX>(A2, Hf, Hj + c0, cc, lane, spm, vmask, colmask, p.n, one);
          bev += (uint32_t)r;
          bodd += (uint32_t)(r >> 32);
        }
      };
      if (dense) {
        uint32_t bev, bodd;
        exact_range(0, L, bev, bodd);
        ev += bev;
        odd += bodd;
        dense = __any_sync(FULL, bev >= (uint32_t)(K / 2) * nbt);
        continue;
      }
      // Long lists (batches of 8 superblocks; pieces that most B states are
      // compatible with) are filtered and verified in segments, so that a
      // lane's pass list sees at most kSeg entries between two verifies and
      // rarely overflows into the exact path.
      // The 17-row kernels (5 key columns: ~17 steps per 4 superblocks on
      // uniform inputs, but all 128 for a piece without a zero key trit on
      // sparse B states) run in segments; the 14-row kernel (C2) does not.
      // TP_BATCH_SEG: entries per segment, a multiple of 6 (C3: 176.7 ms
      // without segments, 172.4 at 66, 170.1 at 48, 169.8 at 36, 171.4 at 24).
#ifndef TP_BATCH_SEG
#define TP_BATCH_SEG 48
#endif
      static_assert(TP_BATCH_SEG % 6 == 0, "segments hold whole filter iterations");
      constexpr bool kSegments = NBAT > 4 || FIX == 17;
      constexpr uint32_t kSeg = (uint32_t)TP_BATCH_SEG;
      uint32_t ib = 0;
      do {
      const uint32_t ie = kSegments ? min(L, ib + kSeg) : L;
      // the packed filter over the list, three entries per iteration: the
      // three zp words of packed word w meet in one halfword-wise minimum
      // (packed_test3), so bit w of M = word w passed for one of the entries
      // i, i + 1, i + 2 (the verify finds which); one or two entries are left
      // for a last iteration
      uint32_t ne = 0;
      auto record = [&](uint32_t M, uint32_t i) {
        // unconditional store (slot ECAP takes the overflow), no branch
        E[min(ne, (uint32_t)ECAP)][lane] = make_uint2(M, i);
        ne += M != 0u ? 1u : 0u;
      };
      auto filter = [&](auto Wc) {
        constexpr int W = decltype(Wc)::value;
        uint32_t i = ib;
#if TP_BATCH_SIX
        // two groups of three entries per iteration and record: bit w of M
        // for entries i..i+2, bit 16 + w for i+3..i+5 (the piece's common
        // widths only: the code has to stay in the instruction cache)
        if constexpr (W <= TP_BATCH_SIX && (FIX == 14 || WIDE)) {
#pragma unroll 1
          for (; i + 6 <= ie; i += 6) {
            const uint4* q = reinterpret_cast<const uint4*>(Hc + i);  // i is even
            const uint4 hab = q[0], hcd = q[1], hef = q[2];
            uint32_t M = 0;
            static_for<W>([&](auto wc) {
              constexpr int w = decltype(wc)::value;
              packed_test3<(1u << w)>(Zp[w], Gp[w], hab.x, hab.y, hab.z, hab.w, hcd.x, hcd.y, M, one, cneg);
              packed_test3<(1u << (16 + w))>(Zp[w], Gp[w], hcd.z, hcd.w, hef.x, hef.y, hef.z, hef.w, M, one, cneg);
            });
            record(M, i);
          }
        }
#endif
#pragma unroll 1
        for (; i + 3 <= ie; i += 3) {
          const uint2 ha = Hc[i], hb = Hc[i + 1], hc = Hc[i + 2];
          uint32_t M = 0;
          static_for<W>([&](auto wc) {
            constexpr int w = decltype(wc)::value;
            packed_test3<(1u << w)>(Zp[w], Gp[w], ha.x, ha.y, hb.x, hb.y, hc.x, hc.y, M, one, cneg);
          });
          record(M, i);
        }
        if (i + 2 == ie) {
          const uint2 ha = Hc[i], hb = Hc[i + 1];
          uint32_t M = 0;
          static_for<W>([&](auto wc) {
            constexpr int w = decltype(wc)::value;
            packed_test2<(1u << w)>(Zp[w], Gp[w], ha.x, ha.y, hb.x, hb.y, M, one, cneg);
          });
          record(M, i);
        } else if (i < ie) {
          const uint2 ha = Hc[i];
          uint32_t M = 0;
          static_for<W>([&](auto wc) {
            constexpr int w = decltype(wc)::value;
            packed_test<(1u << w)>(Zp[w], Gp[w], ha.x, ha.y, M, one, cneg);
          });
          record(M, i);
        }
      };
      using FW = FilterWidths<FIX, KEYS>;
      if constexpr (FW::WA == 16) {
        filter(std::integral_constant<int, 16>{});
      } else {
        if (nwd > (uint32_t)FW::WA) filter(std::integral_constant<int, 16>{});
        else if (nwd > (uint32_t)FW::WB) filter(std::integral_constant<int, FW::WA>{});
        else filter(std::integral_constant<int, FW::WB>{});
      }
      const uint32_t nemax = __reduce_max_sync(FULL, ne);
      if (nemax > (uint32_t)ECAP) {
        // a lane's pass list overflowed (event-dense matrix): the segment exactly
        __syncwarp();
        uint32_t bev, bodd;
        exact_range(ib, ie - ib, bev, bodd);
        ev += bev;
        odd += bodd;
        dense = dense || (p.dense_ok != 0 && __any_sync(FULL, bev >= (uint32_t)(K / 2) * nbt));
      } else if (nemax != 0) {
        // Verify, balanced over the lanes.  The records are compacted row
        // by row into one flat list in place (row r only lands on flat
        // positions < 32 (r + 1), all read by then), tagged with their lane;
        // lane k takes records k, k + 32, ..: it repeats the packed test of
        // the record's words for each of the (up to) three entries against
        // the SOURCE lane's slots (A2; the slots' parities and validity SV
        // in the pass list's overflow row) to find the entry and half that
        // passed, and evaluates those on all columns.
        uint2* Fl = &E[0][0];
        uint2* SV = &E[ECAP][0];
        __syncwarp();
        SV[lane] = make_uint2(spm, vmask);
        uint32_t nrec = 0;
        for (uint32_t r = 0; r < nemax; ++r) {
          const bool has = r < ne;
          const uint2 rec = E[r][lane];
          const uint32_t bal = __ballot_sync(FULL, has);
          __syncwarp();
          if (has) Fl[nrec + __popc(bal & lanemask_lt)] = make_uint2(rec.x, rec.y | (lane << 16));
          nrec += __popc(bal);
        }
        __syncwarp();
        uint32_t bev = 0, bodd = 0;
        for (uint32_t ri = lane; ri < nrec; ri += 32u) {
          const uint2 rec = Fl[ri];
          const uint32_t src = rec.y >> 16;
          const uint2 sv = SV[src];
          uint32_t M = rec.x;
          TP_CHECK((rec.y & 0xFFFFu) < L && src < 32u && (TP_BATCH_SIX || M < 0x10000u));
          while (M) {
            const uint32_t bm = __ffs(M) - 1;
            M &= M - 1;
            // bit w: entries i .. i + 2 of the record; bit 16 + w: i + 3 .. i + 5
            const uint32_t w = bm & 15u, i0 = (rec.y & 0xFFFFu) + 3u * (bm >> 4);
            const uint32_t i1 = min(i0 + 3u, ie);  // a last iteration holds one or two entries
            const uint4 a4 = A2[w][src];
            const uint32_t zk = __byte_perm(a4.x, a4.z, 0x5410), gk = __byte_perm(a4.y, a4.w, 0x5410);
            // which entries and halves passed: bit e + 16 half, branch-free
            uint32_t hit[3];
#pragma unroll
            for (uint32_t e = 0; e < 3u; ++e) {
              const uint2 hq = Hc[min(i0 + e, ie - 1u)];
              uint32_t dq, zq;
              TP_LOP3(dq, zk, gk, hq.y, 0x06);
              TP_LOP3(zq, dq, zk, hq.x, 0x09);
              hit[e] = (zq - 0x00010001u) & ~zq;  // bit 15 / 31: half 0 / 1 has no zero column
            }
            // (a last iteration of one or two entries repeats its last entry)
            uint32_t hits = ((hit[0] >> 15) & 0x00010001u) | (i0 + 1u < i1 ? (hit[1] >> 14) & 0x00020002u : 0u) |
                            (i0 + 2u < i1 ? (hit[2] >> 13) & 0x00040004u : 0u);
            while (hits) {
              const uint32_t bq = __ffs(hits) - 1;
              hits &= hits - 1;
              const uint32_t j = i0 + (bq & 3u), hf = bq >> 4;
              TP_CHECK(j < L);
              uint2 h, hw;
              entry_state(j, h.x, h.y, hw.x, hw.y);
              const uint32_t k = w + 16u * hf;
              const uint2 a = hf ? make_uint2(a4.z, a4.w) : make_uint2(a4.x, a4.y);
              uint32_t d, zp;
              TP_LOP3(d, a.x, a.y, h.y, 0x06);
              TP_LOP3(zp, d, a.x, h.x, 0x09);
              if (zp == 0 && ((sv.y >> k) & 1u)) {
                uint32_t par = 0;
                if constexpr (WIDE) {
                  // the primary columns are nonzero: test the secondary ones
                  const uint32_t rr =
                      bucket_wide_term<FIX, KEYS>(Tm, grp, pbase + 32u * lrow(k) + src, hw, colmask1);
                  if (!rr) continue;
                  par = rr >> 1;
                }
                bev += 1;
                bodd += (__popc((d ^ pair_g2(h.x, h.y)) & colmask) + par + (Hj[j] & 1u) + ((sv.x >> k) & 1u)) & 1u;
              }
            }
          }
        }
        ev += bev;
        odd += bodd;
        // event-dense (e.g. all-ones rows): exact mode for the next batches
        // (the verify's events are spread over the lanes: the warp's total)
        dense = dense || (p.dense_ok != 0 && __reduce_add_sync(FULL, bev) >= 4u * (uint32_t)(K / 2) * nbt);
      }
      if constexpr (!kSegments) break;
      __syncwarp();  // the segment's records are consumed
      ib += kSeg;
      } while (ib < L);  // segments
    }
    warp_flush(p.pm + 2 * b, ev - odd, odd, lane);
    if (bp.tested && lane == 0) {
      const uint32_t words = FilterWidths<FIX, KEYS>::width(nwd);
      atomicAdd(bp.tested, 64ull * words * tested_steps);
    }
    if (!sticky) break;
    c = grab();
    if (c >= p.chunks) break;
    }  // chunks
  }
  queue_done(p, lane);
}

// Batch shapes: NBAT superblocks per list, ECAP pass-list entries per lane.
// Sized so that four 4-warp blocks fit an SM (228 KB of shared memory).
template <bool WIDE, int FIX>
struct BatchShape {
#ifndef TP_BATCH_NB_NARROW
#define TP_BATCH_NB_NARROW 4
#define TP_BATCH_EC_NARROW 10
#endif
// the 17-row A side for n <= 32 (28 <= n <= 32; C3): batches of 8 (states
// recomputed) gain 6 % on uniform inputs but lose on C3's sparse family
// (long lists: more segments, more pass-list overflows): 4
#ifndef TP_BATCH_NB17
#define TP_BATCH_NB17 4
#define TP_BATCH_EC17 10
#endif
// n > 32: batches of 8 superblocks (the 16-byte rows make the room; lists of
// ~34 steps on uniform inputs instead of ~17 halve the per-batch costs of
// the verify: C4 1.66 -> 1.53 ms, C5 window 362 -> 327 ms)
#ifndef TP_BATCH_NBW
#define TP_BATCH_NBW 8
#define TP_BATCH_ECW 6
#endif
  static constexpr int NBAT = WIDE ? TP_BATCH_NBW : FIX == 17 ? TP_BATCH_NB17 : TP_BATCH_NB_NARROW;
  static constexpr int ECAP = WIDE ? TP_BATCH_ECW : FIX == 17 ? TP_BATCH_EC17 : TP_BATCH_EC_NARROW;
  // four blocks per SM: 228 KB of shared memory, 1 KB reserved per block
  static_assert(4 * (4 * BatchSmem<NBAT, ECAP, WIDE, FIX>::kWarp + 1024) <= 228 * 1024,
                "k_walk_batch: four blocks must fit an SM");
};

template <bool WIDE, int FIX, int KEYS>
static cudaError_t launch_batch_k(int grid, const BucketParamsCfg& bc, cudaStream_t st) {
  using Sh = BatchShape<WIDE, FIX>;
  constexpr int bytes = 4 * BatchSmem<Sh::NBAT, Sh::ECAP, WIDE, FIX>::kWarp;
  auto* k = &k_walk_batch<Sh::NBAT, Sh::ECAP, WIDE, FIX, KEYS>;
  static const cudaError_t attr = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (attr != cudaSuccess) return attr;
  k<<<grid, 128, bytes, st>>>(bc);
  return cudaGetLastError();
}

cudaError_t launch_walk_batch(int grid, const BucketParams& bp, BucketCfg c, cudaStream_t st) {
  const BucketParamsCfg bc{bp.fp, bp.tab, bp.ptab, bp.tested, bp.s_end, c.fix, c.keys, bp.chunk_ctr, bp.npieces};
  if (bp.fp.n > 32 && c.fix == 17 && c.keys == 4) return launch_batch_k<true, 17, 4>(grid, bc, st);
  if (bp.fp.n > 32 && c.fix == 17 && c.keys == 5) return launch_batch_k<true, 17, 5>(grid, bc, st);
  if (c.fix == 14 && c.keys == 3) return launch_batch_k<false, 14, 3>(grid, bc, st);
  if (c.fix == 17 && c.keys == 5) return launch_batch_k<false, 17, 5>(grid, bc, st);
  return cudaErrorInvalidValue;
}

// blocks of the batched walk resident per SM (the plan sizes its grid with it)
template <bool WIDE, int FIX, int KEYS>
static int batch_occupancy() {
  using Sh = BatchShape<WIDE, FIX>;
  constexpr int bytes = 4 * BatchSmem<Sh::NBAT, Sh::ECAP, WIDE, FIX>::kWarp;
  auto* k = &k_walk_batch<Sh::NBAT, Sh::ECAP, WIDE, FIX, KEYS>;
  int nb = 0;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 128, bytes) != cudaSuccess) return 0;
  return nb;
}

// the least over the kernels of that width
int walk_batch_blocks_per_sm(bool wide) {
  if (wide) return std::min(batch_occupancy<true, 17, 4>(), batch_occupancy<true, 17, 5>());
  return std::min(batch_occupancy<false, 14, 3>(), batch_occupancy<false, 17, 5>());
}

}  // namespace tp
