// tp_walk_tc.cu -- the pair test on the 5th-generation tensor cores (tcgen05).
//
// Meet in the middle, as in the pair walks: a subset S of the rows splits as
// S = S_A u S_B with S_A in rows 0..7 (256 "A vectors", fixed per matrix) and
// S_B in rows 8..n-1 (walked), and v_S = v_A + v_B.  The term of S is nonzero
// iff no column of v_S is zero, and the number Z of zero columns is a
// bilinear form of the two trit vectors:
//
//   3 [x + y = 0 (mod 3)] = 1 + 2 Re(w^x w^y),   w = exp(2 pi i / 3).
//
// In the basis (1, w) of Z[w], w^y = r + s w with (r, s) = (1,0), (0,1),
// (-1,-1) for y = 0, 1, 2, and 2 Re((p + q w)(r + s w)) = (2p - q) r + (-p - q) s.
// So with the A vector x encoded per column as the bytes (2p - q, -p - q) and
// the B vector y as (r, s), the dot product over all n columns plus n (a few
// constant K slots) is exactly 3 Z.  One tcgen05.mma.kind::f8f6f4 (e4m3
// operands, every value in {0, +-1, +-2, <= 16} is exact) computes it for a
// 128 x 128 block of (A vector, B vector) pairs; the f16 accumulator is
// exact (|partial sums| << 2048).
//
// Per CTA (one per SM, persistent, static item schedule); the arbiter issues
// the highest eligible warp id first, so the latency-critical roles get the
// high ids:
//   warp 18     : TMEM allocation (512 columns = 4 slots of 128); the whole
//                 warp runs the issue loop and one elected lane issues the MMAs
//                 of each sub-tile (one M-tile x the 128 B vectors of a tile,
//                 ks k-steps of 32 bytes) and its commit.
//   warps 16-17 : producers.  Thread j owns B columns j and j + 64: it walks
//                 their B vectors in Gray order over the tile index (one row
//                 add/sub per tile, 3 LOP3 per 4 columns on byte-replicated
//                 (z, g) masks, see below), turns them into operand bytes with
//                 2 LOP3 per 4 columns and stores their rows of the stage.
//                 They also build the A operand at each new item.
//   warps 0..15 : epilogue, four groups of 4, group g owning TMEM slot g.
//                 Each thread owns one TMEM lane (an A vector) and reads its
//                 128 accumulators as 64 packed f16 pairs; the slot is released
//                 as soon as they are in registers.  "Some element is 0" is a
//                 product tree (HMUL2, FMA pipe) over half of them and a min
//                 tree (HMNMX2, ALU pipe) over the other half.  A zero (a
//                 nonzero term, probability (2/3)^n per pair) is evaluated
//                 exactly from the bit planes: sign (-1)^(|S| + #(-1 columns)),
//                 as in chunk_sum (src/_kernels.py:123-127).
// Exact but slower than the packed LOP3 walk on B200,
// so it is opt-in (TRITPERM_TC=1).
//
// B operand bytes from walk masks.  Each column owns one byte of a 32-bit
// word; the trit state (z = [y = 0], g = [y = 2], the z-encoding of
// tp_device.cuh) is replicated in bits 3, 4, 5, 7 of the byte and bits 0, 1,
// 2, 6 hold a frozen dummy (z = g = 0, rows are 0 there).  sub_word works
// bitwise, so the walk step is unchanged, and
//   r byte = (z & 0x38) | (g & ~z)  ->  0x38 (1.0), 0x00, 0xB8 (-1.0) for y = 0, 1, 2
//   s byte = ~z & (0x38 | g)        ->  0x00, 0x38 (1.0), 0xB8 (-1.0)
// are one LOP3 each per 4 columns ((z, g) = (1, 1) is an alternate zero, so g
// only counts where ~z).
//
// The sum over all subsets is order-independent, so a work item (matrix b,
// chunk c) covers the subsets whose bits >= 15 + t equal gray(c0 + c): that is
// exactly the Gray step range [(c0 + c) 2^(15+t), (c0 + c + 1) 2^(15+t)) of
// chunk_sum (src/_kernels.py:90-128), so aligned ranges are supported as well
// as full traversals.
#include <cstdio>
#include "tp_kernels.cuh"

namespace tp {

namespace {

constexpr int kTcStages = 4;       // B operand ring
constexpr int kTcSlots = 4;        // TMEM accumulator slots (128 columns = one 128 x 128 sub-tile each)
// Warp roles.  B200's warp arbiter issues the highest eligible warp id first,
// so the latency-critical roles get the high ids: the MMA issuer is the last
// warp, the producers the two before it, the 16 epilogue warps come first.
constexpr int kTcEpiWarp0 = 0;     // 16 epilogue warps: group (e / 4) owns TMEM slot (e / 4)
constexpr int kTcEpiWarps = 16;
constexpr int kTcProdWarp0 = 16;   // 2 producer warps: thread j builds B columns j and j + 64
constexpr int kTcProdThreads = 64;
constexpr int kTcMmaWarp = 18;     // TMEM allocation; an elected lane issues the MMAs
constexpr int kTcThreads = 32 * (kTcMmaWarp + 1);  // 608

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
// Waiting roles other than the MMA issuer back off between polls, so that
// their barrier traffic does not compete with the tensor core's operand reads.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(64);
  }
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void proxy_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, no swizzle: core matrices of 8 rows
// x 16 bytes; LBO = distance of K-adjacent core matrices, SBO = distance of
// 8-row groups; bit 46 = descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// e4m3 byte of a small nonnegative integer v <= 16 (exact).
__host__ __device__ constexpr uint32_t e4m3_int(uint32_t v) {
  if (v == 0) return 0;
  uint32_t e = 0;
  while ((2u << e) <= v) ++e;
  const uint32_t m = ((v << 3) >> e) & 7u;
  return ((e + 7u) << 3) | m;
}

__device__ __forceinline__ uint32_t spread4(uint32_t nib) {  // bit b of nib -> 0xB8 in byte b
  return ((nib & 0xFu) * 0x00204081u & 0x01010101u) * 0xB8u;
}

__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hmin2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
// A half is "hit" when it is +-0 (a zero accumulator) or NaN (0 * inf in a
// product tree); positive finite values and +inf are not.
__device__ __forceinline__ bool half_hit(uint32_t h) { return ((h & 0x7FFFu) - 1u) >= 0x7C00u; }
__device__ __forceinline__ bool pair_hit(uint32_t x) { return half_hit(x & 0xFFFFu) || half_hit(x >> 16); }

#define TP_TLD32(addr, v, o)                                                                                      \
  asm volatile(                                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"  \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                  \
      : "=r"(v[o + 0]), "=r"(v[o + 1]), "=r"(v[o + 2]), "=r"(v[o + 3]), "=r"(v[o + 4]), "=r"(v[o + 5]),           \
        "=r"(v[o + 6]), "=r"(v[o + 7]), "=r"(v[o + 8]), "=r"(v[o + 9]), "=r"(v[o + 10]), "=r"(v[o + 11]),         \
        "=r"(v[o + 12]), "=r"(v[o + 13]), "=r"(v[o + 14]), "=r"(v[o + 15]), "=r"(v[o + 16]), "=r"(v[o + 17]),     \
        "=r"(v[o + 18]), "=r"(v[o + 19]), "=r"(v[o + 20]), "=r"(v[o + 21]), "=r"(v[o + 22]), "=r"(v[o + 23]),     \
        "=r"(v[o + 24]), "=r"(v[o + 25]), "=r"(v[o + 26]), "=r"(v[o + 27]), "=r"(v[o + 28]), "=r"(v[o + 29]),     \
        "=r"(v[o + 30]), "=r"(v[o + 31])                                                                         \
      : "r"(addr))

struct TcSmem {
  uint64_t full[kTcStages], empty[kTcStages];
  uint64_t tfull[kTcSlots], tempty[kTcSlots];
  uint64_t afull[2], aempty[2];
  uint32_t taddr;
};

// Exact term of one hit (a zero accumulator): v = vA + vB from the bit
// planes (z-encoding; add = sub of the negated vector), sign (-1)^(|S| +
// #(-1 columns)) as in chunk_sum (src/_kernels.py:123-127).  Padding columns
// (bits >= n) are nonzero in both vectors, so only the sign needs the mask.
__device__ __forceinline__ void tc_term(uint32_t zA0, uint32_t gA0, uint32_t zA1, uint32_t gA1, uint4 b,
                                        uint32_t cm0, uint32_t cm1, uint32_t spar, uint32_t& plus, uint32_t& minus,
                                        unsigned long long* err) {
  uint32_t z0 = zA0, g0 = gA0, z1 = zA1, g1 = gA1;
  sub_word(z0, g0, ~b.x, ~b.x ^ b.z);
  sub_word(z1, g1, ~b.y, ~b.y ^ b.w);
  if ((z0 | z1) != 0) {
    atomicAdd(err, 1ull);
    return;
  }
  const uint32_t par = (spar + __popc(g0 & cm0) + __popc(g1 & cm1)) & 1u;
  if (par) ++minus;
  else ++plus;
}

// Rare path of the epilogue (out of line: the hot loop stays small in the
// instruction cache).  The 8 accumulators of one quad (columns j0..j0+7 of
// this lane's A vector); every zero among them is a nonzero term.
static __device__ __noinline__ void tc_quad(const uint32_t (&w)[4], int j0, const uint4* pl, uint32_t zA0,
                                            uint32_t gA0, uint32_t zA1, uint32_t gA1, uint32_t cm0, uint32_t cm1,
                                            uint32_t spar, uint32_t& plus, uint32_t& minus, unsigned long long* err) {
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int jj = j0 + 2 * r + h;  // B column
      if (half_hit(h ? (w[r] >> 16) : (w[r] & 0xFFFFu)))
        tc_term(zA0, gA0, zA1, gA1, pl[jj], cm0, cm1, spar ^ (__popc(jj) & 1u), plus, minus, err);
    }
}

}  // namespace

template <int NW>
__global__ void __launch_bounds__(kTcThreads, 1) k_walk_tc(const TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align the operand area
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int KP = 32 * p.ks;                 // operand row bytes
  const uint32_t SBO = 8u * KP;             // 8-row group stride
  const uint32_t MT = 128u * KP;            // one 128-row operand tile
  uint8_t* sA = base;                       // [2 buffers][2 M-tiles] tiles
  uint8_t* sB = sA + 4 * MT;                // [kTcStages] tiles
  uint32_t* sRow = (uint32_t*)(sB + kTcStages * MT);  // [64][3][NW] byte-mask rows (m, s, a)
  uint4* sPl = (uint4*)(sRow + 64 * 3 * NW);           // [8][128] B vector bit planes (z0, z1, g0, g1)
  RowRec* sRB = (RowRec*)(sPl + 8 * 128);                // [64] bit-plane rows of the current matrix
  TcSmem* S = (TcSmem*)(sRB + 64);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = p.n, t = p.t;
  const unsigned long long tiles = 1ull << t;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kTcStages; ++i) {
      mbar_init(smem_u32(&S->full[i]), kTcProdThreads);
      mbar_init(smem_u32(&S->empty[i]), 1);
    }
    for (int i = 0; i < kTcSlots; ++i) {
      mbar_init(smem_u32(&S->tfull[i]), 1);
      mbar_init(smem_u32(&S->tempty[i]), 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&S->afull[i]), kTcProdThreads);
      mbar_init(smem_u32(&S->aempty[i]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kTcMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&S->taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // constant tail of every B stage row: K slots [2R, 2R + nslots) hold 1.0,
  // the rest of [2R, KP) is 0; padding columns come from the walk itself.
  {
    const int nslots = (n + 15) / 16;
    for (int i = threadIdx.x; i < kTcStages * 128 * KP; i += blockDim.x) {
      const int st = i / (128 * KP), rem = i % (128 * KP), row = rem / KP, kb = rem % KP;
      if (kb >= 2 * p.R) {
        const uint8_t v = (kb < 2 * p.R + nslots) ? 0x38 : 0;
        sB[st * MT + (row >> 3) * SBO + (kb >> 4) * 128 + (row & 7) * 16 + (kb & 15)] = v;
      }
    }
  }
  proxy_fence();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = S->taddr;

  if (warp == kTcMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // Sub-tile (T, mt) = M-tile mt x the 128 B vectors of tile T goes to TMEM
    // slot (2T + mt) mod 4; the B stage is released after both.  The whole
    // warp runs the loop (warp-uniform descriptors live in uniform registers)
    // and one elected lane issues each tcgen05 instruction: a single-lane
    // loop pays a uniform-register round trip per MMA.
    {
      const uint32_t idesc = (16u << 17) | (8u << 24);  // M=128, N=128, e4m3 x e4m3 -> f16, K-major
      const uint64_t dA0 = umma_desc(smem_u32(sA), 128, SBO), dB0 = umma_desc(smem_u32(sB), 128, SBO);
      const uint64_t mt_step = (uint64_t)(MT >> 4);      // descriptor address units (16 B)
      uint32_t bs = 0, bph = 0, sl = 0, sph = 0, seq = 0;
      for (unsigned long long item = blockIdx.x; item < p.items; item += gridDim.x, ++seq) {
        const uint32_t abuf = seq & 1u;
        mbar_wait(smem_u32(&S->afull[abuf]), (seq >> 1) & 1u);
        for (unsigned long long T = 0; T < tiles; ++T) {
          mbar_wait(smem_u32(&S->full[bs]), bph);
          const uint64_t db = dB0 + bs * mt_step;
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            mbar_wait(smem_u32(&S->tempty[sl]), sph ^ 1u);
            tc_fence_after();
            const uint64_t da = dA0 + (abuf * 2 + mt) * mt_step;
            const uint32_t d = tbase + sl * 128u;
            if (elect_one()) {
              for (int k = 0; k < p.ks; ++k)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                    "l"(da + 16 * k), "l"(db + 16 * k), "r"(idesc), "r"((uint32_t)k));
              tc_commit(smem_u32(&S->tfull[sl]));
            }
            __syncwarp();
            if (++sl == kTcSlots) { sl = 0; sph ^= 1u; }
          }
          if (elect_one()) tc_commit(smem_u32(&S->empty[bs]));
          __syncwarp();
          if (++bs == kTcStages) { bs = 0; bph ^= 1u; }
        }
        if (elect_one()) tc_commit(smem_u32(&S->aempty[abuf]));
        __syncwarp();
      }
    }
  } else if (warp >= kTcProdWarp0) {
    // ------------------------------------------------------------ producers
    const int j0 = threadIdx.x - 32 * kTcProdWarp0;  // B columns j0 and j0 + 64
    uint32_t bs = 0, bph = 0, seq = 0;
    long long cur_b = -1;
    uint32_t colmask[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      uint32_t m = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (4 * w + b < n) m |= 0xFFu << (8 * b);
      colmask[w] = m;
    }
    const int nslots = (n + 15) / 16;  // K slots [2R, 2R + nslots) carry the offset n
    const uint32_t pz0i = n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
    const uint32_t pz1i = n <= 32 ? 0u : (n >= 64 ? 0xffffffffu : ((1u << (n - 32)) - 1u));
    for (unsigned long long item = blockIdx.x; item < p.items; item += gridDim.x, ++seq) {
      const unsigned long long b = item / p.chunks, c = item % p.chunks;
      const RowRec* R = p.rows + b * 64;
      const unsigned long long cg = p.c0 + c;
      const unsigned long long P = (cg ^ (cg >> 1)) << (15 + t);
      if ((long long)b != cur_b) {
        asm volatile("bar.sync 1, 64;" ::: "memory");  // every producer is done with the old rows
        for (int i = j0; i < n * NW; i += kTcProdThreads) {
          const int row = i / NW, w = i % NW;
          const unsigned long long m = (unsigned long long)R[row].m[0] | ((unsigned long long)R[row].m[1] << 32);
          const unsigned long long sg = (unsigned long long)R[row].s[0] | ((unsigned long long)R[row].s[1] << 32);
          const uint32_t mb = spread4((uint32_t)(m >> (4 * w))), sb = spread4((uint32_t)(sg >> (4 * w)));
          sRow[(row * 3 + 0) * NW + w] = mb;
          sRow[(row * 3 + 1) * NW + w] = sb;
          sRow[(row * 3 + 2) * NW + w] = mb ^ sb;
        }
        for (int i = j0; i < 64; i += kTcProdThreads) sRB[i] = R[i];
        asm volatile("bar.sync 1, 64;" ::: "memory");
        cur_b = (long long)b;
      }
      // ---- A operand of this item (rows 0..7): 256 vectors, 4 per thread.
      // Bytes per column: r slot (2p - q) = 0x40 (2.0) for x = 0 else 0xB8
      // (-1.0); s slot (-p - q) = 0x40 for x = 2 else 0xB8; then the offset.
      const uint32_t abuf = seq & 1u;
      mbar_wait(smem_u32(&S->aempty[abuf]), ((seq >> 1) & 1u) ^ 1u);
#pragma unroll 1
      for (int k4 = 0; k4 < 4; ++k4) {
        const int a = j0 + kTcProdThreads * k4;
        uint32_t z[NW], g[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) { z[w] = 0xB8B8B8B8u; g[w] = 0; }
#pragma unroll 1
        for (int r = 0; r < 8 && r < n; ++r)
          if ((a >> r) & 1) {
#pragma unroll
            for (int w = 0; w < NW; ++w) sub_word(z[w], g[w], sRow[(r * 3) * NW + w], sRow[(r * 3 + 2) * NW + w]);
          }
        const int row = a & 127;
        uint8_t* tile = sA + (abuf * 2 + (a >> 7)) * MT + (row >> 3) * SBO + (row & 7) * 16;
#pragma unroll 1
        for (int kb4 = 0; kb4 < KP / 4; ++kb4) {
          uint32_t word = 0;
          const int kb = 4 * kb4;
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            if (kb == 4 * w) word = (0xB8B8B8B8u ^ ((z[w] | (z[w] << 1)) & 0xF8F8F8F8u)) & colmask[w];
            if (kb == p.R + 4 * w) {
              const uint32_t gv = g[w] & ~z[w];  // (z, g) = (1, 1) is an alternate zero
              word = (0xB8B8B8B8u ^ ((gv | (gv << 1)) & 0xF8F8F8F8u)) & colmask[w];
            }
          }
          if (kb >= 2 * p.R) {
            word = 0;
            for (int qq = 0; qq < 4; ++qq) {
              const int slot = kb + qq - 2 * p.R;
              if (slot < nslots) {
                const int v = n - 16 * slot;
                word |= e4m3_int(v > 16 ? 16 : v) << (8 * qq);
              }
            }
          }
          *(uint32_t*)(tile + (kb >> 4) * 128 + (kb & 15)) = word;
        }
      }
      proxy_fence();
      mbar_arrive(smem_u32(&S->afull[abuf]));

      // ---- B walk: column jj of tile T is the subset P | gray(T) << 15 | jj << 8
      uint32_t z[2][NW], g[2][NW], pz[2][2], pg[2][2];
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
#pragma unroll
        for (int w = 0; w < NW; ++w) { z[cc][w] = 0xB8B8B8B8u; g[cc][w] = 0; }
        pz[cc][0] = pz0i;
        pz[cc][1] = pz1i;
        pg[cc][0] = pg[cc][1] = 0;
        unsigned long long x = P | ((unsigned long long)(j0 + 64 * cc) << 8);
        while (x) {
          const int r = __ffsll((long long)x) - 1;
          x &= x - 1;
#pragma unroll
          for (int w = 0; w < NW; ++w) sub_word(z[cc][w], g[cc][w], sRow[(r * 3) * NW + w], sRow[(r * 3 + 2) * NW + w]);
          sub_word(pz[cc][0], pg[cc][0], sRB[r].m[0], sRB[r].a[0]);
          if (NW > 8) sub_word(pz[cc][1], pg[cc][1], sRB[r].m[1], sRB[r].a[1]);
        }
      }
      for (unsigned long long T = 0; T < tiles; ++T) {
        if (T) {
          const int tz = __ffsll((long long)T) - 1;
          const int r = 15 + tz;
          const bool enter = ((T ^ (T >> 1)) >> tz) & 1ull;
          const uint32_t* rm = sRow + (r * 3) * NW;
          const uint32_t* rs = sRow + (r * 3 + (enter ? 2 : 1)) * NW;
          const uint32_t bm0 = sRB[r].m[0], bs0 = enter ? sRB[r].a[0] : sRB[r].s[0];
          const uint32_t bm1 = sRB[r].m[1], bs1 = enter ? sRB[r].a[1] : sRB[r].s[1];
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const uint32_t m = rm[w], sw = rs[w];
            sub_word(z[0][w], g[0][w], m, sw);
            sub_word(z[1][w], g[1][w], m, sw);
          }
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            sub_word(pz[cc][0], pg[cc][0], bm0, bs0);
            if (NW > 8) sub_word(pz[cc][1], pg[cc][1], bm1, bs1);
          }
        }
        mbar_wait_sleep(smem_u32(&S->empty[bs]), bph ^ 1u);
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int jj = j0 + 64 * cc;
          uint8_t* rowp = sB + bs * MT + (jj >> 3) * SBO + (jj & 7) * 16;
          // row words: r bytes of columns 4w..4w+3 at word w, s bytes at word NW + w,
          // then the constant tail (rewritten only in the last partial 16-byte chunk)
          uint32_t wd[2 * NW + 3];
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            // (z, g) = (1, 1) is an alternate zero (tp_device.cuh): g counts only where ~z
            wd[w] = (z[cc][w] & 0x38383838u) | (g[cc][w] & ~z[cc][w]);
            wd[NW + w] = ~z[cc][w] & (0x38383838u | g[cc][w]);
          }
#pragma unroll
          for (int qq = 0; qq < 3; ++qq) {
            uint32_t word = 0;
#pragma unroll
            for (int bb = 0; bb < 4; ++bb)
              if (4 * qq + bb < nslots) word |= 0x38u << (8 * bb);
            wd[2 * NW + qq] = word;
          }
#pragma unroll
          for (int ch = 0; ch < (2 * NW + 3) / 4; ++ch)
            *(uint4*)(rowp + ch * 128) = make_uint4(wd[4 * ch], wd[4 * ch + 1], wd[4 * ch + 2], wd[4 * ch + 3]);
          sPl[(T & 7) * 128 + jj] = make_uint4(pz[cc][0], pz[cc][1], pg[cc][0], pg[cc][1]);
        }
        proxy_fence();
        mbar_arrive(smem_u32(&S->full[bs]));
        if (++bs == kTcStages) { bs = 0; bph ^= 1u; }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // Group grp = e / 4 owns TMEM slot grp, i.e. the sub-tiles (T, mt) with
    // mt = grp & 1 and T = grp >> 1 (mod 2); warp e reads lane quarter
    // q = warp % 4 (hardware rule) of all 128 columns: 64 packed f16 pairs.
    const int e = warp - kTcEpiWarp0;
    const int grp = e >> 2, q = warp & 3, mt = grp & 1;
    const unsigned long long t_par = (unsigned long long)(grp >> 1);
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t a = mt * 128 + q * 32 + lane;  // this thread's A vector (rows 0..7)
    const uint32_t cm0 = n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
    const uint32_t cm1 = n <= 32 ? 0u : (n >= 64 ? 0xffffffffu : ((1u << (n - 32)) - 1u));
    const uint32_t col = tbase + lane_off + grp * 128u;
    uint32_t sph = 0;
    for (unsigned long long item = blockIdx.x; item < p.items; item += gridDim.x) {
      const unsigned long long b = item / p.chunks, c = item % p.chunks;
      const unsigned long long cg = p.c0 + c;
      const unsigned long long P = (cg ^ (cg >> 1)) << (15 + t);
      const RowRec* R = p.rows + b * 64;
      uint32_t plus = 0, minus = 0;
      uint32_t zA0 = cm0, zA1 = cm1, gA0 = 0, gA1 = 0;
      {
        RowRec rr[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) rr[r] = R[r];
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if ((a >> r) & 1u) {
            sub_word(zA0, gA0, rr[r].m[0], rr[r].a[0]);
            sub_word(zA1, gA1, rr[r].m[1], rr[r].a[1]);
          }
      }
      const uint32_t spar0 = (__popc(a) + __popcll(P)) & 1u;
      for (unsigned long long T = t_par; T < tiles; T += 2) {
        mbar_wait_sleep(smem_u32(&S->tfull[grp]), sph);
        tc_fence_after();
        uint32_t v[64];
        TP_TLD32(col, v, 0);
        TP_TLD32(col + 64, v, 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // the accumulators are in registers: release the slot before the test
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&S->tempty[grp]));
        sph ^= 1u;
        // quad g = registers 4g..4g+3 = columns 8g..8g+7: products over quads
        // 0..7 (HMUL2, FMA pipe), minima over quads 8..15 (HMNMX2, ALU pipe);
        // a quad holds a zero iff its value is +-0 or NaN.
        uint32_t qv[16];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          qv[g] = hmul2(hmul2(v[4 * g], v[4 * g + 1]), hmul2(v[4 * g + 2], v[4 * g + 3]));
          qv[8 + g] = hmin2(hmin2(v[32 + 4 * g], v[33 + 4 * g]), hmin2(v[34 + 4 * g], v[35 + 4 * g]));
        }
        const uint32_t tp_ = hmul2(hmul2(hmul2(qv[0], qv[1]), hmul2(qv[2], qv[3])),
                                   hmul2(hmul2(qv[4], qv[5]), hmul2(qv[6], qv[7])));
        const uint32_t tm_ = hmin2(hmin2(hmin2(qv[8], qv[9]), hmin2(qv[10], qv[11])),
                                   hmin2(hmin2(qv[12], qv[13]), hmin2(qv[14], qv[15])));
        if (pair_hit(tp_) || pair_hit(tm_)) {
          // rare, per lane: pick each hit quad's registers (compile-time
          // selects, no local memory) and evaluate its zeros exactly
          uint32_t qm = 0;
#pragma unroll
          for (int g = 0; g < 16; ++g)
            if (pair_hit(qv[g])) qm |= 1u << g;
          const uint32_t spar = spar0 ^ (__popcll(T ^ (T >> 1)) & 1u);
          const uint4* pl = sPl + (T & 7) * 128;
          while (qm) {
            const int g = __ffs(qm) - 1;
            qm &= qm - 1;
            uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
            for (int gg = 0; gg < 16; ++gg)
#pragma unroll
              for (int r = 0; r < 4; ++r) w[r] = (gg == g) ? v[4 * gg + r] : w[r];
            tc_quad(w, 8 * g, pl, zA0, gA0, zA1, gA1, cm0, cm1, spar, plus, minus, p.err);
          }
        }
      }
      // per-item counts -> pm[b]
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        plus += __shfl_xor_sync(FULL, plus, o);
        minus += __shfl_xor_sync(FULL, minus, o);
      }
      if (lane == 0 && (plus | minus)) {
        if (plus) atomicAdd(&p.pm[2 * b], (unsigned long long)plus);
        if (minus) atomicAdd(&p.pm[2 * b + 1], (unsigned long long)minus);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kTcMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
}

size_t tc_smem_bytes(int n, int ks) {
  const int NW = (n + 3) / 4;
  const size_t KP = 32 * (size_t)ks;
  size_t b = 1024 + (4 + kTcStages) * 128 * KP + 64 * 3 * NW * 4 + 8 * 128 * 16 + 64 * sizeof(RowRec) + sizeof(TcSmem) + 64;
  if (b < 120 * 1024) b = 120 * 1024;  // one CTA per SM: it owns all 512 TMEM columns
  return b;
}

// K layout: r bytes at [0, n), padding to R = 4 ceil(n/4), s bytes at
// [R, R + n), the offset slots at [2R, 2R + ceil(n/16)).
void tc_layout(int n, int* R, int* ks) {
  *R = 4 * ((n + 3) / 4);
  const int need = 2 * *R + (n + 15) / 16;
  *ks = (need + 31) / 32;
}

template <int NW>
static cudaError_t launch_tc_nw(int grid, const TcParams& p, cudaStream_t st) {
  const size_t smem = tc_smem_bytes(p.n, p.ks);
  // per launch: the attribute belongs to the current device's context
  cudaError_t e = cudaFuncSetAttribute(k_walk_tc<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_walk_tc<NW><<<grid, kTcThreads, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_walk_tc(int grid, const TcParams& p, cudaStream_t st) {
  switch ((p.n + 3) / 4) {
    case 4: return launch_tc_nw<4>(grid, p, st);
    case 5: return launch_tc_nw<5>(grid, p, st);
    case 6: return launch_tc_nw<6>(grid, p, st);
    case 7: return launch_tc_nw<7>(grid, p, st);
    case 8: return launch_tc_nw<8>(grid, p, st);
    case 9: return launch_tc_nw<9>(grid, p, st);
    case 10: return launch_tc_nw<10>(grid, p, st);
    case 11: return launch_tc_nw<11>(grid, p, st);
    case 12: return launch_tc_nw<12>(grid, p, st);
    case 13: return launch_tc_nw<13>(grid, p, st);
    case 14: return launch_tc_nw<14>(grid, p, st);
    case 15: return launch_tc_nw<15>(grid, p, st);
    case 16: return launch_tc_nw<16>(grid, p, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tp
