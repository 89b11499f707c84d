// tp_small.cu -- one thread per matrix for small n (1 <= n <= kSmallMaxN).
//
// For small n a matrix has too few subsets to feed the lane walk (a warp per
// 32 * 2^V steps), and the per-matrix setup of the warp kernels (row table in
// HBM, 2 KB shared-memory copy, seeding) dominates.  Here every thread owns a
// whole matrix: it samples it from the reference's per-trial splitmix64
// stream (src/_kernels.py:212-242, the Monte Carlo path) or packs it from
// caller entries, keeps its rows in shared memory (row-major over threads, so
// row loads are conflict-free), and walks all 2^n - 1 Gray steps itself
// (src/_kernels.py:131-161): rows 0..3 flip at compile-time positions from
// registers, 16 steps per unrolled block, rows >= 4 come from shared memory
// at the block boundary.  Events (full magnitude) are frequent at small n
// ((2/3)^n) and are folded in exactly on every step.
#include <cstdint>

#include "tp_device.cuh"
#include "tp_kernels.cuh"

namespace tp {

struct SmallParams {
  int n;
  long long B;                   // matrices
  const uint8_t* entries;        // [B][n][n] classes, or nullptr: sample
  long long t0;                  // first trial (sampling)
  unsigned long long seed;
  int8_t* cls;                   // [B] classes {0,1,2} (may be null)
  long long* partial;            // [B] raw partial sums (may be null)
  unsigned long long* pm;        // [B][2] (plus, minus), added (may be null)
  long long* hist;               // [3] accumulated (may be null)
};

__device__ __forceinline__ unsigned long long mix64s(unsigned long long z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

// TP_SMALL_SAMPLER 1: a sampled 64-bit word is handled as a whole -- its 32
// two-bit slices are split into a low-bit and a high-bit mask, the slices
// of value 3 are rejected by a branch-free compress of both masks (the
// parallel-suffix method: the moves depend only on the mask and serve both),
// and the accepted trits are appended to two bit streams (nonzero, minus)
// from which a row takes n bits at a time (earlier trit = higher column bit:
// one BREV).  The same trits in the same order as the reference's slice
// loop (src/_kernels.py:212-242; rng.py:49-65), at ~6 instead of ~25
// instructions per trit.  0: the slice loop.
#ifndef TP_SMALL_SAMPLER
#define TP_SMALL_SAMPLER 1
#endif

// bits 0, 2, 4, .. of x gathered into the low 16 bits
__device__ __forceinline__ uint32_t even_bits16(uint32_t x) {
  x &= 0x55555555u;
  x = (x | (x >> 1)) & 0x33333333u;
  x = (x | (x >> 2)) & 0x0F0F0F0Fu;
  x = (x | (x >> 4)) & 0x00FF00FFu;
  x = (x | (x >> 8)) & 0x0000FFFFu;
  return x;
}

// a and b compressed by mask m (the bits of a, b under the 1-bits of m moved
// to the low end, order kept): Hacker's Delight 7-4, the move masks shared
__device__ __forceinline__ void compress2(uint32_t m, uint32_t& a, uint32_t& b) {
  a &= m;
  b &= m;
  uint32_t mk = ~m << 1;
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    uint32_t mp = mk ^ (mk << 1);
    mp ^= mp << 2;
    mp ^= mp << 4;
    mp ^= mp << 8;
    mp ^= mp << 16;
    const uint32_t mv = mp & m;
    m = (m ^ mv) | (mv >> (1 << i));
    uint32_t t = a & mv;
    a = (a ^ t) | (t >> (1 << i));
    t = b & mv;
    b = (b ^ t) | (t >> (1 << i));
    mk &= ~mp;
  }
}

// (Events are rare from n = 12, (2/3)^n < 1 % of the steps, but putting their
// accounting behind a warp vote instead of predicating it into every step
// measured 22 % slower at n = 12..15: the vote and branch per step cost
// more than the ~4 predicated instructions and break the unrolled schedule.)
__global__ void __launch_bounds__(kSmallThreads) k_small(SmallParams p) {
  __shared__ uint32_t Sm[kSmallMaxN][kSmallThreads], Ss[kSmallMaxN][kSmallThreads], Sa[kSmallMaxN][kSmallThreads];
  const int tid = threadIdx.x;
  const long long b = blockIdx.x * (long long)kSmallThreads + tid;
  const bool active = b < p.B;
  const int n = p.n;

  // ---- rows: column k of row t -> bit n-1-k (src/core_f3.py:14-16)
  if (active) {
    if (p.entries) {
      const uint8_t* E = p.entries + b * n * n;
      for (int t = 0; t < n; ++t) {
        uint32_t m = 0, s = 0;
        for (int k = 0; k < n; ++k) {
          const uint32_t v = (uint32_t)E[t * n + k] % 3u;
          const uint32_t bit = 1u << (n - 1 - k);
          if (v) m |= bit;
          if (v == 2) s |= bit;
        }
        Sm[t][tid] = m;
        Ss[t][tid] = s;
        Sa[t][tid] = m ^ s;
      }
    } else {
      const unsigned long long golden = 0x9E3779B97F4A7C15ull;
      unsigned long long state = mix64s(mix64s(p.seed) ^ ((unsigned long long)(p.t0 + b + 1) * golden));
#if TP_SMALL_SAMPLER
      // bit streams of the accepted trits, earliest at bit 0: nonzero, minus
      unsigned long long sm = 0, ss = 0;
      int have = 0;
      const uint32_t rowmask = (1u << n) - 1u;  // n <= kSmallMaxN < 32
      for (int t = 0; t < n; ++t) {
        while (have < n) {  // < 15 + 32 bits in the streams
          state += golden;
          const unsigned long long word = mix64s(state);
          const uint32_t wl = (uint32_t)word, wh = (uint32_t)(word >> 32);
          uint32_t lo = even_bits16(wl) | (even_bits16(wh) << 16);            // bit j: low bit of slice j
          uint32_t hi = even_bits16(wl >> 1) | (even_bits16(wh >> 1) << 16);  // high bit of slice j
          const uint32_t acc = ~(lo & hi);                                    // slices of value 0, 1, 2
          uint32_t mg = lo | hi, sg = hi;                                     // nonzero; value 2 = -1
          compress2(acc, mg, sg);
          sm |= (unsigned long long)mg << have;
          ss |= (unsigned long long)sg << have;
          have += __popc(acc);
        }
        // the row's n trits: trit k -> column k -> bit n-1-k
        const uint32_t m = __brev((uint32_t)sm & rowmask) >> (32 - n);
        const uint32_t s = __brev((uint32_t)ss & rowmask) >> (32 - n);
        sm >>= n;
        ss >>= n;
        have -= n;
        Sm[t][tid] = m;
        Ss[t][tid] = s;
        Sa[t][tid] = m ^ s;
      }
#else
      unsigned long long word = 0;
      int pairs = 0;
      for (int t = 0; t < n; ++t) {
        uint32_t m = 0, s = 0;
        for (int k = 0; k < n; ++k) {
          unsigned long long v;
          for (;;) {
            if (pairs == 0) {
              state += golden;
              word = mix64s(state);
              pairs = 32;
            }
            v = word & 3ull;
            word >>= 2;
            pairs -= 1;
            if (v != 3ull) break;
          }
          const uint32_t bit = 1u << (n - 1 - k);
          if (v) m |= bit;
          if (v == 2) s |= bit;
        }
        Sm[t][tid] = m;
        Ss[t][tid] = s;
        Sa[t][tid] = m ^ s;
      }
#endif
    }
  } else {
    for (int t = 0; t < n; ++t) Sm[t][tid] = Ss[t][tid] = Sa[t][tid] = 0;
  }

  // ---- walk all 2^n - 1 Gray steps of this thread's matrix
  uint32_t z = (n >= 32) ? 0xffffffffu : ((1u << n) - 1u), g = 0;
  uint32_t ev = 0, odd = 0;
  auto event = [&](uint32_t i_parity) {
    if (z == 0) {
      ev += 1;
      odd += (__popc(g) ^ i_parity) & 1u;
    }
  };
  const uint32_t steps = 1u << n;  // steps 1 .. 2^n - 1
  if (n <= 4) {
    for (uint32_t i = 1; i < steps; ++i) {
      const int t = __ffs(i) - 1;
      const bool leave = (i >> (t + 1)) & 1u;
      sub_word(z, g, Sm[t][tid], leave ? Ss[t][tid] : Sa[t][tid]);
      event(i & 1u);
    }
  } else {
    uint32_t RM[4], RS[4], RA[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      RM[r] = Sm[r][tid];
      RS[r] = Ss[r][tid];
      RA[r] = Sa[r][tid];
    }
    for (uint32_t base = 0; base < steps; base += 16) {
      if (base) {  // block boundary step: row 4 + tz(base/16)
        const int t = __ffs(base) - 1;
        const bool leave = (base >> (t + 1)) & 1u;
        sub_word(z, g, Sm[t][tid], leave ? Ss[t][tid] : Sa[t][tid]);
        event(0u);
      }
      // row 3 flips at j = 8; it leaves iff bit 4 of base + 8 (= of base) is set
      const uint32_t X3 = ((base >> 4) & 1u) ? RS[3] : RA[3];
#pragma unroll
      for (int j = 1; j < 16; ++j) {
        const int t = ctz_c(j);
        const bool leave = (t < 3) ? (((j >> (t + 1)) & 1) != 0) : false;
        sub_word(z, g, RM[t], (t == 3) ? X3 : (leave ? RS[t] : RA[t]));
        event((uint32_t)(j & 1));
      }
    }
  }

  // ---- finalise: perm mod 3 = cmod3((-1)^n (plus - minus)) (src/permanent.py:116-119)
  const uint32_t plus = ev - odd, minus = odd;
  int r = -1;
  if (active) {
    int d = (int)(plus % 3u) - (int)(minus % 3u);
    if (d < 0) d += 3;
    if ((n & 1) && d) d = 3 - d;
    r = d;
    if (p.cls) p.cls[b] = (int8_t)r;
    if (p.partial) p.partial[b] = (long long)plus - (long long)minus;
    if (p.pm) {
      atomicAdd(p.pm + 2 * b, (unsigned long long)plus);
      atomicAdd(p.pm + 2 * b + 1, (unsigned long long)minus);
    }
  }
  if (p.hist) {
    __shared__ unsigned int h[3];
    if (tid < 3) h[tid] = 0;
    __syncthreads();
    const uint32_t lane = tid & 31u;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const uint32_t cnt = __popc(__ballot_sync(FULL, r == c));
      if (lane == 0 && cnt) atomicAdd(&h[c], cnt);
    }
    __syncthreads();
    if (tid < 3 && h[tid]) atomicAdd(reinterpret_cast<unsigned long long*>(p.hist + tid), (unsigned long long)h[tid]);
  }
}

cudaError_t launch_small(int n, long long B, const uint8_t* entries, long long t0, unsigned long long seed,
                         int8_t* cls, long long* partial, unsigned long long* pm, long long* hist, cudaStream_t st) {
  if (n < 1 || n > kSmallMaxN) return cudaErrorInvalidValue;
  SmallParams p{n, B, entries, t0, seed, cls, partial, pm, hist};
  const long long grid = (B + kSmallThreads - 1) / kSmallThreads;
  if (grid > 0) k_small<<<(unsigned)grid, kSmallThreads, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace tp
