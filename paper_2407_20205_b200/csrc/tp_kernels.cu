// tp_kernels.cu -- sm_100a kernels of the Gray-code Ryser permanent mod 3.
//
// Work decomposition (north_star): subset S of the rows is written
// S = (gray(a) << 5) | l, where lane l of a warp owns the low 5 subset bits
// and the warp walks the "high step" a in Gray order.  All 32 lanes apply the
// same row at every step (no divergence); only the starting vectors differ.
// Reference steps [32a, 32b) are exactly the subsets
// {(gray(h) << 5) | l : h in [a, b), l in [0, 32)}, so partial sums over
// 32-aligned step ranges are bit-equal to chunk_sum (src/_kernels.py:90-128);
// lane l at high step a is reference step i = 32a + (ginv5(l) ^ 31*(a&1)),
// which the generic kernel uses to mask unaligned [lo, hi).
//
// Kernels (this file): the generic walk, packing, sampling, finalisation,
// self-test and the ALU probe, plus the dispatch over the fast walks:
//   k_walk_lane  (tp_walk_lane.cu)  3 LOP3 per subset, n <= 32
//   k_walk_wide  (tp_walk_wide.cu)  3 LOP3 per subset, primary filter, n > 32
//   k_walk_pair  (tp_walk_pair.cu)  2 LOP3 per subset (meet in the middle)
//   k_walk_generic<NW>  runtime-row walk with per-lane step masking: small n,
//                       unaligned range heads/tails.
//   k_pack              uint8 [B][n][n] classes -> RowRec [B][64].
//   k_sample            splitmix64 per-trial sampler -> RowRec (+ entries).
//   k_finalize          (plus, minus) -> class {0,1,2}, raw partial, histogram.
//   k_selftest_ops      packed primitives on caller words.
#include "tp_walk_common.cuh"

namespace tp {

// ---------------------------------------------------------------------------
// Generic walk: pieces of up to glen high steps (32 reference steps each) of
// two regions, with lanes masked to the reference step range [lo, hi).
// Covers small n, and the unaligned heads and tails of step ranges.
// ---------------------------------------------------------------------------
template <int NW>
__global__ void __launch_bounds__(kWalkThreads) k_walk_generic(GenericParams p) {
  __shared__ RowRec srow[kWalkThreads / 32][64];
  const uint32_t lane = threadIdx.x & 31u;
  RowRec* R = srow[threadIdx.x >> 5];
  const uint32_t lanepar = __popc(lane) & 1u;
  const uint32_t jl = ginv5(lane);
  const unsigned long long per_mat = p.pieces[0] + p.pieces[1];
  const unsigned long long warps = (unsigned long long)gridDim.x * (kWalkThreads / 32);
  for (unsigned long long item = blockIdx.x * (kWalkThreads / 32) + (threadIdx.x >> 5); item < p.items;
       item += warps) {
    const unsigned long long b = item / per_mat;
    unsigned long long q = item - b * per_mat;
    const int r = q < p.pieces[0] ? 0 : 1;
    if (r) q -= p.pieces[0];
    const unsigned long long a0 = (r ? p.reg_a0[1] : p.reg_a0[0]) + q * p.glen;
    const unsigned long long rend = r ? p.reg_a1[1] : p.reg_a1[0];
    const unsigned long long a1 = (a0 + p.glen < rend) ? a0 + p.glen : rend;
    __syncwarp();
    load_rows(R, p.rows + b * 64, lane, p.n);
    __syncwarp();
    uint32_t z[2], g[2];
    seed_state<NW>(R, p.n, a0, lane, p.z0_init, p.z1_init, z, g);
    uint32_t ev = 0, odd = 0;
    for (unsigned long long a = a0; a < a1; ++a) {
      if (a != a0) runtime_step<NW>(R, a, z, g);
      const unsigned long long i = (a << 5) + (jl ^ ((a & 1ull) ? 31u : 0u));
      if ((!p.masked || (i >= p.lo && i < p.hi)) && is_full<NW>(z)) {
        ev += 1;
        odd += (sign_parity<NW>(g) ^ (uint32_t)(a & 1ull) ^ lanepar) & 1u;
      }
    }
    warp_flush(p.pm + 2 * b, ev - odd, odd, lane);
  }
}

// ---------------------------------------------------------------------------
// Packing: one warp per matrix; column k of row t -> plane bit n-1-k
// (src/core_f3.py:14-16), split into two 32-bit words.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void store_row(RowRec* dst, unsigned long long mag, unsigned long long sgn) {
  RowRec r;
  r.m[0] = (uint32_t)mag;
  r.m[1] = (uint32_t)(mag >> 32);
  r.s[0] = (uint32_t)sgn;
  r.s[1] = (uint32_t)(sgn >> 32);
  r.a[0] = r.m[0] ^ r.s[0];
  r.a[1] = r.m[1] ^ r.s[1];
  r.pad[0] = 0;
  r.pad[1] = 0;
  *dst = r;
}

// One warp per matrix, one lane per row (rows lane and lane + 32): each lane
// reads its row's n bytes (independent loads, so a single matrix -- C1 -- is
// packed in one load latency rather than 64 dependent ones) and writes its
// RowRec; rows >= n are zero.
__global__ void k_pack(const uint8_t* __restrict__ entries, long long B, int n, RowRec* __restrict__ rows) {
  const uint32_t lane = threadIdx.x & 31u;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long b = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); b < B; b += warps) {
    const uint8_t* E = entries + b * (long long)n * n;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = (int)lane + 32 * h;
      unsigned long long mag = 0, sgn = 0;
      if (t < n) {
        const uint8_t* row = E + (long long)t * n;
        for (int k = 0; k < n; ++k) {
          const uint32_t v = (uint32_t)__ldg(row + k) % 3u;
          const unsigned long long bit = 1ull << (n - 1 - k);  // column k -> bit n-1-k (src/core_f3.py:14-16)
          if (v) mag |= bit;
          if (v == 2u) sgn |= bit;
        }
      }
      store_row(rows + b * 64 + t, mag, sgn);
    }
  }
}

// ---------------------------------------------------------------------------
// Device sampler: the reference's per-trial splitmix64 stream
// (src/rng.py:25-71, src/_kernels.py:212-242), one thread per trial.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

__global__ void k_sample(int n, long long t0, long long count, unsigned long long seed, RowRec* __restrict__ rows,
                         uint8_t* __restrict__ entries_out) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= count) return;
  const unsigned long long trial = (unsigned long long)(t0 + k);
  const unsigned long long golden = 0x9E3779B97F4A7C15ull;
  unsigned long long state = mix64(mix64(seed) ^ ((trial + 1ull) * golden));
  unsigned long long word = 0;
  int pairs = 0;
  RowRec* dst = rows ? rows + k * 64 : nullptr;
  for (int i = 0; i < n; ++i) {
    unsigned long long mag = 0, sgn = 0;
    for (int col = 0; col < n; ++col) {
      unsigned long long v;
      for (;;) {
        if (pairs == 0) {
          state += golden;
          word = mix64(state);
          pairs = 32;
        }
        v = word & 3ull;
        word >>= 2;
        pairs -= 1;
        if (v != 3ull) break;
      }
      if (v != 0) {
        const unsigned long long bit = 1ull << (n - 1 - col);
        mag |= bit;
        if (v == 2) sgn |= bit;
      }
      if (entries_out) entries_out[k * (long long)n * n + i * n + col] = (uint8_t)v;  // class {0,1,2}
    }
    if (dst) store_row(dst + i, mag, sgn);
  }
  if (dst)
    for (int i = n; i < 64; ++i) store_row(dst + i, 0, 0);
}

// ---------------------------------------------------------------------------
// Finalisation: perm mod 3 = cmod3((-1)^n (plus - minus)) (src/permanent.py:116-119),
// computed from plus and minus separately so it is exact for every n <= 64.
// ---------------------------------------------------------------------------
__global__ void k_finalize(const unsigned long long* __restrict__ pm, long long B, int n, int8_t* __restrict__ cls,
                           long long* __restrict__ partial, long long* __restrict__ hist) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int r = -1;
  if (b < B) {
    const unsigned long long P = pm[2 * b], M = pm[2 * b + 1];
    int d = (int)(P % 3ull) - (int)(M % 3ull);
    if (d < 0) d += 3;
    if ((n & 1) && d) d = 3 - d;
    r = d;
    if (cls) cls[b] = (int8_t)r;
    if (partial) partial[b] = (long long)(P - M);
  }
  if (hist) {
    const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const uint32_t cnt = __popc(__ballot_sync(FULL, r == c));
      if (lane == 0 && cnt) atomicAdd(reinterpret_cast<unsigned long long*>(hist + c), (unsigned long long)cnt);
    }
  }
}

__global__ void k_selftest_ops(const uint32_t* __restrict__ in, int count, int op, uint32_t* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  uint32_t mag = in[4 * k], sgn = in[4 * k + 1], m2 = in[4 * k + 2], s2 = in[4 * k + 3];
  if (op == 0) {
    add_ref_word(mag, sgn, m2, s2);
  } else {
    uint32_t z = ~mag, g = sgn;
    sub_word(z, g, m2, op == 1 ? s2 : (m2 ^ s2));
    mag = ~z;
    sgn = g;
  }
  out[2 * k] = mag;
  out[2 * k + 1] = sgn;
}

// ---------------------------------------------------------------------------
// ALU roofline probe: 8 independent lop3 chains per thread, register
// resident; measures the LOP3 issue rate the walk is bounded by.
// ---------------------------------------------------------------------------
constexpr int kPeakInner = 16;
__global__ void __launch_bounds__(256) k_alu_peak(uint32_t* out, int iters, uint32_t b, uint32_t c) {
  uint32_t a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 8u + (uint32_t)k + blockIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < kPeakInner; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) TP_LOP3(a[k], a[k], b, c, 0x96);
  }
  uint32_t r = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) r ^= a[k];
  if (r == 0x12345678u) out[blockIdx.x] = r;  // keep the chains live
}

cudaError_t run_alu_peak(int sm_count, uint32_t* scratch, cudaStream_t st, double* ops_per_s, double* ms) {
  const int grid = sm_count * 8, iters = 2048;
  cudaEvent_t e0, e1;
  cudaError_t e;
  if ((e = cudaEventCreate(&e0)) != cudaSuccess) return e;
  if ((e = cudaEventCreate(&e1)) != cudaSuccess) return e;
  k_alu_peak<<<grid, 256, 0, st>>>(scratch, 64, 0x5a5a5a5au, 0x3c3c3c3cu);  // warm-up
  cudaEventRecord(e0, st);
  k_alu_peak<<<grid, 256, 0, st>>>(scratch, iters, 0x5a5a5a5au, 0x3c3c3c3cu);
  cudaEventRecord(e1, st);
  if ((e = cudaEventSynchronize(e1)) != cudaSuccess) return e;
  float t = 0;
  cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double ops = (double)grid * 256 * iters * kPeakInner * 8;
  *ops_per_s = ops / (t * 1e-3);
  *ms = t;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Host-side launch wrappers (called by the runtime in tp_runtime.cu).
// ---------------------------------------------------------------------------
cudaError_t launch_lane(int V, int grid, const FastParams& p, cudaStream_t st);
const void* lane_symbol(int V);
cudaError_t launch_wide(int KB, int V, int grid, const FastParams& p, cudaStream_t st);
const void* wide_symbol(int KB, int V);
cudaError_t launch_pair(int KB, int V, bool wide, int grid, const FastParams& p, cudaStream_t st);
const void* pair_symbol(int KB, int V, bool wide);
cudaError_t launch_packed(int V, int grid, const FastParams& p, cudaStream_t st);
const void* packed_symbol(int V);

const void* walk_fast_symbol(int v) {
  if (fast_is_lane(v)) return lane_symbol(fast_v(v));
  if (fast_is_pair(v)) return pair_symbol(fast_kb(v), fast_v(v), fast_pair_wide(v));
  if (fast_is_packed(v)) return packed_symbol(packed_which(v));
  return wide_symbol(fast_kb(v), fast_v(v));
}

const void* walk_generic_symbol(int nw) {
  return nw == 1 ? reinterpret_cast<const void*>(&k_walk_generic<1>)
                 : reinterpret_cast<const void*>(&k_walk_generic<2>);
}

cudaError_t launch_walk_fast(int v, int grid, const FastParams& p, cudaStream_t st) {
  if (fast_is_lane(v)) return launch_lane(fast_v(v), grid, p, st);
  if (fast_is_pair(v)) return launch_pair(fast_kb(v), fast_v(v), fast_pair_wide(v), grid, p, st);
  if (fast_is_packed(v)) return launch_packed(packed_which(v), grid, p, st);
  return launch_wide(fast_kb(v), fast_v(v), grid, p, st);
}

cudaError_t launch_walk_generic(int nw, int grid, const GenericParams& p, cudaStream_t st) {
  if (nw == 1) k_walk_generic<1><<<grid, kWalkThreads, 0, st>>>(p);
  else k_walk_generic<2><<<grid, kWalkThreads, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_pack(const uint8_t* entries, long long B, int n, RowRec* rows, int grid, cudaStream_t st) {
  k_pack<<<grid, 256, 0, st>>>(entries, B, n, rows);
  return cudaGetLastError();
}

cudaError_t launch_sample(int n, long long t0, long long count, unsigned long long seed, RowRec* rows,
                          uint8_t* entries_out, cudaStream_t st) {
  const int threads = 128;
  const long long grid = (count + threads - 1) / threads;
  k_sample<<<(unsigned)grid, threads, 0, st>>>(n, t0, count, seed, rows, entries_out);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const unsigned long long* pm, long long B, int n, int8_t* cls, long long* partial,
                            long long* hist, cudaStream_t st) {
  const int threads = 256;
  const long long grid = (B + threads - 1) / threads;
  k_finalize<<<(unsigned)grid, threads, 0, st>>>(pm, B, n, cls, partial, hist);
  return cudaGetLastError();
}

cudaError_t launch_selftest(const uint32_t* in, int count, int op, uint32_t* out, cudaStream_t st) {
  k_selftest_ops<<<(count + 127) / 128, 128, 0, st>>>(in, count, op, out);
  return cudaGetLastError();
}

}  // namespace tp
