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
// Kernels
//   k_walk_fast<NW,V>   persistent, dynamic work queue over (matrix, chunk)
//                       items; the walk is unrolled in 2^V-step superblocks
//                       whose V low rows live in registers; 3*NW LOP3 per
//                       subset (ALU pipe) + predicated IMADs (FMA pipe).
//   k_walk_generic<NW>  runtime-row walk with per-lane step masking: small n,
//                       unaligned range heads/tails, and the fast kernel's
//                       exact per-block replay logic in scalar form.
//   k_pack              uint8 [B][n][n] classes -> RowRec [B][64].
//   k_sample            splitmix64 per-trial sampler -> RowRec (+ entries).
//   k_finalize          (plus, minus) -> class {0,1,2}, raw partial, histogram.
//   k_selftest_ops      packed primitives on caller words.
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
__device__ __forceinline__ unsigned long long next_item(unsigned long long* queue, uint32_t lane) {
  unsigned long long item = 0;
  if (lane == 0) item = atomicAdd(queue, 1ull);
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
// Lane walk, n <= 32: one subset per lane, one 32-bit word per plane.
// Superblocks of 2^V high steps: the first 2^V - 1 steps flip rows 5..5+V-1
// at compile-time positions (register operands, fully unrolled); the step
// into the next superblock flips row 5+V+tz(kb) (shared memory, uniform).
// Events (full magnitude, z == 0) are recorded per step parity with two
// predicated IMADs (count, sign word); a lane with two events of one parity
// in a superblock forces an exact replay of that superblock.
// ---------------------------------------------------------------------------
template <int V, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) k_walk_lane(FastParams p) {
  __shared__ RowRec Rs[WARPS][64];
  const uint32_t lane = threadIdx.x & 31u;
  RowRec* R = Rs[threadIdx.x >> 5];
  const uint32_t lanepar = __popc(lane) & 1u;
  const uint32_t one = p.one;
  const unsigned long long t_start = p.trace ? clock64() : 0;
  unsigned long long n_items = 0;

  for (;;) {
    const unsigned long long item = next_item(p.queue, lane);
    if (item >= p.items) break;
    ++n_items;
    const unsigned long long b = item / p.chunks;
    const unsigned long long A0 = p.F0 + (item - b * p.chunks) * p.L;
    const unsigned long long B0 = A0 >> V;
    __syncwarp();
    load_rows(R, p.rows + b * 64, lane, p.n);
    __syncwarp();

    uint32_t SM[V], SS[V], SA[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      SM[v] = R[5 + v].m[0];
      SS[v] = R[5 + v].s[0];
      SA[v] = R[5 + v].a[0];
    }
    uint32_t z[2], g[2];
    seed_state<1>(R, p.n, A0, lane, p.z0_init, 0u, z, g);

    uint32_t ev = 0, odd = 0;
    uint32_t cnt0 = 0, cnt1 = 0, slot0 = 0, slot1 = 0;
    record_slot(z[0], g[0], cnt0, slot0, one);
    bool dense = false;  // warp-uniform: exact accumulation mode for event-dense inputs
    for (uint32_t kb = 0; kb < p.nblk; ++kb) {
      const uint32_t ze = z[0], ge = g[0];
      // row 5+V-1 flips at j = 2^(V-1); it leaves iff bit 0 of B0+kb (= of kb) is set
      const uint32_t SX = (kb & 1u) ? SS[V - 1] : SA[V - 1];
      if (!dense) {
#pragma unroll
        for (int j = 1; j < (1 << V); ++j) {
          const int t = ctz_c(j);
          const bool leave = (t + 1 < V) ? (((j >> (t + 1)) & 1) != 0) : false;
          const uint32_t sop = (t == V - 1) ? SX : (leave ? SS[t] : SA[t]);
          sub_word(z[0], g[0], SM[t], sop);
          if (j & 1) record_slot(z[0], g[0], cnt1, slot1, one);
          else record_slot(z[0], g[0], cnt0, slot0, one);
        }
        // fold this superblock's events in exactly
        if (__any_sync(FULL, (cnt0 | cnt1) != 0)) {
          uint32_t bev = 0, bodd = 0;
          if (cnt0 == 1) { bev += 1; bodd += (__popc(slot0) ^ lanepar) & 1u; }
          if (cnt1 == 1) { bev += 1; bodd += (__popc(slot1) ^ 1u ^ lanepar) & 1u; }
          if (__any_sync(FULL, cnt0 > 1 || cnt1 > 1)) {
            const unsigned long long r = replay_block<1>(R, ze, 0u, ge, 0u, (B0 + kb) << V, 1 << V, lanepar);
            bev = (uint32_t)r;
            bodd = (uint32_t)(r >> 32);
            dense = true;  // events are dense here: accumulate exactly from now on
          }
          ev += bev;
          odd += bodd;
        }
      } else {
        // Exact block for event-dense matrices (e.g. all-ones rows): every
        // full step is folded in as it happens.  Two halves of 2^(V-1)
        // steps keep the unrolled body small; the middle step flips row
        // 5+V-1 (direction SX), and in half h the step j' = 2^(V-2) flips
        // row 5+V-2, leaving iff h == 1.
        uint32_t bev = 0, bodd = 0;
        if (cnt0 == 1) { bev += 1; bodd += (__popc(slot0) ^ lanepar) & 1u; }  // entry step
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          if (h == 1) {
            sub_word(z[0], g[0], SM[V - 1], SX);
            if (z[0] == 0) { bev += 1; bodd += (__popc(g[0]) ^ lanepar) & 1u; }
          }
          const uint32_t SH = h ? SS[V - 2] : SA[V - 2];
#pragma unroll
          for (int j = 1; j < (1 << (V - 1)); ++j) {
            const int t = ctz_c(j);
            const bool leave = (t + 2 < V) ? (((j >> (t + 1)) & 1) != 0) : false;
            const uint32_t sop = (t == V - 2) ? SH : (leave ? SS[t] : SA[t]);
            sub_word(z[0], g[0], SM[t], sop);
            if (z[0] == 0) { bev += 1; bodd += (__popc(g[0]) ^ (uint32_t)(j & 1) ^ lanepar) & 1u; }
          }
        }
        ev += bev;
        odd += bodd;
        dense = __any_sync(FULL, bev >= 4);
      }
      cnt0 = cnt1 = 0;
      if (kb + 1 < p.nblk) {
        const uint32_t u = kb + 1;
        const int t = __ffs(u) - 1;
        const RowRec& row = R[5 + V + t];
        sub_word(z[0], g[0], row.m[0], entry_leave(u, t, p, B0) ? row.s[0] : row.a[0]);
        record_slot(z[0], g[0], cnt0, slot0, one);
      }
    }
    warp_flush(p.pm + 2 * b, ev - odd, odd, lane);
  }
  trace_end(p, t_start, n_items, blockIdx.x * WARPS + (threadIdx.x >> 5), lane);
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

template <int KB, int V, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) k_walk_wide(FastParams p) {
  constexpr int K = 1 << KB;
  constexpr int FIX = 5 + KB;
  __shared__ RowRec Rs[WARPS][64];
  const uint32_t lane = threadIdx.x & 31u;
  RowRec* R = Rs[threadIdx.x >> 5];
  const uint32_t lanepar = __popc(lane) & 1u;
  const uint32_t one = p.one, zero = p.one - 1u;
  const unsigned long long t_start = p.trace ? clock64() : 0;
  unsigned long long n_items = 0;

  for (;;) {
    const unsigned long long item = next_item(p.queue, lane);
    if (item >= p.items) break;
    ++n_items;
    const unsigned long long b = item / p.chunks;
    const unsigned long long A0 = p.F0 + (item - b * p.chunks) * p.L;
    const unsigned long long B0 = A0 >> V;
    __syncwarp();
    load_rows(R, p.rows + b * 64, lane, p.n);
    __syncwarp();

    uint32_t SM[V], SS[V], SA[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      SM[v] = R[FIX + v].m[0];
      SS[v] = R[FIX + v].s[0];
      SA[v] = R[FIX + v].a[0];
    }
    // seed the K slots in Gray order of k: one primary-row update per slot
    uint32_t z[K], g[K];
    {
      uint32_t zz[2], gg[2];
      wide_subset_state<KB>(R, p.n, A0, lane, p.z0_init, p.z1_init, zz, gg);
      uint32_t zc = zz[0], gc = gg[0];
      static_for<K>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        if constexpr (i > 0) {
          constexpr int t = ctz_c(i);
          constexpr bool leave = ((gray_c(i - 1) >> t) & 1) != 0;
          sub_word(zc, gc, R[5 + t].m[0], leave ? R[5 + t].s[0] : R[5 + t].a[0]);
        }
        z[gray_c(i)] = zc;
        g[gray_c(i)] = gc;
      });
    }

    uint32_t ev = 0, odd = 0;
    uint32_t cnt = 0, rec = 0;
    static_for<K>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      record_hit<(uint32_t)k>(z[k], cnt, rec, one, zero);
    });
    // Dense mode (warp-uniform): after a superblock needed a replay, the
    // secondary words are materialised and every subset is evaluated
    // exactly (both words, per step) until events thin out again.
    uint32_t z1[K], g1[K];
    bool dense = false, have_sec = false;
    for (uint32_t kb = 0; kb < p.nblk; ++kb) {
      const unsigned long long B = B0 + kb;
      if (!dense) {
        const uint32_t SX = (kb & 1u) ? SS[V - 1] : SA[V - 1];
        static_for<(1 << V) - 1>([&](auto jc) {
          constexpr int j = decltype(jc)::value + 1;
          constexpr int t = ctz_c(j);
          constexpr bool leave = (t + 1 < V) ? (((j >> (t + 1)) & 1) != 0) : false;
          const uint32_t sop = (t == V - 1) ? SX : (leave ? SS[t] : SA[t]);
          static_for<K>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            sub_word(z[k], g[k], SM[t], sop);
            record_hit<(uint32_t)((j << KB) | k)>(z[k], cnt, rec, one, zero);
          });
        });
        if (__any_sync(FULL, cnt != 0)) {
          uint32_t bev = 0, bodd = 0;
          if (__any_sync(FULL, cnt > 1)) {
            const unsigned long long r = replay_wide<KB>(R, p.n, B << V, 1 << V, lane, p.z0_init, p.z1_init);
            bev = (uint32_t)r;
            bodd = (uint32_t)(r >> 32);
            dense = true;  // primary hits are dense here: switch to the exact walk
            have_sec = false;
          } else if (cnt == 1) {
            const uint32_t j = rec >> KB, k = rec & (K - 1);
            uint32_t zz[2], gg[2];
            wide_subset_state<KB>(R, p.n, (B << V) + j, (k << 5) | lane, p.z0_init, p.z1_init, zz, gg);
            if ((zz[0] | zz[1]) == 0) {
              bev = 1;
              bodd = (__popc(gg[0]) + __popc(gg[1]) + j + __popc(k) + lanepar) & 1u;
            }
          }
          ev += bev;
          odd += bodd;
        }
      } else {
        if (!have_sec) {
          // secondary words of every slot at this superblock's entry (from scratch)
          static_for<K>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            uint32_t zz[2], gg[2];
            wide_subset_state<KB>(R, p.n, B << V, ((uint32_t)k << 5) | lane, p.z0_init, p.z1_init, zz, gg);
            z1[k] = zz[1];
            g1[k] = gg[1];
          });
          have_sec = true;
        }
        uint32_t bev = 0, bodd = 0;
        static_for<K>([&](auto kc) {  // the entry subset of each slot
          constexpr int k = decltype(kc)::value;
          if ((z[k] | z1[k]) == 0) {
            bev += 1;
            bodd += (__popc(g[k]) + __popc(g1[k]) + (uint32_t)__popc(k) + lanepar) & 1u;
          }
        });
#pragma unroll 1
        for (int j = 1; j < (1 << V); ++j) {
          const int t = __ffs(j) - 1;
          const bool leave = (t + 1 < V) ? (((j >> (t + 1)) & 1) != 0) : ((kb & 1u) != 0);
          const RowRec& row = R[FIX + t];
          const uint32_t m0 = row.m[0], m1 = row.m[1];
          const uint32_t s0 = leave ? row.s[0] : row.a[0], s1 = leave ? row.s[1] : row.a[1];
          static_for<K>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            sub_word(z[k], g[k], m0, s0);
            sub_word(z1[k], g1[k], m1, s1);
            if ((z[k] | z1[k]) == 0) {
              bev += 1;
              bodd += (__popc(g[k]) + __popc(g1[k]) + (uint32_t)j + (uint32_t)__popc(k) + lanepar) & 1u;
            }
          });
        }
        ev += bev;
        odd += bodd;
        dense = __any_sync(FULL, bev >= 4);
      }
      cnt = 0;
      if (kb + 1 < p.nblk) {
        const uint32_t u = kb + 1;
        const int t = __ffs(u) - 1;
        const RowRec& row = R[FIX + V + t];
        const bool leave = entry_leave(u, t, p, B0);
        const uint32_t m = row.m[0], s = leave ? row.s[0] : row.a[0];
        if (dense) {
          const uint32_t m1 = row.m[1], s1 = leave ? row.s[1] : row.a[1];
          static_for<K>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            sub_word(z[k], g[k], m, s);
            if (have_sec) sub_word(z1[k], g1[k], m1, s1);
          });
        } else {
          have_sec = false;
          static_for<K>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            sub_word(z[k], g[k], m, s);
            record_hit<(uint32_t)k>(z[k], cnt, rec, one, zero);
          });
        }
      }
    }
    warp_flush(p.pm + 2 * b, ev - odd, odd, lane);
  }
  trace_end(p, t_start, n_items, blockIdx.x * WARPS + (threadIdx.x >> 5), lane);
}

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
__device__ __forceinline__ uint32_t pair_g2(uint32_t z2, uint32_t u2) {  // g2 = ~(u2 ^ z2)
  uint32_t g;
  TP_LOP3(g, z2, u2, 0u, 0xC3);
  return g;
}

template <int KB, int V, int WARPS, bool WIDE>
__global__ void __launch_bounds__(32 * WARPS) k_walk_pair(FastParams p) {
  constexpr int K = 1 << KB;
  constexpr int FIX = 5 + KB;
  constexpr int SB = 1 << V;
  __shared__ RowRec Rs[WARPS][64];
  // B-side states of the current superblock: (z2, u2) of the primary word and,
  // for n > 32 in dense mode, (z2s, u2s) of the secondary word.
  __shared__ uint4 Hs[WARPS][SB];
  // A-side words per slot and lane: the primary (z1, g1) for n <= 32 (single
  // hits), the secondary word for n > 32 (dense mode).
  __shared__ uint2 As[WARPS][K][32];
  const uint32_t lane = threadIdx.x & 31u;
  RowRec* R = Rs[threadIdx.x >> 5];
  uint4* H = Hs[threadIdx.x >> 5];
  uint2 (*A)[32] = As[threadIdx.x >> 5];
  const uint32_t lanepar = __popc(lane) & 1u;
  const uint32_t one = p.one;
  const uint32_t colmask = p.z0_init;   // real columns of the primary word
  const uint32_t colmask1 = p.z1_init;  // real columns of the secondary word (n > 32)
  const unsigned long long t_start = p.trace ? clock64() : 0;
  unsigned long long n_items = 0;

  for (;;) {
    const unsigned long long item = next_item(p.queue, lane);
    if (item >= p.items) break;
    ++n_items;
    const unsigned long long b = item / p.chunks;
    const unsigned long long A0 = p.F0 + (item - b * p.chunks) * p.L;
    const unsigned long long B0 = A0 >> V;
    __syncwarp();
    load_rows(R, p.rows + b * 64, lane, p.n);
    __syncwarp();

    uint32_t SM[V], SS[V], SA[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      SM[v] = R[FIX + v].m[0];
      SS[v] = R[FIX + v].s[0];
      SA[v] = R[FIX + v].a[0];
    }
    // A side: v1 for S1 = (k << 5) | lane, k in Gray order (one row per slot)
    uint32_t z1[K], g1[K];
    {
      uint32_t zz[2], gg[2];
      wide_subset_state<KB>(R, p.n, 0ull, lane, p.z0_init, p.z1_init, zz, gg);
      uint32_t zc = zz[0], gc = gg[0], zc1 = zz[1], gc1 = gg[1];
      static_for<K>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        if constexpr (i > 0) {
          constexpr int t = ctz_c(i);
          constexpr bool leave = ((gray_c(i - 1) >> t) & 1) != 0;
          sub_word(zc, gc, R[5 + t].m[0], leave ? R[5 + t].s[0] : R[5 + t].a[0]);
          if (WIDE) sub_word(zc1, gc1, R[5 + t].m[1], leave ? R[5 + t].s[1] : R[5 + t].a[1]);
        }
        z1[gray_c(i)] = zc;
        g1[gray_c(i)] = gc;
        A[gray_c(i)][lane] = WIDE ? make_uint2(zc1, gc1) : make_uint2(zc, gc);
      });
    }
    // B side: v2 for S2 = gray(A0) on rows >= h (low bits empty)
    uint32_t z2, u2;
    {
      uint32_t zz[2], gg[2];
      wide_subset_state<KB>(R, p.n, A0, 0u, p.z0_init, p.z1_init, zz, gg);
      z2 = zz[0];
      u2 = pair_u2(zz[0], gg[0]);
    }
    uint32_t ev = 0, odd = 0;
    // Exact evaluation of every pair of the current superblock from the
    // B-side history H: replays (n <= 32) and dense mode (all n).
    auto exact_block = [&](uint32_t& bev, uint32_t& bodd) {
      bev = bodd = 0;
      for (int j = 0; j < SB; ++j) {
        const uint4 h = H[j];
        const uint32_t gh = pair_g2(h.x, h.y);
#pragma unroll
        for (int q = 0; q < K; ++q) {
          uint32_t d, zp;
          TP_LOP3(d, z1[q], g1[q], h.y, 0x06);
          TP_LOP3(zp, d, z1[q], h.x, 0x09);
          if (zp == 0) {
            if (WIDE) {  // primary columns all nonzero: test the secondary word
              const uint2 a2 = A[q][lane];
              uint32_t d1, zp1;
              TP_LOP3(d1, a2.x, a2.y, h.w, 0x06);
              TP_LOP3(zp1, d1, a2.x, h.z, 0x09);
              if (zp1 == 0) {
                bev += 1;
                bodd += (__popc(d ^ gh) + __popc((d1 ^ pair_g2(h.z, h.w)) & colmask1) + (uint32_t)j +
                         (uint32_t)__popc(q) + lanepar) & 1u;
              }
            } else {
              bev += 1;
              bodd += (__popc((d ^ gh) & colmask) + (uint32_t)j + (uint32_t)__popc(q) + lanepar) & 1u;
            }
          }
        }
      }
    };
    bool dense = false;  // warp-uniform: skip the filter pass on event-dense matrices
    for (uint32_t kb = 0; kb < p.nblk; ++kb) {
      const unsigned long long B = B0 + kb;
      const uint32_t SX = (kb & 1u) ? SS[V - 1] : SA[V - 1];
      const uint32_t CX = (kb & 1u) ? SA[V - 1] : SS[V - 1];
      if (dense) {
        // walk the B side only, recording its states, then evaluate exactly
        uint32_t z2s = 0, u2s = 0;
        if (WIDE) {  // secondary B word at the superblock entry, from scratch
          uint32_t zz[2], gg[2];
          wide_subset_state<KB>(R, p.n, B << V, 0u, p.z0_init, p.z1_init, zz, gg);
          z2s = zz[1];
          u2s = pair_u2(zz[1], gg[1]);
        }
        __syncwarp();
        if (lane == 0) H[0] = make_uint4(z2, u2, z2s, u2s);
        static_for<SB - 1>([&](auto jc) {
          constexpr int j = decltype(jc)::value + 1;
          constexpr int t = ctz_c(j);
          constexpr bool leave = (t + 1 < V) ? (((j >> (t + 1)) & 1) != 0) : false;
          const uint32_t sop = (t == V - 1) ? SX : (leave ? SS[t] : SA[t]);
          const uint32_t cop = (t == V - 1) ? CX : (leave ? SA[t] : SS[t]);
          sub_word_u(z2, u2, SM[t], sop, cop);
          if (WIDE) {
            const RowRec& row = R[FIX + t];
            const bool lv = (t == V - 1) ? ((kb & 1u) != 0) : leave;
            sub_word_u(z2s, u2s, row.m[1], lv ? row.s[1] : row.a[1], lv ? row.a[1] : row.s[1]);
          }
          if (lane == 0) H[j] = make_uint4(z2, u2, z2s, u2s);
        });
        __syncwarp();
        uint32_t bev, bodd;
        exact_block(bev, bodd);
        ev += bev;
        odd += bodd;
        dense = __any_sync(FULL, bev >= (uint32_t)K / 2);
      } else {
        uint32_t rec = 0;
        if (!WIDE) {
          __syncwarp();
          if (lane == 0) H[0] = make_uint4(z2, u2, 0u, 0u);
        }
        static_for<K>([&](auto kc) {
          constexpr int k = decltype(kc)::value;
          pair_test<(((uint32_t)k) << 16) | 1u>(z1[k], g1[k], z2, u2, rec, one);
        });
        static_for<SB - 1>([&](auto jc) {
          constexpr int j = decltype(jc)::value + 1;
          constexpr int t = ctz_c(j);
          constexpr bool leave = (t + 1 < V) ? (((j >> (t + 1)) & 1) != 0) : false;
          const uint32_t sop = (t == V - 1) ? SX : (leave ? SS[t] : SA[t]);
          const uint32_t cop = (t == V - 1) ? CX : (leave ? SA[t] : SS[t]);
          sub_word_u(z2, u2, SM[t], sop, cop);
          if (!WIDE) {
            if (lane == 0) H[j] = make_uint4(z2, u2, 0u, 0u);
          }
          static_for<K>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            pair_test<((uint32_t)((j << KB) | k) << 16) | 1u>(z1[k], g1[k], z2, u2, rec, one);
          });
        });
        if (__any_sync(FULL, rec != 0)) {
          if (!WIDE) __syncwarp();
          const uint32_t cnt = rec & 0xffffu;
          uint32_t bev = 0, bodd = 0;
          if (__any_sync(FULL, cnt > 1)) {
            // exact re-evaluation of every pair of the superblock
            if (WIDE) {
              const unsigned long long r = replay_wide<KB>(R, p.n, B << V, SB, lane, p.z0_init, p.z1_init);
              bev = (uint32_t)r;
              bodd = (uint32_t)(r >> 32);
            } else {
              exact_block(bev, bodd);
            }
            // switch to the exact mode only when events are really dense
            // (e.g. all-ones rows: 2/3 of all pairs), not on a stray double hit
            dense = p.dense_ok != 0 && __any_sync(FULL, bev >= (uint32_t)K / 2);
          } else if (cnt == 1) {
            const uint32_t id = rec >> 16, j = id >> KB, k = id & (K - 1);
            if (WIDE) {
              uint32_t zz[2], gg[2];
              wide_subset_state<KB>(R, p.n, (B << V) + j, (k << 5) | lane, p.z0_init, p.z1_init, zz, gg);
              if ((zz[0] | zz[1]) == 0) {
                bev = 1;
                bodd = (__popc(gg[0]) + __popc(gg[1]) + j + __popc(k) + lanepar) & 1u;
              }
            } else {
              // the hit is exact for n <= 32; its sign word is d ^ g2(step j)
              const uint2 a1 = A[k][lane];
              const uint4 h = H[j];
              uint32_t d;
              TP_LOP3(d, a1.x, a1.y, h.y, 0x06);
              bev = 1;
              bodd = (__popc((d ^ pair_g2(h.x, h.y)) & colmask) + j + __popc(k) + lanepar) & 1u;
            }
          }
          ev += bev;
          odd += bodd;
        }
      }
      if (kb + 1 < p.nblk) {
        const uint32_t u = kb + 1;
        const int t = __ffs(u) - 1;
        const RowRec& row = R[FIX + V + t];
        const bool lv = entry_leave(u, t, p, B0);
        sub_word_u(z2, u2, row.m[0], lv ? row.s[0] : row.a[0], lv ? row.a[0] : row.s[0]);
      }
    }
    warp_flush(p.pm + 2 * b, ev - odd, odd, lane);
  }
  trace_end(p, t_start, n_items, blockIdx.x * WARPS + (threadIdx.x >> 5), lane);
}

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

__global__ void k_pack(const uint8_t* __restrict__ entries, long long B, int n, RowRec* __restrict__ rows) {
  const uint32_t lane = threadIdx.x & 31u;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long b = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); b < B; b += warps) {
    const uint8_t* E = entries + b * (long long)n * n;
    for (int t = 0; t < 64; ++t) {
      unsigned long long mag = 0, sgn = 0;
      if (t < n) {
        uint32_t v0 = lane < (uint32_t)n ? (uint32_t)E[t * n + lane] % 3u : 0u;
        uint32_t v1 = lane + 32 < (uint32_t)n ? (uint32_t)E[t * n + lane + 32] % 3u : 0u;
        const unsigned long long m = (unsigned long long)__ballot_sync(FULL, v0 != 0) |
                                     ((unsigned long long)__ballot_sync(FULL, v1 != 0) << 32);
        const unsigned long long s = (unsigned long long)__ballot_sync(FULL, v0 == 2) |
                                     ((unsigned long long)__ballot_sync(FULL, v1 == 2) << 32);
        mag = __brevll(m) >> (64 - n);
        sgn = __brevll(s) >> (64 - n);
      }
      if (lane == 0) store_row(rows + b * 64 + t, mag, sgn);
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
// Walk variants (see tp_kernels.cuh FastVariant).
#define TP_FAST_VARIANTS(X)              \
  X(kLaneV5W4, k_walk_lane<5, 4>)        \
  X(kLaneV7W4, k_walk_lane<7, 4>)        \
  X(kLaneV8W4, k_walk_lane<8, 4>)        \
  X(kWideK2V7W4, k_walk_wide<1, 7, 4>)   \
  X(kWideK4V6W4, k_walk_wide<2, 6, 4>)   \
  X(kWideK8V5W4, k_walk_wide<3, 5, 4>)   \
  X(kWideK8V6W4, k_walk_wide<3, 6, 4>)    \
  X(kPairK32V4W4, k_walk_pair<5, 4, 4, false>) \
  X(kPairK16V5W4, k_walk_pair<4, 5, 4, false>) \
  X(kPairWideK32V4W4, k_walk_pair<5, 4, 4, true>) \
  X(kPairWideK16V5W4, k_walk_pair<4, 5, 4, true>) \
  X(kPairK32V3W4, k_walk_pair<5, 3, 4, false>) \
  X(kPairK16V4W4, k_walk_pair<4, 4, 4, false>) \
  X(kPairWideK32V3W4, k_walk_pair<5, 3, 4, true>)

const void* walk_fast_symbol(int variant) {
  switch (variant) {
#define X(id, ...) \
  case id:         \
    return reinterpret_cast<const void*>(&__VA_ARGS__);
    TP_FAST_VARIANTS(X)
#undef X
    default: return nullptr;
  }
}

const void* walk_generic_symbol(int nw) {
  return nw == 1 ? reinterpret_cast<const void*>(&k_walk_generic<1>)
                 : reinterpret_cast<const void*>(&k_walk_generic<2>);
}

cudaError_t launch_walk_fast(int variant, int grid, const FastParams& p, cudaStream_t st) {
  const int threads = 32 * fast_warps(variant);
  switch (variant) {
#define X(id, ...)                                  \
  case id:                                          \
    __VA_ARGS__<<<grid, threads, 0, st>>>(p);       \
    break;
    TP_FAST_VARIANTS(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
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
