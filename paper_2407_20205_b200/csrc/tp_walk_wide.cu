// tp_walk_wide.cu -- the wide walk (3 LOP3 per subset over the 32 primary
// columns, K slots per lane), n > 32.
#include "tp_walk_common.cuh"

namespace tp {

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
    const unsigned long long item = next_item(p, lane, n_items, blockIdx.x * WARPS + (threadIdx.x >> 5));
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
  queue_done(p, lane);
  trace_end(p, t_start, n_items, blockIdx.x * WARPS + (threadIdx.x >> 5), lane);
}

cudaError_t launch_wide(int KB, int V, int grid, const FastParams& p, cudaStream_t st) {
  if (KB == 2 && V == 6) {
    k_walk_wide<2, 6, 4><<<grid, 128, 0, st>>>(p);
    return cudaGetLastError();
  }
  return cudaErrorInvalidValue;
}

const void* wide_symbol(int KB, int V) {
  return (KB == 2 && V == 6) ? reinterpret_cast<const void*>(&k_walk_wide<2, 6, 4>) : nullptr;
}

}  // namespace tp
