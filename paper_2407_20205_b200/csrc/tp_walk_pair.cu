// tp_walk_pair.cu -- the pair walk (meet in the middle, 2 LOP3 per subset).
#include "tp_walk_common.cuh"

namespace tp {

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
#pragma unroll 1
      for (int j = 0; j < SB; ++j) {
        const uint4 h = H[j];
        const uint32_t gh = pair_g2(h.x, h.y);
        if (WIDE) {
#pragma unroll
          for (int q = 0; q < K; ++q) {
            uint32_t d, zp;
            TP_LOP3(d, z1[q], g1[q], h.y, 0x06);
            TP_LOP3(zp, d, z1[q], h.x, 0x09);
            if (zp == 0) {  // primary columns all nonzero: test the secondary word
              const uint2 a2 = A[q][lane];
              uint32_t d1, zp1;
              TP_LOP3(d1, a2.x, a2.y, h.w, 0x06);
              TP_LOP3(zp1, d1, a2.x, h.z, 0x09);
              if (zp1 == 0) {
                bev += 1;
                bodd += (__popc(d ^ gh) + __popc((d1 ^ pair_g2(h.z, h.w)) & colmask1) + (uint32_t)j +
                         (uint32_t)__popc(q) + lanepar) & 1u;
              }
            }
          }
        } else {
          // Branch-free exact fold: per pair the test (2 LOP3), the sign word
          // (d ^ g2) & colmask (1 LOP3), and predicated popc / and / two IMAD
          // counters split by the static parity of popc(q).
          uint32_t n0 = 0, a0 = 0, n1 = 0, a1 = 0;
#pragma unroll
          for (int q = 0; q < K; ++q) {
            if (__popc(q) & 1) exact_fold(z1[q], g1[q], h.x, h.y, gh, colmask, n1, a1, one);
            else exact_fold(z1[q], g1[q], h.x, h.y, gh, colmask, n0, a0, one);
          }
          // term is odd iff popc(sgn) + j + popc(q) + lane parity is odd
          const uint32_t pj = ((uint32_t)j ^ lanepar) & 1u;
          bev += n0 + n1;
          bodd += pj ? (n0 - a0) + a1 : a0 + (n1 - a1);
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
        // The B states of the whole superblock, one per lane (step j = lane mod
        // SB): relative to the entry, step j adds the rows FIX + r for the bits r
        // of gray(j); row FIX+V-1 leaves instead when bit 0 of the superblock
        // index is set.  V row updates per warp replace SB-1 sequential steps;
        // each step then broadcasts its state with two shuffles.
        uint32_t zj = z2, uj = u2;
        {
          const uint32_t j = lane & (SB - 1), gj = j ^ (j >> 1);
#pragma unroll
          for (int r = 0; r < V; ++r) {
            if ((gj >> r) & 1u) {
              const bool lv = (r == V - 1) && (kb & 1u);
              sub_word_u(zj, uj, SM[r], lv ? SS[r] : SA[r], lv ? SA[r] : SS[r]);
            }
          }
        }
        if (!WIDE) {
          __syncwarp();
          if (lane < (uint32_t)SB) H[lane] = make_uint4(zj, uj, 0u, 0u);
        }
        static_for<K>([&](auto kc) {
          constexpr int k = decltype(kc)::value;
          pair_test<(((uint32_t)k) << 16) | 1u>(z1[k], g1[k], z2, u2, rec, one);
        });
        static_for<SB - 1>([&](auto jc) {
          constexpr int j = decltype(jc)::value + 1;
          z2 = __shfl_sync(FULL, zj, j);
          u2 = __shfl_sync(FULL, uj, j);
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
  queue_done(p, lane);
  trace_end(p, t_start, n_items, blockIdx.x * WARPS + (threadIdx.x >> 5), lane);
}

cudaError_t launch_pair(int KB, int V, bool wide, int grid, const FastParams& p, cudaStream_t st) {
  if (KB != 5) return cudaErrorInvalidValue;
  if (!wide && V == 3) k_walk_pair<5, 3, 4, false><<<grid, 128, 0, st>>>(p);
  else if (!wide && V == 4) k_walk_pair<5, 4, 4, false><<<grid, 128, 0, st>>>(p);
  else if (wide && V == 3) k_walk_pair<5, 3, 4, true><<<grid, 128, 0, st>>>(p);
  else if (wide && V == 4) k_walk_pair<5, 4, 4, true><<<grid, 128, 0, st>>>(p);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

const void* pair_symbol(int KB, int V, bool wide) {
  if (KB != 5) return nullptr;
  if (!wide && V == 3) return reinterpret_cast<const void*>(&k_walk_pair<5, 3, 4, false>);
  if (!wide && V == 4) return reinterpret_cast<const void*>(&k_walk_pair<5, 4, 4, false>);
  if (wide && V == 3) return reinterpret_cast<const void*>(&k_walk_pair<5, 3, 4, true>);
  if (wide && V == 4) return reinterpret_cast<const void*>(&k_walk_pair<5, 4, 4, true>);
  return nullptr;
}

}  // namespace tp
