// tp_walk_lane.cu -- the lane walk (3 LOP3 per subset), n <= 32.
#include "tp_walk_common.cuh"

namespace tp {

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
      // row 5+V-1 flips at j = 2^(V-1); it leaves iff bit 0 of B0+kb is set
      // (B0 may be odd: lane-walk items can be a single superblock)
      const uint32_t SX = (((uint32_t)B0 + kb) & 1u) ? SS[V - 1] : SA[V - 1];
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
  queue_done(p, lane);
  trace_end(p, t_start, n_items, blockIdx.x * WARPS + (threadIdx.x >> 5), lane);
}

template <int V>
static cudaError_t launch_lane_v(int grid, const FastParams& p, cudaStream_t st) {
  k_walk_lane<V, 4><<<grid, 128, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_lane(int V, int grid, const FastParams& p, cudaStream_t st) {
  switch (V) {
    case 5: return launch_lane_v<5>(grid, p, st);
    case 8: return launch_lane_v<8>(grid, p, st);
    default: return cudaErrorInvalidValue;
  }
}

const void* lane_symbol(int V) {
  switch (V) {
    case 5: return reinterpret_cast<const void*>(&k_walk_lane<5, 4>);
    case 8: return reinterpret_cast<const void*>(&k_walk_lane<8, 4>);
    default: return nullptr;
  }
}

}  // namespace tp
