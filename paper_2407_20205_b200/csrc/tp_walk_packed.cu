// tp_walk_packed.cu -- the pair walk with a packed 16-column filter (n <= 32).
//
// Same meet-in-the-middle split as tp_walk_pair.cu (A side = rows 0..9 fixed
// per lane in K = 32 slots, B side walked), but the filter tests two pairs per
// 32-bit word: the low 16 columns of slot w sit in the low half of packed word
// w and those of slot w + 16 in the high half, and the B state's low 16
// columns are duplicated into both halves.  Per word:
//
//   d  = ~z1 & (g1 ^ u2)              lop3 0x06
//   zp = ~d & ~(z1 ^ z2)              lop3 0x09   (zero columns of the sums)
//   t  = zp - 0x00010001              imad (FMA pipe)
//   P  = (t & ~zp & 0x80008000) != 0  lop3 -> predicate: a half without zero columns
//   @P m += bit(j, w)                 imad (FMA pipe)
//
// i.e. 1.5 LOP3 per pair instead of 2, and 2.5 instructions per pair.  A
// pass (probability (2/3)^16 per pair on uniform inputs) is verified exactly
// on all 32 columns after each superblock: one ballot per pair of pass masks
// compacts the nonzero ones into a per-warp list, and lane e walks the pass
// bits of entry e against the full A words and the group's B states (both in
// shared memory).  Terms are evaluated only there, so the counts are exact.
// Event-dense matrices switch to an exact mode as in the pair walk; the cold
// paths (dense fold, n > 32 primary hits) are out of line so that they do not
// take registers from the filter loop.  V = 4 (512 pairs per lane and
// superblock) is the default for n >= 16 when the job fills the GPU.
//
// WIDE (n > 32): the filter and the verify cover the 32 primary columns; a
// verified primary hit (probability (2/3)^32) is evaluated over all n columns
// from scratch, as in the wide pair walk.
#include "tp_walk_common.cuh"

namespace tp {

// Exact fold of the B states Hb[0..SB) against the lane's 32 slots (full A
// words in shared memory): the dense mode.  Not inlined, so that its
// registers do not constrain the filter loop's allocation.
template <int SB>
static __device__ __noinline__ unsigned long long packed_exact_block(const uint4 (*A)[32], const uint2* Hb,
                                                                     uint32_t lane, uint32_t colmask, uint32_t one) {
  constexpr int NW = 16;
  uint32_t bev = 0, bodd = 0;
#pragma unroll 1
  for (int j = 0; j < SB; ++j) {
    const uint2 h = Hb[j];
    const uint32_t gh = pair_g2(h.x, h.y);
    uint32_t n0 = 0, a0 = 0, n1 = 0, a1 = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      // re-read per step (volatile): hoisting all 16 loads out of the j loop
      // would leave the fold one temporary register and serialise it
      uint4 a;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w)
                   : "r"((uint32_t)__cvta_generic_to_shared(&A[w][lane])));
      if (__popc(w) & 1) exact_fold(a.x, a.y, h.x, h.y, gh, colmask, n1, a1, one);
      else exact_fold(a.x, a.y, h.x, h.y, gh, colmask, n0, a0, one);
      if (__popc(w + NW) & 1) exact_fold(a.z, a.w, h.x, h.y, gh, colmask, n1, a1, one);
      else exact_fold(a.z, a.w, h.x, h.y, gh, colmask, n0, a0, one);
    }
    // term parity: popc(sign word) + j + popc(slot) + lane parity
    const uint32_t pj = ((uint32_t)j ^ __popc(lane)) & 1u;
    bev += n0 + n1;
    bodd += pj ? (n0 - a0) + a1 : a0 + (n1 - a1);
  }
  return (unsigned long long)bev | ((unsigned long long)bodd << 32);
}

// Term of one subset for n > 32, from scratch: bit 0 = all n columns
// nonzero, bits 2.. = popc of the sign words (0 when not full).  Not inlined
// (a primary hit has probability (2/3)^32; keeps the hot code small).
template <int KB>
static __device__ __noinline__ uint32_t wide_hit_term(const RowRec* R, int n, unsigned long long a, uint32_t low,
                                                      uint32_t z0i, uint32_t z1i) {
  uint32_t zz[2], gg[2];
  wide_subset_state<KB>(R, n, a, low, z0i, z1i, zz, gg);
  if ((zz[0] | zz[1]) != 0) return 0u;
  return 1u | ((uint32_t)(__popc(gg[0]) + __popc(gg[1])) << 2);
}

__device__ __forceinline__ uint32_t lanemask_lt() {  // %lanemask_lt: read where needed, holds no register
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// (z2, u2) of the primary word at B-side index a (low bits empty), from
// scratch; out of line (dense superblocks of the wide walk).
template <int KB>
static __device__ __noinline__ uint2 wide_b_entry(const RowRec* R, int n, unsigned long long a, uint32_t z0i,
                                                  uint32_t z1i) {
  uint32_t zz[2], gg[2];
  wide_subset_state<KB>(R, n, a, 0u, z0i, z1i, zz, gg);
  return make_uint2(zz[0], pair_u2(zz[0], gg[0]));
}

template <int V, int WARPS, int MINB, bool WIDE>
__global__ void __launch_bounds__(32 * WARPS, MINB) k_walk_packed(FastParams p) {
  constexpr int KB = 5;
  constexpr int K = 1 << KB;
  constexpr int NW = K / 2;  // packed words
  constexpr int FIX = 5 + KB;
  constexpr int SB = 1 << V;
  constexpr int LG = 5 - V;  // a group of G superblocks fills the warp's lanes
  constexpr int G = 1 << LG;
  constexpr int MQ = SB / 2;  // pass masks per superblock (2 steps x 16 words each)
  static_assert(V >= 1 && V <= 5, "superblock");
  __shared__ RowRec Rs[WARPS][WIDE ? 64 : 32];
  __shared__ uint2 Hs[WARPS][32];             // B states (z2, u2) of the group, lane = (c << V) | j
  __shared__ uint4 As[WARPS][NW][32];         // full A words: slot w and slot w + 16
  constexpr uint32_t LCAP = 64;                 // verify list capacity (uniform inputs: ~22 entries)
  __shared__ uint4 Ls[WARPS][LCAP];              // verify list: ((lane << 4) | mask pair, mask, mask, -)
  __shared__ uint2 HPs[WARPS][32];               // packed (low 16 columns doubled) B states of the group
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t wid = threadIdx.x >> 5;
  RowRec* R = Rs[wid];
  uint2* H = Hs[wid];
  uint4 (*A)[32] = As[wid];
  uint4* Lst = Ls[wid];
  uint2* HP = HPs[wid];
  const uint32_t one = p.one;
  const uint32_t cneg = 0xfffeffffu * one;  // -0x00010001, runtime so ptxas keeps the IMAD
  const uint32_t colmask = p.z0_init;
  const uint32_t zero = one - 1u;  // runtime 0: keeps the first record of a mask an IMAD
  const unsigned long long t_start = p.trace ? clock64() : 0;
  unsigned long long n_items = 0;

  for (;;) {
    const unsigned long long item = next_item(p, lane, n_items, blockIdx.x * WARPS + wid);
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
    // A side: v1 for S1 = (k << 5) | lane, k in Gray order; packed low halves
    uint32_t Zp[NW], Gp[NW];
    {
      uint32_t z1[K], g1[K];
      uint32_t zz[2], gg[2];
      wide_subset_state<KB>(R, p.n, 0ull, lane, p.z0_init, p.z1_init, zz, gg);
      uint32_t zc = zz[0], gc = gg[0];
      static_for<K>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        if constexpr (i > 0) {
          constexpr int t = ctz_c(i);
          constexpr bool leave = ((gray_c(i - 1) >> t) & 1) != 0;
          sub_word(zc, gc, R[5 + t].m[0], leave ? R[5 + t].s[0] : R[5 + t].a[0]);
        }
        z1[gray_c(i)] = zc;
        g1[gray_c(i)] = gc;
      });
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        Zp[w] = __byte_perm(z1[w], z1[w + NW], 0x5410);
        Gp[w] = __byte_perm(g1[w], g1[w + NW], 0x5410);
        A[w][lane] = make_uint4(z1[w], g1[w], z1[w + NW], g1[w + NW]);
      }
    }
    // B side: v2 for S2 = gray(A0) on rows >= FIX (low bits empty)
    uint32_t z2, u2;
    {
      uint32_t zz[2], gg[2];
      wide_subset_state<KB>(R, p.n, A0, 0u, p.z0_init, p.z1_init, zz, gg);
      z2 = zz[0];
      u2 = pair_u2(zz[0], gg[0]);
    }
    __syncwarp();
    uint32_t ev = 0, odd = 0;

    // a verified pass with a full primary word: exact for n <= 32; for n > 32
    // the subset's n-column vector is recomputed and tested
    auto hit = [&](uint32_t d, uint32_t gh, uint32_t j, uint32_t k, uint32_t src, uint32_t srcpar,
                   unsigned long long sb, uint32_t& bev, uint32_t& bodd) {
      if (!WIDE) {
        bev += 1;
        bodd += (__popc((d ^ gh) & colmask) + j + __popc(k) + srcpar) & 1u;
      } else {
        const uint32_t r = wide_hit_term<KB>(R, p.n, (sb << V) + j, (k << 5) | src, p.z0_init, p.z1_init);
        bev += r & 1u;
        bodd += (r & 1u) & ((r >> 2) + j + __popc(k) + srcpar);
      }
    };
    bool dense = false;   // warp-uniform: exact mode on event-dense matrices
    bool have = false;    // lanes hold the packed B states of the current group
    uint32_t hoff = 0;    // superblocks since those states were computed
    for (uint32_t kb = 0; kb < p.nblk; ++kb) {
      const unsigned long long B = B0 + kb;
      if (WIDE && dense) {
        // exact replay of the superblock; the next superblock's entry state
        // from scratch (both out of line: keeps the hot code small)
        const unsigned long long r = replay_wide<KB>(R, p.n, B << V, SB, lane, p.z0_init, p.z1_init);
        ev += (uint32_t)r;
        odd += (uint32_t)(r >> 32);
        dense = __any_sync(FULL, (uint32_t)r >= (uint32_t)K / 2);
        have = false;
        if (kb + 1 < p.nblk) {
          const uint2 st = wide_b_entry<KB>(R, p.n, (B + 1) << V, p.z0_init, p.z1_init);
          z2 = st.x;
          u2 = st.y;
        }
        continue;
      }
      if (dense) {
        const uint32_t SX = (kb & 1u) ? SS[V - 1] : SA[V - 1];
        const uint32_t CX = (kb & 1u) ? SA[V - 1] : SS[V - 1];
        __syncwarp();
        if (lane == 0) H[0] = make_uint2(z2, u2);
        static_for<SB - 1>([&](auto jc) {
          constexpr int j = decltype(jc)::value + 1;
          constexpr int t = ctz_c(j);
          constexpr bool leave = (t + 1 < V) ? (((j >> (t + 1)) & 1) != 0) : false;
          const uint32_t sop = (t == V - 1) ? SX : (leave ? SS[t] : SA[t]);
          const uint32_t cop = (t == V - 1) ? CX : (leave ? SA[t] : SS[t]);
          sub_word_u(z2, u2, SM[t], sop, cop);
          if (lane == 0) H[j] = make_uint2(z2, u2);
        });
        __syncwarp();
        uint32_t bev, bodd;
        if (WIDE) {
          const unsigned long long r = replay_wide<KB>(R, p.n, B << V, SB, lane, p.z0_init, p.z1_init);
          bev = (uint32_t)r;
          bodd = (uint32_t)(r >> 32);
        } else {
          const unsigned long long r = packed_exact_block<SB>(A, H, lane, colmask, one);
          bev = (uint32_t)r;
          bodd = (uint32_t)(r >> 32);
        }
        ev += bev;
        odd += bodd;
        dense = __any_sync(FULL, bev >= (uint32_t)K / 2);
        have = false;
      } else {
        if (!have) {
          // B states of the rest of this superblock's aligned group, one per
          // lane (see tp_walk_pair.cu): lane (c << V) | j holds Gray index
          // y = ((B + c) << V) | j, reached from the entry of B by the rows
          // FIX + r for the bits r of gray(y) ^ gray(B << V).
          uint32_t zj = z2, uj = u2;
          const unsigned long long yB = B << V, y = ((B + (lane >> V)) << V) | (lane & (SB - 1));
          const uint32_t gB = (uint32_t)(yB ^ (yB >> 1)), D = ((uint32_t)(y ^ (y >> 1)) ^ gB) & 31u;
#pragma unroll
          for (int r = 0; r < V + LG; ++r) {
            if ((D >> r) & 1u) {
              const bool lv = ((gB >> r) & 1u) != 0;
              if (r < V) {
                sub_word_u(zj, uj, SM[r], lv ? SS[r] : SA[r], lv ? SA[r] : SS[r]);
              } else {
                const RowRec& row = R[FIX + r];
                sub_word_u(zj, uj, row.m[0], lv ? row.s[0] : row.a[0], lv ? row.a[0] : row.s[0]);
              }
            }
          }
          __syncwarp();
          H[lane] = make_uint2(zj, uj);
          HP[lane] = make_uint2(__byte_perm(zj, zj, 0x1010), __byte_perm(uj, uj, 0x1010));
          __syncwarp();
          have = true;
          hoff = 0;
        }
        uint32_t Mc[MQ];
#pragma unroll
        for (int q = 0; q < MQ; ++q) Mc[q] = zero;
        // the packed B states of steps j, j+1 in one uniform 16-byte load
        const uint4* HP4 = reinterpret_cast<const uint4*>(HP + (hoff << V));
        static_for<SB / 2>([&](auto ic) {
          constexpr int i = decltype(ic)::value;
          const uint4 hp = HP4[i];
          static_for<NW>([&](auto wc) {
            constexpr int w = decltype(wc)::value;
            packed_test<(1u << w)>(Zp[w], Gp[w], hp.x, hp.y, Mc[i], one, cneg);
          });
          static_for<NW>([&](auto wc) {
            constexpr int w = decltype(wc)::value;
            packed_test<(1u << (16 + w))>(Zp[w], Gp[w], hp.z, hp.w, Mc[i], one, cneg);
          });
        });
        const bool gend = ((B + 1) & (G - 1)) == 0;
        // verify this superblock's passes: every nonzero mask becomes one list
        // entry (ballot compaction), and lane e walks the bits of entry e
        constexpr int MP = MQ / 2;  // mask pairs
        uint32_t bq[MP], tot = 0;
#pragma unroll
        for (int q = 0; q < MP; ++q) {
          bq[q] = __ballot_sync(FULL, (Mc[2 * q] | Mc[2 * q + 1]) != 0u);
          tot += __popc(bq[q]);
        }
        if (tot > LCAP) {
          // too many passes for the list (event-dense matrix): evaluate the
          // superblock exactly and let the dense test decide the next mode
          uint32_t bev, bodd;
          if (WIDE) {
            const unsigned long long r = replay_wide<KB>(R, p.n, B << V, SB, lane, p.z0_init, p.z1_init);
            bev = (uint32_t)r;
            bodd = (uint32_t)(r >> 32);
          } else {
            const unsigned long long r = packed_exact_block<SB>(A, H + (hoff << V), lane, colmask, one);
            bev = (uint32_t)r;
            bodd = (uint32_t)(r >> 32);
          }
          ev += bev;
          odd += bodd;
          dense = p.dense_ok != 0 && __any_sync(FULL, bev >= (uint32_t)K / 2);
        } else if (tot) {
          uint32_t base = 0;
#pragma unroll
          for (int q = 0; q < MP; ++q) {
            if (Mc[2 * q] | Mc[2 * q + 1])
              Lst[base + __popc(bq[q] & lanemask_lt())] = make_uint4((lane << 4) | (uint32_t)q, Mc[2 * q], Mc[2 * q + 1], 0u);
            base += __popc(bq[q]);
          }
          __syncwarp();
          uint32_t bev = 0, bodd = 0;
          const uint32_t hblk = hoff << V;
          for (uint32_t e = lane; e < tot; e += 32) {
            const uint4 ent = Lst[e];
            const uint32_t src = ent.x >> 4, jb = 4 * (ent.x & 15u);
            const uint32_t srcpar = __popc(src) & 1u;
            uint32_t m0 = ent.y, m1 = ent.z;
            while (m0 | m1) {
              // bit b of mask 2q + h: step 4q + 2h + (b >> 4), word b & 15
              const uint32_t hsel = m0 ? 0u : 1u;
              const uint32_t mm = m0 ? m0 : m1;
              const uint32_t bit = __ffs(mm) - 1;
              if (hsel) m1 &= m1 - 1; else m0 &= m0 - 1;
              const uint32_t j = jb + 2 * hsel + (bit >> 4), w = bit & 15u;
              const uint4 av = A[w][src];
              const uint2 h = H[hblk + j];
              const uint32_t gh = pair_g2(h.x, h.y);
              uint32_t d, zp;
              TP_LOP3(d, av.x, av.y, h.y, 0x06);
              TP_LOP3(zp, d, av.x, h.x, 0x09);
              if (zp == 0) hit(d, gh, j, w, src, srcpar, B, bev, bodd);
              TP_LOP3(d, av.z, av.w, h.y, 0x06);
              TP_LOP3(zp, d, av.z, h.x, 0x09);
              if (zp == 0) hit(d, gh, j, w + NW, src, srcpar, B, bev, bodd);
            }
          }
          ev += bev;
          odd += bodd;
          // switch to the exact mode when events are dense (e.g. all-ones rows)
          dense = p.dense_ok != 0 && __reduce_add_sync(FULL, bev) >= (uint32_t)(32 * K * SB) / 8u;
          __syncwarp();
        }
        if (dense || gend) {
          have = false;
          // (z2, u2) = state of step SB-1 of this superblock, for the entry step
          const uint2 h = H[(hoff << V) + SB - 1];
          z2 = h.x;
          u2 = h.y;
        } else {
          ++hoff;
        }
      }
      // enter superblock kb+1 when the next superblock needs (z2, u2)
      if (!have && kb + 1 < p.nblk) {
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
  trace_end(p, t_start, n_items, blockIdx.x * WARPS + wid, lane);
}

// which: 0 = V 3, 1 = V 4 (n <= 32); 2 = V 4 wide (n > 32).  4 CTAs/SM.
cudaError_t launch_packed(int which, int grid, const FastParams& p, cudaStream_t st) {
  if (which == 0) k_walk_packed<3, 4, 4, false><<<grid, 128, 0, st>>>(p);
  else if (which == 1) k_walk_packed<4, 4, 4, false><<<grid, 128, 0, st>>>(p);
  else if (which == 2) k_walk_packed<4, 4, 4, true><<<grid, 128, 0, st>>>(p);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

const void* packed_symbol(int which) {
  if (which == 0) return reinterpret_cast<const void*>(&k_walk_packed<3, 4, 4, false>);
  if (which == 1) return reinterpret_cast<const void*>(&k_walk_packed<4, 4, 4, false>);
  if (which == 2) return reinterpret_cast<const void*>(&k_walk_packed<4, 4, 4, true>);
  return nullptr;
}

}  // namespace tp
