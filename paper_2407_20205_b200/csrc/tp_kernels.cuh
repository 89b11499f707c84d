// tp_kernels.cuh -- kernel parameter blocks and launch entry points shared by
// tp_kernels.cu (device code) and tp_runtime.cu (host runtime + C ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "tp_device.cuh"

namespace tp {

constexpr int kWalkThreads = 256;  // 8 warps per CTA
constexpr int kSmallMaxN = 15;      // thread-per-matrix kernel (tp_small.cu) for n <= 15
constexpr int kSmallThreads = 128;
// Fast-walk variants.  Lane walk (n <= 32): one subset per lane, superblock
// 2^V high steps of 32 reference steps.  Wide walk (n > 32): 2^KB subsets per
// lane, superblock 2^V high steps of 32 * 2^KB reference steps.
// Variant = (kind, KB, V, warps per CTA); each warp takes its own items.
// The unrolled superblock body is (2^V - 1) * 2^KB steps: keep it <= ~20 KB of
// SASS so it stays resident in the instruction cache.
enum FastVariant {
  kLaneV7W4 = 0,
  kLaneV8W4 = 1,
  kWideK2V7W4 = 2,
  kWideK4V6W4 = 3,
  kWideK8V5W4 = 4,
  kWideK8V6W4 = 5,
  kLaneV5W4 = 6,
  kPairK32V4W4 = 7,      // pair walk (meet in the middle), n <= 32
  kPairK16V5W4 = 8,
  kPairWideK32V4W4 = 9,  // pair walk, n > 32 (primary-column filter)
  kPairWideK16V5W4 = 10,
  kPairK32V3W4 = 11,
  kPairK16V4W4 = 12,
  kPairWideK32V3W4 = 13,
  kNumFast = 14
};
constexpr bool fast_is_pair(int v) { return v >= kPairK32V4W4 && v <= kPairWideK32V3W4; }
constexpr bool fast_pair_wide(int v) {
  return v == kPairWideK32V4W4 || v == kPairWideK16V5W4 || v == kPairWideK32V3W4;
}
constexpr bool fast_is_lane(int v) { return v <= kLaneV8W4 || v == kLaneV5W4; }
constexpr int fast_v(int v) {
  return (v == kPairK32V3W4 || v == kPairWideK32V3W4) ? 3
       : (v == kPairK32V4W4 || v == kPairWideK32V4W4 || v == kPairK16V4W4) ? 4
       : (v == kPairK16V5W4 || v == kPairWideK16V5W4) ? 5
       : v == kLaneV5W4 ? 5
       : v == kLaneV7W4 ? 7
       : v == kLaneV8W4 ? 8
       : v == kWideK2V7W4 ? 7
       : v == kWideK4V6W4 ? 6
       : v == kWideK8V5W4 ? 5
                          : 6;
}
constexpr int fast_kb(int v) {
  return (v == kPairK32V4W4 || v == kPairWideK32V4W4 || v == kPairK32V3W4 || v == kPairWideK32V3W4) ? 5
       : (v == kPairK16V5W4 || v == kPairWideK16V5W4 || v == kPairK16V4W4) ? 4
       : fast_is_lane(v) ? 0 : v == kWideK2V7W4 ? 1 : v == kWideK4V6W4 ? 2 : 3;
}
constexpr int fast_warps(int) { return 4; }

// Fast walk: items are L-aligned chunks [F0 + c*L, F0 + (c+1)*L) of every
// matrix's fast region, in fast units (32 * 2^KB reference steps); L =
// nblk * 2^V, nblk a power of two >= 2, F0 a multiple of L.
struct FastParams {
  const RowRec* rows;           // [B][64]
  unsigned long long* pm;       // [B][2] (plus, minus) accumulators
  unsigned long long* queue;    // dynamic work counter (zeroed before launch)
  unsigned long long F0, L, chunks, items;
  uint32_t nblk;                // superblocks per item
  int lognblk;
  int n;
  uint32_t z0_init, z1_init;    // zero-indicator of an empty vector (padding = 0)
  uint32_t one;                 // runtime 1
  unsigned long long* trace;    // optional per-warp trace (smid, t_start, t_end, items); nullptr = off
  int dense_ok;                 // allow the exact (dense-event) mode
};

// Generic walk: regions [reg_a0[r], reg_a1[r]) of 32-step high steps, cut
// into pieces of glen high steps; one warp per (matrix, piece).
struct GenericParams {
  const RowRec* rows;
  unsigned long long* pm;
  unsigned long long reg_a0[2], reg_a1[2], pieces[2];
  unsigned long long glen;
  unsigned long long lo, hi;    // reference step range for lane masking
  int masked;                   // 0: every lane of every piece is in range
  unsigned long long items;     // B * (pieces[0] + pieces[1])
  int n;
  uint32_t z0_init, z1_init;
};

const void* walk_fast_symbol(int variant);
const void* walk_generic_symbol(int nw);
cudaError_t launch_walk_fast(int variant, int grid, const FastParams& p, cudaStream_t st);
cudaError_t launch_walk_generic(int nw, int grid, const GenericParams& p, cudaStream_t st);
cudaError_t launch_pack(const uint8_t* entries, long long B, int n, RowRec* rows, int grid, cudaStream_t st);
cudaError_t launch_sample(int n, long long t0, long long count, unsigned long long seed, RowRec* rows,
                          uint8_t* entries_out, cudaStream_t st);
cudaError_t launch_finalize(const unsigned long long* pm, long long B, int n, int8_t* cls, long long* partial,
                            long long* hist, cudaStream_t st);
cudaError_t run_alu_peak(int sm_count, uint32_t* scratch, cudaStream_t st, double* ops_per_s, double* ms);
cudaError_t launch_small(int n, long long B, const uint8_t* entries, long long t0, unsigned long long seed,
                         int8_t* cls, long long* partial, unsigned long long* pm, long long* hist, cudaStream_t st);
cudaError_t launch_census(int n, int grid, unsigned long long configs, unsigned long long* n0, cudaStream_t st);
cudaError_t launch_selftest(const uint32_t* in, int count, int op, uint32_t* out, cudaStream_t st);

}  // namespace tp
