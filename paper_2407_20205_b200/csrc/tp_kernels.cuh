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
// Fast-walk variants: (kind, KB, V); all run 4 warps per CTA and each warp
// takes its own items.  The unrolled superblock body stays near 20 KB of
// SASS so it lives in the instruction cache.
//   lane: one subset per lane, superblock 2^V high steps of 32 steps;
//   wide: 2^KB subsets per lane (primary-column filter, n > 32);
//   pair: 2^KB fixed A-side vectors per lane, B side walked (2 LOP3/subset);
//         pair_wide = primary-column filter for n > 32.
enum FastVariant {
  kLaneV5 = 0,
  kLaneV8 = 1,
  kWideK4V6 = 2,
  kPairK32V3 = 3,
  kPairK32V4 = 4,
  kPairWideK32V3 = 5,
  kPairWideK32V4 = 6,
  kPackedK32V3 = 7,
  kPackedK32V4 = 8,
  kPackedWideK32V4 = 9,
  kNumFast = 10
};
constexpr bool fast_is_lane(int v) { return v == kLaneV5 || v == kLaneV8; }
constexpr bool fast_is_pair(int v) { return v >= kPairK32V3 && v <= kPairWideK32V4; }
constexpr bool fast_pair_wide(int v) { return v == kPairWideK32V3 || v == kPairWideK32V4; }
constexpr bool fast_is_packed(int v) { return v == kPackedK32V3 || v == kPackedK32V4 || v == kPackedWideK32V4; }
constexpr int packed_which(int v) { return v == kPackedK32V3 ? 0 : v == kPackedK32V4 ? 1 : 2; }
constexpr int fast_v(int v) {
  return v == kLaneV5 ? 5 : v == kLaneV8 ? 8 : v == kWideK4V6 ? 6
       : (v == kPairK32V3 || v == kPairWideK32V3 || v == kPackedK32V3) ? 3 : 4;
}
constexpr int fast_kb(int v) { return fast_is_lane(v) ? 0 : v == kWideK4V6 ? 2 : 5; }
constexpr int fast_warps(int) { return 4; }

// Fast walk: items are L-aligned chunks [F0 + c*L, F0 + (c+1)*L) of every
// matrix's fast region, in fast units (32 * 2^KB reference steps); L =
// nblk * 2^V, nblk a power of two >= 2, F0 a multiple of L.
struct FastParams {
  const RowRec* rows;           // [B][64]
  unsigned long long* pm;       // [B][2] (plus, minus) accumulators
  // Work queue {next item, warps done}; the last warp out resets both to 0,
  // so the counter needs no memset between launches.
  unsigned long long* queue;
  unsigned long long F0, L, chunks, items;
  uint32_t nblk;                // superblocks per item
  int lognblk;
  int n;
  uint32_t z0_init, z1_init;    // zero-indicator of an empty vector (padding = 0)
  uint32_t one;                 // runtime 1
  unsigned long long* trace;    // optional per-warp trace (smid, t_start, t_end, items); nullptr = off
  int dense_ok;                 // allow the exact (dense-event) mode
  int static_items;             // items <= warps of the grid: warp w takes item w, no queue
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

// Tensor-core pair test (tp_walk_tc.cu): full traversals and chunk-aligned
// ranges, n >= 18.  Item i = (matrix i / chunks, chunk c0 + i % chunks); a
// chunk is 2^(15+t) subsets = 2^t tiles of 256 A vectors x 128 B vectors.
struct TcParams {
  const RowRec* rows;           // [B][64]
  unsigned long long* pm;       // [B][2] (plus, minus) accumulators
  unsigned long long* err;      // count of tensor hits the exact check rejected (must stay 0)
  unsigned long long items, chunks, c0;
  int n, t;                     // tiles per item = 2^t
  int R, ks;                    // K layout (tc_layout)
};
void tc_layout(int n, int* R, int* ks);
size_t tc_smem_bytes(int n, int ks);
cudaError_t launch_walk_tc(int grid, const TcParams& p, cudaStream_t st);

// Bucketed pair walk (tp_walk_bucket.cu): 21 <= n <= 64, full traversals and
// the superblock-aligned middle of ranges.  Items (matrix, piece, chunk);
// chunk c covers B-side superblocks [F0 + c * nblk, min(F0 + (c + 1) * nblk,
// s_end)) (superblocks of 2^bucket_v B steps, a B step = 2^FIX reference
// steps).  tab/ptab come from launch_bucket_group: per matrix a compact
// table of the A side's two halves sorted by their key-column pattern (the
// pieces' slots are decoded from it, nothing per piece is materialised).
struct BucketParams {
  FastParams fp;                // items = B * bucket_pieces(cfg) * chunks; F0, nblk in superblocks
  const void* tab;              // [B][bucket_tab_bytes] half tables (offsets, subsets, vectors)
  const uint32_t* ptab;         // [B][pieces] bucket | count << 8 | piece-in-bucket << 20 (count 0 = unused)
  unsigned long long* tested;   // += pairs actually tested (compatible steps x 1024), or nullptr
  unsigned long long s_end;     // end of the superblock region
  // k_walk_batch, n > 32 ("sticky" pieces): a chunk counter per piece; items
  // are tickets t, piece t % npieces (matrix fastest), and a warp that joins
  // a piece takes its chunks from the counter until they run out
  unsigned int* chunk_ctr = nullptr;
  unsigned long long npieces = 0;
};
struct BucketCfg {
  int fix;   // A side: rows 0..fix-1
  int keys;  // key columns: 3^keys buckets
};
BucketCfg bucket_cfg(int n, bool packed, bool batch, unsigned long long B = 1);
int bucket_pieces(BucketCfg c);
size_t bucket_tab_bytes(BucketCfg c, bool wide);  // per matrix
int bucket_v(bool packed);
cudaError_t launch_bucket_group(const RowRec* rows, long long B, int n, BucketCfg c, bool packed, void* tab,
                                uint32_t* ptab, cudaStream_t st);
cudaError_t launch_walk_bucket(int grid, const BucketParams& bp, bool packed, cudaStream_t st);
const void* walk_bucket_symbol(bool packed);
cudaError_t launch_walk_batch(int grid, const BucketParams& bp, BucketCfg c, cudaStream_t st);  // tp_walk_batch.cu
int walk_batch_blocks_per_sm(bool wide);

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
