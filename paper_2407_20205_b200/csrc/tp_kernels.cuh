// tp_kernels.cuh -- kernel parameter blocks and launch entry points shared by
// tp_kernels.cu (device code) and tp_runtime.cu (host runtime + C ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "tp_device.cuh"

namespace tp {

constexpr int kWalkThreads = 256;  // 8 warps per CTA
// Fast-walk variants (words per plane NW, superblock = 2^V high steps).
enum FastVariant { kFast1V7 = 0, kFast1V8 = 1, kFast2V6 = 2, kFast2V7 = 3, kNumFast = 4 };
constexpr int fast_nw(int v) { return v <= kFast1V8 ? 1 : 2; }
constexpr int fast_v(int v) { return v == kFast1V7 ? 7 : v == kFast1V8 ? 8 : v == kFast2V6 ? 6 : 7; }

// Fast walk over [F0, F1) high steps (multiples of 2^V) of every matrix,
// chunked into items of L high steps.
struct FastParams {
  const RowRec* rows;           // [B][64]
  unsigned long long* pm;       // [B][2] (plus, minus) accumulators
  unsigned long long* queue;    // dynamic work counter (zeroed before launch)
  unsigned long long F0, F1, L, chunks, items;
  int n;
  uint32_t z0_init, z1_init;    // zero-indicator of an empty vector (padding = 0)
  uint32_t one;                 // runtime 1
};

constexpr int kMaxSeg = 4;
struct GenericParams {
  const RowRec* rows;
  unsigned long long* pm;
  unsigned long long seg_a0[kMaxSeg], seg_a1[kMaxSeg];
  unsigned long long lo, hi;    // reference step range for lane masking
  int masked;                   // 0: every lane of every segment is in range
  unsigned long long items;     // B * nseg
  int nseg;
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
cudaError_t launch_selftest(const uint32_t* in, int count, int op, uint32_t* out, cudaStream_t st);

}  // namespace tp
