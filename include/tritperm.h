/*
 * tritperm.h -- C ABI of the B200-native Gray-code Ryser permanent mod 3.
 *
 * Library: paper_2407_20205_b200/lib/libtritperm_b200.so (sm_100a kernels,
 * static cudart).  Plain pointers and sizes only; no torch types.
 *
 * Each entry point replaces one native (numba) dispatcher of the reference
 * package tritperm (/root/reference/pkg/src/tritperm, cited src/<file>:<line>):
 *
 *   tp_range_sum        <- _kernels.chunk_sum        src/_kernels.py:90-128
 *                          (called at src/permanent.py:194,248,251)
 *   tp_range_sum_ex     <- _kernels.chunk_sum for n = 64 (the reference's
 *                          big-int twin, src/permanent.py:157-178,192-196)
 *   tp_range_sum_multi  <- the ThreadPool fan-out of perm_mod3_parallel
 *                          src/permanent.py:232-255 (one range per device)
 *   tp_range_sum_nccl   <- the same, with sum(partials) (:255) as one
 *                          ncclAllReduce of the counters across the devices
 *   tp_mc_zero_count    <- _kernels.mc_zero_count    src/_kernels.py:245-255
 *                          (called at src/experiments.py:180,183,186)
 *   tp_mc_sample_entries<- _kernels.mc_sample_entries src/_kernels.py:258-272
 *                          (called at tests/test_rng.py:53)
 *   tp_perm_batch       <- new: per-matrix perm mod 3 + histogram for a batch
 *                          (the per-trial loop of mc_zero_count,
 *                          src/_kernels.py:251-254, over caller matrices)
 *
 * Conventions (identical to the reference):
 *   - packed planes: mags[t], sgns[t] are row t of the matrix; column k is bit
 *     n-1-k (src/core_f3.py:14-16, src/permanent.py:94-100);
 *   - steps are Gray-code steps i; step i visits subset gray(i)=i^(i>>1) and
 *     carries sign (-1)^(popcount(sgn)+i) when every column is nonzero
 *     (src/_kernels.py:111-127).  Step 0 (empty subset) contributes 0;
 *   - partial sum over [lo,hi) = plus - minus, bit-equal to chunk_sum;
 *   - perm mod 3 = cmod3((-1)^n * (plus - minus))  (src/permanent.py:116-119);
 *     classes are {0,1,2} with 2 == -1.
 *
 * Errors: every function returns 0 on success and a negative TP_E* code on
 * failure; tp_last_error() returns a thread-local message.  Validation that
 * the reference does in Python (ValueError) is repeated here so a caller that
 * skips the Python layer still gets a clean error instead of a fault.
 * Calls are synchronous unless named *_async; synchronous calls run on a
 * library-owned stream and a cached workspace per device and are serialised
 * per device.  *_async calls enqueue on the caller's `stream` argument, a
 * cudaStream_t with the usual CUDA meaning (NULL/0 = the legacy default
 * stream), and return without synchronising.  Every device buffer an
 * *_async call needs internally (row records, bucket tables) is allocated
 * stream-ordered on that stream (cudaMallocAsync/cudaFreeAsync) and private
 * to the call: concurrent calls on different streams never share memory,
 * the calls may be captured into CUDA graphs, and no call synchronises the
 * device.
 */
#ifndef TRITPERM_H
#define TRITPERM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TP_OK 0
#define TP_E_INVALID (-1)   /* bad argument (maps to ValueError)            */
#define TP_E_CUDA (-2)      /* CUDA runtime error (maps to RuntimeError)     */
#define TP_E_NODEV (-3)     /* no usable sm_100 device                       */

#define TP_MAX_N 64

/* ABI version (major*100 + minor). */
int tp_version(void);

/* Thread-local message for the last failing call on this thread. */
const char *tp_last_error(void);

/* Number of visible CUDA devices that can run the sm_100a kernels. */
int tp_device_count(int *count);

/* SM count, max SM clock (kHz) and compute capability of `device`. */
int tp_device_info(int device, int *sm_count, int *max_clock_khz, int *cc_major, int *cc_minor);

/* Partial Ryser sum over steps [lo, hi) of one matrix given as reference
 * planes (n <= 63, 0 <= lo <= hi <= 2^n).  Replaces _kernels.chunk_sum
 * (src/_kernels.py:90-128): *plus - *minus == chunk_sum(mags,sgns,n,lo,hi). */
int tp_range_sum(const uint64_t *mags, const uint64_t *sgns, int n,
                 uint64_t lo, uint64_t hi, int device,
                 uint64_t *plus, uint64_t *minus);

/* tp_range_sum extended to n = 64, where the end 2^64 does not fit a
 * uint64: the range is [lo, hi) if hi_is_2_64 == 0 (any lo <= hi), or
 * [lo, 2^64) if hi_is_2_64 != 0 (then n must be 64 and hi 0).  For n <= 63 it
 * is tp_range_sum. */
int tp_range_sum_ex(const uint64_t *mags, const uint64_t *sgns, int n,
                    uint64_t lo, uint64_t hi, int hi_is_2_64, int device,
                    uint64_t *plus, uint64_t *minus);

/* Same, asynchronous: the counters {plus, minus} are ADDED into the device
 * buffer d_pm[2] on `stream`.  Used by the one-process-per-GPU path, which all-reduces d_pm
 * with NCCL. */
int tp_range_sum_async(const uint64_t *mags, const uint64_t *sgns, int n,
                       uint64_t lo, uint64_t hi, int device,
                       uint64_t *d_pm, void *stream);

/* [lo, hi) split into ndev contiguous parts (split_steps rule,
 * src/permanent.py:221-229), one per listed device, run concurrently from one
 * host thread, counters summed on the host.  Result is invariant to ndev. */
int tp_range_sum_multi(const uint64_t *mags, const uint64_t *sgns, int n,
                       uint64_t lo, uint64_t hi, const int *devices, int ndev,
                       uint64_t *plus, uint64_t *minus);

/* Same split, but the per-device counters meet on the devices in ONE
 * in-place ncclAllReduce (uint64[2], sum) over a communicator clique the
 * library creates once per device list (ncclCommInitAll, cached) and device
 * 0's copy is read back.  NCCL is dlopen'ed on first use (libnccl.so.2);
 * TP_E_CUDA if it is unavailable.  Devices are locked in ascending id order. */
int tp_range_sum_nccl(const uint64_t *mags, const uint64_t *sgns, int n,
                      uint64_t lo, uint64_t hi, const int *devices, int ndev,
                      uint64_t *plus, uint64_t *minus);

/* Batch of B matrices, uint8 entries [B][n][n] (host memory; values reduced
 * mod 3, so {0,1,2} classes or any non-negative integers), 1 <= n <= 64.
 * Outputs (each may be NULL): out_class[B] in {0,1,2}, out_partial[B] raw
 * partial sums over [1,2^n) (n <= 62), hist[3] counts of each class. */
int tp_perm_batch(const uint8_t *entries, int64_t B, int n, int device,
                  int8_t *out_class, int64_t *out_partial, int64_t *hist);

/* Device-pointer variant, asynchronous on `stream`.
 * d_entries: device uint8 [B][n][n].  d_class (int8[B]), d_pm (uint64[B][2]
 * plus/minus) and d_hist (int64[3]) are device buffers, each may be NULL;
 * d_hist is accumulated into (caller zeroes it).  Returns the number of
 * kernel launches issued in *launches (may be NULL). */
int tp_perm_batch_async(const uint8_t *d_entries, int64_t B, int n, int device,
                        int8_t *d_class, uint64_t *d_pm, int64_t *d_hist,
                        void *stream, int *launches);

/* The three stages of tp_perm_batch_async as separate calls (for callers
 * that keep packed rows resident, and for per-stage timing).  All are
 * asynchronous on `stream`.
 *   tp_pack_async:     d_entries uint8 [B][n][n] -> d_rows (B * TP_ROWREC_BYTES
 *                      bytes; the kernels' packed row records, 64 per matrix).
 *   tp_walk_async:     full Gray walk of every matrix; ADDS (plus, minus) into
 *                      d_pm uint64 [B][2] (caller zeroes it first).
 *   tp_finalize_async: d_pm -> d_class int8 [B] (may be NULL), d_hist int64[3]
 *                      accumulated (may be NULL). */
#define TP_ROWREC_BYTES 2048
int tp_pack_async(const uint8_t *d_entries, int64_t B, int n, int device,
                  void *d_rows, void *stream);
int tp_walk_async(const void *d_rows, int64_t B, int n, int device,
                  uint64_t *d_pm, void *stream, int *launches);
/* Range walk [lo, hi) of ONE matrix whose rows are already packed on the
 * device (d_rows from tp_pack_async with B = 1); ADDS {plus, minus} into
 * d_pm[2].  Same contract as tp_range_sum_async without the host planes. */
int tp_walk_range_async(const void *d_rows, int n, uint64_t lo, uint64_t hi, int device,
                        uint64_t *d_pm, void *stream, int *launches);
int tp_finalize_async(const uint64_t *d_pm, int64_t B, int n, int device,
                      int8_t *d_class, int64_t *d_hist, void *stream);

/* Exact census over all 3^(n^2) matrices, 1 <= n <= 6: counts of
 * perm mod 3 = 0, +1, -1.  Replaces exact_count_kernel (src/_kernels.py:164-209,
 * which enumerates and stops at n = 4); here two Laplace expansions reduce
 * it to 3^((n-2) n) rank computations over F3 (see csrc/tp_census.cu). */
int tp_exact_census(int n, int device, int64_t *zeros, int64_t *plus, int64_t *minus);

/* Which walk kernel serves full traversals of `batch` matrices of size n
 * (batch = 1: a single matrix or a range), and its ALU-pipe op count per
 * subset term (3 LOP3 for the lane/wide walks, 2 for the pair walks, 1.5 for
 * the packed walks).  For the bucketed walk (21 <= n <= 64: batches, single
 * matrices and the aligned middle of ranges that fill the GPU) the count is
 * per TESTED pair (k_walk_batch: 4/3 = 2 LOP3 + 1/3 VIMNMX3 + 1/3 LOP3 per
 * packed word of two pairs; k_walk_bucket: 1.5): it skips the pairs its key
 * columns prove zero, and tp_walk_tested reports how many it tested. */
int tp_walk_info(int n, long long batch, char *name, int name_len, double *lop3_per_term);

/* Pairs tested by the bucketed walk on `device` since the last call (the
 * counter is read and reset).  Diagnostics for the roofline accounting. */
int tp_walk_tested(int device, uint64_t *pairs);

/* Diagnostics: measured LOP3 throughput of `device` (ops/s, the ALU-pipe
 * roofline denominator) from a register-resident lop3 chain kernel timed
 * with CUDA events, and the kernel's duration in ms. */
int tp_alu_peak(int device, double *lop3_ops_per_s, double *ms);

/* Debug: when d_trace != NULL, every later fast-walk launch records per warp
 * (SM id, clock64 at start, clock64 at end, items) into the device buffer
 * d_trace[4 * warp] (uint64).  NULL switches tracing off. */
int tp_debug_trace(void *d_trace);

/* Monte Carlo tally over trials [t0, t1) with the reference's per-trial
 * splitmix64 streams (src/rng.py, src/_kernels.py:212-242), sampled on the
 * device.  *zeros == mc_zero_count(n, t0, t1, seed); hist[3] (may be NULL)
 * gets the per-class counts.  1 <= n <= 64. */
int tp_mc_zero_count(int n, int64_t t0, int64_t t1, uint64_t seed, int device,
                     int64_t *zeros, int64_t *hist);

/* Per-trial classes for trials [t0,t0+count) into host out_class[count]. */
int tp_mc_classes(int n, int64_t t0, int64_t count, uint64_t seed, int device,
                  int8_t *out_class);

/* uint8 classes {0,1,2} (2 == -1) of trials [t0, t0+count), row-major
 * [count][n][n], sampled on the device with the reference stream
 * (src/rng.py:68-71 sample_square).  out is host memory, or device memory
 * when out_on_device != 0 (then the call is asynchronous on `stream`). */
int tp_sample_classes(int n, int64_t t0, int64_t count, uint64_t seed, int device,
                      uint8_t *out, int out_on_device, void *stream);

/* Centred entries {-1,0,1} (row-major, n*n) of one trial, sampled on the
 * device (audit hook; replaces _kernels.mc_sample_entries). */
int tp_mc_sample_entries(int n, int64_t trial, uint64_t seed, int device,
                         int8_t *out);

/* Device self-test of the packed primitives on 32-bit words, evaluated with
 * the same lop3 sequences the walk kernels use:
 *   op 0 = add_reps formula   (src/core_f3.py:123-131, bit-exact incl. the
 *          sign bit of zero results, i.e. ADD_TABLE_ROWS),
 *   op 1 = sub_reps formula   (src/core_f3.py:134-138; the walk's step),
 *   op 2 = walk ADD = sub_reps of the negated row (m2, m2^s2); equal to
 *          add_reps on every decoded trit, may differ on zero-sign bits.
 * in[k*4+{0,1,2,3}] = mag1,sgn1,mag2,sgn2; out[k*2+{0,1}] = mag,sgn of the
 * result (standard encoding). */
int tp_selftest_ops(const uint32_t *in, int count, int op, int device, uint32_t *out);

#ifdef __cplusplus
}
#endif

#endif /* TRITPERM_H */
