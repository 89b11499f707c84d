// tp_runtime.cu -- host runtime and C ABI (include/tritperm.h).
//
// The runtime replaces the reference's Python/numba orchestration
// (src/permanent.py:181-255, src/experiments.py:158-190): it plans a step
// range into fast (superblock-aligned) and generic (masked) work, owns one
// stream per device, launches the sm_100a kernels and folds the per-matrix
// (plus, minus) counters into classes.
//
// Memory.  Every buffer a call enqueues work on is private to that call and
// stream-ordered: cudaMallocAsync on the call's stream before the first
// launch, cudaFreeAsync after the last (struct Scratch), from the device's
// default memory pool (kept warm: release threshold kPoolKeep).  So two
// *_async calls in flight on different streams never share memory, a call
// captured into a CUDA graph gets graph-owned allocations, and no call ever
// synchronises the device.  Only synchronous calls (which return after their
// own stream drained, serialised per device) reuse the grow-only d.ws.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tritperm.h"
#include "tp_kernels.cuh"

using tp::RowRec;

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

#define TP_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) return fail(TP_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                    \
  } while (0)

struct Device {
  int id = -1;
  bool ready = false;
  int sm_count = 0;
  int max_clock_khz = 0;
  int cc_major = 0, cc_minor = 0;
  int fast_blocks_per_sm[tp::kNumFast] = {};  // indexed by FastVariant
  int generic_blocks_per_sm[3] = {0, 0, 0};
  cudaStream_t stream = nullptr;
  void* ws = nullptr;  // grow-only workspace
  size_t ws_size = 0;
  // Work-queue counters for the fast walk, used round-robin so that walks
  // enqueued on different streams never share a counter.
  static constexpr int kQueues = 64;
  unsigned long long* queues = nullptr;
  int next_queue = 0;
  unsigned long long* tc_err = nullptr;  // tensor-path self-check counter (must stay 0)
  unsigned long long* bucket_tested = nullptr;  // pairs tested by the bucketed walk (tp_walk_tested)
  int bucket_blocks_per_sm = 0;
  int batch_blocks_per_sm[2] = {0, 0};  // k_walk_batch, n <= 32 / n > 32
  // Pinned staging for the synchronous single-range call (tp_range_sum): the
  // row table and zeroed counters go up in one async copy, the counters come
  // back in one (guarded by mu).
  static constexpr size_t kStageBytes = 64 * sizeof(RowRec) + 2 * sizeof(unsigned long long);
  void* stage = nullptr;
  std::mutex mu;
};

Device g_dev[64];
std::mutex g_init_mu;

int ensure_device(int dev, Device** out) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(TP_E_NODEV, "no CUDA device available (%s)", e == cudaSuccess ? "count=0" : cudaGetErrorString(e));
  if (dev < 0 || dev >= count || dev >= 64) return fail(TP_E_INVALID, "device %d out of range [0,%d)", dev, count);
  Device& d = g_dev[dev];
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (!d.ready) {
    TP_CUDA(cudaSetDevice(dev));
    cudaDeviceProp prop;
    TP_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10 || prop.minor != 0)
      return fail(TP_E_NODEV, "device %d is sm_%d%d; this build carries sm_100a code only", dev, prop.major,
                  prop.minor);
    d.id = dev;
    d.sm_count = prop.multiProcessorCount;
    TP_CUDA(cudaDeviceGetAttribute(&d.max_clock_khz, cudaDevAttrClockRate, dev));
    d.cc_major = prop.major;
    d.cc_minor = prop.minor;
    for (int v = 0; v < tp::kNumFast; ++v) {
      TP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.fast_blocks_per_sm[v], tp::walk_fast_symbol(v),
                                                            32 * tp::fast_warps(v), 0));
      if (d.fast_blocks_per_sm[v] < 1) return fail(TP_E_CUDA, "walk kernels cannot be resident on device %d", dev);
    }
    for (int nw = 1; nw <= 2; ++nw) {
      TP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.generic_blocks_per_sm[nw],
                                                            tp::walk_generic_symbol(nw), tp::kWalkThreads, 0));
      if (d.generic_blocks_per_sm[nw] < 1) return fail(TP_E_CUDA, "walk kernels cannot be resident on device %d", dev);
    }
    TP_CUDA(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
    TP_CUDA(cudaMalloc(&d.queues, 2 * Device::kQueues * sizeof(unsigned long long)));
    TP_CUDA(cudaMemset(d.queues, 0, 2 * Device::kQueues * sizeof(unsigned long long)));
    TP_CUDA(cudaMalloc(&d.tc_err, sizeof(unsigned long long)));
    TP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.bucket_blocks_per_sm, tp::walk_bucket_symbol(true), 128, 0));
    if (d.bucket_blocks_per_sm < 1) return fail(TP_E_CUDA, "bucket walk cannot be resident on device %d", dev);
    for (int w = 0; w < 2; ++w) {
      d.batch_blocks_per_sm[w] = tp::walk_batch_blocks_per_sm(w != 0);
      if (d.batch_blocks_per_sm[w] < 1) return fail(TP_E_CUDA, "batched walk cannot be resident on device %d", dev);
    }
    TP_CUDA(cudaMemset(d.tc_err, 0, sizeof(unsigned long long)));
    TP_CUDA(cudaMalloc(&d.bucket_tested, sizeof(unsigned long long)));
    TP_CUDA(cudaMemset(d.bucket_tested, 0, sizeof(unsigned long long)));
    TP_CUDA(cudaMallocHost(&d.stage, Device::kStageBytes));
    // stream-ordered scratch comes from the default pool: keep up to
    // kPoolKeep bytes cached across calls instead of returning them at
    // every synchronisation
    cudaMemPool_t pool;
    TP_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = (uint64_t)2 << 30;  // kPoolKeep
    TP_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    d.ready = true;
  }
  *out = &d;
  return TP_OK;
}

// Grow-only workspace of the SYNCHRONOUS calls only (each drains its stream
// before returning, and they are serialised by d.mu, so nothing in flight
// can still use the old buffer).  Caller holds d.mu and has set the device.
int ensure_ws(Device& d, size_t bytes) {
  if (d.ws_size >= bytes) return TP_OK;
  if (d.ws) {
    TP_CUDA(cudaFree(d.ws));
    d.ws = nullptr;
    d.ws_size = 0;
  }
  size_t sz = std::max<size_t>(bytes, 1 << 20);
  TP_CUDA(cudaMalloc(&d.ws, sz));
  d.ws_size = sz;
  return TP_OK;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Stream-ordered per-call scratch (see the header comment): take() enqueues
// a cudaMallocAsync on the call's stream, and the destructor a cudaFreeAsync
// of everything taken, after the call's launches.
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {}
  Scratch(const Scratch&) = delete;
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
  // 0 or TP_E_CUDA (message set, error state cleared)
  int take(size_t bytes, void** out) {
    void* p = nullptr;
    const cudaError_t e = cudaMallocAsync(&p, std::max<size_t>(bytes, 256), st);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(TP_E_CUDA, "cudaMallocAsync(%zu bytes): %s", bytes, cudaGetErrorString(e));
    }
    ptrs.push_back(p);
    *out = p;
    return TP_OK;
  }
};

// Workspace carve-up for a batch of B matrices.
struct Carve {
  size_t off = 0;
  template <class T>
  T* take(char* base, size_t count) {
    off = align_up(off, 256);
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += count * sizeof(T);
    return p;
  }
};

uint32_t zmask(int bits) {
  if (bits <= 0) return 0u;
  if (bits >= 32) return 0xffffffffu;
  return (1u << bits) - 1u;
}

// ---------------------------------------------------------------------------
// Planner: one reference step range [lo, hi) for every matrix of a batch.
// ---------------------------------------------------------------------------
struct Plan {
  int nw = 1;
  int variant = 0;
  bool fast = false;
  tp::FastParams fp{};
  tp::GenericParams gp{};
  int fast_grid = 0, generic_grid = 0;
  bool bucket = false;  // bucketed pair walk covers the whole plan
  tp::BucketParams bkp{};
  int bucket_grid = 0;
  long long bucket_B = 0;
  bool bucket_packed = true;
  bool bucket_batch = false;  // k_walk_batch instead of k_walk_bucket
  tp::BucketCfg bucket_cfg{14, 2};
  void* bucket_tab = nullptr;
  uint32_t* bucket_ptab = nullptr;
  bool host_last = false;  // n = 64, range end 2^64: step 2^64-1 is left to the host (range_sum_impl)
  bool tc = false;  // tensor-core pair test covers the whole plan
  tp::TcParams tcp{};
  int tc_grid = 0;
};

// Tensor-core pair test (tp_walk_tc.cu) for full traversals, opt-in with
// TRITPERM_TC=1: exact, but slower than the packed LOP3 walk on B200 (its
// 128 x 128 x 64 sub-tiles turn TMEM over faster than the MMA/epilogue
// handshake allows).
// Bucketed pair walk (tp_walk_bucket.cu), the default for 21 <= n <= 64 (full
// traversals and the superblock-aligned middle of ranges): TRITPERM_BUCKET=0
// selects the packed walk, =2 the bucketed walk with unpacked pair tests
// (n <= 31).
int bucket_mode() {
  const char* e = getenv("TRITPERM_BUCKET");  // read per call: tests switch it at run time
  return e ? atoi(e) : 1;
}

// Same size rule as the packed walk: the job must fill the GPU
// (B * 2^n >= 2^26; make_plan applies it to the region of a range).
bool bucket_applies(int n, unsigned long long B) {
  const int m = bucket_mode();
  // n >= 32 only with the packed filter (its verify tests the padding-slot
  // mask: there is no padding column); the unpacked pair tests need n <= 31
  return n >= 21 && n <= (m == 2 ? 31 : 64) && B > 0 && (n >= 26 || (B << (n - 15)) >= 2048ull) && m > 0;
}

// The packed bucketed walk runs as k_walk_batch (tp_walk_batch.cu: the
// compatible steps of several superblocks batched into one filter loop);
// TRITPERM_BATCH=0 selects k_walk_bucket (one filter loop per superblock).
bool batch_mode() {
  const char* e = getenv("TRITPERM_BATCH");  // read per call: tests switch it at run time
  return e ? atoi(e) != 0 : true;
}

int tc_mode() {
  const char* e = getenv("TRITPERM_TC");  // read per call: tests switch it at run time
  return e ? atoi(e) : 0;
}

// Superblock size per n: longer superblocks amortise the per-block work, but
// raise the chance that one lane sees two events of the same step parity in a
// block (which forces an exact replay); events have probability (2/3)^n.
// Override with TRITPERM_FAST_VARIANT for measurements.
int choose_variant(int n, unsigned long long B) {
  const char* e = getenv("TRITPERM_FAST_VARIANT");  // read per call: tests switch it at run time
  const int forced = e ? atoi(e) : -1;
  if (forced >= 0 && forced < tp::kNumFast) {
    const bool for_narrow = tp::fast_is_lane(forced) || forced == tp::kPackedK32V3 || forced == tp::kPackedK32V4 ||
                            (tp::fast_is_pair(forced) && !tp::fast_pair_wide(forced));
    if (for_narrow == (n <= 32)) return forced;
  }
  // The packed walk needs enough work to fill the GPU with its items (at
  // least 32 fast units = 2^15 subsets each): B * 2^(n-15) >= 2048.  Smaller
  // jobs (one matrix up to n = 25, small batches) run the lane walk, whose
  // items are 32x shorter.
  if (n <= 32) {
    const bool packed = n >= 16 && (B << (n - 15)) >= 2048ull;
    return packed ? tp::kPackedK32V4 : tp::kLaneV5;
  }
  return tp::kPackedWideK32V4;
}

// Optional CTA trace buffer for the fast walks (tp_debug_trace).
unsigned long long* g_trace = nullptr;

unsigned long long* take_queue(Device& d) {
  unsigned long long* q = d.queues + 2 * d.next_queue;
  d.next_queue = (d.next_queue + 1) % Device::kQueues;
  return q;
}

// full = true: the whole range [0, 2^n) of every matrix (n <= 64), planned
// directly in high steps so n = 64 does not overflow; lo/hi are then unused.
// Otherwise the reference step range [lo, hi), or [lo, 2^64) when end64 (n =
// 64, hi ignored; the generic walk's masks cannot express the last step, so
// a plan whose generic tail reaches it sets host_last).
//
// Layout: the fast kernel takes the L-aligned part of the fully covered fast
// units; the generic kernel takes the rest (range heads/tails, small n) in
// pieces of kGenericPiece high steps so it parallelises.  The bucketed
// walk's tables are taken from the call's stream-ordered scratch `sc`.
constexpr unsigned long long kGenericPiece = 64;

int make_plan(Device& d, int n, unsigned long long B, unsigned long long lo, unsigned long long hi, bool full,
              const RowRec* rows, unsigned long long* pm, Scratch& sc, Plan& pl, bool end64 = false) {
  pl = Plan();
  pl.nw = n <= 32 ? 1 : 2;
  // Bucketed pair walk over the superblocks [s0, s1) the step range covers
  // completely (superblock = 2^(14 + bv) reference steps); range heads and
  // tails go to the generic walk.  Items (matrix, piece, chunk of nblk
  // superblocks).
  bool bucket_mid = false;
  unsigned long long mid0 = 0, mid1 = 0;  // bucket region in 32-step units (ranges)
  if (bucket_applies(n, B) && (full || end64 || lo < hi)) {
    const bool packed = n > 31 || bucket_mode() != 2;  // 2: the unpacked pair tests
    const bool batch = packed && batch_mode();
    const tp::BucketCfg cfg = tp::bucket_cfg(n, packed, batch, B);
    const int fix = cfg.fix;  // A side: rows 0..fix-1
    const int P = tp::bucket_pieces(cfg);
    const int bv = tp::bucket_v(packed);
    const int sbl = fix + bv;  // log2 reference steps per superblock
    unsigned long long s0 = 0, s1 = 0;
    if (full) {
      s1 = 1ull << (n - sbl);
    } else {
      const unsigned long long lo0 = lo == 1 ? 0 : lo;  // step 0 contributes 0
      s0 = (lo0 >> sbl) + ((lo0 & ((1ull << sbl) - 1)) ? 1 : 0);
      s1 = end64 ? 1ull << (64 - sbl) : hi >> sbl;
    }
    // the region must fill the GPU: B * 2^(sbl) * (s1 - s0) >= 2^26
    const bool big = s1 > s0 && (s1 - s0 >= (1ull << (26 - sbl)) || B * (s1 - s0) >= (1ull << (26 - sbl)));
    const unsigned long long total = big ? s1 - s0 : 0;
    // Items per warp: at least 4 (fill the grid); items longer than 1024
    // superblocks are split further, up to ~128 per warp, so that uneven items
    // (event-dense matrices in exact mode run ~4x longer) balance through the
    // dynamic queue.  Short items (C2: one matrix's whole B side of 64
    // superblocks) stay whole: their per-item setup is not free.
    static const unsigned long long per_warp = [] {
      const char* e = getenv("TRITPERM_BUCKET_ITEMS");  // tuning knob: the ~128 above
      return (unsigned long long)(e && atoi(e) > 0 ? atoi(e) : 128);
    }();
    const int bps = batch ? d.batch_blocks_per_sm[n > 32 ? 1 : 0] : d.bucket_blocks_per_sm;
    const unsigned long long warps = (unsigned long long)d.sm_count * bps * 4;
    unsigned long long nblk = std::min<unsigned long long>(std::max<unsigned long long>(total, 1), 1ull << 16);
    auto items_of = [&](unsigned long long nb) { return B * (unsigned long long)P * ((total + nb - 1) / nb); };
    // (TRITPERM_BUCKET_MIN_ITEMS: items per warp at least, default 4.  One
    // 36x36 matrix ends with a tail of 14.7 of 16 warps active, but 16 or 64
    // items per warp cost more in per-item setup than the tail: C4 2.81 ms at
    // 4, 2.91 at 16, 4.14 at 64; C3 and C5 unchanged)
    static const unsigned long long min_items = [] {
      const char* e = getenv("TRITPERM_BUCKET_MIN_ITEMS");
      return (unsigned long long)(e && atoi(e) > 0 ? atoi(e) : 4);
    }();
    while (nblk > 1 && (items_of(nblk) < min_items * warps || (nblk > 1024 && items_of(nblk) < per_warp * warps)))
      nblk = (nblk + 1) / 2;
    // k_walk_batch, n > 32: sticky pieces (a warp keeps its decoded piece and
    // takes chunk after chunk of it from the piece's counter), so chunks can
    // be short without paying the per-piece set-up for each: at least 16
    // chunks per warp, of at least 16 superblocks.  Only where the items
    // above are few per warp (their tail shows: C4 1.90 -> 1.76 ms); long
    // jobs with many items (C5) measured 2 % slower with it.
    // TRITPERM_STICKY: 0 off, 1 this rule, 2 always (n > 32)
    const char* se = getenv("TRITPERM_STICKY");  // read per call: tests switch it at run time
    const int sticky_mode = se ? atoi(se) : 1;
    const bool sticky = batch && n > 32 &&
                        (sticky_mode == 2 || (sticky_mode == 1 && items_of(nblk) < 64 * warps));
    if (sticky) {
      nblk = std::min<unsigned long long>(std::max<unsigned long long>(total, 1), 1024);
      while (nblk > 16 && items_of(nblk) < 16 * warps) nblk /= 2;
    }
    const unsigned long long chunks = (total + nblk - 1) / nblk;
    if (big) {
      // per matrix: the half table (2-14 KB) and the piece table; no cap,
      // any batch fits (C2: 33 MB; a 65,536-trial n >= 33 slab: 0.9 GB)
      const size_t tb = align_up(tp::bucket_tab_bytes(cfg, n > 32) * (size_t)B, 256);
      void* mem = nullptr;
      const size_t pb = align_up((size_t)B * P * sizeof(uint32_t), 256);
      if (int rc = sc.take(tb + pb + (sticky ? (size_t)B * P * sizeof(unsigned int) : 0), &mem)) return rc;
      pl.bucket = true;
      pl.bucket_packed = packed;
      pl.bucket_batch = batch;
      pl.bucket_B = (long long)B;
      pl.bucket_cfg = cfg;
      pl.bucket_tab = mem;
      pl.bucket_ptab = reinterpret_cast<uint32_t*>(static_cast<char*>(mem) + tb);
      if (sticky) {
        pl.bkp.chunk_ctr = reinterpret_cast<unsigned int*>(static_cast<char*>(mem) + tb + pb);
        pl.bkp.npieces = B * (unsigned long long)P;
      }
      tp::FastParams& f = pl.bkp.fp;
      f.rows = rows;
      f.pm = pm;
      f.queue = take_queue(d);
      f.F0 = s0;
      f.L = nblk << bv;
      f.chunks = chunks;
      f.items = B * (unsigned long long)P * chunks;
      if (sticky) {  // tickets: every piece at least twice, about 4 per warp
        const unsigned long long np = B * (unsigned long long)P;
        f.items = np * std::max<unsigned long long>(2, (4 * warps + np - 1) / np);
      }
      f.nblk = (uint32_t)nblk;  // superblocks of 2^bv B steps
      f.lognblk = 0;
      f.n = n;
      f.z0_init = zmask(std::min(n, 32));
      f.z1_init = zmask(n - 32);
      f.one = 1u;
      f.trace = nullptr;
      f.dense_ok = 1;
      f.static_items = 0;
      pl.bkp.tab = pl.bucket_tab;
      pl.bkp.ptab = pl.bucket_ptab;
      pl.bkp.tested = d.bucket_tested;
      pl.bkp.s_end = s1;
      const unsigned long long ctas = (unsigned long long)d.sm_count * bps;
      pl.bucket_grid = (int)std::max<unsigned long long>(1, std::min(ctas, (f.items + 3) / 4));
      if (full) return TP_OK;
      bucket_mid = true;
      mid0 = s0 << (sbl - 5);
      mid1 = s1 << (sbl - 5);
    }
  }
  // Full traversals of n >= 18 (at least 8 tiles per matrix) go to the tensor
  // cores.  Tiles per item 2^t: as long as the grid still gets >= 8 items per CTA.
  if (!bucket_mid && full && n >= 18 && B > 0 && tc_mode() != 0) {
    const int tmax = n - 15;
    const unsigned long long want = 8ull * (unsigned long long)d.sm_count;
    int t = tmax;
    while (t > 3 && (B << (tmax - t)) < want) --t;
    pl.tc = true;
    pl.tcp.rows = rows;
    pl.tcp.pm = pm;
    pl.tcp.err = d.tc_err;
    pl.tcp.n = n;
    pl.tcp.t = t;
    pl.tcp.chunks = 1ull << (tmax - t);
    pl.tcp.items = B * pl.tcp.chunks;
    pl.tcp.c0 = 0;
    tp::tc_layout(n, &pl.tcp.R, &pl.tcp.ks);
    pl.tc_grid = (int)std::min<unsigned long long>(pl.tcp.items, (unsigned long long)d.sm_count);
    return TP_OK;
  }
  pl.variant = choose_variant(n, B);
  const int V = tp::fast_v(pl.variant);
  const int U = tp::fast_kb(pl.variant);  // log2(fast unit / 32 reference steps)
  const uint32_t z0 = zmask(std::min(n, 32)), z1 = zmask(n - 32);

  pl.gp.rows = rows;
  pl.gp.pm = pm;
  pl.gp.n = n;
  pl.gp.z0_init = z0;
  pl.gp.z1_init = z1;
  pl.gp.glen = kGenericPiece;
  unsigned long long a_lo, a_hi, A0, A1;  // touched / fully covered high steps (32-step units)
  if (full) {
    const unsigned long long H = n >= 5 ? (1ull << (n - 5)) : 1ull;
    a_lo = A0 = 0;
    a_hi = A1 = H;
    pl.gp.lo = 0;
    pl.gp.hi = n >= 5 ? ~0ull : (1ull << n);  // n < 5: lanes >= 2^n inactive
    pl.gp.masked = n < 5 ? 1 : 0;
  } else {
    if (lo >= hi && !end64) return TP_OK;
    if (lo == 1) lo = 0;  // step 0 (the empty subset) contributes 0 for n >= 1
    a_lo = lo >> 5;  // (no lo + 31 / hi + 31: n = 64 bounds may be within 31 of 2^64)
    a_hi = end64 ? 1ull << 59 : (hi >> 5) + ((hi & 31) ? 1 : 0);
    A0 = (lo >> 5) + ((lo & 31) ? 1 : 0);
    A1 = end64 ? 1ull << 59 : hi >> 5;
    pl.gp.lo = lo;
    pl.gp.hi = end64 ? ~0ull : hi;  // end64: the mask keeps i < 2^64 - 1
    pl.gp.masked = 1;
  }
  if (B == 0) return TP_OK;

  // Fast region, in fast units of 2^U high steps, superblocks of 2^V units.
  const unsigned long long A0u = (A0 + (1ull << U) - 1) >> U, A1u = A1 >> U;
  const unsigned long long SBu = 1ull << V;
  unsigned long long F0 = 0, F1 = 0, L = 0;
  if (!bucket_mid && n >= 5 + U + V + 1 && A0u < A1u) {
    const int bps = d.fast_blocks_per_sm[pl.variant];
    const unsigned long long warps = (unsigned long long)d.sm_count * bps * tp::fast_warps(pl.variant);
    const unsigned long long want_items = warps * 32;  // dynamic queue: a few dozen per warp
    const unsigned long long Lmax = 1ull << (20 - U);   // per-item counters stay 32-bit
    auto aligned_chunks = [&](unsigned long long Lc) {
      const unsigned long long f0 = (A0u + Lc - 1) / Lc * Lc, f1 = A1u / Lc * Lc;
      return f1 > f0 ? (f1 - f0) / Lc : 0ull;
    };
    // items of >= 2 superblocks keep B0 even for the pair/packed walks; the
    // lane walk takes single-superblock items (short jobs: more parallelism)
    L = (tp::fast_is_lane(pl.variant) ? 1 : 2) * SBu;
    if (aligned_chunks(L) == 0) L = 0;
    while (L && 2 * L <= Lmax && aligned_chunks(2 * L) * B >= want_items) L <<= 1;
    if (L) {
      F0 = (A0u + L - 1) / L * L;
      F1 = A1u / L * L;
    }
  }
  unsigned long long g0a = a_lo, g0b = a_hi, g1a = 0, g1b = 0;  // generic regions (32-step units)
  if (bucket_mid) {  // range head and tail around the bucket region
    g0b = mid0;
    g1a = mid1;
    g1b = a_hi;
  }
  if (L) {
    g0b = F0 << U;
    g1a = F1 << U;
    g1b = a_hi;
    pl.fast = true;
    pl.fp.rows = rows;
    pl.fp.pm = pm;
    pl.fp.queue = take_queue(d);
    pl.fp.F0 = F0;
    pl.fp.L = L;
    pl.fp.chunks = (F1 - F0) / L;
    pl.fp.items = pl.fp.chunks * B;
    pl.fp.nblk = (uint32_t)(L >> V);
    pl.fp.lognblk = 0;
    while ((1u << pl.fp.lognblk) < pl.fp.nblk) pl.fp.lognblk++;
    pl.fp.n = n;
    pl.fp.z0_init = z0;
    pl.fp.z1_init = z1;
    pl.fp.one = 1u;
    pl.fp.trace = g_trace;
    {
      static int dense_ok = -1;
      if (dense_ok < 0) {
        const char* e = getenv("TRITPERM_NO_DENSE");
        dense_ok = (e && atoi(e)) ? 0 : 1;
      }
      pl.fp.dense_ok = dense_ok;
    }
    const int bps = d.fast_blocks_per_sm[pl.variant];
    const unsigned long long ctas = (unsigned long long)d.sm_count * bps;
    const unsigned long long wpc = tp::fast_warps(pl.variant);
    pl.fast_grid = (int)std::max<unsigned long long>(1, std::min(ctas, (pl.fp.items + wpc - 1) / wpc));
    pl.fp.static_items = pl.fp.items <= (unsigned long long)pl.fast_grid * wpc ? 1 : 0;
  }
  auto pieces = [&](unsigned long long x0, unsigned long long x1) {
    return x1 > x0 ? (x1 - x0 + kGenericPiece - 1) / kGenericPiece : 0ull;
  };
  pl.gp.reg_a0[0] = g0a;
  pl.gp.reg_a1[0] = g0b;
  pl.gp.pieces[0] = pieces(g0a, g0b);
  pl.gp.reg_a0[1] = g1a;
  pl.gp.reg_a1[1] = g1b;
  pl.gp.pieces[1] = pieces(g1a, g1b);
  pl.gp.items = (pl.gp.pieces[0] + pl.gp.pieces[1]) * B;
  if (pl.gp.items) {
    const unsigned long long max_grid = (unsigned long long)d.sm_count * d.generic_blocks_per_sm[pl.nw];
    const unsigned long long need = (pl.gp.items + 7) / 8;
    pl.generic_grid = (int)std::max<unsigned long long>(1, std::min(max_grid, need));
  }
  // end64: the generic tail, if it reaches the end, masks out step 2^64 - 1
  pl.host_last = end64 && pl.gp.pieces[1] > 0 && g1b == (1ull << 59);
  if (end64 && pl.gp.pieces[1] == 0 && pl.gp.pieces[0] > 0 && g0b == (1ull << 59)) pl.host_last = true;
  return TP_OK;
}

// Enqueue the walk of plan `pl`; returns launches in *launches.
int run_plan(const Plan& pl, cudaStream_t st, int* launches) {
  int nl = 0;
  if (pl.bucket) {  // (ranges: plus the generic head and tail below)
    TP_CUDA(tp::launch_bucket_group(pl.bkp.fp.rows, pl.bucket_B, pl.bkp.fp.n, pl.bucket_cfg, pl.bucket_packed,
                                    pl.bucket_tab, pl.bucket_ptab, st));
    if (pl.bkp.chunk_ctr) TP_CUDA(cudaMemsetAsync(pl.bkp.chunk_ctr, 0, pl.bkp.npieces * sizeof(unsigned int), st));
    if (pl.bucket_batch) TP_CUDA(tp::launch_walk_batch(pl.bucket_grid, pl.bkp, pl.bucket_cfg, st));
    else TP_CUDA(tp::launch_walk_bucket(pl.bucket_grid, pl.bkp, pl.bucket_packed, st));
    nl += 2;
  }
  if (pl.tc) {
    TP_CUDA(tp::launch_walk_tc(pl.tc_grid, pl.tcp, st));
    if (launches) *launches += 1;
    return TP_OK;
  }
  if (pl.fast) {
    TP_CUDA(tp::launch_walk_fast(pl.variant, pl.fast_grid, pl.fp, st));
    nl++;
  }
  if (pl.gp.items) {
    TP_CUDA(tp::launch_walk_generic(pl.nw, pl.generic_grid, pl.gp, st));
    nl++;
  }
  if (launches) *launches += nl;
  return TP_OK;
}

void planes_to_rows(const uint64_t* mags, const uint64_t* sgns, int n, RowRec* out) {
  for (int t = 0; t < 64; ++t) {
    const uint64_t m = t < n ? mags[t] : 0, s = t < n ? sgns[t] : 0;
    RowRec r;
    r.m[0] = (uint32_t)m;
    r.m[1] = (uint32_t)(m >> 32);
    r.s[0] = (uint32_t)s;
    r.s[1] = (uint32_t)(s >> 32);
    r.a[0] = r.m[0] ^ r.s[0];
    r.a[1] = r.m[1] ^ r.s[1];
    r.pad[0] = r.pad[1] = 0;
    out[t] = r;
  }
}

int check_planes(const uint64_t* mags, const uint64_t* sgns, int n) {
  if (!mags || !sgns) return fail(TP_E_INVALID, "mags/sgns must not be NULL");
  const uint64_t window = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
  for (int t = 0; t < n; ++t)
    if ((mags[t] & ~window) || (sgns[t] & ~window))
      return fail(TP_E_INVALID, "row %d has bits outside the %d-bit window", t, n);
  return TP_OK;
}

// Enqueue one range of one matrix on device d (caller holds d.mu, device
// set); the counters are added into d_pm[0..1].  Rows go into the call's
// own scratch (stream-ordered on st).
int enqueue_range(Device& d, const uint64_t* mags, const uint64_t* sgns, int n, uint64_t lo, uint64_t hi,
                  unsigned long long* d_pm, cudaStream_t st) {
  Scratch sc(st);
  void* mem = nullptr;
  if (int rc = sc.take(64 * sizeof(RowRec), &mem)) return rc;
  RowRec* rows = static_cast<RowRec*>(mem);
  RowRec h[64];
  planes_to_rows(mags, sgns, n, h);
  TP_CUDA(cudaMemcpyAsync(rows, h, sizeof h, cudaMemcpyHostToDevice, st));
  Plan pl;
  if (int rc = make_plan(d, n, 1, lo, hi, false, rows, d_pm, sc, pl)) return rc;
  // The H2D above is from pageable memory: it returns once `h` is staged,
  // so `h` may go out of scope before the stream runs.
  return run_plan(pl, st, nullptr);
}

// end64: the range end is 2^64 (n = 64 only; hi must then be 0); allow64:
// the caller can take n = 64 (tp_range_sum_ex), whose every u64 hi is <= 2^n.
int check_range(int n, uint64_t lo, uint64_t hi, bool end64 = false, bool allow64 = false) {
  if (end64) {
    if (n != 64 || hi != 0) return fail(TP_E_INVALID, "an end of 2^64 needs n = 64 and hi = 0");
    return TP_OK;
  }
  if (n == 64 && allow64) {
    if (lo > hi) return fail(TP_E_INVALID, "need lo <= hi, got lo=%llu hi=%llu", (unsigned long long)lo,
                             (unsigned long long)hi);
    return TP_OK;
  }
  if (n < 1 || n > 63) return fail(TP_E_INVALID, "range API needs 1 <= n <= 63 (n = 64: tp_range_sum_ex), got n=%d", n);
  const uint64_t last = 1ull << n;
  if (!(lo <= hi && hi <= last))
    return fail(TP_E_INVALID, "need 0 <= lo <= hi <= 2**n, got lo=%llu hi=%llu n=%d", (unsigned long long)lo,
                (unsigned long long)hi, n);
  return TP_OK;
}

// Term of the last step 2^64 - 1 of an n = 64 walk: subset gray(2^64 - 1) =
// {row 63}; full iff row 63 has no zero entry; sign (-1)^(popc(sgn) + 1).
void last_step_term(const uint64_t* mags, const uint64_t* sgns, uint64_t* plus, uint64_t* minus) {
  if (mags[63] != ~0ull) return;
  if (__builtin_popcountll(sgns[63]) & 1) ++*plus;
  else ++*minus;
}

// The synchronous single-range call behind tp_range_sum / tp_range_sum_ex.
int range_sum_impl(const uint64_t* mags, const uint64_t* sgns, int n, uint64_t lo, uint64_t hi, bool end64,
                   int device, uint64_t* plus, uint64_t* minus, bool allow64 = false) {
  int rc = check_range(n, lo, hi, end64, allow64);
  if (rc) return rc;
  if ((rc = check_planes(mags, sgns, n))) return rc;
  if (!plus || !minus) return fail(TP_E_INVALID, "plus/minus must not be NULL");
  Device* d;
  if ((rc = ensure_device(device, &d))) return rc;
  std::lock_guard<std::mutex> lk(d->mu);
  TP_CUDA(cudaSetDevice(device));
  // device layout = staging layout: 64 RowRec, then the (plus, minus) counters
  if ((rc = ensure_ws(*d, Device::kStageBytes))) return rc;
  RowRec* hrows = static_cast<RowRec*>(d->stage);
  unsigned long long* hpm = reinterpret_cast<unsigned long long*>(hrows + 64);
  planes_to_rows(mags, sgns, n, hrows);
  hpm[0] = hpm[1] = 0;
  RowRec* rows = static_cast<RowRec*>(d->ws);
  unsigned long long* pm = reinterpret_cast<unsigned long long*>(rows + 64);
  TP_CUDA(cudaMemcpyAsync(rows, hrows, Device::kStageBytes, cudaMemcpyHostToDevice, d->stream));
  Plan pl;
  {
    Scratch sc(d->stream);
    if ((rc = make_plan(*d, n, 1, lo, hi, false, rows, pm, sc, pl, end64))) return rc;
    if ((rc = run_plan(pl, d->stream, nullptr))) return rc;
  }
  TP_CUDA(cudaMemcpyAsync(hpm, pm, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, d->stream));
  TP_CUDA(cudaStreamSynchronize(d->stream));
  *plus = hpm[0];
  *minus = hpm[1];
  if (pl.host_last) last_step_term(mags, sgns, plus, minus);
  return TP_OK;
}

// ---------------------------------------------------------------------------
// NCCL, loaded on first use (dlopen of libnccl.so.2: the copy torch already
// loaded if any, else the system one), so the library has no link-time
// dependency on it.  One communicator clique per device list, cached.
// ---------------------------------------------------------------------------
struct Nccl {
  bool tried = false, ok = false;
  std::string why;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::map<std::vector<int>, std::vector<ncclComm_t>> comms;
};
Nccl g_nccl;
std::mutex g_nccl_mu;

int nccl_load() {
  Nccl& N = g_nccl;
  if (!N.tried) {
    N.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      N.why = dlerror() ? dlerror() : "dlopen failed";
    } else {
      N.CommInitAll = reinterpret_cast<decltype(N.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
      N.AllReduce = reinterpret_cast<decltype(N.AllReduce)>(dlsym(h, "ncclAllReduce"));
      N.GroupStart = reinterpret_cast<decltype(N.GroupStart)>(dlsym(h, "ncclGroupStart"));
      N.GroupEnd = reinterpret_cast<decltype(N.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
      N.GetErrorString = reinterpret_cast<decltype(N.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
      N.ok = N.CommInitAll && N.AllReduce && N.GroupStart && N.GroupEnd && N.GetErrorString;
      if (!N.ok) N.why = "libnccl.so.2 lacks a required symbol";
    }
  }
  if (!N.ok) return fail(TP_E_CUDA, "NCCL unavailable: %s", N.why.c_str());
  return TP_OK;
}

#define TP_NCCL(call)                                                                                  \
  do {                                                                                                 \
    ncclResult_t r_ = (call);                                                                          \
    if (r_ != ncclSuccess) return fail(TP_E_CUDA, "%s: %s", #call, g_nccl.GetErrorString(r_));         \
  } while (0)

// Multi-device split of one range (shared by tp_range_sum_multi and
// tp_range_sum_nccl): part k of split_steps' rule goes to devices[k]; every
// part is enqueued before any is waited on.  use_nccl: the per-device
// counters meet in one ncclAllReduce over the clique and device 0's copy is
// read; otherwise each device's counters are read and summed on the host.
int range_sum_multi_impl(const uint64_t* mags, const uint64_t* sgns, int n, uint64_t lo, uint64_t hi,
                         const int* devices, int ndev, bool use_nccl, uint64_t* plus, uint64_t* minus) {
  int rc = check_range(n, lo, hi);
  if (rc) return rc;
  if ((rc = check_planes(mags, sgns, n))) return rc;
  if (!devices || ndev < 1) return fail(TP_E_INVALID, "need at least one device");
  if (!plus || !minus) return fail(TP_E_INVALID, "plus/minus must not be NULL");
  for (int k = 0; k < ndev; ++k)
    for (int q = 0; q < k; ++q)
      if (devices[q] == devices[k]) return fail(TP_E_INVALID, "device %d listed twice", devices[k]);
  std::vector<Device*> ds(ndev);
  for (int k = 0; k < ndev; ++k)
    if ((rc = ensure_device(devices[k], &ds[k]))) return rc;
  std::unique_lock<std::mutex> nlk;
  std::vector<ncclComm_t>* comms = nullptr;
  if (use_nccl) {
    nlk = std::unique_lock<std::mutex>(g_nccl_mu);
    if ((rc = nccl_load())) return rc;
    const std::vector<int> key(devices, devices + ndev);
    auto it = g_nccl.comms.find(key);
    if (it == g_nccl.comms.end()) {  // communicator init is outside every timed path: once per device list
      std::vector<ncclComm_t> c(ndev);
      TP_NCCL(g_nccl.CommInitAll(c.data(), ndev, devices));
      it = g_nccl.comms.emplace(key, std::move(c)).first;
    }
    comms = &it->second;
  }
  // lock the devices in ascending id order (concurrent calls listing the
  // same devices in different orders cannot deadlock)
  std::vector<int> order(ndev);
  for (int k = 0; k < ndev; ++k) order[k] = k;
  std::sort(order.begin(), order.end(), [&](int x, int y) { return devices[x] < devices[y]; });
  std::vector<std::unique_lock<std::mutex>> locks;
  for (int k : order) locks.emplace_back(ds[k]->mu);
  std::vector<unsigned long long*> pms(ndev);
  std::vector<RowRec> h(64);
  planes_to_rows(mags, sgns, n, h.data());
  // Split [lo, hi) like split_steps (src/permanent.py:221-229) and enqueue
  // every part before waiting on any, so the devices run concurrently.
  const unsigned long long total = hi - lo;
  for (int k = 0; k < ndev; ++k) {
    Device& d = *ds[k];
    TP_CUDA(cudaSetDevice(d.id));
    Carve cv;
    cv.take<RowRec>(nullptr, 64);
    cv.take<unsigned long long>(nullptr, 2);
    if ((rc = ensure_ws(d, cv.off))) return rc;
    char* base = static_cast<char*>(d.ws);
    Carve c2;
    RowRec* rows = c2.take<RowRec>(base, 64);
    pms[k] = c2.take<unsigned long long>(base, 2);
    const unsigned long long plo = lo + (unsigned long long)((unsigned __int128)total * k / ndev);
    const unsigned long long phi = lo + (unsigned long long)((unsigned __int128)total * (k + 1) / ndev);
    TP_CUDA(cudaMemsetAsync(pms[k], 0, 2 * sizeof(unsigned long long), d.stream));
    TP_CUDA(cudaMemcpyAsync(rows, h.data(), 64 * sizeof(RowRec), cudaMemcpyHostToDevice, d.stream));
    Plan pl;
    Scratch sc(d.stream);
    if ((rc = make_plan(d, n, 1, plo, phi, false, rows, pms[k], sc, pl))) return rc;
    if ((rc = run_plan(pl, d.stream, nullptr))) return rc;
  }
  unsigned long long P = 0, M = 0;
  if (use_nccl) {
    // the reference's sum(partials) (src/permanent.py:255) as one in-place
    // all-reduce of the 16-byte counters over the clique
    TP_NCCL(g_nccl.GroupStart());
    for (int k = 0; k < ndev; ++k)
      TP_NCCL(g_nccl.AllReduce(pms[k], pms[k], 2, ncclUint64, ncclSum, (*comms)[k], ds[k]->stream));
    TP_NCCL(g_nccl.GroupEnd());
    unsigned long long hp[2];
    TP_CUDA(cudaSetDevice(ds[0]->id));
    TP_CUDA(cudaMemcpyAsync(hp, pms[0], sizeof hp, cudaMemcpyDeviceToHost, ds[0]->stream));
    for (int k = 0; k < ndev; ++k) {
      TP_CUDA(cudaSetDevice(ds[k]->id));
      TP_CUDA(cudaStreamSynchronize(ds[k]->stream));
    }
    P = hp[0];
    M = hp[1];
  } else {
    for (int k = 0; k < ndev; ++k) {
      Device& d = *ds[k];
      TP_CUDA(cudaSetDevice(d.id));
      unsigned long long hp[2];
      TP_CUDA(cudaMemcpyAsync(hp, pms[k], sizeof hp, cudaMemcpyDeviceToHost, d.stream));
      TP_CUDA(cudaStreamSynchronize(d.stream));
      P += hp[0];
      M += hp[1];
    }
  }
  *plus = P;
  *minus = M;
  return TP_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int tp_version(void) { return 200; }

const char* tp_last_error(void) { return g_err; }

int tp_device_count(int* count) {
  if (!count) return fail(TP_E_INVALID, "count must not be NULL");
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *count = 0;
    return fail(TP_E_NODEV, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  int ok = 0;
  for (int i = 0; i < c; ++i) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, i) == cudaSuccess && p.major == 10 && p.minor == 0) ok++;
  }
  *count = ok;
  return TP_OK;
}

int tp_device_info(int device, int* sm_count, int* max_clock_khz, int* cc_major, int* cc_minor) {
  Device* d;
  int rc = ensure_device(device, &d);
  if (rc) return rc;
  if (sm_count) *sm_count = d->sm_count;
  if (max_clock_khz) *max_clock_khz = d->max_clock_khz;
  if (cc_major) *cc_major = d->cc_major;
  if (cc_minor) *cc_minor = d->cc_minor;
  return TP_OK;
}

int tp_range_sum(const uint64_t* mags, const uint64_t* sgns, int n, uint64_t lo, uint64_t hi, int device,
                 uint64_t* plus, uint64_t* minus) {
  return range_sum_impl(mags, sgns, n, lo, hi, false, device, plus, minus);
}


int tp_range_sum_ex(const uint64_t* mags, const uint64_t* sgns, int n, uint64_t lo, uint64_t hi, int hi_is_2_64,
                    int device, uint64_t* plus, uint64_t* minus) {
  return range_sum_impl(mags, sgns, n, lo, hi, hi_is_2_64 != 0, device, plus, minus, true);
}

int tp_range_sum_async(const uint64_t* mags, const uint64_t* sgns, int n, uint64_t lo, uint64_t hi, int device,
                       uint64_t* d_pm, void* stream) {
  int rc = check_range(n, lo, hi);
  if (rc) return rc;
  if ((rc = check_planes(mags, sgns, n))) return rc;
  if (!d_pm) return fail(TP_E_INVALID, "d_pm must not be NULL");
  Device* d;
  if ((rc = ensure_device(device, &d))) return rc;
  std::lock_guard<std::mutex> lk(d->mu);
  TP_CUDA(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);  // 0 = legacy default stream, as in CUDA
  return enqueue_range(*d, mags, sgns, n, lo, hi, reinterpret_cast<unsigned long long*>(d_pm), st);
}

int tp_range_sum_multi(const uint64_t* mags, const uint64_t* sgns, int n, uint64_t lo, uint64_t hi,
                       const int* devices, int ndev, uint64_t* plus, uint64_t* minus) {
  return range_sum_multi_impl(mags, sgns, n, lo, hi, devices, ndev, false, plus, minus);
}

int tp_range_sum_nccl(const uint64_t* mags, const uint64_t* sgns, int n, uint64_t lo, uint64_t hi,
                      const int* devices, int ndev, uint64_t* plus, uint64_t* minus) {
  return range_sum_multi_impl(mags, sgns, n, lo, hi, devices, ndev, true, plus, minus);
}

int tp_perm_batch_async(const uint8_t* d_entries, int64_t B, int n, int device, int8_t* d_class, uint64_t* d_pm,
                        int64_t* d_hist, void* stream, int* launches) {
  if (n < 1 || n > TP_MAX_N) return fail(TP_E_INVALID, "need 1 <= n <= %d, got %d", TP_MAX_N, n);
  if (B < 0) return fail(TP_E_INVALID, "batch size must be >= 0");
  if (B > 0 && !d_entries) return fail(TP_E_INVALID, "d_entries must not be NULL");
  if (launches) *launches = 0;
  if (B == 0) return TP_OK;
  Device* d;
  int rc = ensure_device(device, &d);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(d->mu);
  TP_CUDA(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);  // 0 = legacy default stream, as in CUDA
  Scratch sc(st);
  void* mem = nullptr;
  const size_t rbytes = align_up((size_t)B * 64 * sizeof(RowRec), 256);
  if ((rc = sc.take(rbytes + (d_pm ? 0 : (size_t)B * 2 * sizeof(unsigned long long)), &mem))) return rc;
  RowRec* rows = static_cast<RowRec*>(mem);
  unsigned long long* pm = d_pm ? reinterpret_cast<unsigned long long*>(d_pm)
                                : reinterpret_cast<unsigned long long*>(static_cast<char*>(mem) + rbytes);
  int nl = 0;
  TP_CUDA(cudaMemsetAsync(pm, 0, (size_t)B * 2 * sizeof(unsigned long long), st));
  if (n <= tp::kSmallMaxN) {  // thread per matrix: pack + walk + finalise in one kernel
    TP_CUDA(tp::launch_small(n, B, d_entries, 0, 0, d_class, nullptr, pm, reinterpret_cast<long long*>(d_hist), st));
    if (launches) *launches = 1;
    return TP_OK;
  }
  const int pack_grid = (int)std::min<long long>((B + 7) / 8, (long long)d->sm_count * 8);
  TP_CUDA(tp::launch_pack(d_entries, B, n, rows, pack_grid, st));
  nl++;
  Plan pl;
  if ((rc = make_plan(*d, n, (unsigned long long)B, 0, 0, true, rows, pm, sc, pl))) return rc;
  if ((rc = run_plan(pl, st, &nl))) return rc;
  if (d_class || d_hist) {
    TP_CUDA(tp::launch_finalize(pm, B, n, d_class, nullptr, reinterpret_cast<long long*>(d_hist), st));
    nl++;
  }
  if (launches) *launches = nl;
  return TP_OK;
}

int tp_pack_async(const uint8_t* d_entries, int64_t B, int n, int device, void* d_rows, void* stream) {
  if (n < 1 || n > TP_MAX_N) return fail(TP_E_INVALID, "need 1 <= n <= %d, got %d", TP_MAX_N, n);
  if (B < 0) return fail(TP_E_INVALID, "batch size must be >= 0");
  if (B > 0 && (!d_entries || !d_rows)) return fail(TP_E_INVALID, "buffers must not be NULL");
  if (B == 0) return TP_OK;
  Device* d;
  int rc = ensure_device(device, &d);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(d->mu);
  TP_CUDA(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);  // 0 = legacy default stream, as in CUDA
  const int pack_grid = (int)std::min<long long>((B + 7) / 8, (long long)d->sm_count * 8);
  TP_CUDA(tp::launch_pack(d_entries, B, n, static_cast<RowRec*>(d_rows), pack_grid, st));
  return TP_OK;
}

int tp_walk_async(const void* d_rows, int64_t B, int n, int device, uint64_t* d_pm, void* stream, int* launches) {
  if (n < 1 || n > TP_MAX_N) return fail(TP_E_INVALID, "need 1 <= n <= %d, got %d", TP_MAX_N, n);
  if (B < 0) return fail(TP_E_INVALID, "batch size must be >= 0");
  if (B > 0 && (!d_rows || !d_pm)) return fail(TP_E_INVALID, "buffers must not be NULL");
  if (launches) *launches = 0;
  if (B == 0) return TP_OK;
  Device* d;
  int rc = ensure_device(device, &d);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(d->mu);
  TP_CUDA(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);  // 0 = legacy default stream, as in CUDA
  Scratch sc(st);
  Plan pl;
  if ((rc = make_plan(*d, n, (unsigned long long)B, 0, 0, true, static_cast<const RowRec*>(d_rows),
                      reinterpret_cast<unsigned long long*>(d_pm), sc, pl)))
    return rc;
  return run_plan(pl, st, launches);
}

int tp_walk_range_async(const void* d_rows, int n, uint64_t lo, uint64_t hi, int device, uint64_t* d_pm,
                        void* stream, int* launches) {
  int rc = check_range(n, lo, hi);
  if (rc) return rc;
  if (!d_rows || !d_pm) return fail(TP_E_INVALID, "buffers must not be NULL");
  if (launches) *launches = 0;
  Device* d;
  if ((rc = ensure_device(device, &d))) return rc;
  std::lock_guard<std::mutex> lk(d->mu);
  TP_CUDA(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Scratch sc(st);
  Plan pl;
  if ((rc = make_plan(*d, n, 1, lo, hi, false, static_cast<const RowRec*>(d_rows),
                      reinterpret_cast<unsigned long long*>(d_pm), sc, pl)))
    return rc;
  return run_plan(pl, st, launches);
}

int tp_finalize_async(const uint64_t* d_pm, int64_t B, int n, int device, int8_t* d_class, int64_t* d_hist,
                      void* stream) {
  if (n < 1 || n > TP_MAX_N) return fail(TP_E_INVALID, "need 1 <= n <= %d, got %d", TP_MAX_N, n);
  if (B < 0) return fail(TP_E_INVALID, "batch size must be >= 0");
  if (B > 0 && !d_pm) return fail(TP_E_INVALID, "d_pm must not be NULL");
  if (B == 0) return TP_OK;
  Device* d;
  int rc = ensure_device(device, &d);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(d->mu);
  TP_CUDA(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);  // 0 = legacy default stream, as in CUDA
  TP_CUDA(tp::launch_finalize(reinterpret_cast<const unsigned long long*>(d_pm), B, n, d_class, nullptr,
                              reinterpret_cast<long long*>(d_hist), st));
  return TP_OK;
}

// Debug: when d_trace != NULL, fast-walk launches record per warp
// (smid, clock64 start, clock64 end, items) into d_trace[4*warp].
int tp_debug_trace(void* d_trace) {
  g_trace = static_cast<unsigned long long*>(d_trace);
  return TP_OK;
}

int tp_exact_census(int n, int device, int64_t* zeros, int64_t* plus, int64_t* minus) {
  if (n < 1 || n > 6) return fail(TP_E_INVALID, "exact census supports 1 <= n <= 6, got n=%d", n);
  if (!zeros || !plus || !minus) return fail(TP_E_INVALID, "outputs must not be NULL");
  if (n == 1) {  // perm = the entry
    *zeros = *plus = *minus = 1;
    return TP_OK;
  }
  Device* d;
  int rc = ensure_device(device, &d);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(d->mu);
  TP_CUDA(cudaSetDevice(device));
  if ((rc = ensure_ws(*d, 256))) return rc;
  unsigned long long* n0 = static_cast<unsigned long long*>(d->ws);
  unsigned long long configs = 1;
  for (int e = 0; e < (n - 2) * n; ++e) configs *= 3ull;
  TP_CUDA(cudaMemsetAsync(n0, 0, sizeof(unsigned long long), d->stream));
  const unsigned long long blocks = (configs + 255) / 256;
  const int grid = (int)std::min<unsigned long long>(blocks, (unsigned long long)d->sm_count * 16);
  TP_CUDA(tp::launch_census(n, grid, configs, n0, d->stream));
  unsigned long long N0 = 0;
  TP_CUDA(cudaMemcpyAsync(&N0, n0, sizeof N0, cudaMemcpyDeviceToHost, d->stream));
  TP_CUDA(cudaStreamSynchronize(d->stream));
  unsigned long long p3 = 1, q3 = 1;  // 3^(n-1), 3^(n(n-1))
  for (int e = 0; e < n - 1; ++e) p3 *= 3ull;
  for (int e = 0; e < n * (n - 1); ++e) q3 *= 3ull;
  *zeros = (int64_t)(p3 * q3 + 2ull * p3 * N0);
  *plus = *minus = (int64_t)(p3 * (q3 - N0));
  return TP_OK;
}

int tp_walk_info(int n, long long batch, char* name, int name_len, double* lop3_per_term) {
  if (n < 1 || n > TP_MAX_N) return fail(TP_E_INVALID, "need 1 <= n <= %d, got %d", TP_MAX_N, n);
  if (batch < 1) return fail(TP_E_INVALID, "need batch >= 1, got %lld", batch);
  const int v = choose_variant(n, (unsigned long long)batch);
  if (bucket_applies(n, (unsigned long long)batch)) {
    // ALU-pipe ops per TESTED pair: the bucketed walk skips the incompatible
    // steps, so the tested fraction (tp_walk_tested) scales this per term
    const bool packed = bucket_mode() != 2;
    if (name && name_len > 0) {
      if (packed && batch_mode()) snprintf(name, (size_t)name_len, "k_walk_batch<packed> V=%d", tp::bucket_v(packed));
      else snprintf(name, (size_t)name_len, "k_walk_bucket<%s> V=%d", packed ? "packed" : "pair", tp::bucket_v(packed));
    }
    // k_walk_batch tests three entries per packed word with one zero-field
    // test (packed_test3): per word and entry 2 LOP3 + 1/3 VIMNMX3 + 1/3
    // LOP3 = 8/3 ALU-pipe ops for two pairs
    if (lop3_per_term) *lop3_per_term = !packed ? 2.0 : batch_mode() ? 4.0 / 3.0 : 1.5;
    return TP_OK;
  }
  const char* kind;
  double ops;
  if (n <= tp::kSmallMaxN) {
    kind = "k_small";  // batch / Monte Carlo path; ranges use the lane walk
    ops = 3.0;
  } else if (tp::fast_is_pair(v)) {
    kind = tp::fast_pair_wide(v) ? "k_walk_pair<wide>" : "k_walk_pair";
    ops = 2.0;
  } else if (tp::fast_is_packed(v)) {
    kind = v == tp::kPackedWideK32V4 ? "k_walk_packed<wide>" : "k_walk_packed";  // 3 LOP3 per word of two pairs
    ops = 1.5;
  } else if (tp::fast_is_lane(v)) {
    kind = "k_walk_lane";
    ops = 3.0;
  } else {
    kind = "k_walk_wide";
    ops = 3.0;
  }
  if (name && name_len > 0) snprintf(name, (size_t)name_len, "%s KB=%d V=%d", kind, tp::fast_kb(v), tp::fast_v(v));
  if (lop3_per_term) *lop3_per_term = ops;
  return TP_OK;
}

int tp_walk_tested(int device, uint64_t* pairs) {
  if (!pairs) return fail(TP_E_INVALID, "pairs must not be NULL");
  Device* d;
  int rc = ensure_device(device, &d);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(d->mu);
  TP_CUDA(cudaSetDevice(device));
  unsigned long long v = 0;
  TP_CUDA(cudaMemcpy(&v, d->bucket_tested, sizeof v, cudaMemcpyDeviceToHost));
  TP_CUDA(cudaMemset(d->bucket_tested, 0, sizeof v));
  *pairs = v;
  return TP_OK;
}

int tp_alu_peak(int device, double* lop3_ops_per_s, double* ms) {
  if (!lop3_ops_per_s) return fail(TP_E_INVALID, "lop3_ops_per_s must not be NULL");
  Device* d;
  int rc = ensure_device(device, &d);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(d->mu);
  TP_CUDA(cudaSetDevice(device));
  if ((rc = ensure_ws(*d, 1 << 20))) return rc;
  double ops = 0, t = 0;
  TP_CUDA(tp::run_alu_peak(d->sm_count, static_cast<uint32_t*>(d->ws), d->stream, &ops, &t));
  *lop3_ops_per_s = ops;
  if (ms) *ms = t;
  return TP_OK;
}

int tp_perm_batch(const uint8_t* entries, int64_t B, int n, int device, int8_t* out_class, int64_t* out_partial,
                  int64_t* hist) {
  if (n < 1 || n > TP_MAX_N) return fail(TP_E_INVALID, "need 1 <= n <= %d, got %d", TP_MAX_N, n);
  if (B < 0) return fail(TP_E_INVALID, "batch size must be >= 0");
  if (B > 0 && !entries) return fail(TP_E_INVALID, "entries must not be NULL");
  if (out_partial && n > 62) return fail(TP_E_INVALID, "raw partial sums only fit int64 for n <= 62");
  if (hist) hist[0] = hist[1] = hist[2] = 0;
  if (B == 0) return TP_OK;
  Device* d;
  int rc = ensure_device(device, &d);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(d->mu);
  TP_CUDA(cudaSetDevice(device));
  cudaStream_t st = d->stream;
  const size_t ebytes = (size_t)B * n * n;
  Carve cv;
  cv.take<RowRec>(nullptr, (size_t)B * 64);
  cv.take<unsigned long long>(nullptr, 1);
  cv.take<unsigned long long>(nullptr, (size_t)B * 2);
  cv.take<uint8_t>(nullptr, ebytes);
  cv.take<int8_t>(nullptr, (size_t)B);
  cv.take<long long>(nullptr, (size_t)B);
  cv.take<long long>(nullptr, 3);
  if ((rc = ensure_ws(*d, cv.off))) return rc;
  char* base = static_cast<char*>(d->ws);
  Carve c2;
  RowRec* rows = c2.take<RowRec>(base, (size_t)B * 64);
  unsigned long long* pm = c2.take<unsigned long long>(base, (size_t)B * 2);
  uint8_t* dent = c2.take<uint8_t>(base, ebytes);
  int8_t* dcls = c2.take<int8_t>(base, (size_t)B);
  long long* dpart = c2.take<long long>(base, (size_t)B);
  long long* dhist = c2.take<long long>(base, 3);
  TP_CUDA(cudaMemcpyAsync(dent, entries, ebytes, cudaMemcpyHostToDevice, st));
  TP_CUDA(cudaMemsetAsync(dhist, 0, 3 * sizeof(long long), st));
  if (n <= tp::kSmallMaxN) {
    TP_CUDA(tp::launch_small(n, B, dent, 0, 0, dcls, dpart, nullptr, dhist, st));
  } else {
    TP_CUDA(cudaMemsetAsync(pm, 0, (size_t)B * 2 * sizeof(unsigned long long), st));
    const int pack_grid = (int)std::min<long long>((B + 7) / 8, (long long)d->sm_count * 8);
    TP_CUDA(tp::launch_pack(dent, B, n, rows, pack_grid, st));
    Plan pl;
    Scratch sc(st);
    if ((rc = make_plan(*d, n, (unsigned long long)B, 0, 0, true, rows, pm, sc, pl))) return rc;
    if ((rc = run_plan(pl, st, nullptr))) return rc;
    TP_CUDA(tp::launch_finalize(pm, B, n, dcls, dpart, dhist, st));
  }
  if (out_class) TP_CUDA(cudaMemcpyAsync(out_class, dcls, (size_t)B, cudaMemcpyDeviceToHost, st));
  if (out_partial) TP_CUDA(cudaMemcpyAsync(out_partial, dpart, (size_t)B * 8, cudaMemcpyDeviceToHost, st));
  long long hh[3];
  unsigned long long tcerr = 0;
  TP_CUDA(cudaMemcpyAsync(hh, dhist, sizeof hh, cudaMemcpyDeviceToHost, st));
  TP_CUDA(cudaMemcpyAsync(&tcerr, d->tc_err, sizeof tcerr, cudaMemcpyDeviceToHost, st));
  TP_CUDA(cudaStreamSynchronize(st));
  if (tcerr) {
    TP_CUDA(cudaMemset(d->tc_err, 0, sizeof(unsigned long long)));
    return fail(TP_E_CUDA, "tensor path self-check failed on %llu terms", tcerr);
  }
  if (hist) {
    hist[0] = hh[0];
    hist[1] = hh[1];
    hist[2] = hh[2];
  }
  return TP_OK;
}

// Monte Carlo: device sampler -> walk -> finalize, in slabs so the RowRec
// workspace stays bounded.
static int mc_run(int n, int64_t t0, int64_t count, uint64_t seed, int device, int8_t* out_class, int64_t* hist) {
  if (n < 1 || n > TP_MAX_N) return fail(TP_E_INVALID, "need 1 <= n <= %d, got %d", TP_MAX_N, n);
  if (t0 < 0 || count < 0) return fail(TP_E_INVALID, "trial range must be non-negative");
  if (hist) hist[0] = hist[1] = hist[2] = 0;
  if (count == 0) return TP_OK;
  Device* d;
  int rc = ensure_device(device, &d);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(d->mu);
  TP_CUDA(cudaSetDevice(device));
  cudaStream_t st = d->stream;
  const bool small = n <= tp::kSmallMaxN;  // thread-per-trial kernel needs no row table
  // slabs large enough that mid-size n get whole-matrix items (row table 2 KB per trial)
  const int64_t slab = std::min<int64_t>(count, small ? (1ll << 24) : n <= 22 ? (1ll << 20) : (1ll << 16));
  const size_t nrows = small ? 0 : (size_t)slab * 64, npm = small ? 0 : (size_t)slab * 2;
  Carve cv;
  cv.take<RowRec>(nullptr, nrows);
  cv.take<unsigned long long>(nullptr, npm);
  cv.take<int8_t>(nullptr, (size_t)slab);
  cv.take<long long>(nullptr, 3);
  if ((rc = ensure_ws(*d, cv.off))) return rc;
  char* base = static_cast<char*>(d->ws);
  Carve c2;
  RowRec* rows = c2.take<RowRec>(base, nrows);
  unsigned long long* pm = c2.take<unsigned long long>(base, npm);
  int8_t* dcls = c2.take<int8_t>(base, (size_t)slab);
  long long* dhist = c2.take<long long>(base, 3);
  TP_CUDA(cudaMemsetAsync(dhist, 0, 3 * sizeof(long long), st));
  for (int64_t s0 = 0; s0 < count; s0 += slab) {
    const int64_t B = std::min<int64_t>(slab, count - s0);
    if (n <= tp::kSmallMaxN) {  // sample + walk + finalise, thread per trial
      TP_CUDA(tp::launch_small(n, B, nullptr, t0 + s0, seed, out_class ? dcls : nullptr, nullptr, nullptr, dhist, st));
    } else {
      TP_CUDA(cudaMemsetAsync(pm, 0, (size_t)B * 2 * sizeof(unsigned long long), st));
      TP_CUDA(tp::launch_sample(n, t0 + s0, B, seed, rows, nullptr, st));
      Plan pl;
      Scratch sc(st);
      if ((rc = make_plan(*d, n, (unsigned long long)B, 0, 0, true, rows, pm, sc, pl))) return rc;
      if ((rc = run_plan(pl, st, nullptr))) return rc;
      TP_CUDA(tp::launch_finalize(pm, B, n, dcls, nullptr, dhist, st));
    }
    if (out_class) TP_CUDA(cudaMemcpyAsync(out_class + s0, dcls, (size_t)B, cudaMemcpyDeviceToHost, st));
    if (out_class) TP_CUDA(cudaStreamSynchronize(st));
  }
  long long hh[3];
  unsigned long long tcerr = 0;
  TP_CUDA(cudaMemcpyAsync(hh, dhist, sizeof hh, cudaMemcpyDeviceToHost, st));
  TP_CUDA(cudaMemcpyAsync(&tcerr, d->tc_err, sizeof tcerr, cudaMemcpyDeviceToHost, st));
  TP_CUDA(cudaStreamSynchronize(st));
  if (tcerr) {
    TP_CUDA(cudaMemset(d->tc_err, 0, sizeof(unsigned long long)));
    return fail(TP_E_CUDA, "tensor path self-check failed on %llu terms", tcerr);
  }
  if (hist) {
    hist[0] = hh[0];
    hist[1] = hh[1];
    hist[2] = hh[2];
  }
  return TP_OK;
}

int tp_mc_zero_count(int n, int64_t t0, int64_t t1, uint64_t seed, int device, int64_t* zeros, int64_t* hist) {
  if (!zeros) return fail(TP_E_INVALID, "zeros must not be NULL");
  if (t1 < t0) return fail(TP_E_INVALID, "need t0 <= t1");
  int64_t h[3];
  int rc = mc_run(n, t0, t1 - t0, seed, device, nullptr, h);
  if (rc) return rc;
  *zeros = h[0];
  if (hist) {
    hist[0] = h[0];
    hist[1] = h[1];
    hist[2] = h[2];
  }
  return TP_OK;
}

int tp_mc_classes(int n, int64_t t0, int64_t count, uint64_t seed, int device, int8_t* out_class) {
  if (!out_class && count > 0) return fail(TP_E_INVALID, "out_class must not be NULL");
  return mc_run(n, t0, count, seed, device, out_class, nullptr);
}

int tp_sample_classes(int n, int64_t t0, int64_t count, uint64_t seed, int device, uint8_t* out, int out_on_device,
                      void* stream) {
  if (n < 1 || n > TP_MAX_N) return fail(TP_E_INVALID, "need 1 <= n <= %d, got %d", TP_MAX_N, n);
  if (t0 < 0 || count < 0) return fail(TP_E_INVALID, "trial range must be non-negative");
  if (count > 0 && !out) return fail(TP_E_INVALID, "out must not be NULL");
  if (count == 0) return TP_OK;
  Device* d;
  int rc = ensure_device(device, &d);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(d->mu);
  TP_CUDA(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);  // 0 = legacy default stream, as in CUDA
  if (out_on_device) {
    TP_CUDA(tp::launch_sample(n, t0, count, seed, nullptr, out, st));
    return TP_OK;
  }
  const size_t bytes = (size_t)count * n * n;
  if ((rc = ensure_ws(*d, bytes))) return rc;
  uint8_t* ent = static_cast<uint8_t*>(d->ws);
  TP_CUDA(tp::launch_sample(n, t0, count, seed, nullptr, ent, st));
  TP_CUDA(cudaMemcpyAsync(out, ent, bytes, cudaMemcpyDeviceToHost, st));
  TP_CUDA(cudaStreamSynchronize(st));
  return TP_OK;
}

int tp_mc_sample_entries(int n, int64_t trial, uint64_t seed, int device, int8_t* out) {
  if (!out) return fail(TP_E_INVALID, "out must not be NULL");
  int rc = tp_sample_classes(n, trial, 1, seed, device, reinterpret_cast<uint8_t*>(out), 0, nullptr);
  if (rc) return rc;
  for (int k = 0; k < n * n; ++k)
    if (out[k] == 2) out[k] = -1;  // centred, as src/_kernels.py:258-272 returns
  return TP_OK;
}

int tp_selftest_ops(const uint32_t* in, int count, int op, int device, uint32_t* out) {
  if (count < 0 || (count > 0 && (!in || !out))) return fail(TP_E_INVALID, "bad buffers");
  if (op < 0 || op > 2) return fail(TP_E_INVALID, "op must be 0 (add), 1 (sub) or 2 (walk add)");
  if (count == 0) return TP_OK;
  Device* d;
  int rc = ensure_device(device, &d);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(d->mu);
  TP_CUDA(cudaSetDevice(device));
  Carve cv;
  cv.take<uint32_t>(nullptr, (size_t)count * 4);
  cv.take<uint32_t>(nullptr, (size_t)count * 2);
  if ((rc = ensure_ws(*d, cv.off))) return rc;
  char* base = static_cast<char*>(d->ws);
  Carve c2;
  uint32_t* din = c2.take<uint32_t>(base, (size_t)count * 4);
  uint32_t* dout = c2.take<uint32_t>(base, (size_t)count * 2);
  TP_CUDA(cudaMemcpyAsync(din, in, (size_t)count * 16, cudaMemcpyHostToDevice, d->stream));
  TP_CUDA(tp::launch_selftest(din, count, op, dout, d->stream));
  TP_CUDA(cudaMemcpyAsync(out, dout, (size_t)count * 8, cudaMemcpyDeviceToHost, d->stream));
  TP_CUDA(cudaStreamSynchronize(d->stream));
  return TP_OK;
}

}  // extern "C"
