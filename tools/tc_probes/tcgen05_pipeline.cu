// Pipeline microbenchmark: MMA issuer + producer + epilogue handshakes, no real work.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  do asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(su(b)), "r"(ph) : "memory");
  while (!done);
}
__device__ __forceinline__ void commit(uint64_t* b) { asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(b)) : "memory"); }

// NEPI: number of epilogue warps per slot (each arrives once); MMA warp = last warp
template <int NEPI, int KS, int DATA = 0, int FENCE = 1>
__global__ void k(int tiles, long long* cyc, uint32_t* tr) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr;
  __shared__ __align__(8) uint64_t full[4], empty[4], tfull[4], tempty[4];
  const int nw = blockDim.x / 32, warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int mmaw = nw - 1, prodw = nw - 2;
  for (int i = threadIdx.x; i < 65536; i += blockDim.x) {
    const uint32_t h = (uint32_t)i * 2654435761u;
    const uint8_t vals[4] = {0x38, 0xB8, 0x40, 0xC0};
    sm[i] = DATA == 0 ? ((i * 7) & 0x38) : DATA == 1 ? vals[(h >> 13) & 3] : 0;
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (warp == mmaw) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su(&taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; i++) { init(&full[i], 32); init(&empty[i], 1); init(&tfull[i], 1); init(&tempty[i], NEPI); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  long long t0 = clock64();
  if (warp == mmaw) {
    if (lane == 0) {
      uint32_t idesc = (16u << 17) | (8u << 24);
      uint32_t a0 = su(sm), b0 = a0 + 32768;
      uint32_t bs = 0, bph = 0, sl = 0, sph = 0;
      for (int T = 0; T < tiles; T++) {
        wait(&full[bs], bph);
        for (int mt = 0; mt < 2; mt++) {
          const int idx = 2 * T + mt;
          if (blockIdx.x == 0 && idx < 64) tr[idx * 8 + 0] = (uint32_t)clock64();
          wait(&tempty[sl], sph ^ 1);
          if (blockIdx.x == 0 && idx < 64) tr[idx * 8 + 1] = (uint32_t)clock64();
          if (FENCE) asm volatile("tcgen05.fence::after_thread_sync;");
          for (int k = 0; k < KS; k++) {
            uint64_t da = umma_desc(a0 + mt * 8192 + k * 256, 128, 512);
            uint64_t db = umma_desc(b0 + bs * 8192 + k * 256, 128, 512);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
              :: "r"(taddr + sl * 128), "l"(da), "l"(db), "r"(idesc), "r"(k));
          }
          commit(&tfull[sl]);
          if (blockIdx.x == 0 && idx < 64) tr[idx * 8 + 2] = (uint32_t)clock64();
          if (++sl == 4) { sl = 0; sph ^= 1; }
        }
        commit(&empty[bs]);
        if (++bs == 4) { bs = 0; bph ^= 1; }
      }
    }
  } else if (warp == prodw) {
    uint32_t bs = 0, bph = 0;
    for (int T = 0; T < tiles; T++) {
      wait(&empty[bs], bph ^ 1);
      asm volatile("fence.proxy.async.shared::cta;");
      arrive(&full[bs]);
      if (++bs == 4) { bs = 0; bph ^= 1; }
    }
  } else if (warp < 4 * NEPI) {
    const int grp = warp / NEPI;  // slot
    uint32_t sph = 0;
    for (int T = grp >> 1; T < tiles; T += 2) {
      const int idx = 2 * T + (grp & 1);
      wait(&tfull[grp], sph);
      if (blockIdx.x == 0 && idx < 64 && lane == 0 && (warp % NEPI) == 0) tr[idx * 8 + 3] = (uint32_t)clock64();
      asm volatile("tcgen05.fence::after_thread_sync;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) arrive(&tempty[grp]);
      if (blockIdx.x == 0 && idx < 64 && lane == 0 && (warp % NEPI) == 0) tr[idx * 8 + 4] = (uint32_t)clock64();
      sph ^= 1;
    }
  }
  long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 32 * mmaw) cyc[blockIdx.x] = t1 - t0;
  if (warp == mmaw) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(taddr));
}
int main() {
  long long* cyc; cudaMalloc(&cyc, 8 * 1024);
  uint32_t* tr; cudaMalloc(&tr, 64 * 8 * 4);
  auto run = [&](auto kern, int threads, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    int tiles = 4096;
    kern<<<148, threads, 120 * 1024>>>(16, cyc, tr);
    kern<<<148, threads, 120 * 1024>>>(tiles, cyc, tr);
    cudaError_t e = cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%s: %s %.0f clk/tile\n", name, cudaGetErrorString(e), (double)c / tiles);
    uint32_t h[512]; cudaMemcpy(h, tr, sizeof h, cudaMemcpyDeviceToHost);
    printf("  idx  pre   go   committed  epi_obs  epi_arr\n");
    for (int i = 16; i < 32; i++) printf("  %2d %6d %6d %6d %6d %6d\n", i, (int)(h[i*8]-h[0]), (int)(h[i*8+1]-h[0]), (int)(h[i*8+2]-h[0]), (int)(h[i*8+3]-h[0]), (int)(h[i*8+4]-h[0]));
  };
  run(k<4, 2>, 32 * 18, "KS=2 NEPI=4 (18 warps)");
  return 0;
}
