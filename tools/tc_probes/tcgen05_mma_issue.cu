// MMA throughput microbenchmark: tcgen05.mma kind::f8f6f4 M=128 N=128 K=32, SS, no swizzle.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
template <int F16, int NN, int BATCH>
__global__ void k(int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 65536; i += blockDim.x) sm[i] = (i * 7) & 0x38;
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    uint32_t idesc = ((F16 ? 0u : 1u) << 4) | ((uint32_t)(NN >> 3) << 17) | (8u << 24);
    uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sm), b0 = a0 + 32768;
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
      for (int m = 0; m < BATCH; m++) {
        uint64_t da = umma_desc(a0 + (m & 1) * 256, 128, 512);
        uint64_t db = umma_desc(b0 + (m & 1) * 256, 128, 512);
        uint32_t d = taddr + (m & 3) * 128;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
          :: "r"(d), "l"(da), "l"(db), "r"(idesc), "r"(m & 1));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(&bar)));
      uint32_t done = 0;
      while (!done) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(ph));
      ph ^= 1;
    }
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(taddr));
}

template <int SPREAD, int COMMITS>
__global__ void k2(int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr;
  __shared__ __align__(8) uint64_t bar[8];
  for (int i = threadIdx.x; i < 131072; i += blockDim.x) sm[i] = (i * 7) & 0x38;
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { for (int i = 0; i < 8; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&bar[i]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    uint32_t idesc = (16u << 17) | (8u << 24);
    uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sm), b0 = a0 + 65536;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
      for (int mt = 0; mt < 2; mt++) {
        for (int k = 0; k < 2; k++) {
          uint32_t aoff = SPREAD ? ((it & 1) * 2 + mt) * 8192 : 0;
          uint32_t boff = SPREAD ? (it & 3) * 8192 : 0;
          uint64_t da = umma_desc(a0 + aoff + k * 256, 128, 512);
          uint64_t db = umma_desc(b0 + boff + k * 256, 128, 512);
          uint32_t d = taddr + ((2 * it + mt) & 3) * 128;
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
            :: "r"(d), "l"(da), "l"(db), "r"(idesc), "r"(k));
        }
        if (COMMITS) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(&bar[mt])));
      }
      if (COMMITS) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(&bar[2])));
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(&bar[7])));
    uint32_t done = 0;
    while (!done) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(&bar[7])), "r"(0));
    cyc[blockIdx.x] = clock64() - t0;
    cyc[256 + blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(taddr));
}
int main() {
  long long* cyc; cudaMalloc(&cyc, 8 * 1024);
  auto run = [&](auto kern, const char* name, int batch, int nn) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    int iters = 2000;
    kern<<<148, 128, 140 * 1024>>>(10, cyc);
    kern<<<148, 128, 140 * 1024>>>(iters, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double per = (double)c / (iters * (double)batch);
    printf("%s: %s  %.1f clk per MMA (M=128 N=%d K=32) -> %.0f MAC/clk\n", name, cudaGetErrorString(e), per, nn, 128.0 * nn * 32 / per);
  };
  auto run2 = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int iters = 2000;
    kern<<<148, 128, 200 * 1024>>>(10, cyc);
    kern<<<148, 128, 200 * 1024>>>(iters, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    long long c[512]; cudaMemcpy(c, cyc, 8 * 512, cudaMemcpyDeviceToHost);
    printf("%s: %s  %.1f clk per MMA total, issue loop %.1f clk per MMA\n", name, cudaGetErrorString(e), (double)c[0] / (iters * 4.0), (double)c[256] / (iters * 4.0));
  };
  run2(k2<0, 0>, "pattern same-addr no-commit");
  run2(k2<0, 1>, "pattern same-addr commits");
  run2(k2<1, 0>, "pattern spread no-commit");
  run2(k2<1, 1>, "pattern spread commits");
  run(k<1, 128, 4>, "f16 N128 batch4", 4, 128);
  run(k<1, 128, 16>, "f16 N128 batch16", 16, 128);
  run(k<0, 128, 16>, "f32 N128 batch16", 16, 128);

  return 0;
}
