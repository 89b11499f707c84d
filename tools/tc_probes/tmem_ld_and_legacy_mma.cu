// Microbenchmarks: tcgen05.ld (TMEM read) throughput and legacy IMMA throughput on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int X>
__device__ __forceinline__ void tld(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void tld<32>(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
    : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),
      "=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31])
    : "r"(taddr));
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_tmem(uint32_t* out, int iters, long long* cyc) {
  __shared__ uint32_t s_taddr;
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&s_taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t taddr = s_taddr;
  uint32_t lane_base = (uint32_t)((warp % 4) * 32) << 16;
  uint32_t col0 = ((warp / 4) % 2) * 256;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    uint32_t r[32];
    tld<32>(taddr + lane_base + col0 + (i & 7) * 32, r);
    asm volatile("tcgen05.wait::ld.sync.aligned;");
acc ^= r[0] ^ r[31];
  }
  long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(taddr));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// 4 independent IMMA m16n8k32 s8 chains per warp.
__global__ void k_imma(const uint32_t* in, int* out, int iters) {
  uint32_t a0 = in[threadIdx.x & 31], a1 = in[(threadIdx.x + 1) & 31], a2 = in[(threadIdx.x + 2) & 31], a3 = in[(threadIdx.x + 3) & 31];
  uint32_t b0 = in[(threadIdx.x + 4) & 31], b1 = in[(threadIdx.x + 5) & 31];
  int d[4][4] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int c = 0; c < 4; c++)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
  for (int c = 0; c < 4; c++) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// e4m3 m16n8k32 f32 legacy
__global__ void k_fmma(const uint32_t* in, float* out, int iters) {
  uint32_t a0 = in[threadIdx.x & 31], a1 = in[(threadIdx.x + 1) & 31], a2 = in[(threadIdx.x + 2) & 31], a3 = in[(threadIdx.x + 3) & 31];
  uint32_t b0 = in[(threadIdx.x + 4) & 31], b1 = in[(threadIdx.x + 5) & 31];
  float d[4][4] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int c = 0; c < 4; c++)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.f32.e4m3.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int c = 0; c < 4; c++) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out; cudaMalloc(&out, 1 << 24);
  long long* cyc; cudaMalloc(&cyc, 8 * 1024);
  uint32_t* in; cudaMalloc(&in, 4096); cudaMemset(in, 1, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  auto run_tmem = [&](auto kern, int nw, const char* name) {
    int iters = 20000;
    kern<<<nsm, nw * 32>>>(out, 100, cyc);
    cudaEventRecord(e0);
    kern<<<nsm, nw * 32>>>(out, iters, cyc);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double bytes = (double)nsm * nw * 32 * 32 * 4.0 * iters;
    printf("%s: err=%s %.3f ms  %.1f TB/s total, %.1f B/clk/SM (clock64 %lld cyc)\n", name, cudaGetErrorString(cudaGetLastError()), ms,
           bytes / ms / 1e9, bytes / nsm / ((double)c), c);
  };
  run_tmem(k_tmem<4>, 4, "tcgen05.ld 32x32b.x32 4 warps");
  run_tmem(k_tmem<8>, 8, "tcgen05.ld 32x32b.x32 8 warps");
  run_tmem(k_tmem<16>, 16, "tcgen05.ld 32x32b.x32 16 warps");
  for (int nw : {4, 8, 16}) {
    int iters = 20000;
    k_imma<<<nsm, nw * 32>>>(in, (int*)out, 100);
    cudaEventRecord(e0);
    k_imma<<<nsm, nw * 32>>>(in, (int*)out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double macs = (double)nsm * nw * 4 * iters * 16 * 8 * 32;
    printf("IMMA s8 m16n8k32 %d warps/SM: err=%s %.3f ms  %.1f TMAC/s  %.0f MAC/clk/SM at %d MHz\n", nw, cudaGetErrorString(cudaGetLastError()), ms, macs / ms / 1e9,
           macs / ms / 1e-3 / nsm / (clk * 1e3), clk / 1000);
    k_fmma<<<nsm, nw * 32>>>(in, (float*)out, 100);
    cudaEventRecord(e0);
    k_fmma<<<nsm, nw * 32>>>(in, (float*)out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("QMMA e4m3 m16n8k32 %d warps/SM: err=%s %.3f ms  %.1f TMAC/s  %.0f MAC/clk/SM\n", nw, cudaGetErrorString(cudaGetLastError()), ms, macs / ms / 1e9,
           macs / ms / 1e-3 / nsm / (clk * 1e3));
  }
  return 0;
}
