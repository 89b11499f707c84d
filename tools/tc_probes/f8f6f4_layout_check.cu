// Prototype: tcgen05.mma kind::f8f6f4 (e4m3) M=128 N=128 K=64, f16 or f32 accumulate, SWIZZLE_NONE K-major.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version for sm100
  return d;  // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

// canonical no-swizzle K-major: row r, byte kb -> (r/8)*SBO + (kb/16)*LBO + (r%8)*16 + kb%16
__device__ __forceinline__ uint32_t canon_off(int r, int kb, int LBO, int SBO) {
  return (r >> 3) * SBO + (kb >> 4) * LBO + (r & 7) * 16 + (kb & 15);
}

template <bool F16ACC, int LBO, int SBO>
__global__ void k_proto(const uint8_t* A, const uint8_t* B, uint32_t* out_raw, uint32_t* out_pack) {
  constexpr int M = 128, N = 128, K = 64;
  __shared__ __align__(1024) uint8_t sA[M * K];
  __shared__ __align__(1024) uint8_t sB[N * K];
  __shared__ uint32_t s_taddr;
  __shared__ __align__(8) uint64_t mbar;
  int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < M * K; i += blockDim.x) sA[canon_off(i / K, i % K, LBO, SBO)] = A[i];
  for (int i = tid; i < N * K; i += blockDim.x) sB[canon_off(i / K, i % K, LBO, SBO)] = B[i];
  asm volatile("fence.proxy.async.shared::cta;");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"((uint32_t)__cvta_generic_to_shared(&s_taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t taddr = s_taddr;
  if (tid == 0) {
    uint32_t idesc = 0;
    idesc |= (F16ACC ? 0u : 1u) << 4;  // c_format
    idesc |= 0u << 7;                   // a e4m3
    idesc |= 0u << 10;                  // b e4m3
    idesc |= (uint32_t)(N >> 3) << 17;
    idesc |= (uint32_t)(M >> 4) << 24;
    uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sA), b0 = (uint32_t)__cvta_generic_to_shared(sB);
    for (int ks = 0; ks < K / 32; ks++) {
      uint64_t da = smem_desc(a0 + ks * 2 * LBO, LBO, SBO);
      uint64_t db = smem_desc(b0 + ks * 2 * LBO, LBO, SBO);
      uint32_t acc = ks > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
                   :: "r"(taddr), "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(&mbar)));
  }
  // wait phase 0
  {
    uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(mb), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // each warp reads its 32 lanes; 128 columns
  uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  for (int c = 0; c < 128; c += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]) : "r"(taddr + lane_base + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; j++) out_raw[tid * 128 + c + j] = r[j];
  }
  for (int c = 0; c < 128; c += 16) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]) : "r"(taddr + lane_base + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; j++) out_pack[tid * 64 + c / 2 + j] = r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(taddr));
}

static float e4m3_to_f(uint8_t b) {
  int s = b >> 7, e = (b >> 3) & 15, m = b & 7;
  float v = e ? ldexpf(1.0f + m / 8.0f, e - 7) : ldexpf(m / 8.0f, -6);
  return s ? -v : v;
}
static float h2f(uint16_t h) {
  int s = h >> 15, e = (h >> 10) & 31, m = h & 1023;
  float v = e ? ldexpf(1.0f + m / 1024.0f, e - 15) : ldexpf(m / 1024.0f, -14);
  return s ? -v : v;
}

int main() {
  const int M = 128, N = 128, K = 64;
  uint8_t vals[5] = {0x00, 0x38, 0xB8, 0x40, 0xC0};  // 0, 1, -1, 2, -2
  uint8_t *hA = (uint8_t*)malloc(M * K), *hB = (uint8_t*)malloc(N * K);
  srand(1);
  for (int i = 0; i < M * K; i++) hA[i] = vals[rand() % 3];
  for (int i = 0; i < N * K; i++) hB[i] = vals[rand() % 5];
  float* ref = (float*)malloc(M * N * 4);
  for (int i = 0; i < M; i++)
    for (int j = 0; j < N; j++) {
      float s = 0;
      for (int k = 0; k < K; k++) s += e4m3_to_f(hA[i * K + k]) * e4m3_to_f(hB[j * K + k]);
      ref[i * N + j] = s;
    }
  uint8_t *dA, *dB; uint32_t *draw, *dpack;
  cudaMalloc(&dA, M * K); cudaMalloc(&dB, N * K); cudaMalloc(&draw, M * 128 * 4); cudaMalloc(&dpack, M * 64 * 4);
  cudaMemcpy(dA, hA, M * K, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, N * K, cudaMemcpyHostToDevice);
  uint32_t* hraw = (uint32_t*)malloc(M * 128 * 4); uint32_t* hpack = (uint32_t*)malloc(M * 64 * 4);
  for (int variant = 0; variant < 4; variant++) {
    bool f16 = variant & 1; bool swap = variant & 2;
    cudaMemset(draw, 0xEE, M * 128 * 4);
    if (!f16 && !swap) k_proto<false, 128, 512><<<1, 128>>>(dA, dB, draw, dpack);
    if (f16 && !swap) k_proto<true, 128, 512><<<1, 128>>>(dA, dB, draw, dpack);
    if (!f16 && swap) k_proto<false, 1024, 128><<<1, 128>>>(dA, dB, draw, dpack);
    if (f16 && swap) k_proto<true, 1024, 128><<<1, 128>>>(dA, dB, draw, dpack);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant f16=%d swapLBO=%d: %s\n", f16, swap, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    cudaMemcpy(hraw, draw, M * 128 * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hpack, dpack, M * 64 * 4, cudaMemcpyDeviceToHost);
    int bad = 0, badp = 0;
    for (int i = 0; i < M; i++)
      for (int j = 0; j < N; j++) {
        float got = f16 ? h2f(hraw[i * 128 + j] & 0xFFFF) : __builtin_bit_cast(float, hraw[i * 128 + j]);
        if (got != ref[i * N + j]) { if (bad < 3) printf("  raw (%d,%d) got %g (0x%08x) want %g\n", i, j, got, hraw[i*128+j], ref[i * N + j]); bad++; }
        if (f16) {
          uint32_t w = hpack[i * 64 + j / 2];
          float gp = h2f((j & 1) ? (w >> 16) : (w & 0xFFFF));
          if (gp != ref[i * N + j]) { if (badp < 3) printf("  pack (%d,%d) got %g want %g\n", i, j, gp, ref[i * N + j]); badp++; }
        }
      }
    printf("  raw mismatches %d, pack mismatches %d; sample raw[0..3]=%08x %08x %08x %08x\n", bad, badp, hraw[0], hraw[1], hraw[2], hraw[3]);
  }
  return 0;
}
