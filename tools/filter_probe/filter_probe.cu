// filter_probe.cu -- micro-benchmark of packed pair-test formulations for the
// bucketed walk's filter loop (tp_walk_bucket.cu).  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o filter_probe filter_probe.cu
//   ./filter_probe            (prints tests/clk/SM per variant and checks the masks)
// Each warp holds 16 packed A words (two slots' low 16 columns each) in
// registers and streams pairs of doubled B states from shared memory; a
// "test" is one packed word against one B state (two pairs).
//   V0  the current test: 2 LOP3, IMAD (zp - 0x00010001), LOP3.P, @P IMAD into M
//   V1  2 LOP3, HSET2.EQ (f16x2 zero compare), HFMA2 into three f16x2 accumulators
//   V2  2 LOP3, HSETP2 (two predicates), OR, @P IMAD into M
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define FULL 0xffffffffu
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

#include <utility>
template <typename F, int... I>
__device__ __forceinline__ void sfor_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void sfor(F&& f) { sfor_impl(f, std::make_integer_sequence<int, N>{}); }

__device__ __forceinline__ uint32_t zp_of(uint32_t z1, uint32_t g1, uint32_t z2, uint32_t u2) {
  uint32_t d, zp;
  asm("lop3.b32 %0, %1, %2, %3, 0x06;" : "=r"(d) : "r"(z1), "r"(g1), "r"(u2));
  asm("lop3.b32 %0, %1, %2, %3, 0x09;" : "=r"(zp) : "r"(d), "r"(z1), "r"(z2));
  return zp;
}

template <uint32_t BIT>
__device__ __forceinline__ void t_v0(uint32_t z1, uint32_t g1, uint32_t z2, uint32_t u2, uint32_t& m, uint32_t one, uint32_t cneg) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 d, zp, t, h;\n\t"
      "lop3.b32 d, %1, %2, %4, 0x06;\n\t"
      "lop3.b32 zp, d, %1, %3, 0x09;\n\t"
      "mad.lo.u32 t, zp, %5, %6;\n\t"
      "lop3.b32 h, t, 0x80008000, zp, 0x40;\n\t"
      "setp.ne.u32 p, h, 0;\n\t"
      "@p mad.lo.u32 %0, %5, %7, %0;\n\t}"
      : "+r"(m) : "r"(z1), "r"(g1), "r"(z2), "r"(u2), "r"(one), "r"(cneg), "n"(BIT));
}

// f16 weight 2^k as f16x2 bits
__host__ __device__ constexpr uint32_t h2pow(int k) { return (uint32_t)((15 + k) << 10) * 0x10001u; }

template <uint32_t C>
__device__ __forceinline__ void t_v1(uint32_t z1, uint32_t g1, uint32_t z2, uint32_t u2, uint32_t& acc) {
  asm volatile(
      "{\n\t.reg .b32 d, zp, r;\n\t"
      "lop3.b32 d, %1, %2, %4, 0x06;\n\t"
      "lop3.b32 zp, d, %1, %3, 0x09;\n\t"
      "set.eq.f16x2.f16x2 r, zp, %6;\n\t"
      "fma.rn.f16x2 %0, r, %5, %0;\n\t}"
      : "+r"(acc) : "r"(z1), "r"(g1), "r"(z2), "r"(u2), "r"(C), "r"(0u));
}

template <uint32_t BIT>
__device__ __forceinline__ void t_v2(uint32_t z1, uint32_t g1, uint32_t z2, uint32_t u2, uint32_t& m, uint32_t one) {
  asm volatile(
      "{\n\t.reg .pred p, q, pq;\n\t.reg .b32 d, zp;\n\t"
      "lop3.b32 d, %1, %2, %4, 0x06;\n\t"
      "lop3.b32 zp, d, %1, %3, 0x09;\n\t"
      "setp.eq.f16x2 p|q, zp, %7;\n\t"
      "or.pred pq, p, q;\n\t"
      "@pq mad.lo.u32 %0, %5, %6, %0;\n\t}"
      : "+r"(m) : "r"(z1), "r"(g1), "r"(z2), "r"(u2), "r"(one), "n"(BIT), "r"(0u));
}

// V3: fields are 15 bits (A z bits 15/31 set, B z bits 15/31 clear, so zp
// bits 15/31 are 0); t = zp - 0x00010001 borrows into bit 15 / 31 iff a field
// is zero; the two tests of word w (steps a, b) share one LOP3.P
template <uint32_t BIT>
__device__ __forceinline__ void t_v3(uint32_t z1, uint32_t g1, uint32_t za, uint32_t ua, uint32_t zb, uint32_t ub,
                                     uint32_t& m, uint32_t one, uint32_t cneg) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 da, zpa, ta, db, zpb, tb, h;\n\t"
      "lop3.b32 da, %1, %2, %4, 0x06;\n\t"
      "lop3.b32 zpa, da, %1, %3, 0x09;\n\t"
      "lop3.b32 db, %1, %2, %6, 0x06;\n\t"
      "lop3.b32 zpb, db, %1, %5, 0x09;\n\t"
      "mad.lo.u32 ta, zpa, %7, %8;\n\t"
      "mad.lo.u32 tb, zpb, %7, %8;\n\t"
      "lop3.b32 h, ta, tb, 0x80008000, 0xA8;\n\t"
      "setp.ne.u32 p, h, 0;\n\t"
      "@p mad.lo.u32 %0, %7, %9, %0;\n\t}"
      : "+r"(m) : "r"(z1), "r"(g1), "r"(za), "r"(ua), "r"(zb), "r"(ub), "r"(one), "r"(cneg), "n"(BIT));
}

// V4: three B entries against word w share one zero-field test: the
// halfword-wise minimum of the three zp words (VIMNMX3.U16x2) has a zero
// field iff one of them has; bit w of m = a pass of word w by any of the three
template <uint32_t BIT>
__device__ __forceinline__ void t_v4(uint32_t z1, uint32_t g1, uint32_t za, uint32_t ua, uint32_t zb, uint32_t ub,
                                     uint32_t zc, uint32_t uc, uint32_t& m, uint32_t one, uint32_t cneg) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 da, zpa, db, zpb, dc, zpc, mn, t, h;\n\t"
      "lop3.b32 da, %1, %2, %4, 0x06;\n\t"
      "lop3.b32 zpa, da, %1, %3, 0x09;\n\t"
      "lop3.b32 db, %1, %2, %6, 0x06;\n\t"
      "lop3.b32 zpb, db, %1, %5, 0x09;\n\t"
      "lop3.b32 dc, %1, %2, %8, 0x06;\n\t"
      "lop3.b32 zpc, dc, %1, %7, 0x09;\n\t"
      "min.u16x2 mn, zpa, zpb;\n\t"
      "min.u16x2 mn, mn, zpc;\n\t"
      "mad.lo.u32 t, mn, %9, %10;\n\t"
      "lop3.b32 h, t, 0x80008000, mn, 0x40;\n\t"
      "setp.ne.u32 p, h, 0;\n\t"
      "@p mad.lo.u32 %0, %9, %11, %0;\n\t}"
      : "+r"(m) : "r"(z1), "r"(g1), "r"(za), "r"(ua), "r"(zb), "r"(ub), "r"(zc), "r"(uc), "r"(one), "r"(cneg), "n"(BIT));
}

// decode the three V1 accumulators into the V0 mask layout (bit w: step a word w,
// bit 16 + w: step b word w); index i = w (a) or 16 + w (b), acc0: i 0..10,
// acc1: i 11..21, acc2: i 22..31, weight 2^(i - base)
__device__ __forceinline__ uint32_t v1_mask(uint32_t a0, uint32_t a1, uint32_t a2) {
  auto dec = [](uint32_t a) -> uint32_t {
    const uint32_t lo = (uint32_t)__half2float(__ushort_as_half((unsigned short)(a & 0xffff)));
    const uint32_t hi = (uint32_t)__half2float(__ushort_as_half((unsigned short)(a >> 16)));
    return lo | hi;
  };
  return dec(a0) | (dec(a1) << 11) | (dec(a2) << 22);
}

struct Out { unsigned long long hits, sum; };

template <int V, int MINB = 4>
__global__ void __launch_bounds__(128, MINB) k_probe(const uint32_t* A, const uint2* B, int nB, int reps, uint32_t* masks, int record, unsigned long long* res) {
  __shared__ __align__(16) uint2 Hc[4][1024];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = lane; i < nB; i += 32) {
    const uint2 b = B[i];
    Hc[warp][i] = make_uint2(__byte_perm(b.x, b.x, 0x1010), __byte_perm(b.y, b.y, 0x1010));
  }
  uint32_t Zp[16], Gp[16];
  const uint32_t gl = blockIdx.x * 128 + threadIdx.x;
#pragma unroll
  for (int w = 0; w < 16; ++w) { Zp[w] = A[(gl % 4096) * 32 + 2 * w]; Gp[w] = A[(gl % 4096) * 32 + 2 * w + 1]; }
  __syncwarp();
  const uint32_t one = res ? 1u : 0u;  // runtime 1
  const uint32_t cneg = 0xfffeffffu * one;
  unsigned long long hits = 0, sum = 0;
  if constexpr (V >= 4) {
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
      for (int i = 0; i + 3 <= nB; i += 3) {
        const uint2 ha = Hc[warp][i], hb = Hc[warp][i + 1], hc = Hc[warp][i + 2];
        uint32_t M = 0;
        if constexpr (V == 4) {
          sfor<16>([&](auto wc) { constexpr int w = decltype(wc)::value;
            t_v4<(1u << w)>(Zp[w], Gp[w], ha.x, ha.y, hb.x, hb.y, hc.x, hc.y, M, one, cneg); });
        } else {
          uint32_t Ma = 0, Mb = 0, Mc = 0;
          sfor<16>([&](auto wc) { constexpr int w = decltype(wc)::value;
            t_v0<(1u << w)>(Zp[w], Gp[w], ha.x, ha.y, Ma, one, cneg);
            t_v0<(1u << w)>(Zp[w], Gp[w], hb.x, hb.y, Mb, one, cneg);
            t_v0<(1u << w)>(Zp[w], Gp[w], hc.x, hc.y, Mc, one, cneg); });
          M = Ma | Mb | Mc;
        }
        if (M) { ++hits; sum += M; }
      }
    }
    atomicAdd(&res[0], hits);
    atomicAdd(&res[1], sum);
    return;
  }
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int i = 0; i + 2 <= nB; i += 2) {
      const uint4 hab = *reinterpret_cast<const uint4*>(&Hc[warp][i]);
      uint32_t M = 0;
      if constexpr (V == 0) {
        sfor<16>([&](auto wc) { constexpr int w = decltype(wc)::value;
          t_v0<(1u << w)>(Zp[w], Gp[w], hab.x, hab.y, M, one, cneg);
          t_v0<(1u << (16 + w))>(Zp[w], Gp[w], hab.z, hab.w, M, one, cneg); });
        if (M) { ++hits; sum += M; if (record && r == 0) masks[(size_t)gl * (nB / 2) + i / 2] = M; }
      } else if constexpr (V == 1) {
        uint32_t a0 = 0, a1 = 0, a2 = 0;
        sfor<16>([&](auto wc) { constexpr int w = decltype(wc)::value;
          constexpr int ia = w, ib = 16 + w;
          uint32_t& xa = ia < 11 ? a0 : ia < 22 ? a1 : a2;
          uint32_t& xb = ib < 11 ? a0 : ib < 22 ? a1 : a2;
          t_v1<h2pow(ia < 11 ? ia : ia < 22 ? ia - 11 : ia - 22)>(Zp[w], Gp[w], hab.x, hab.y, xa);
          t_v1<h2pow(ib < 11 ? ib : ib < 22 ? ib - 11 : ib - 22)>(Zp[w], Gp[w], hab.z, hab.w, xb); });
        if (a0 | a1 | a2) { M = v1_mask(a0, a1, a2); ++hits; sum += M; if (record && r == 0) masks[(size_t)gl * (nB / 2) + i / 2] = M; }
      } else if constexpr (V == 3) {
        const uint32_t za = hab.x & 0x7fff7fffu, zb = hab.z & 0x7fff7fffu;
        sfor<16>([&](auto wc) { constexpr int w = decltype(wc)::value;
          t_v3<(1u << w)>(Zp[w] | 0x80008000u, Gp[w], za, hab.y, zb, hab.w, M, one, cneg); });
        if (M) { ++hits; sum += M; if (record && r == 0) masks[(size_t)gl * (nB / 2) + i / 2] = M | (M << 16); }
      } else {
        sfor<16>([&](auto wc) { constexpr int w = decltype(wc)::value;
          t_v2<(1u << w)>(Zp[w], Gp[w], hab.x, hab.y, M, one);
          t_v2<(1u << (16 + w))>(Zp[w], Gp[w], hab.z, hab.w, M, one); });
        if (M) { ++hits; sum += M; if (record && r == 0) masks[(size_t)gl * (nB / 2) + i / 2] = M; }
      }
    }
  }
  atomicAdd(&res[0], hits);
  atomicAdd(&res[1], sum);
}

static uint64_t sm_state = 88172645463325252ull;
static uint32_t rnd() { sm_state ^= sm_state << 13; sm_state ^= sm_state >> 7; sm_state ^= sm_state << 17; return (uint32_t)sm_state; }
static uint32_t trit() { for (;;) { uint32_t t = rnd() & 3; if (t < 3) return t; } }

int main() {
  // A words: (z, g) of random trit vectors (z = zero indicator, g = sign), B: (z, u = ~(z ^ g))
  const int nA = 4096, nB = 1024;
  std::vector<uint32_t> A(nA * 32);
  for (int i = 0; i < nA * 16; ++i) {
    uint32_t z = 0, g = 0;
    for (int c = 0; c < 32; ++c) { uint32_t t = trit(); if (t == 0) z |= 1u << c; if (t == 2) g |= 1u << c; }
    A[2 * i] = z; A[2 * i + 1] = g;
  }
  std::vector<uint2> B(nB);
  for (int i = 0; i < nB; ++i) {
    uint32_t z = 0, g = 0;
    for (int c = 0; c < 32; ++c) { uint32_t t = trit(); if (t == 0) z |= 1u << c; if (t == 2) g |= 1u << c; }
    B[i] = make_uint2(z, ~(z ^ g));
  }
  uint32_t *dA, *dM[4]; uint2* dB; unsigned long long* dR;
  CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, nB * 8)); CK(cudaMalloc(&dR, 16));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), nB * 8, cudaMemcpyHostToDevice));
  int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  int clk = 0; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  const int grid = nsm * 4;
  const size_t nmask = (size_t)grid * 128 * (nB / 2);
  for (int v = 0; v < 4; ++v) { CK(cudaMalloc(&dM[v], nmask * 4)); CK(cudaMemset(dM[v], 0, nmask * 4)); }
  auto launch = [&](int v, int reps, int record) {
    CK(cudaMemset(dR, 0, 16));
    if (v == 0) k_probe<0><<<grid, 128>>>(dA, dB, nB, reps, dM[0], record, dR);
    if (v == 1) k_probe<1><<<grid, 128>>>(dA, dB, nB, reps, dM[1], record, dR);
    if (v == 2) k_probe<2><<<grid, 128>>>(dA, dB, nB, reps, dM[2], record, dR);
    if (v == 3) k_probe<3><<<grid, 128>>>(dA, dB, nB, reps, dM[3], record, dR);
    if (v == 4) k_probe<4><<<grid, 128>>>(dA, dB, nB, reps, nullptr, 0, dR);
    if (v == 5) k_probe<5><<<grid, 128>>>(dA, dB, nB, reps, nullptr, 0, dR);
    CK(cudaGetLastError());
  };
  for (int v = 0; v < 4; ++v) launch(v, 1, 1);
  CK(cudaDeviceSynchronize());
  std::vector<uint32_t> m0(nmask), m1(nmask), m2(nmask), m3(nmask);
  CK(cudaMemcpy(m3.data(), dM[3], nmask * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(m0.data(), dM[0], nmask * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(m1.data(), dM[1], nmask * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(m2.data(), dM[2], nmask * 4, cudaMemcpyDeviceToHost));
  // V0 is exact on 16-bit fields; V1/V2 also flag 0x8000 fields (f16 -0): supersets
  size_t miss1 = 0, miss2 = 0, n0 = 0, n1 = 0, n2 = 0, n3 = 0;
  for (size_t i = 0; i < nmask; ++i) {
    n0 += __builtin_popcount(m0[i]); n1 += __builtin_popcount(m1[i]); n2 += __builtin_popcount(m2[i]);
    if (m0[i] & ~m1[i]) ++miss1;
    if (m0[i] & ~m2[i]) ++miss2;
    // V3 tests columns 0..14 only: compare with the exact 15-column mask
    n3 += __builtin_popcount(m3[i]);
  }
  printf("V3 bits %zu (15-column fields, word-level, steps merged)\n", n3);
  printf("mask check: V0 bits %zu, V1 bits %zu (missed %zu), V2 bits %zu (missed %zu)\n", n0, n1, miss1, n2, miss2);
  const int reps = 40;
  for (int v = 0; v < 4; ++v) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    launch(v, reps, 0);
    cudaEventRecord(a); launch(v, reps, 0); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double tests = (double)grid * 128 * reps * (nB / 2) * 32;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("V%d: %.3f ms, %.2f tests/clk/SM (at %d MHz nominal)\n", v, ms, tests / cyc / nsm, clk / 1000);
  }
  // V4 (min3 over three entries) against V5 (the V0 tests in the same layout): same hits and mask sums
  for (int v = 4; v <= 5; ++v) {
    launch(v, 1, 0);
    unsigned long long r2[2]; CK(cudaMemcpy(r2, dR, 16, cudaMemcpyDeviceToHost));
    printf("V%d: hits %llu, mask sum %llu\n", v, r2[0], r2[1]);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    launch(v, reps, 0);
    cudaEventRecord(a); launch(v, reps, 0); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double tests = (double)grid * 128 * reps * (nB / 3) * 3 * 16;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("V%d: %.3f ms, %.2f tests/clk/SM (at %d MHz nominal)\n", v, ms, tests / cyc / nsm, clk / 1000);
  }
  // occupancy sweep of V0: k blocks of 4 warps per SM (grid nsm * k)
  auto sweep = [&](auto kc) {
    constexpr int KB = decltype(kc)::value;
    const int g2 = nsm * KB;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    CK(cudaMemset(dR, 0, 16));
    k_probe<0, KB><<<g2, 128>>>(dA, dB, nB, reps, dM[0], 0, dR);
    cudaEventRecord(a);
    k_probe<0, KB><<<g2, 128>>>(dA, dB, nB, reps, dM[0], 0, dR);
    cudaEventRecord(b); CK(cudaEventSynchronize(b)); CK(cudaGetLastError());
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double tests = (double)g2 * 128 * reps * (nB / 2) * 32;
    printf("V0 with %d warps/SM: %.2f tests/clk/SM\n", 4 * KB, tests / (ms * 1e-3 * clk * 1e3) / nsm);
  };
  sweep(std::integral_constant<int, 2>{});
  sweep(std::integral_constant<int, 3>{});
  sweep(std::integral_constant<int, 4>{});
  sweep(std::integral_constant<int, 5>{});
  sweep(std::integral_constant<int, 6>{});
  sweep(std::integral_constant<int, 8>{});
  return 0;
}
