// tp_census.cu -- exact census of perm mod 3 over all n x n matrices
// (reference: exact_count_kernel, src/_kernels.py:164-209,
// and exact_zero_count, src/experiments.py:113-140, which brute-forces all
// 3^(n^2) matrices and stops at n = 4).
//
// Two Laplace expansions collapse the enumeration:
//  * along the last row: perm(A) = r . C with C_j = perm(A without row n,
//    column j).  For fixed rows 1..n-1, r . C is 0 for all 3^n last rows if
//    C = 0, otherwise each value 0, 1, 2 is taken 3^(n-1) times;
//  * along row n-1: C = D r' with D_jk = perm(rows 1..n-2, columns
//    without j and k), a symmetric zero-diagonal n x n matrix over F3, so
//    #{r' : C = 0} = 3^(n - rank D).
// Hence, with N0 = sum over the 3^((n-2) n) configurations w of rows 1..n-2
// of 3^(n - rank_F3 D(w)):
//    z(n)    = 3^(n-1) * 3^(n(n-1)) + 2 * 3^(n-1) * N0
//    plus(n) = minus(n) = 3^(n-1) * (3^(n(n-1)) - N0).
// The (n-2) x (n-2) permanents D_jk are Ryser sums over the 2^(n-2) row
// subsets of w, sharing the subset column sums across all pairs (j, k).
// One thread per configuration w; n <= 6 (3^24 configurations for n = 6).
#include <cstdint>

#include "tp_kernels.cuh"

namespace tp {

// F3 rank of a symmetric n x n matrix (entries 0..2), by elimination.
template <int N>
__device__ __forceinline__ int rank_f3(int (&M)[N][N]) {
  int rank = 0;
  for (int col = 0; col < N && rank < N; ++col) {
    int piv = -1;
#pragma unroll
    for (int r = 0; r < N; ++r)
      if (piv < 0 && r >= rank && M[r][col] != 0) piv = r;
    if (piv < 0) continue;
#pragma unroll
    for (int c = 0; c < N; ++c) {
      const int t = M[piv][c];
      M[piv][c] = M[rank][c];
      M[rank][c] = t;
    }
    const int inv = M[rank][col];  // 1 or 2; 2 * 2 = 1 mod 3, so inv = itself
#pragma unroll
    for (int r = 0; r < N; ++r) {
      if (r != rank && M[r][col] != 0) {
        const int f = (M[r][col] * inv) % 3;  // factor so that M[r][col] becomes 0
#pragma unroll
        for (int c = 0; c < N; ++c) M[r][c] = (M[r][c] + 3 * 3 - f * M[rank][c]) % 3;
      }
    }
    ++rank;
  }
  return rank;
}

template <int N>
__global__ void __launch_bounds__(256) k_census(unsigned long long configs, unsigned long long* n0_out) {
  constexpr int NR = N - 2;  // rows of w
  constexpr int NP = N * (N - 1) / 2;
  unsigned long long acc = 0;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long idx = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; idx < configs;
       idx += stride) {
    // decode w (NR x N trits, base 3, row-major)
    int w[NR > 0 ? NR : 1][N];
    unsigned long long x = idx;
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        w[r][c] = (int)(x % 3ull);
        x /= 3ull;
      }
    // Ryser over row subsets of w: D_jk = (-1)^NR sum_S (-1)^|S| prod_{c != j,k} v_S[c]
    int D[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) D[q] = 0;
    int v[N];
#pragma unroll
    for (int c = 0; c < N; ++c) v[c] = 0;
    for (int i = 0; i < (1 << NR); ++i) {  // i = 0 is the empty subset (all-zero v; contributes for NR = 0)
      if (i > 0) {
        const int t = __ffs(i) - 1;
        const bool leave = ((i ^ (i >> 1)) >> t & 1) == 0;  // bit t of gray(i) cleared -> row t left
#pragma unroll
        for (int c = 0; c < N; ++c) v[c] = (v[c] + (leave ? 3 - w[t][c] : w[t][c])) % 3;
      }
      const int sgn_set = (i & 1) ? 2 : 1;  // (-1)^|S| in F3; |gray(i)| has the parity of i
      // zeros among the N column sums, and the product of the nonzero ones
      int nz = 0, z0 = -1, z1 = -1, prod = 1;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        if (v[c] == 0) {
          if (nz == 0) z0 = c;
          else if (nz == 1) z1 = c;
          ++nz;
        } else {
          prod = (prod * v[c]) % 3;
        }
      }
      if (nz > 2) continue;
      int q = 0;
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int k = j + 1; k < N; ++k, ++q) {
          // product over columns other than j, k (nonzero elements are self-inverse)
          int term;
          if (nz == 0) term = (prod * v[j] * v[k]) % 3;
          else if (nz == 1) term = (z0 == j) ? (prod * v[k]) % 3 : (z0 == k) ? (prod * v[j]) % 3 : 0;
          else term = (z0 == j && z1 == k) ? prod : 0;
          D[q] = (D[q] + term * sgn_set) % 3;
        }
    }
    int M[N][N];
    int q = 0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      M[j][j] = 0;
#pragma unroll
      for (int k = j + 1; k < N; ++k, ++q) {
        const int d = (NR & 1) ? (3 - D[q]) % 3 : D[q];
        M[j][k] = d;
        M[k][j] = d;
      }
    }
    const int rk = rank_f3<N>(M);
    unsigned long long pw = 1;
    for (int e = 0; e < N - rk; ++e) pw *= 3ull;
    acc += pw;
  }
  // block reduction
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  __shared__ unsigned long long part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += part[k];
    atomicAdd(n0_out, s);
  }
}

cudaError_t launch_census(int n, int grid, unsigned long long configs, unsigned long long* n0, cudaStream_t st) {
  switch (n) {
    case 2: k_census<2><<<grid, 256, 0, st>>>(configs, n0); break;
    case 3: k_census<3><<<grid, 256, 0, st>>>(configs, n0); break;
    case 4: k_census<4><<<grid, 256, 0, st>>>(configs, n0); break;
    case 5: k_census<5><<<grid, 256, 0, st>>>(configs, n0); break;
    case 6: k_census<6><<<grid, 256, 0, st>>>(configs, n0); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace tp
