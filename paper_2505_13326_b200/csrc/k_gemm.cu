// SIMT GEMM, fp32 accumulate: C[m][n] (+)= sum_k A[m][k] B[n][k] (+ bias[n]).
// The fp32 parity mode uses it for every projection (tcgen05 kind::tf32 would not hold
// 1e-5); the bf16 mode uses the tcgen05 kernel (k_gemm_tc.cu) when it applies.
#include "kernels.h"

namespace {
constexpr int BM = 64, BN = 64, BK = 16;

template <typename T>
__global__ void __launch_bounds__(256) k_gemm_simt(const T* __restrict__ A, const T* __restrict__ B,
                                                   const float* __restrict__ bias, float* __restrict__ C,
                                                   int M, int N, int K, int mode) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
    for (int i = threadIdx.x; i < BM * BK; i += 256) {
      int mm = i / BK, kk = i % BK;
      int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? to_f(A[(long long)gm * K + gk]) : 0.f;
      int gn = n0 + mm;
      Bs[kk][mm] = (gn < N && gk < K) ? to_f(B[(long long)gn * K + gk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      float v = acc[i][j] + (bias ? bias[gn] : 0.f);
      float* c = C + (long long)gm * N + gn;
      *c = mode == GEMM_ACCUM ? *c + v : v;
    }
  }
}
}  // namespace

template <typename T>
void launch_gemm_simt(const T* A, const T* B, const float* bias, float* C, int M, int N, int K, int mode,
                      cudaStream_t s) {
  if (M <= 0 || N <= 0) return;
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
  k_gemm_simt<T><<<grid, 256, 0, s>>>(A, B, bias, C, M, N, K, mode);
}
template void launch_gemm_simt<float>(const float*, const float*, const float*, float*, int, int, int, int,
                                      cudaStream_t);
template void launch_gemm_simt<bf16>(const bf16*, const bf16*, const float*, float*, int, int, int, int,
                                     cudaStream_t);
