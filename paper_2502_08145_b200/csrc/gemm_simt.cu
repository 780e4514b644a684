// gemm_simt.cu — fp32 SIMT GEMM for the fp32 test mode.
//
// tcgen05 kind::tf32 rounds fp32 inputs to a 10-bit mantissa, so the fp32 mode
// (tolerance 1e-5, bit-exact on integer inputs) runs plain FFMA: 64x64 tiles,
// BK = 16, 256 threads each owning a 4x4 block of C.
#include <cuda_runtime.h>

#include <cstdint>

#include "gemm.h"

namespace axonn {
namespace {

constexpr int TM = 64, TN = 64, TK = 16;

// a(m,k), b(k,n) index maps per op: NN A[m][k] B[k][n]; NT A[m][k] B[n][k];
// TN A[k][m] B[k][n].
template <int OP>
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, int64_t lda,
                                                       const float* __restrict__ B, int64_t ldb,
                                                       float* __restrict__ C, int64_t ldc, int M,
                                                       int N, int K) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int idx = threadIdx.x; idx < TK * TM; idx += 256) {
      int kk, mm;
      if (OP == 2) { mm = idx % TM; kk = idx / TM; } else { kk = idx % TK; mm = idx / TK; }
      const int m = m0 + mm, k = k0 + kk;
      float v = 0.f;
      if (m < M && k < K) v = (OP == 2) ? A[static_cast<int64_t>(k) * lda + m]
                                        : A[static_cast<int64_t>(m) * lda + k];
      As[kk][mm] = v;
    }
    for (int idx = threadIdx.x; idx < TK * TN; idx += 256) {
      int kk, nn;
      if (OP == 1) { kk = idx % TK; nn = idx / TK; } else { nn = idx % TN; kk = idx / TN; }
      const int n = n0 + nn, k = k0 + kk;
      float v = 0.f;
      if (n < N && k < K) v = (OP == 1) ? B[static_cast<int64_t>(n) * ldb + k]
                                        : B[static_cast<int64_t>(k) * ldb + n];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
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
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < N) C[static_cast<int64_t>(m) * ldc + n] = acc[i][j];
    }
  }
}

}  // namespace

GemmStatus gemm_f32_simt(int op, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                         const float* B, int64_t ldb, float* C, int64_t ldc, cudaStream_t stream) {
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return GemmStatus::kBadShape;
  dim3 grid(static_cast<unsigned>((N + TN - 1) / TN), static_cast<unsigned>((M + TM - 1) / TM));
  const int m = static_cast<int>(M), n = static_cast<int>(N), k = static_cast<int>(K);
  switch (op) {
    case 0: gemm_f32_kernel<0><<<grid, 256, 0, stream>>>(A, lda, B, ldb, C, ldc, m, n, k); break;
    case 1: gemm_f32_kernel<1><<<grid, 256, 0, stream>>>(A, lda, B, ldb, C, ldc, m, n, k); break;
    case 2: gemm_f32_kernel<2><<<grid, 256, 0, stream>>>(A, lda, B, ldb, C, ldc, m, n, k); break;
    default: return GemmStatus::kBadOp;
  }
  return cudaGetLastError() == cudaSuccess ? GemmStatus::kOk : GemmStatus::kLaunch;
}

}  // namespace axonn
