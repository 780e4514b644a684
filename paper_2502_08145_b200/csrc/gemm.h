// gemm.h — internal launch interface of the local-product kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace axonn {

enum class GemmStatus { kOk = 0, kBadShape, kBadAlignment, kTensorMap, kBadOp, kLaunch };

// bf16 x bf16 -> bf16 (fp32 accumulate) on tcgen05; op 0 = NN, 1 = NT, 2 = TN.
// red_mc != nullptr: instead of storing C, add the bf16-rounded tile into
// every rank's copy of a multicast-mapped buffer (multimem.red; C/ldc give the
// local layout, N % 8 == 0).
GemmStatus gemm_bf16_tc(int op, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                        const void* B, int64_t ldb, void* C, int64_t ldc, int num_sms,
                        cudaStream_t stream, void* red_mc = nullptr);

// fp32 SIMT FMA (test mode, no TF32): same op codes.
GemmStatus gemm_f32_simt(int op, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                         const float* B, int64_t ldb, float* C, int64_t ldc, cudaStream_t stream);

}  // namespace axonn
