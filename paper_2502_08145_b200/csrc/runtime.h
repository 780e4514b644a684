// runtime.h — internal hooks of the host runtime (axonn.cpp) used by the
// single-GPU loopback (loopback.cpp).  Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/axonn.h"
#include "gemm.h"

namespace axonn {

// One local product through the runtime's instrumented launch path
// (run_gemm in axonn.cpp): status + thread-local message on failure.
axonn_status_t rt_gemm(int op, int dtype, int64_t M, int64_t N, int64_t K, const void* A,
                       int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                       cudaStream_t st, const EpiTarget* epi, const SideSum* side = nullptr);
axonn_status_t rt_fail(axonn_status_t s, const char* msg);
void rt_count_launch();
int rt_num_sms();

axonn_status_t loopback_step(const axonn_fc_desc_t* d, const int g[4], const void* const* I,
                             const void* const* What, const void* const* dO, void* const* O,
                             void* const* dI, void* const* dW, int flags, cudaStream_t st,
                             int* paths);

}  // namespace axonn
