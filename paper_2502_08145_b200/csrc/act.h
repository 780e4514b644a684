// act.h — GeLU of the GPT block's MLP (see act.cu; reading R18).
#pragma once

#include <cuda_runtime.h>

namespace axonn {

#if defined(__CUDACC__)
// GELU(x) = x Φ(x) and GELU'(x) = Φ(x) + x φ(x) in fp32 (erff, expf).
__device__ __forceinline__ float gelu_f(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  return 0.5f * (1.0f + erff(x * 0.70710678118654752f)) +
         x * 0.39894228040143268f * expf(-0.5f * x * x);
}
#endif

// z (bf16, n % 8 == 0) := GELU(z) in place; zsave (optional) := the old z.
cudaError_t gelu_forward_inplace(void* z, void* zsave, long long n, int num_sms, cudaStream_t st);
// dz := bf16(dO * GELU'(z)) (bf16, n % 8 == 0).
cudaError_t gelu_backward(const void* dO, const void* z, void* dz, long long n, int num_sms,
                          cudaStream_t st);

}  // namespace axonn
