// act.cu — GeLU between fc1 and fc2 (reading R18).
//
// The GPT block's MLP applies GELU(x) = x Φ(x), Φ(x) = (1 + erf(x/√2)) / 2,
// to fc1's output (PAPER.md:715-720 cite GPT-3).  With the activation on a
// layer, Alg. 1's output becomes O = GELU(Z), Z = all-reduce(Ô) (line 4), and
// the backward first forms dZ = dO ⊙ GELU'(Z), GELU'(x) = Φ(x) + x φ(x), which
// then takes dO's place in lines 11 and 13.  Z is rounded to bf16 where Alg. 1
// rounds O (R8); A = bf16(GELU(Z)) and dZ = bf16(dO · GELU'(Z)) are computed
// in fp32 from the bf16 values.
//
// Both kernels are elementwise and HBM-bound (16-B units, grid-stride):
//   forward:  read Z, write A (in place) and Z's copy for backward: 6 B/elem
//   backward: read dO, Z; write dZ: 6 B/elem
// The exchange all-reduce applies GELU in its local-sum pass instead
// (sym.cu k_owner_reduce, OwnerOut::act), so no separate pass runs there.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "act.h"

namespace axonn {
namespace {

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// z: in/out (A replaces Z); zsave: Z's copy (may be null)
__global__ void k_gelu_fwd(uint4* __restrict__ z, uint4* __restrict__ zsave, long long n16) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n16;
       i += stride) {
    const uint4 v = z[i];
    if (zsave) zsave[i] = v;
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = pack(gelu_f(bf_lo(w[q])), gelu_f(bf_hi(w[q])));
    z[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

__global__ void k_gelu_bwd(const uint4* __restrict__ dO, const uint4* __restrict__ z,
                           uint4* __restrict__ dz, long long n16) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n16;
       i += stride) {
    const uint4 g = dO[i], v = z[i];
    const uint32_t gw[4] = {g.x, g.y, g.z, g.w}, zw[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      o[q] = pack(bf_lo(gw[q]) * gelu_grad_f(bf_lo(zw[q])), bf_hi(gw[q]) * gelu_grad_f(bf_hi(zw[q])));
    dz[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

unsigned grid_for(long long n16, int num_sms) {
  long long blocks = (n16 + 255) / 256;
  if (blocks > 8LL * num_sms) blocks = 8LL * num_sms;
  return static_cast<unsigned>(blocks < 1 ? 1 : blocks);
}

}  // namespace

cudaError_t gelu_forward_inplace(void* z, void* zsave, long long n, int num_sms, cudaStream_t st) {
  if (n % 8) return cudaErrorInvalidValue;
  if (n == 0) return cudaSuccess;
  const long long n16 = n / 8;
  k_gelu_fwd<<<grid_for(n16, num_sms), 256, 0, st>>>(static_cast<uint4*>(z),
                                                    static_cast<uint4*>(zsave), n16);
  return cudaGetLastError();
}

cudaError_t gelu_backward(const void* dO, const void* z, void* dz, long long n, int num_sms,
                          cudaStream_t st) {
  if (n % 8) return cudaErrorInvalidValue;
  if (n == 0) return cudaSuccess;
  const long long n16 = n / 8;
  k_gelu_bwd<<<grid_for(n16, num_sms), 256, 0, st>>>(static_cast<const uint4*>(dO),
                                                    static_cast<const uint4*>(z),
                                                    static_cast<uint4*>(dz), n16);
  return cudaGetLastError();
}

}  // namespace axonn
