// sym.cu — NVLink symmetric memory for the fused GEMM + all-reduce path.
//
// For an axis communicator of P ranks (all inside one NVSwitch domain) this
// file provides
//   * a device communicator with an NVLS multicast team (ncclDevCommCreate,
//     lsaMultimem) and one LSA barrier;
//   * symmetric buffers (ncclMemAlloc + ncclCommWindowRegister) and their
//     multicast address, which the GEMM epilogue targets with
//     multimem.red.add so that NVSwitch sums every rank's partial tile into
//     every rank's copy (Alg. 1 lines 4 / 12 fused into lines 3 / 11);
//   * a one-CTA barrier kernel (release/acquire at system scope) that orders
//     "buffer zeroed on every rank" before the GEMM and "every rank's
//     reductions landed" after it.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "act.h"
#include "sym.h"

namespace axonn {
namespace {

// Programmatic dependent launch for the small kernels between the GEMMs
// (barriers, owner phases, gathers, waits): launched early when the previous
// kernel in the stream allows it, they wait for its completion before any
// memory access and let the next kernel be scheduled at once.  No-ops
// without the launch attribute (AXONN_PDL=0).
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void k_mc_ptr(ncclWindow_t w, ncclDevComm dc, void** out) {
  out[0] = ncclGetLsaMultimemPointer(w, 0, dc);
  out[1] = ncclGetLocalPointer(w, 0);
}

__global__ void k_peer_ptr(ncclWindow_t w, int peer, void** out) {
  out[0] = ncclGetLsaPointer(w, 0, peer);
}

// NVLink primitive throughput probe: every thread moves 16-B vectors.
__global__ void k_probe(uint4* local, uint64_t target, size_t n16, int mode) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n16; i += stride) {
    uint4 v = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
    const uint64_t a = target + 16 * i;
    if (mode == 0) {
      asm volatile("multimem.red.relaxed.sys.global.add.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(a),
                   "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    } else if (mode == 1) {
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(a),
                   "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    } else if (mode == 2) {
      *reinterpret_cast<uint4*>(a) = v;               // plain store to a peer (LSA) address
    } else if (mode == 5) {                           // unicast red.add into a peer (kRedPair)
      asm volatile("red.relaxed.sys.global.add.noftz.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(a),
                   "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    } else if (mode == 6) {                           // local red.add (kRedPair's own output)
      asm volatile("red.relaxed.gpu.global.add.noftz.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(
                       reinterpret_cast<uint64_t>(local + i)),
                   "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    } else if (mode == 3) {
      uint32_t x0, x1, x2, x3;
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                   : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "l"(a) : "memory");
      local[i] = make_uint4(x0, x1, x2, x3);
    } else {
      local[i] = v;                                    // local HBM store, for reference
    }
  }
}

// Owner phase of a P-rank fused reduction: sum the P slots this rank
// received (fixed order src = 0..P-1, fp32, one RNE rounding to bf16) and
// send the result where `out` says (OwnerOut, sym.h): its own copy (+ the
// peer's on 2-rank axes), every rank's copy through multimem.st, or the
// owners of a second reduction axis (RS_z feeding the data-parallel sum).
// Every element is reduced by exactly one rank, so all replicas hold the
// same bits.  F32 = false: 16-B units of 8 bf16, summed in fp32 in rank order
// and rounded once (RNE); F32 = true: 4 fp32, summed in fp32 in rank order
// (fp32 gradient reduction, reading R17).
template <bool F32>
__global__ void k_owner_reduce(const uint4* __restrict__ recv0, const uint4* __restrict__ recv1,
                               const int* __restrict__ par, long long n16, int P,
                               const __grid_constant__ OwnerOut out) {
  pdl_enter();
  constexpr int UNIT = F32 ? 4 : 8;  // elements per 16-B unit
  // kExchange double buffering: the barrier before this kernel advanced the
  // parity counter past the value the producing GEMM read
  const uint4* __restrict__ recv = (par && ((*par - 1) & 1)) ? recv1 : recv0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  long long i0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (!F32 && P == 2 && out.fast && out.mode == kOwnPlain && out.n_dst == 1 && !out.act) {
    // the 2-rank exchange's local sum (HBM-bound): 4 units per thread per
    // step, 8 loads in flight; slot 0 + slot 1 in fp32, one RNE rounding
    uint4* __restrict__ dst = reinterpret_cast<uint4*>(out.dst[0]);
    for (; i0 + 3 * stride < n16; i0 += 4 * stride) {
      uint4 a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = recv[i0 + u * stride];
        b[u] = recv[n16 + i0 + u * stride];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t x[4] = {a[u].x, a[u].y, a[u].z, a[u].w}, y[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          __nv_bfloat162 h = __floats2bfloat162_rn(
              (0.f + __uint_as_float(x[q] << 16)) + __uint_as_float(y[q] << 16),
              (0.f + __uint_as_float(x[q] & 0xFFFF0000u)) + __uint_as_float(y[q] & 0xFFFF0000u));
          o[q] = *reinterpret_cast<uint32_t*>(&h);
        }
        dst[i0 + u * stride] = make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
  }
  for (long long i = i0; i < n16; i += stride) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int src = 0; src < P; ++src) {
      const uint4 v = recv[src * n16 + i];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (F32) {
          acc[q] += __uint_as_float(w[q]);
        } else {
          acc[2 * q] += __uint_as_float(w[q] << 16);
          acc[2 * q + 1] += __uint_as_float(w[q] & 0xFFFF0000u);
        }
      }
    }
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (F32) {
        o[q] = __float_as_uint(acc[q]);
      } else {
        __nv_bfloat162 h = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
        o[q] = *reinterpret_cast<uint32_t*>(&h);
      }
    }
    const uint4 r = make_uint4(o[0], o[1], o[2], o[3]);
    if (out.mode == kOwnMc) {
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(
                       out.dst[0] + static_cast<unsigned long long>(i) * 16),
                   "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3])
                   : "memory");
    } else if (out.mode == kOwnScatter) {
      const long long f = i * UNIT;  // element index inside this owner's slice
      const int ow = static_cast<int>(f / out.slice2);
      const long long off = static_cast<long long>(out.me2) * out.slice2 + (f - ow * out.slice2);
      *reinterpret_cast<uint4*>(out.dst[ow] + static_cast<unsigned long long>(off) * (16 / UNIT)) = r;
    } else {
      for (int d = 0; d < out.n_dst; ++d)
        reinterpret_cast<uint4*>(out.dst[d])[i] = r;
      if (!F32 && out.act) {  // GELU of the rounded sum (act.cu, R18)
        uint32_t a[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          __nv_bfloat162 hh = __floats2bfloat162_rn(gelu_f(__uint_as_float(o[q] << 16)),
                                                    gelu_f(__uint_as_float(o[q] & 0xFFFF0000u)));
          a[q] = *reinterpret_cast<uint32_t*>(&hh);
        }
        reinterpret_cast<uint4*>(out.act_dst)[i] = make_uint4(a[0], a[1], a[2], a[3]);
      }
    }
  }
  if (!out.local) asm volatile("fence.acq_rel.sys;" ::: "memory");  // remote writes performed
}

// AG_z pull on the SMs: dst[q*n16 + i] = src[q][i] for the P ranks' staged
// slices (LSA peer addresses; q == me is local).  Used when nothing runs
// beside the gather (a forward that was not prefetched), where the copy
// engines' serialised per-peer copies are slower than every SM pulling.
struct PullSrc {
  const uint4* p[8];
};
__global__ void k_gather_pull(PullSrc src, int P, long long n16, uint4* __restrict__ dst) {
  pdl_enter();
  const long long total = static_cast<long long>(P) * n16;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += stride) {
    const int q = static_cast<int>(idx / n16);
    dst[idx] = src.p[q][idx - q * n16];
  }
}

// kPairSum completion (gemm.h): wait until every chunk of this call has been
// finalised — by this rank's epilogue or the peer's — then advance the call
// count.  A bounded spin: a lost chunk traps (a launch error) instead of
// hanging the device.
__global__ void k_pair_wait(const uint32_t* done, uint32_t* calls, uint32_t total) {
  pdl_enter();
  if (threadIdx.x != 0) return;
  const uint32_t c = *calls;
  const uint32_t target = (c + 1u) * total;
  long long spins = 0;
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(done) : "memory");
    if (static_cast<int32_t>(v - target) >= 0) break;
    __nanosleep(256);
    if (++spins > (1LL << 27)) __trap();
  }
  *calls = c + 1u;
}

// kXSum sweep (see sym.h): one warp per 32x128 output unit, grid-stride.
__global__ void k_xsum_sweep(const char* __restrict__ recv0, const char* __restrict__ recv1,
                             char* __restrict__ out, int* ctrl, int M, int N, long long U,
                             int* calls, unsigned* fin) {
  pdl_enter();
  const int c = *reinterpret_cast<volatile int*>(calls);
  const int epoch = c + 1;
  const char* s0 = (c & 1) ? recv1 : recv0;
  const char* s1 = s0 + static_cast<uint64_t>(M) * N * 2;
  const int* peerflag = ctrl;
  const int* done = ctrl + U;
  const int lane = threadIdx.x & 31;
  const int upr = (N + 127) / 128;
  const long long nw = static_cast<long long>(gridDim.x) * (blockDim.x / 32);
  for (long long u = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; u < U;
       u += nw) {
    if (*reinterpret_cast<const volatile int*>(done + u) == epoch) continue;
    long long spins = 0;
    for (;;) {
      int f;
      asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(f) : "l"(peerflag + u) : "memory");
      if (__all_sync(0xffffffffu, f == epoch)) break;
      __nanosleep(256);
      if (++spins > (1LL << 26)) __trap();  // the peer never delivered: fail loudly
    }
    const int r0 = static_cast<int>(u / upr) * 32, c0 = static_cast<int>(u % upr) * 128;
    for (int i = 0; i < 16; ++i) {
      const int v = lane + 32 * i;
      const int row = r0 + (v >> 4), col = c0 + (v & 15) * 8;
      if (row < M && col < N) {
        const uint64_t off = (static_cast<uint64_t>(row) * N + col) * 2;
        uint4 a, b;
        asm volatile("ld.global.cg.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(s0 + off) : "memory");
        asm volatile("ld.global.cg.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(s1 + off) : "memory");
        const uint32_t x[4] = {a.x, a.y, a.z, a.w}, y[4] = {b.x, b.y, b.z, b.w};
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // slot 0 + slot 1 in fp32, one RNE rounding (R19)
          const float lo = __uint_as_float(x[q] << 16) + __uint_as_float(y[q] << 16);
          const float hi = __uint_as_float(x[q] & 0xFFFF0000u) + __uint_as_float(y[q] & 0xFFFF0000u);
          __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
          o[q] = *reinterpret_cast<uint32_t*>(&h);
        }
        *reinterpret_cast<uint4*>(out + off) = make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
  }
  // the last CTA out advances the call counter (every CTA has read it)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(fin, 1u) == gridDim.x - 1) {
      *fin = 0;
      *calls = epoch;
      __threadfence();
    }
  }
}

__global__ void k_barrier(ncclDevComm dc, uint32_t index, int* ctr) {
  pdl_enter();
  ncclLsaBarrierSession<ncclCoopCta> b(ncclCoopCta(), dc, ncclTeamTagLsa(), index);
  b.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  // kExchange parity: the next call's epilogue targets the other buffers
  if (ctr && threadIdx.x == 0) *ctr += 1;
}

}  // namespace

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, cudaStream_t st,
                       Args... args) {
  static const bool pdl = [] {
    const char* v = std::getenv("AXONN_PDL");
    return !(v && std::atoi(v) == 0);
  }();
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(block);
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&lc, kern, static_cast<KArgs>(args)...);
}

struct SymAxisImpl {
  ncclComm_t comm = nullptr;
  ncclDevComm dev;
};

bool sym_axis_init(ncclComm_t comm, SymAxis* out, std::string* why) {
  out->impl = nullptr;
  auto* im = new SymAxisImpl();
  im->comm = comm;
  ncclDevCommRequirements reqs;
  std::memset(&reqs, 0, sizeof reqs);
  reqs.lsaMultimem = true;
  reqs.lsaBarrierCount = 2;  // one barrier sequence per issuing stream (see sym_barrier)
  ncclResult_t r = ncclDevCommCreate(comm, &reqs, &im->dev);
  if (r != ncclSuccess) {
    *why = std::string("ncclDevCommCreate: ") + ncclGetErrorString(r);
    delete im;
    return false;
  }
  if (im->dev.lsaSize != im->dev.nRanks || im->dev.lsaMultimem.mcBasePtr == nullptr) {
    *why = "axis group is not one load/store (NVLink) domain with multicast";
    ncclDevCommDestroy(comm, &im->dev);
    delete im;
    return false;
  }
  out->impl = im;
  out->nranks = im->dev.nRanks;
  return true;
}

void sym_axis_destroy(SymAxis* a) {
  if (!a->impl) return;
  ncclDevCommDestroy(a->impl->comm, &a->impl->dev);
  delete a->impl;
  a->impl = nullptr;
}

bool sym_mem_alloc(size_t bytes, SymBuf* out, std::string* why) {
  *out = SymBuf();
  static const bool fail_test = [] {  // test hook: exercise the NCCL fallback
    const char* v = std::getenv("AXONN_SYM_ALLOC_FAIL");
    return v && std::atoi(v) != 0;
  }();
  if (fail_test) {
    *why = "AXONN_SYM_ALLOC_FAIL set";
    return false;
  }
  bytes = (bytes + (2u << 20) - 1) & ~static_cast<size_t>((2u << 20) - 1);
  void* p = nullptr;
  ncclResult_t r = ncclMemAlloc(&p, bytes);
  if (r != ncclSuccess) {
    *why = std::string("ncclMemAlloc: ") + ncclGetErrorString(r);
    return false;
  }
  out->ptr = p;
  out->bytes = bytes;
  return true;
}

bool sym_register(SymAxis* a, SymBuf* b, std::string* why) {
  if (!a->impl || !b->ptr) {
    *why = !a->impl ? "axis has no symmetric-memory communicator" : "nothing allocated";
    return false;
  }
  ncclWindow_t win = nullptr;
  ncclResult_t r = ncclCommWindowRegister(a->impl->comm, b->ptr, b->bytes, &win,
                                          NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess) {
    *why = std::string("ncclCommWindowRegister: ") + ncclGetErrorString(r);
    return false;
  }
  b->win = win;
  void** dptr = nullptr;
  void* host[2] = {nullptr, nullptr};
  cudaError_t e = cudaMalloc(&dptr, 2 * sizeof(void*));
  if (e == cudaSuccess) {
    k_mc_ptr<<<1, 1>>>(win, a->impl->dev, dptr);
    e = cudaMemcpy(host, dptr, sizeof host, cudaMemcpyDeviceToHost);
    cudaFree(dptr);
  }
  // host[1] is this rank's slot in NCCL's flat LSA mapping: another virtual
  // address of the same physical pages as ptr.  The window stays registered
  // on failure (sym_free deregisters it) so every rank's calls stay matched.
  if (e != cudaSuccess || host[0] == nullptr) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "multicast address of the window unavailable (%s, mc=%p)",
                  cudaGetErrorString(e), host[0]);
    *why = buf;
    return false;
  }
  b->mc = host[0];
  return true;
}

bool sym_alloc(SymAxis* a, size_t bytes, SymBuf* out, std::string* why) {
  if (!a->impl) {
    *why = "axis has no symmetric-memory communicator";
    return false;
  }
  if (!sym_mem_alloc(bytes, out, why)) return false;
  if (!sym_register(a, out, why)) {
    sym_free(a, out);
    return false;
  }
  return true;
}

void sym_free(SymAxis* a, SymBuf* b) {
  if (!b->ptr) return;
  if (a->impl && b->win) ncclCommWindowDeregister(a->impl->comm, static_cast<ncclWindow_t>(b->win));
  ncclMemFree(b->ptr);
  *b = SymBuf();
}

void* sym_peer_ptr(SymBuf* b, int peer) {
  void** d = nullptr;
  void* h = nullptr;
  if (cudaMalloc(&d, sizeof(void*)) != cudaSuccess) return nullptr;
  k_peer_ptr<<<1, 1>>>(static_cast<ncclWindow_t>(b->win), peer, d);
  cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h;
}

cudaError_t sym_probe(SymAxis* a, SymBuf* b, int mode, int peer, int ctas, int iters, float* ms) {
  uint64_t target = reinterpret_cast<uint64_t>(b->mc);
  if (mode == 2 || mode == 5) target = reinterpret_cast<uint64_t>(sym_peer_ptr(b, peer));
  if (mode == 4) target = reinterpret_cast<uint64_t>(b->ptr);
  const size_t n16 = b->bytes / 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  sym_barrier(a, 0, 0);
  k_probe<<<ctas, 512>>>(static_cast<uint4*>(b->ptr), target, n16, mode);
  sym_barrier(a, 0, 0);
  cudaEventRecord(e0, 0);
  for (int i = 0; i < iters; ++i) k_probe<<<ctas, 512>>>(static_cast<uint4*>(b->ptr), target, n16, mode);
  cudaEventRecord(e1, 0);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  *ms /= iters;
  sym_barrier(a, 0, 0);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaDeviceSynchronize();
}

cudaError_t sym_owner_reduce(const void* recv, long long slice, int P, bool f32,
                             const OwnerOut& out, int num_sms, cudaStream_t st, const int* par,
                             const void* recv_alt) {
  const int es = f32 ? 4 : 2;
  if (P < 1 || P > 8 || (slice * es) % 16 || out.n_dst < 0 || out.n_dst > 8 ||
      (out.mode == kOwnScatter && (out.slice2 <= 0 || (out.slice2 * es) % 16)))
    return cudaErrorInvalidValue;
  const long long n16 = slice * es / 16;
  long long blocks = (n16 + 255) / 256;
  if (blocks > 4LL * num_sms) blocks = 4LL * num_sms;
  if (blocks < 1) blocks = 1;
  auto kern = f32 ? k_owner_reduce<true> : k_owner_reduce<false>;
  return launch_pdl(kern, static_cast<unsigned>(blocks), 256, st, reinterpret_cast<const uint4*>(recv),
                    reinterpret_cast<const uint4*>(recv_alt ? recv_alt : recv), par, n16, P, out);
}

cudaError_t sym_gather_copy(const void* const* src, int P, size_t bytes, void* dst,
                            cudaStream_t st) {
  for (int q = 0; q < P; ++q) {
    cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + q * bytes, src[q], bytes,
                                    cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int fused_mode(int P, int es, int64_t rows, int64_t cols, int64_t kdim, int red_min_k,
               bool exchange2, bool pairsum2, int xsum2, int redpair2) {
  const int64_t n = rows * cols;
  const int unit = 16 / es;  // elements per 16-B epilogue unit
  // not fused: a 1-rank axis, an empty output, rows not a whole number of
  // 16-B units, or an empty product (K == 0 writes zeros; nothing to scatter)
  if (P < 2 || n <= 0 || cols % unit || kdim <= 0) return kStore;
  // 2-rank bf16: the sum finished inside the epilogue (no post pass, no barrier)
  if (es == 2 && P == 2 && pairsum2) return kPairSum;
  // 2-rank bf16: exchange, summed inside the GEMM as partials land
  if (es == 2 && P == 2 && (xsum2 == 1 || (xsum2 == 2 && kdim < red_min_k))) return kXSum;
  // 2-rank bf16: unicast reductions into both ranks' outputs
  if (es == 2 && P == 2 && (redpair2 == 1 || (redpair2 == 2 && kdim < red_min_k))) return kRedPair;
  // multimem.red.add sums bf16 here; fp32 always takes the scatter + owner phase
  if (es == 2 && P == 2 && kdim >= red_min_k) return kMcRed;
  // 2-rank axes: exchange whole partials, then sum locally (no owner broadcast)
  if (P == 2 && exchange2) return kExchange;
  if (n % (static_cast<int64_t>(unit) * P)) return kStore;
  return kScatter;
}

EpiTarget epi_exchange(int P, int me, long long n, const unsigned long long* recv,
                       const unsigned long long* recv_alt, const int* par) {
  EpiTarget t;
  t.mode = kExchange;
  t.P = P;
  t.me = me;
  t.slice = n;
  for (int q = 0; q < P && q < 8; ++q) {
    t.peer[q] = recv[q];
    t.peer_alt[q] = recv_alt ? recv_alt[q] : recv[q];
  }
  t.par = par;
  return t;
}

EpiTarget epi_xsum(int me, long long rows, long long cols, const unsigned long long* recv,
                   const unsigned long long* recv_alt, void* out, void* ctrl, void* peer_ctrl) {
  EpiTarget t;
  t.mode = kXSum;
  t.P = 2;
  t.me = me;
  t.slice = rows * cols;
  const long long U = xsum_units(rows, cols);
  for (int q = 0; q < 2; ++q) {
    t.peer[q] = recv[q];
    t.peer_alt[q] = recv_alt[q];
  }
  t.peer[2] = reinterpret_cast<unsigned long long>(out);
  t.peer[3] = reinterpret_cast<unsigned long long>(ctrl);
  t.peer[4] = reinterpret_cast<unsigned long long>(peer_ctrl);
  t.peer[5] = reinterpret_cast<unsigned long long>(static_cast<char*>(ctrl) + U * 4);
  t.par = reinterpret_cast<const int*>(static_cast<char*>(ctrl) + xsum_calls_off(U));
  return t;
}

EpiTarget epi_red(unsigned long long mc) {
  EpiTarget t;
  t.mode = kMcRed;
  t.mc = mc;
  return t;
}

EpiTarget epi_scatter(int P, int me, long long slice, const unsigned long long* peer) {
  EpiTarget t;
  t.mode = kScatter;
  t.P = P;
  t.me = me;
  t.slice = slice;
  for (int q = 0; q < P && q < 8; ++q) t.peer[q] = peer[q];
  return t;
}

cudaError_t sym_gather_pull(const void* const* src, int P, size_t bytes, void* dst, int num_sms,
                            cudaStream_t st) {
  if (P < 1 || P > 8 || bytes % 16) return cudaErrorInvalidValue;
  PullSrc ps{};
  for (int q = 0; q < P; ++q) ps.p[q] = static_cast<const uint4*>(src[q]);
  const long long n16 = static_cast<long long>(bytes / 16);
  long long blocks = (P * n16 + 255) / 256;
  if (blocks > 4LL * num_sms) blocks = 4LL * num_sms;
  if (blocks < 1) blocks = 1;
  return launch_pdl(k_gather_pull, static_cast<unsigned>(blocks), 256, st, ps, P, n16,
                    static_cast<uint4*>(dst));
}

cudaError_t sym_pair_wait(const void* done, void* calls, uint32_t total, cudaStream_t st) {
  return launch_pdl(k_pair_wait, 1, 32, st, static_cast<const uint32_t*>(done),
                    static_cast<uint32_t*>(calls), total);
}

cudaError_t sym_xsum_sweep(const void* recv0, const void* recv1, void* out, void* ctrl,
                           long long rows, long long cols, int num_sms, cudaStream_t st) {
  const long long U = xsum_units(rows, cols);
  if (U <= 0) return cudaSuccess;
  char* c = static_cast<char*>(ctrl);
  long long blocks = (U + 7) / 8;
  if (blocks > 2LL * num_sms) blocks = 2LL * num_sms;
  return launch_pdl(k_xsum_sweep, static_cast<unsigned>(blocks), 256, st,
                    static_cast<const char*>(recv0), static_cast<const char*>(recv1),
                    static_cast<char*>(out), reinterpret_cast<int*>(c), static_cast<int>(rows),
                    static_cast<int>(cols), U, reinterpret_cast<int*>(c + xsum_calls_off(U)),
                    reinterpret_cast<unsigned*>(c + xsum_fin_off(U)));
}

cudaError_t sym_barrier(SymAxis* a, cudaStream_t st, int index, int* ctr) {
  return launch_pdl(k_barrier, 1, 32, st, a->impl->dev, static_cast<uint32_t>(index), ctr);
}

}  // namespace axonn
