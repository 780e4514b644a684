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
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "sym.h"

namespace axonn {
namespace {

__global__ void k_mc_ptr(ncclWindow_t w, ncclDevComm dc, void** out) {
  out[0] = ncclGetLsaMultimemPointer(w, 0, dc);
  out[1] = ncclGetLocalPointer(w, 0);
}

__global__ void k_barrier(ncclDevComm dc) {
  ncclLsaBarrierSession<ncclCoopCta> b(ncclCoopCta(), dc, ncclTeamTagLsa(), 0);
  b.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

}  // namespace

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
  reqs.lsaBarrierCount = 1;
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

bool sym_alloc(SymAxis* a, size_t bytes, SymBuf* out, std::string* why) {
  *out = SymBuf();
  if (!a->impl) {
    *why = "axis has no symmetric-memory communicator";
    return false;
  }
  bytes = (bytes + (2u << 20) - 1) & ~static_cast<size_t>((2u << 20) - 1);
  void* p = nullptr;
  ncclResult_t r = ncclMemAlloc(&p, bytes);
  if (r != ncclSuccess) {
    *why = std::string("ncclMemAlloc: ") + ncclGetErrorString(r);
    return false;
  }
  ncclWindow_t win = nullptr;
  r = ncclCommWindowRegister(a->impl->comm, p, bytes, &win, NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess) {
    ncclMemFree(p);
    *why = std::string("ncclCommWindowRegister: ") + ncclGetErrorString(r);
    return false;
  }
  void** dptr = nullptr;
  void* host[2] = {nullptr, nullptr};
  if (cudaMalloc(&dptr, 2 * sizeof(void*)) != cudaSuccess) {
    *why = "cudaMalloc";
    return false;
  }
  k_mc_ptr<<<1, 1>>>(win, a->impl->dev, dptr);
  cudaError_t e = cudaMemcpy(host, dptr, sizeof host, cudaMemcpyDeviceToHost);
  cudaFree(dptr);
  // host[1] is this rank's slot in NCCL's flat LSA mapping: another virtual
  // address of the same physical pages as p.
  if (e != cudaSuccess || host[0] == nullptr) {
    ncclCommWindowDeregister(a->impl->comm, win);
    ncclMemFree(p);
    char buf[160];
    std::snprintf(buf, sizeof buf, "multicast address of the window unavailable (%s, mc=%p)",
                  cudaGetErrorString(e), host[0]);
    *why = buf;
    return false;
  }
  out->ptr = p;
  out->mc = host[0];
  out->bytes = bytes;
  out->win = win;
  return true;
}

void sym_free(SymAxis* a, SymBuf* b) {
  if (!b->ptr) return;
  if (a->impl) ncclCommWindowDeregister(a->impl->comm, static_cast<ncclWindow_t>(b->win));
  ncclMemFree(b->ptr);
  *b = SymBuf();
}

cudaError_t sym_barrier(SymAxis* a, cudaStream_t st) {
  k_barrier<<<1, 32, 0, st>>>(a->impl->dev);
  return cudaGetLastError();
}

}  // namespace axonn
