// sym.h — symmetric NVLink memory for the fused GEMM + all-reduce (see sym.cu).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>
#include <string>

namespace axonn {

struct SymAxisImpl;

struct SymAxis {
  SymAxisImpl* impl = nullptr;  // null: no fused path on this axis
  int nranks = 0;
};

struct SymBuf {
  void* ptr = nullptr;  // this rank's copy (device pointer)
  void* mc = nullptr;   // multicast address: a multimem.red lands in every rank's copy
  size_t bytes = 0;
  void* win = nullptr;  // ncclWindow_t
};

bool sym_axis_init(ncclComm_t comm, SymAxis* out, std::string* why);
void sym_axis_destroy(SymAxis* a);
bool sym_alloc(SymAxis* a, size_t bytes, SymBuf* out, std::string* why);
void sym_free(SymAxis* a, SymBuf* b);
// Diagnostics: device address of `peer`'s copy; NVLink primitive throughput
// probe over the whole buffer (mode 0 multimem.red bf16, 1 multimem.st,
// 2 plain store to peer, 3 multimem.ld_reduce, 4 local store).
void* sym_peer_ptr(SymBuf* b, int peer);
cudaError_t sym_probe(SymAxis* a, SymBuf* b, int mode, int peer, int ctas, int iters, float* ms);
// Owner phase of the P-rank fused all-reduce / reduce-scatter (see sym.cu):
// recv holds P slots of `slice` elements (bf16, or fp32 when f32); the sum
// goes to every rank's out[me*slice ...] (multicast), or to out_local when it
// is non-null (and also to out_peer with plain NVLink stores when that is
// non-null: 2-rank axes).
cudaError_t sym_owner_reduce(const SymBuf* recv, const SymBuf* out, long long slice, int P,
                             int me, int num_sms, cudaStream_t st, void* out_local = nullptr,
                             void* out_peer = nullptr, bool f32 = false);
// All-gather pull on the SMs: dst = src[0] | src[1] | ... | src[P-1], each
// `bytes` long (bytes % 16 == 0; src are LSA peer addresses or local).
cudaError_t sym_gather_pull(const void* const* src, int P, size_t bytes, void* dst, int num_sms,
                            cudaStream_t st);
// One-CTA cross-rank barrier on `st` (system-scope release/acquire).  Each
// `index` (0 or 1) is its own barrier sequence: every rank must issue the
// barriers of one index in the same order, and all barriers of one index must
// be issued on one stream (the epoch state is not safe under concurrency).
cudaError_t sym_barrier(SymAxis* a, cudaStream_t st, int index = 0);

}  // namespace axonn
