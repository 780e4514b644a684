// sym.h — symmetric NVLink memory for the fused GEMM + collective paths (see sym.cu).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>
#include <cstdint>
#include <string>

#include "gemm.h"

namespace axonn {

struct SymAxisImpl;

struct SymAxis {
  SymAxisImpl* impl = nullptr;  // null: no fused path on this axis
  int nranks = 0;
};

struct SymBuf {
  void* ptr = nullptr;  // this rank's copy (device pointer)
  void* mc = nullptr;   // multicast address: a multimem.red / .st lands in every rank's copy
  size_t bytes = 0;
  void* win = nullptr;  // ncclWindow_t (null until sym_register)
};

bool sym_axis_init(ncclComm_t comm, SymAxis* out, std::string* why);
void sym_axis_destroy(SymAxis* a);
// Two phases, so that every rank makes the same sequence of collective calls
// even when a local allocation fails (the caller agrees on the local results
// before any registration):
//   sym_mem_alloc  local: ncclMemAlloc of `bytes` rounded up to 2 MiB;
//   sym_register   collective over the axis: window registration + the
//                  window's multicast address.
bool sym_mem_alloc(size_t bytes, SymBuf* out, std::string* why);
bool sym_register(SymAxis* a, SymBuf* b, std::string* why);
// Both phases (diagnostics only: the probe allocates on every rank alike).
bool sym_alloc(SymAxis* a, size_t bytes, SymBuf* out, std::string* why);
void sym_free(SymAxis* a, SymBuf* b);
// Device address of `peer`'s copy of a registered buffer (LSA), or null.
void* sym_peer_ptr(SymBuf* b, int peer);
// NVLink primitive throughput probe over the whole buffer (mode 0
// multimem.red bf16, 1 multimem.st, 2 plain store to peer, 3
// multimem.ld_reduce, 4 local store).
cudaError_t sym_probe(SymAxis* a, SymBuf* b, int mode, int peer, int ctas, int iters, float* ms);

// Where the owner phase of a fused reduction sends the reduced 16-B units of
// its slice (unit u covers elements [u*U, u*U+U), U = 16 / element bytes):
//   kOwnPlain    plain stores to dst[0 .. n_dst) + 16u (own copy, and the
//                peer's copy on 2-rank axes);
//   kOwnMc       multimem.st at dst[0] + 16u (every rank's copy, NVLS);
//   kOwnScatter  the reduced slice is itself reduced over a second axis
//                (RS_z followed by the data-parallel sum):
//                element f of the slice goes to its owner o = f / slice2 on
//                that axis, at dst[o] + (me2*slice2 + f - o*slice2) * es —
//                the same addressing as the GEMM's kScatter epilogue.
enum OwnMode { kOwnPlain = 0, kOwnMc = 1, kOwnScatter = 2 };
struct OwnerOut {
  int mode = kOwnPlain;
  int n_dst = 0;
  unsigned long long dst[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int me2 = 0;
  long long slice2 = 0;
  // kOwnPlain, bf16 only: also write GELU(sum) to act_dst + 16u (the sum
  // itself still goes to dst[], e.g. Z saved for the backward; reading R18)
  int act = 0;
  unsigned long long act_dst = 0;
  // every destination is this rank's own memory (the exchange's local sum):
  // no system-scope fence at the end
  int local = 0;
  // 2-rank bf16 local sum: the 4-units-per-thread loop (AXONN_SUM_FAST=0: the generic one)
  int fast = 1;
};
// Owner phase: sum the P slots of `slice` elements in `recv` (bf16, or fp32
// when f32) in rank order 0..P-1 in fp32, round once (bf16), write per `out`.
// With `par` (kExchange double buffering) the slots come from recv_alt when
// (*par - 1) is odd: the barrier before the reduce advanced the counter.
cudaError_t sym_owner_reduce(const void* recv, long long slice, int P, bool f32,
                             const OwnerOut& out, int num_sms, cudaStream_t st,
                             const int* par = nullptr, const void* recv_alt = nullptr);
// All-gather pull on the SMs: dst = src[0] | src[1] | ... | src[P-1], each
// `bytes` long (bytes % 16 == 0; src are LSA peer addresses or local).
cudaError_t sym_gather_pull(const void* const* src, int P, size_t bytes, void* dst, int num_sms,
                            cudaStream_t st);
// All-gather on the copy engines (no SMs): one cudaMemcpyAsync per rank's
// slice, in z order: dst[q*bytes ...] = src[q].
cudaError_t sym_gather_copy(const void* const* src, int P, size_t bytes, void* dst,
                            cudaStream_t st);
// One-CTA cross-rank barrier on `st` (system-scope release/acquire).  Each
// `index` (0 or 1) is its own barrier sequence: every rank must issue the
// barriers of one index in the same order, and all barriers of one index must
// be issued on one stream (the epoch state is not safe under concurrency).
// `ctr` (optional): incremented by one thread after the barrier (kExchange parity).
cudaError_t sym_barrier(SymAxis* a, cudaStream_t st, int index = 0, int* ctr = nullptr);

// Fused-reduction plan shared by the multi-GPU path (axonn.cpp) and the
// single-GPU loopback (loopback.cpp): the epilogue mode of a rows x cols
// output of a GEMM with contraction length kdim reduced over P ranks with
// es-byte elements.  kStore means "not fused" (NCCL, or no reduction when
// P == 1).  2-rank bf16 axes use multimem.red when kdim >= red_min_k, else
// (exchange2) the exchange of whole partials, else the scatter + owner phase.
// xsum2: 1 = 2-rank bf16 axes sum inside the GEMM (kXSum) at every K;
// 2 = only below red_min_k (multimem.red above); 0 = never.
// redpair2: 1 = 2-rank bf16 axes reduce by unicast red.add into both ranks'
// outputs (kRedPair) at every K; 2 = only below red_min_k; 0 = never.
int fused_mode(int P, int es, int64_t rows, int64_t cols, int64_t kdim, int red_min_k,
               bool exchange2, bool pairsum2, int xsum2 = 0, int redpair2 = 0);
// kXSum: the control block (per rank, symmetric): [0, 4U) the flags the peer
// raises per 32x128 output unit, [4U, 8U) this rank's done marks, then the
// call counter (the parity of the receive set, the flag epoch) and the
// sweep's finished-CTA counter.  Zeroed once at creation.
inline long long xsum_units(long long rows, long long cols) {
  return ((rows + 31) / 32) * ((cols + 127) / 128);
}
inline size_t xsum_ctrl_bytes(long long units) { return static_cast<size_t>(units) * 8 + 256; }
inline size_t xsum_calls_off(long long units) { return static_cast<size_t>(units) * 8 + 128; }
inline size_t xsum_fin_off(long long units) { return static_cast<size_t>(units) * 8 + 192; }
// The sums the GEMM left open: every unit not marked done waits for the
// peer's flag, then slot 0 + slot 1 of the receive set -> RNE -> out.  The
// last CTA advances the call counter.  recv0 / recv1: this rank's receive
// sets (2 slots of rows*cols bf16 each).
cudaError_t sym_xsum_sweep(const void* recv0, const void* recv1, void* out, void* ctrl,
                           long long rows, long long cols, int num_sms, cudaStream_t st);
// kXSum epilogue target: recv[q] / recv_alt[q] rank q's receive sets, out this
// rank's output, ctrl / peer_ctrl the control blocks (xsum_ctrl_bytes).
EpiTarget epi_xsum(int me, long long rows, long long cols, const unsigned long long* recv,
                   const unsigned long long* recv_alt, void* out, void* ctrl, void* peer_ctrl);
// kPairSum: the control block of a pair-sum reduction (per rank, symmetric):
// [0, 4*chunks) arbitration tickets (rank 0's copy is the shared one),
// then the done counter and the call counter.
inline size_t pair_ctrl_bytes(long long chunks) { return static_cast<size_t>(chunks) * 4 + 256; }
inline size_t pair_done_off(long long chunks) { return static_cast<size_t>(chunks) * 4 + 128; }
inline size_t pair_calls_off(long long chunks) { return static_cast<size_t>(chunks) * 4 + 192; }
// Wait until *done reaches (*calls + 1) * total, then advance *calls (one thread).
cudaError_t sym_pair_wait(const void* done, void* calls, uint32_t total, cudaStream_t st);
// Epilogue targets: multimem.red into `mc`; scatter of 16-B units to the
// owners' receive slots peer[0..P) (owner o = flat / slice).
EpiTarget epi_red(unsigned long long mc);
EpiTarget epi_scatter(int P, int me, long long slice, const unsigned long long* peer);
// All-reduce by exchange (2-rank axes): every rank's whole partial into slot
// `me` of every rank's receive buffer (recv[q]: rank q's buffer of P slots of
// n elements; recv_alt: the second set, chosen when *par is odd).
EpiTarget epi_exchange(int P, int me, long long n, const unsigned long long* recv,
                       const unsigned long long* recv_alt, const int* par);

}  // namespace axonn
