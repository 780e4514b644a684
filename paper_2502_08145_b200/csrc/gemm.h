// gemm.h — internal launch interface of the local-product kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace axonn {

// Where the epilogue sends each bf16 tile (see gemm_tc.cu):
//   kStore     C[M][N] local stores;
//   kMcRed     multimem.red.add into every rank's copy of a multicast buffer
//              (2-rank fused all-reduce);
//   kScatter   plain NVLink stores of each 16-B vector into its owner rank's
//              receive slot: owner o = flat index / slice, destination
//              peer[o] + (me * slice + flat - o * slice) (fused reduce-scatter;
//              needs ldc == N and slice % 8 == 0);
//   kExchange  every rank's whole partial to every rank of the axis: plain
//              stores of each 16-B vector to slot `me` of each rank's receive
//              buffer, peer[q] + (me * slice + flat) (slice = M*N, ldc == N);
//              the post phase is a local sum of the P slots (2-rank axes).
//              With `par` set, the kernel reads *par and targets peer_alt
//              instead when it is odd (device-side double buffering).
//   kPairSum   2-rank all-reduce finished inside the epilogue: each warp's
//              32x64 chunk goes to the peer's receive buffer (peer[1]), then
//              one lane takes a ticket on the chunk's arbitration counter
//              (atomic at mc + 4*chunk, shared by both ranks); the rank that
//              arrives second adds the peer's partial (its own receive
//              buffer, peer[0]) and writes the rounded sum to both ranks'
//              outputs (peer[2] own, peer[3] peer's), then counts the chunk
//              done on both ranks (peer[4] own counter, peer[5] peer's).
//              slice = chunks per row of 64 columns.  bf16, ldc == N.
//   kXSum      2-rank all-reduce by exchange, summed inside the GEMM: each
//              16-B vector goes to slot `me` of both ranks' receive buffers
//              (peer[q]: rank q's, slots of `slice` = M*N elements; peer_alt
//              when *par is odd), as kExchange.  Per finished 32x128 output
//              unit u (row/32 * ceil(N/128) + col/128) the warp raises the
//              peer's flag (peer[4] + 4u) = epoch (*par + 1) after a system
//              fence; a little later (never waiting) it sums units whose own
//              flag (peer[3] + 4u, raised by the peer) shows the epoch: slot
//              0 + slot 1 in fp32, one RNE rounding, to the output peer[2],
//              and marks them done (peer[5] + 4u).  What is still open when
//              the kernel ends is summed by sym_xsum_sweep, which also
//              advances *par.  No barrier, no pass over the whole output.
//   kRedPair   2-rank all-reduce by unicast reductions: each 16-B bf16 vector
//              is red.add-ed into this rank's output (mc + offset) and into
//              the peer's (peer[0] + offset, over NVLink); both outputs are
//              zeroed (and a barrier passed) before the GEMM, so every element
//              ends as RNE(a + b) on both ranks, bit-identical to NCCL.
//   kRedLocal  red.global.add of each 16-B bf16 vector at mc + offset: the
//              single-GPU loopback's stand-in for kMcRed when the device
//              has no multicast support (axonn_loopback_step).
struct EpiTarget {
  int mode = 0;
  int P = 0, me = 0;
  long long slice = 0;
  unsigned long long mc = 0;
  unsigned long long peer[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long peer_alt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int* par = nullptr;
};
enum EpiMode { kStore = 0, kMcRed = 1, kScatter = 2, kRedLocal = 3, kExchange = 4, kPairSum = 5,
               kXSum = 6, kRedPair = 7 };

// A memory-bound task the GEMM's idle helper warps (2 and 3 of every CTA)
// run beside its tiles: the local sum of a 2-rank exchange all-reduce whose
// partials a PREVIOUS GEMM left in this rank's receive set (slot 0 + slot 1
// in fp32, one RNE rounding -> out; the backward's dI sum run inside the dW
// GEMM that follows it, Alg. 1 lines 12-13).  Cross-rank: one CTA raises
// the peer's arrive word to epoch p + 1 (p = *par at kernel start: the set
// the producing GEMM used) and waits for its own, then opens `go` for the
// helpers; the last helper warp out advances *par.  arrive_peer == null: no
// barrier (the single-GPU loopback, where stream order stands in for it).
struct SideSum {
  const void* recv0 = nullptr;  // this rank's receive sets: 2 slots of n16 16-B units each
  const void* recv1 = nullptr;
  void* out = nullptr;
  long long n16 = 0;            // 0: no side task
  int* par = nullptr;
  int* arrive_own = nullptr;    // raised by the peer
  int* arrive_peer = nullptr;   // the peer's (NVLink) arrive word
  int* go = nullptr;
  unsigned* fin = nullptr;
};

enum class GemmStatus { kOk = 0, kBadShape, kBadAlignment, kTensorMap, kBadOp, kLaunch };

// bf16 x bf16 -> bf16 (fp32 accumulate) on tcgen05; op 0 = NN, 1 = NT, 2 = TN.
// out_f32: C is fp32 (op 2 only: the dW product of fp32 gradient reduction).
GemmStatus gemm_bf16_tc(int op, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                        const void* B, int64_t ldb, void* C, int64_t ldc, int num_sms,
                        cudaStream_t stream, const EpiTarget* epi = nullptr, bool out_f32 = false,
                        const SideSum* side = nullptr);

// The launch error behind the last GemmStatus::kLaunch on this thread (the
// launch helpers consume cudaGetLastError()).
cudaError_t gemm_last_launch_error();
// launches that used the stream-K tail (axonn_stream_k_launches)
long long gemm_stream_k_launches();
// the stream-K items of one CTA pair (axonn_stream_k_items); returns the count
int gemm_stream_k_items(int sk_tiles, int num_kb, int cluster, int nclusters, int* tile, int* role,
                        int* kb0, int* kb1, int cap);

// fp32 SIMT FMA (test mode, no TF32): same op codes.
GemmStatus gemm_f32_simt(int op, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                         const float* B, int64_t ldb, float* C, int64_t ldc, cudaStream_t stream);

}  // namespace axonn
