// axonn.cpp — host runtime behind include/axonn.h.
//
// One process per GPU.  The runtime owns:
//   * the world NCCL communicator and the four axis sub-communicators
//     (X, Y, Z, DATA; ncclCommSplit with key = axis coordinate, so NCCL rank
//     order is the coordinate order of PAPER.md:505-510);
//   * one high-priority communication stream per axis;
//   * layer handles (Alg. 1 state: cached I, gathered W, dW partial, events);
//   * GEMM instrumentation (CUDA events on the launching stream).
// Scheduling of one layer (Alg. 1, with the paper's overlap
// optimisations PAPER.md:644-680):
//   forward : [Z stream]  all-gather_z(W_hat) -> W          (OAG: may be prefetched)
//             [caller]    wait AG; GEMM chunk c of I x W; record chunk event
//             [fwd stream] per chunk: wait chunk event; all-reduce that chunk
//             [caller]    wait last all-reduce
//   backward: [caller]    GEMM dO x W^T -> dI
//             [bwd stream] wait; all-reduce(dI)                (OAR, overlaps next GEMM)
//             [caller]    GEMM I^T x dO -> dW partial
//             [Z stream]  wait; reduce-scatter_z -> dW_hat     (ORS: not waited here)
//             [D stream]  wait RS; all-reduce_data(dW_hat)     (per layer)
//             [caller]    wait all-reduce(dI)
//   grads_sync: caller waits every pending RS / DP all-reduce.
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <algorithm>
#include <set>
#include <string>
#include <vector>

#include "../../include/axonn.h"
#include "act.h"
#include "gemm.h"
#include "perf_model.h"
#include "runtime.h"
#include "sym.h"

namespace {

thread_local std::string g_err;

axonn_status_t fail(axonn_status_t s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(AXONN_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(e_));         \
  } while (0)

#define NCCL_TRY(expr)                                                                     \
  do {                                                                                     \
    ncclResult_t r_ = (expr);                                                              \
    if (r_ != ncclSuccess)                                                                 \
      return fail(AXONN_ERR_NCCL, "%s failed: %s", #expr, ncclGetErrorString(r_));         \
  } while (0)

#define STATUS_TRY(expr)                  \
  do {                                    \
    axonn_status_t s_ = (expr);           \
    if (s_ != AXONN_OK) return s_;        \
  } while (0)

enum Axis { AX_X = 0, AX_Y = 1, AX_Z = 2, AX_D = 3 };

struct ProfRec {
  cudaEvent_t start, stop;
  double flops;
};

struct State {
  bool booted = false;
  int rank = 0, world = 1, device = -1, num_sms = 0, gemm_sms = 0;
  ncclComm_t world_comm = nullptr;
  bool grid = false;
  int g[4] = {1, 1, 1, 1};
  int c[4] = {0, 0, 0, 0};
  ncclComm_t axis_comm[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaStream_t cstream[4] = {nullptr, nullptr, nullptr, nullptr};
  axonn::SymAxis sym[4];          // NVLS symmetric memory per axis (fused all-reduce)
  std::string sym_why[4];         // why an axis has no fused path
  int* flag_dev = nullptr;        // agree_all scratch
  std::vector<cudaEvent_t> pending_grads;
  std::set<struct ::axonn_fc*> handles;
  bool profiling = false;
  int64_t comm_bytes[5] = {0, 0, 0, 0, 0};  // ring bytes sent per rank: ag_z, rs_z, ar_fwd, ar_bwd, ar_d
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> prof_free;
  // background zeroing of kRedPair outputs (copy engines): a stream and a
  // zero source the copies read from
  cudaStream_t zstream = nullptr;
  void* zsrc = nullptr;
  size_t zsrc_bytes = 0;
};

State S;
std::recursive_mutex g_mu;
std::atomic<int64_t> g_launches{0};

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
// Activations and weights (O, dI, W, AG_z, AR_x/y): the dtype's storage.
inline size_t elem_size(int dtype) { return dtype == AXONN_F32 ? 4 : 2; }
inline ncclDataType_t nccl_type(int dtype) {
  return dtype == AXONN_F32 ? ncclFloat32 : ncclBfloat16;
}
// The weight gradient (dWpart, dŴ, RS_z, data-parallel AR): fp32 for
// AXONN_BF16_GRADF32 (reading R17).
inline int act_dtype(int dtype) { return dtype == AXONN_BF16_GRADF32 ? AXONN_BF16 : dtype; }
inline int grad_dtype(int dtype) { return dtype == AXONN_BF16 ? AXONN_BF16 : AXONN_F32; }
inline bool valid_dtype(int d) { return d == AXONN_BF16 || d == AXONN_F32 || d == AXONN_BF16_GRADF32; }

// Fail loudly unless the current device is an sm_100 part (the kernels are
// compiled for sm_100a only; there is no other path).
axonn_status_t ensure_device() {
  if (S.num_sms > 0) return AXONN_OK;
  int dev = 0, major = 0, minor = 0, sms = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (major != 10 || minor != 0)
    return fail(AXONN_ERR_CUDA, "libaxonn kernels are built for sm_100a; device %d is sm_%d%d",
                dev, major, minor);
  S.device = dev;
  S.num_sms = sms;
  if (S.gemm_sms <= 0 || S.gemm_sms > sms) S.gemm_sms = sms;
  return AXONN_OK;
}


// Events that order work ACROSS calls (ev_rsdone: the previous fused RS_z
// owner phase; ev_wdone: the previous deferred data-parallel reduction).
// Under stream capture they become external event nodes, so a graph replay
// waits on the previous iteration's (or the eager run's) real record exactly
// as eager execution does; a plain capture would reject the dependency on
// uncaptured work (or drop it).
bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive;
}
cudaError_t record_xcall(cudaEvent_t e, cudaStream_t st) {
  return capturing(st) ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal)
                       : cudaEventRecord(e, st);
}
cudaError_t wait_xcall(cudaStream_t st, cudaEvent_t e) {
  return cudaStreamWaitEvent(st, e, capturing(st) ? cudaEventWaitExternal : 0);
}

// Per-rank bytes a ring collective sends (Assumption-1):
// all-gather (p-1)*count, reduce-scatter (p-1)*recvcount, all-reduce
// 2(p-1)/p*count — the quantities of Eqs. 1-5.
void count_comm(int kind, int p, size_t count, int dtype) {
  const int64_t b = static_cast<int64_t>(elem_size(dtype));
  const int64_t c = static_cast<int64_t>(count);
  int64_t bytes = 0;
  if (kind == 0 || kind == 1) bytes = (p - 1) * c * b;           // AG: count = sendcount; RS: recvcount
  else bytes = (2 * (p - 1) * c * b) / p;                         // AR
  S.comm_bytes[kind] += bytes;
}

axonn_status_t check_async_nccl() {
  for (int a = 0; a < 4; ++a) {
    if (!S.axis_comm[a]) continue;
    ncclResult_t ar = ncclSuccess;
    NCCL_TRY(ncclCommGetAsyncError(S.axis_comm[a], &ar));
    if (ar != ncclSuccess && ar != ncclInProgress)
      return fail(AXONN_ERR_NCCL, "asynchronous NCCL error on axis %d: %s", a,
                  ncclGetErrorString(ar));
  }
  return AXONN_OK;
}

// One local product on `st`, instrumented.  K == 0 writes zeros.
axonn_status_t run_gemm(int op, int dtype, int64_t M, int64_t N, int64_t K, const void* A,
                        int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                        cudaStream_t st, const axonn::EpiTarget* epi = nullptr,
                        const axonn::SideSum* side = nullptr) {
  STATUS_TRY(ensure_device());
  if (M == 0 || N == 0) return AXONN_OK;
  const size_t es = dtype == AXONN_BF16_GRADF32 ? 4 : elem_size(dtype);  // of C
  if (K == 0) {
    // a zero partial: nothing to add into a fused (pre-zeroed) reduction buffer
    if (epi && epi->mode == axonn::kScatter)
      return fail(AXONN_ERR_UNSUPPORTED, "fused reduce-scatter of an empty product");
    if (!epi || epi->mode == axonn::kStore)
      CUDA_TRY(cudaMemset2DAsync(C, ldc * es, 0, N * es, M, st));
    return AXONN_OK;
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // Inside a CUDA-graph capture a plain event record is only a dependency
  // marker; timing events must become external event-record nodes.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (S.profiling) CUDA_TRY(cudaStreamIsCapturing(st, &cap));
  auto record = [&](cudaEvent_t e) {
    return cap == cudaStreamCaptureStatusActive
               ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal)
               : cudaEventRecord(e, st);
  };
  if (S.profiling) {
    for (cudaEvent_t* e : {&e0, &e1}) {
      if (!S.prof_free.empty()) {
        *e = S.prof_free.back();
        S.prof_free.pop_back();
      } else {
        CUDA_TRY(cudaEventCreate(e));
      }
    }
    CUDA_TRY(record(e0));
  }
  axonn::GemmStatus gs;
  if (dtype == AXONN_BF16 || dtype == AXONN_BF16_GRADF32)
    gs = axonn::gemm_bf16_tc(op, M, N, K, A, lda, B, ldb, C, ldc, S.gemm_sms, st, epi,
                             dtype == AXONN_BF16_GRADF32, side);
  else
    gs = axonn::gemm_f32_simt(op, M, N, K, static_cast<const float*>(A), lda,
                              static_cast<const float*>(B), ldb, static_cast<float*>(C), ldc, st);
  switch (gs) {
    case axonn::GemmStatus::kOk: break;
    case axonn::GemmStatus::kBadAlignment:
      return fail(AXONN_ERR_ARG, "gemm: bf16 operands need 16-byte aligned bases and ld %% 8 == 0");
    case axonn::GemmStatus::kBadShape:
      return fail(AXONN_ERR_SHAPE, "gemm: dimension exceeds 2^31-1");
    case axonn::GemmStatus::kTensorMap:
      return fail(AXONN_ERR_CUDA, "gemm: cuTensorMapEncodeTiled failed");
    case axonn::GemmStatus::kBadOp:
      return fail(AXONN_ERR_ARG, dtype == AXONN_BF16_GRADF32
                                     ? "gemm: fp32 output is implemented for op 2 (TN) only"
                                     : "gemm: op must be 0 (NN), 1 (NT) or 2 (TN)");
    default: {
      cudaError_t e = axonn::gemm_last_launch_error();
      if (e == cudaSuccess) e = cudaGetLastError();
      return fail(AXONN_ERR_CUDA, "gemm launch failed: %s", cudaGetErrorString(e));
    }
  }
  g_launches.fetch_add(1);
  if (S.profiling) {
    CUDA_TRY(record(e1));
    S.prof.push_back({e0, e1, 2.0 * static_cast<double>(M) * N * K});
  }
  return AXONN_OK;
}

int coords_to_rank(const int g[4], const int c[4]) {
  return c[0] + g[0] * (c[1] + g[1] * (c[2] + g[2] * c[3]));
}

axonn_status_t check_grid_args(int gx, int gy, int gz, int gd) {
  if (gx < 1 || gy < 1 || gz < 1 || gd < 1)
    return fail(AXONN_ERR_CONFIG, "configuration error: factors (%d,%d,%d,%d) must be >= 1", gx,
                gy, gz, gd);
  return AXONN_OK;
}

axonn_status_t geometry_of(const axonn_fc_desc_t* d, const int g[4], int rank,
                           axonn_geometry_t* out) {
  if (!d || !out) return fail(AXONN_ERR_ARG, "NULL argument");
  if (d->m < 0 || d->k < 0 || d->n < 0) return fail(AXONN_ERR_ARG, "negative dimension");
  if (!valid_dtype(d->dtype))
    return fail(AXONN_ERR_ARG, "dtype must be AXONN_BF16, AXONN_F32 or AXONN_BF16_GRADF32");
  if (d->act != AXONN_ACT_NONE && d->act != AXONN_ACT_GELU)
    return fail(AXONN_ERR_ARG, "act must be AXONN_ACT_NONE or AXONN_ACT_GELU");
  const int G = g[0] * g[1] * g[2] * g[3];
  if (rank < 0 || rank >= G) return fail(AXONN_ERR_ARG, "rank %d outside grid of %d", rank, G);
  const bool t = d->transposed != 0;
  const int ga = t ? g[AX_X] : g[AX_Y];
  const int gb = t ? g[AX_Y] : g[AX_X];
  const char* na = t ? "Gx" : "Gy";
  const char* nb = t ? "Gy" : "Gx";
  const int64_t zd = static_cast<int64_t>(g[AX_Z]) * g[AX_D];
  if (d->m % zd)
    return fail(AXONN_ERR_SHAPE, "m=%lld not divisible by Gz*Gd=%lld", (long long)d->m,
                (long long)zd);
  if (d->k % ga) return fail(AXONN_ERR_SHAPE, "k=%lld not divisible by %s=%d", (long long)d->k, na, ga);
  if (d->n % gb) return fail(AXONN_ERR_SHAPE, "n=%lld not divisible by %s=%d", (long long)d->n, nb, gb);
  const int64_t k_l = d->k / ga, n_l = d->n / gb;
  if ((k_l * n_l) % g[AX_Z])
    return fail(AXONN_ERR_SHAPE, "k_l*n_l=%lld not divisible by Gz=%d", (long long)(k_l * n_l),
                g[AX_Z]);
  int c[4];
  int r = rank;
  for (int a = 0; a < 4; ++a) {
    c[a] = r % g[a];
    r /= g[a];
  }
  const int ia = t ? c[AX_X] : c[AX_Y];  // contraction-block index
  const int ib = t ? c[AX_Y] : c[AX_X];  // output-column-block index
  out->m_l = d->m / zd;
  out->k_l = k_l;
  out->n_l = n_l;
  out->row0 = (static_cast<int64_t>(c[AX_D]) * g[AX_Z] + c[AX_Z]) * out->m_l;
  out->in_col0 = ia * k_l;
  out->out_col0 = ib * n_l;
  out->what_len = k_l * n_l / g[AX_Z];
  out->what_off = c[AX_Z] * out->what_len;
  return AXONN_OK;
}

}  // namespace

// ============================================================== layer handle
struct axonn_fc {
  axonn_fc_desc_t d;
  axonn_geometry_t geo;
  int ax_fwd, ax_bwd;         // axis of the forward / backward-dI all-reduce
  void* wbuf = nullptr;       // gathered W_{j,i} when Gz > 1
  void* zbuf = nullptr;       // act: Z = all-reduce(Ô) kept for the backward (R18)
  void* dzbuf = nullptr;      // act: dZ = dO ⊙ GELU'(Z)
  void* dwpart = nullptr;     // dW partial when Gz > 1
  const void* I = nullptr;    // cached I_{k,j} (caller-owned)
  const void* W = nullptr;    // W_{j,i} used by the last forward
  bool have_fwd = false;
  bool prefetched = false;
  cudaEvent_t ev_in = nullptr, ev_ag = nullptr, ev_ar = nullptr, ev_dw = nullptr,
              ev_rs = nullptr, ev_grad = nullptr;
  std::vector<cudaEvent_t> ev_chunk;
  // fused all-reduces (epi.mode == kStore: NCCL path)
  struct Fused {
    int axis = 0;
    int es = 2;                // element bytes: 2 (bf16), 4 (fp32 dŴ, AXONN_BF16_GRADF32)
    size_t elems = 0;
    void* out_peer = nullptr;  // 2-rank scatter mode: the peer's copy of our slice
    axonn::SymBuf out;    // every rank's result (handle-owned output buffer)
    axonn::SymBuf recv;   // P-rank scatter mode: P slots of elems / P; exchange: P slots of elems
    axonn::SymBuf recv2;  // exchange mode: the second receive buffer (device-side parity)
    int* par = nullptr;   // exchange mode: parity counter, advanced by the post barrier
    axonn::SymBuf ctrl;   // pair-sum mode: arbitration tickets + done / call counters;
                          // exchange mode: the side-sum words (arrive, go, finished)
    int* side_arrive_peer = nullptr;  // exchange mode: the peer's arrive word (LSA)
    // kRedPair: the output was zeroed in the background once its last reader
    // (the next layer's backward) was enqueued; the next use waits for it
    bool prezeroed = false;
    cudaEvent_t ev_zeroed = nullptr;
    long long chunks = 0; // pair-sum mode: 32 x 64 output chunks
    int64_t cols = 0;     // row length of the reduced output
    axonn::EpiTarget epi;
  };
  Fused fo;   // O   over the forward axis      (Alg. 1 line 4 fused into line 3)
  Fused fi;   // dI  over the backward axis     (line 12 fused into line 11)
  Fused fw;   // dŴ  over DATA when Gz == 1     (PAPER.md:313-317 fused into line 13)
  Fused fz;   // RS_z fused into line 13: the epilogue scatters to the slice owners
  Fused fd;   // dŴ over DATA when Gz > 1: the RS_z owner phase scatters its reduced
              // slice to the DATA owners (PAPER.md:313-317 fused into line 14)
  axonn::SymBuf wstage;        // AG_z over copy engines: symmetric staging copy of Ŵ
  std::vector<void*> wpeer;    // every Z rank's staging address (LSA)
  std::string fused_why;            // non-empty: fused buffers fell back to NCCL
  cudaEvent_t ev_rsdone = nullptr;  // last fused RS_z finished reading its slots
  cudaEvent_t ev_wdone = nullptr;   // last deferred data-parallel reduction finished
};

namespace {

// Barrier index 0: barriers issued on the caller's stream (and, for Z, the Z
// stream, which is the only stream issuing Z barriers); index 1: the deferred
// data-parallel reductions on the DATA stream.
axonn_status_t fused_barrier(int axis, cudaStream_t st, int index) {
  CUDA_TRY(axonn::sym_barrier(&S.sym[axis], st, index));
  g_launches.fetch_add(1);
  return AXONN_OK;
}

// Fused all-reduce of a rows x cols output over `axis` (see sym.cu):
// 2 ranks: multimem.red straight from the epilogue (RNE(a + b), exact
// commutative: bit-identical to NCCL); P >= 3: the epilogue scatters 16-B
// vectors to their owner rank, the owner sums the P slots in rank order and
// multicasts the result (every element reduced once: replicas bit-identical).
// `kdim` is the contraction length of the producing GEMM: its output leaves the
// epilogue at ~(GEMM flop rate)/K bytes/s.  2-rank axes use multimem.red when
// that rate stays well inside what NVLS reductions sustain from the epilogue
// (K >= AXONN_RED_MIN_K, default 8192): fully overlapped, no extra pass.
// Shorter K (e.g. the transposed proj layer, K = h/Gx) uses the scatter mode,
// whose epilogue traffic is half as large and goes out as plain stores.
//
// Buffers are created in two phases: fused_plan records the
// symmetric buffers a layer needs; axonn_fc_create allocates them locally,
// agrees on the outcome over the world, and only then registers the windows
// (collective), so every rank makes the same sequence of collective calls.
struct SymReq {
  int axis;
  size_t bytes;
  axonn::SymBuf* buf;
};

void fused_plan(axonn_fc::Fused* f, int axis, int64_t rows, int64_t cols, int64_t kdim, int es,
                std::vector<SymReq>* reqs) {
  f->axis = axis;
  f->es = es;
  f->epi = axonn::EpiTarget();
  if (!S.sym[axis].impl) return;
  const int mode = axonn::fused_mode(S.g[axis], es, rows, cols, kdim,
                                     env_int("AXONN_RED_MIN_K", 8192),
                                     env_int("AXONN_EXCHANGE", 1) != 0,
                                     env_int("AXONN_PAIRSUM", 0) != 0,
                                     env_int("AXONN_XSUM", 0), env_int("AXONN_REDPAIR", 2));
  if (mode == axonn::kStore) return;
  f->elems = static_cast<size_t>(rows * cols);
  f->cols = cols;
  if (mode == axonn::kXSum) {
    // two receive sets of 2 slots (the call counter's parity picks one), the
    // output, and the flag / done / counter block
    f->epi.mode = mode;
    reqs->push_back({axis, f->elems * es, &f->out});
    reqs->push_back({axis, f->elems * es * 2, &f->recv});
    reqs->push_back({axis, f->elems * es * 2, &f->recv2});
    reqs->push_back({axis, axonn::xsum_ctrl_bytes(axonn::xsum_units(rows, cols)), &f->ctrl});
    return;
  }
  if (mode == axonn::kPairSum) {
    f->chunks = ((rows + 31) / 32) * ((cols + 63) / 64);
    f->epi.mode = mode;
    reqs->push_back({axis, f->elems * es, &f->out});
    reqs->push_back({axis, f->elems * es, &f->recv});
    reqs->push_back({axis, axonn::pair_ctrl_bytes(f->chunks), &f->ctrl});
    return;
  }
  f->epi.mode = mode;  // targets are bound after registration (fused_bind)
  reqs->push_back({axis, f->elems * es, &f->out});
  if (mode == axonn::kScatter) reqs->push_back({axis, f->elems * es, &f->recv});
  if (mode == axonn::kExchange) {
    const int P = S.g[axis];
    reqs->push_back({axis, f->elems * es * P, &f->recv});
    reqs->push_back({axis, f->elems * es * P, &f->recv2});
    reqs->push_back({axis, 256, &f->ctrl});  // side-sum words (SideSum)
  }
}

// After registration: the epilogue targets (multicast address, or every
// rank's receive slot) and, on 2-rank scatter axes, the peer's output copy.
bool fused_bind(axonn_fc::Fused* f, std::string* why) {
  if (f->epi.mode == axonn::kStore) return true;
  if (f->epi.mode == axonn::kMcRed) {
    f->epi = axonn::epi_red(reinterpret_cast<unsigned long long>(f->out.mc));
    return true;
  }
  if (f->epi.mode == axonn::kRedPair) {
    void* pout = axonn::sym_peer_ptr(&f->out, 1 - S.c[f->axis]);
    if (!pout) {
      *why = "peer address of the output window unavailable";
      return false;
    }
    axonn::EpiTarget t;
    t.mode = axonn::kRedPair;
    t.P = 2;
    t.me = S.c[f->axis];
    t.mc = reinterpret_cast<unsigned long long>(f->out.ptr);
    t.peer[0] = reinterpret_cast<unsigned long long>(pout);
    f->epi = t;
    return true;
  }
  const int P = S.g[f->axis], me = S.c[f->axis];
  if (f->epi.mode == axonn::kXSum) {
    unsigned long long recv[2], alt[2];
    for (int q = 0; q < 2; ++q) {
      recv[q] = reinterpret_cast<unsigned long long>(axonn::sym_peer_ptr(&f->recv, q));
      alt[q] = reinterpret_cast<unsigned long long>(axonn::sym_peer_ptr(&f->recv2, q));
    }
    void* pctrl = axonn::sym_peer_ptr(&f->ctrl, 1 - me);
    if (!recv[0] || !recv[1] || !alt[0] || !alt[1] || !pctrl) {
      *why = "peer address of an exchange-sum window unavailable";
      return false;
    }
    const long long rows = static_cast<long long>(f->elems) / f->cols;
    if (cudaMemset(f->ctrl.ptr, 0, axonn::xsum_ctrl_bytes(axonn::xsum_units(rows, f->cols))) !=
            cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
      *why = "zeroing the exchange-sum control block failed";
      return false;
    }
    f->epi = axonn::epi_xsum(me, rows, f->cols, recv, alt, f->out.ptr, f->ctrl.ptr, pctrl);
    f->epi.mc = static_cast<unsigned long long>(env_int("AXONN_XSUM_OPT", 0));  // experiments
    return true;
  }
  if (f->epi.mode == axonn::kPairSum) {
    char* precv = static_cast<char*>(axonn::sym_peer_ptr(&f->recv, 1 - me));
    char* pout = static_cast<char*>(axonn::sym_peer_ptr(&f->out, 1 - me));
    char* pctrl = static_cast<char*>(axonn::sym_peer_ptr(&f->ctrl, 1 - me));
    char* arb = static_cast<char*>(axonn::sym_peer_ptr(&f->ctrl, 0));
    if (!precv || !pout || !pctrl || !arb) {
      *why = "peer address of a pair-sum window unavailable";
      return false;
    }
    if (cudaMemset(f->ctrl.ptr, 0, axonn::pair_ctrl_bytes(f->chunks)) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
      *why = "zeroing the pair-sum control block failed";
      return false;
    }
    axonn::EpiTarget t;
    t.mode = axonn::kPairSum;
    t.P = 2;
    t.me = me;
    t.slice = (f->cols + 63) / 64;
    t.mc = reinterpret_cast<unsigned long long>(arb);
    const size_t done = axonn::pair_done_off(f->chunks);
    // AXONN_PAIRSUM=1 push: our partial goes to the peer's receive buffer
    // (peer[1]) and the second arriver reads the peer's from ours (peer[0]);
    // =2 pull: our partial stays in our own buffer and the second arriver
    // reads the peer's over NVLink from the peer's buffer — per rank half the
    // NVLink bytes of push on average (the first arriver sends nothing)
    const bool pull = env_int("AXONN_PAIRSUM", 0) == 2;
    t.peer[0] = reinterpret_cast<unsigned long long>(pull ? static_cast<void*>(precv) : f->recv.ptr);
    t.peer[1] = reinterpret_cast<unsigned long long>(pull ? f->recv.ptr : static_cast<void*>(precv));
    t.peer[2] = reinterpret_cast<unsigned long long>(f->out.ptr);
    t.peer[3] = reinterpret_cast<unsigned long long>(pout);
    t.peer[4] = reinterpret_cast<unsigned long long>(static_cast<char*>(f->ctrl.ptr) + done);
    t.peer[5] = reinterpret_cast<unsigned long long>(pctrl + done);
    f->epi = t;
    return true;
  }
  unsigned long long peer[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int q = 0; q < P; ++q) {
    peer[q] = reinterpret_cast<unsigned long long>(axonn::sym_peer_ptr(&f->recv, q));
    if (!peer[q]) {
      *why = "peer address of the receive window unavailable";
      return false;
    }
  }
  if (f->epi.mode == axonn::kExchange) {
    unsigned long long alt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int q = 0; q < P; ++q) {
      alt[q] = reinterpret_cast<unsigned long long>(axonn::sym_peer_ptr(&f->recv2, q));
      if (!alt[q]) {
        *why = "peer address of the receive window unavailable";
        return false;
      }
    }
    if (cudaMalloc(&f->par, sizeof(int)) != cudaSuccess || cudaMemset(f->par, 0, sizeof(int)) != cudaSuccess) {
      *why = "cudaMalloc of the exchange parity counter failed";
      return false;
    }
    f->epi = axonn::epi_exchange(P, me, static_cast<long long>(f->elems), peer, alt, f->par);
    if (P == 2 && f->ctrl.ptr) {
      f->side_arrive_peer = static_cast<int*>(axonn::sym_peer_ptr(&f->ctrl, 1 - me));
      if (!f->side_arrive_peer || cudaMemset(f->ctrl.ptr, 0, 256) != cudaSuccess ||
          cudaDeviceSynchronize() != cudaSuccess) {
        *why = "exchange side-sum words unavailable";
        return false;
      }
    }
    return true;
  }
  f->epi = axonn::epi_scatter(P, me, static_cast<long long>(f->elems) / P, peer);
  if (P == 2) {  // the owner sends its reduced slice to the peer with plain stores
    char* peer_out = static_cast<char*>(axonn::sym_peer_ptr(&f->out, 1 - me));
    if (!peer_out) {
      *why = "peer address of the output window unavailable";
      return false;
    }
    f->out_peer = peer_out + static_cast<size_t>(me) * f->epi.slice * f->es;
  }
  return true;
}

// Where the owner phase of a scatter-mode reduction writes its slice: its
// own copy (+ the peer's on 2-rank axes), or every copy through multimem.st.
axonn::OwnerOut owner_out(const axonn_fc::Fused& f) {
  axonn::OwnerOut o;
  const size_t off = static_cast<size_t>(f.epi.me) * f.epi.slice * f.es;
  if (f.out_peer) {
    o.mode = axonn::kOwnPlain;
    o.n_dst = 2;
    o.dst[0] = reinterpret_cast<unsigned long long>(static_cast<char*>(f.out.ptr) + off);
    o.dst[1] = reinterpret_cast<unsigned long long>(f.out_peer);
  } else {
    o.mode = axonn::kOwnMc;
    o.n_dst = 1;
    o.dst[0] = reinterpret_cast<unsigned long long>(f.out.mc) + off;
  }
  return o;
}

axonn_status_t fused_barrier(int axis, cudaStream_t st, int index = 0);

// Back to the NCCL path: free a fused record's windows and clear its target.
void fused_reset(axonn_fc::Fused* f) {
  axonn::sym_free(&S.sym[f->axis], &f->out);
  axonn::sym_free(&S.sym[f->axis], &f->recv);
  axonn::sym_free(&S.sym[f->axis], &f->recv2);
  axonn::sym_free(&S.sym[f->axis], &f->ctrl);
  if (f->par) cudaFree(f->par);
  f->par = nullptr;
  f->epi = axonn::EpiTarget();
  f->out_peer = nullptr;
  f->side_arrive_peer = nullptr;
  if (f->ev_zeroed) cudaEventDestroy(f->ev_zeroed);
  f->ev_zeroed = nullptr;
  f->prezeroed = false;
  f->elems = 0;
}

// *ok := AND over every rank of the world (host; synchronous; no-op at 1 rank).
axonn_status_t agree_all(bool* ok) {
  if (S.world <= 1 || !S.world_comm) return AXONN_OK;
  if (!S.flag_dev) CUDA_TRY(cudaMalloc(&S.flag_dev, sizeof(int)));
  int v = *ok ? 1 : 0;
  cudaStream_t st = S.cstream[AX_X];  // the library's own stream, never under capture
  CUDA_TRY(cudaMemcpyAsync(S.flag_dev, &v, sizeof v, cudaMemcpyHostToDevice, st));
  NCCL_TRY(ncclAllReduce(S.flag_dev, S.flag_dev, 1, ncclInt32, ncclMin, S.world_comm, st));
  CUDA_TRY(cudaMemcpyAsync(&v, S.flag_dev, sizeof v, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *ok = v != 0;
  return AXONN_OK;
}

axonn_status_t fused_pre(axonn_fc::Fused& f, cudaStream_t st) {
  if ((f.epi.mode == axonn::kRedPair || f.epi.mode == axonn::kMcRed) && f.prezeroed) {
    // zeroed on the copy engines after its last reader; every rank's zeroing
    // is ordered before its barrier, so after it every copy is zero
    f.prezeroed = false;
    CUDA_TRY(cudaStreamWaitEvent(st, f.ev_zeroed, 0));
    return fused_barrier(f.axis, st);
  }
  if (f.epi.mode == axonn::kMcRed || f.epi.mode == axonn::kRedPair) {
    // zero every rank's copy, and order that before any rank's reductions
    CUDA_TRY(cudaMemsetAsync(f.out.ptr, 0, f.elems * f.es, st));
    return fused_barrier(f.axis, st);
  }
  return AXONN_OK;  // scatter: the previous use's final barrier already freed the slots
}

// `buf` (a layer input or output gradient the caller passed) is read for the
// last time by work already enqueued on `st`.  If it is the red.add output of
// some layer (kRedPair or multimem.red), zero it now on the copy engines, off
// the critical path; its next fused_pre then only waits for that
// (AXONN_PREZERO=0: zero inline).
axonn_status_t prezero_after(const void* buf, cudaStream_t st) {
  static const bool on = env_int("AXONN_PREZERO", 1) != 0;
  if (!on || !buf) return AXONN_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(st, &cs));
  if (cs != cudaStreamCaptureStatusNone) return AXONN_OK;  // graphs: zero inline at the next use
  for (axonn_fc* o : S.handles) {
    for (axonn_fc::Fused* f : {&o->fo, &o->fi}) {
      const bool red = f->epi.mode == axonn::kRedPair || f->epi.mode == axonn::kMcRed;
      if (!red || f->out.ptr != buf || f->prezeroed) continue;
      const size_t bytes = f->elems * f->es;
      if (!S.zstream)
        CUDA_TRY(cudaStreamCreateWithFlags(&S.zstream, cudaStreamNonBlocking));
      if (S.zsrc_bytes < (size_t(32) << 20)) {
        if (S.zsrc) CUDA_TRY(cudaFree(S.zsrc));
        S.zsrc_bytes = size_t(32) << 20;
        CUDA_TRY(cudaMalloc(&S.zsrc, S.zsrc_bytes));
        CUDA_TRY(cudaMemset(S.zsrc, 0, S.zsrc_bytes));
        CUDA_TRY(cudaDeviceSynchronize());
      }
      if (!f->ev_zeroed) CUDA_TRY(cudaEventCreateWithFlags(&f->ev_zeroed, cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(f->ev_zeroed, st));
      CUDA_TRY(cudaStreamWaitEvent(S.zstream, f->ev_zeroed, 0));
      for (size_t o2 = 0; o2 < bytes; o2 += S.zsrc_bytes)
        CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(f->out.ptr) + o2, S.zsrc,
                                 std::min(S.zsrc_bytes, bytes - o2), cudaMemcpyDeviceToDevice,
                                 S.zstream));
      CUDA_TRY(cudaEventRecord(f->ev_zeroed, S.zstream));
      f->prezeroed = true;
    }
  }
  return AXONN_OK;
}

axonn_status_t fused_post(axonn_fc::Fused& f, cudaStream_t st, int index = 0,
                          void* act_z = nullptr) {
  if (f.epi.mode == axonn::kXSum) {
    // the GEMM summed what had landed; the sweep sums the rest as the peer's
    // flags come up (no barrier) and advances the call counter
    const long long rows = static_cast<long long>(f.elems) / f.cols;
    CUDA_TRY(axonn::sym_xsum_sweep(f.recv.ptr, f.recv2.ptr, f.out.ptr, f.ctrl.ptr, rows, f.cols,
                                   S.num_sms, st));
    g_launches.fetch_add(1);
    return AXONN_OK;
  }
  if (f.epi.mode == axonn::kPairSum) {
    // the epilogues of both ranks finished the sums; wait for the peer's
    // share of the chunks (no barrier, no pass over the output)
    char* c = static_cast<char*>(f.ctrl.ptr);
    CUDA_TRY(axonn::sym_pair_wait(c + axonn::pair_done_off(f.chunks),
                                  c + axonn::pair_calls_off(f.chunks),
                                  static_cast<uint32_t>(f.chunks), st));
    g_launches.fetch_add(1);
    return AXONN_OK;
  }
  if (f.epi.mode == axonn::kExchange) {
    // every rank's whole partial has landed in our slots (the barrier also
    // advances the parity counter); the sum is local, in slot order, so all
    // ranks hold the same bits and nothing crosses NVLink after the barrier
    CUDA_TRY(axonn::sym_barrier(&S.sym[f.axis], st, index, f.par));
    g_launches.fetch_add(1);
    axonn::OwnerOut o;
    o.n_dst = 1;
    o.local = 1;
    o.fast = env_int("AXONN_SUM_FAST", 1);
    o.dst[0] = reinterpret_cast<unsigned long long>(f.out.ptr);
    if (act_z) {  // the GeLU rides on the local sum: Z to act_z, GELU(Z) to the output
      o.dst[0] = reinterpret_cast<unsigned long long>(act_z);
      o.act = 1;
      o.act_dst = reinterpret_cast<unsigned long long>(f.out.ptr);
    }
    CUDA_TRY(axonn::sym_owner_reduce(f.recv.ptr, static_cast<long long>(f.elems), f.epi.P,
                                     f.es == 4, o, S.num_sms, st, f.par, f.recv2.ptr));
    g_launches.fetch_add(1);
    return AXONN_OK;
  }
  STATUS_TRY(fused_barrier(f.axis, st, index));  // every rank's epilogue writes have landed
  if (f.epi.mode == axonn::kScatter) {
    CUDA_TRY(axonn::sym_owner_reduce(f.recv.ptr, f.epi.slice, f.epi.P, f.es == 4, owner_out(f),
                                     S.num_sms, st));
    g_launches.fetch_add(1);
    STATUS_TRY(fused_barrier(f.axis, st, index));  // every owner's broadcast has landed
  }
  return AXONN_OK;
}

// inline: a forward that was not prefetched needs W_{j,i} at once, so the
// gather runs on the caller's stream itself with every SM pulling (Z barrier
// sequence 1), independent of prefetches queued on the Z stream (sequence 0).
// Staging reuse stays ordered across the two sequences: every gather's
// completion is joined into the caller's stream before its forward GEMM.
// Returns with h->prefetched = false and nothing to wait for.
axonn_status_t gather_inline(axonn_fc* h, const void* W_hat, cudaStream_t st) {
  const size_t bytes = static_cast<size_t>(h->geo.what_len) * elem_size(h->d.dtype);
  STATUS_TRY(fused_barrier(AX_Z, st, 1));  // peers are done reading my previous staging
  CUDA_TRY(cudaMemcpyAsync(h->wstage.ptr, W_hat, bytes, cudaMemcpyDeviceToDevice, st));
  STATUS_TRY(fused_barrier(AX_Z, st, 1));  // every rank's Ŵ is staged
  std::vector<const void*> src(S.g[AX_Z]);
  for (int q = 0; q < S.g[AX_Z]; ++q) src[q] = q == S.c[AX_Z] ? W_hat : h->wpeer[q];
  CUDA_TRY(axonn::sym_gather_pull(src.data(), S.g[AX_Z], bytes, h->wbuf, S.num_sms, st));
  g_launches.fetch_add(1);
  count_comm(0, S.g[AX_Z], static_cast<size_t>(h->geo.what_len), h->d.dtype);
  return AXONN_OK;
}

axonn_status_t issue_allgather(axonn_fc* h, const void* W_hat, cudaStream_t st) {
  if (S.g[AX_Z] == 1) {
    h->prefetched = true;
    return AXONN_OK;
  }
  const size_t S_el = static_cast<size_t>(h->geo.what_len);
  CUDA_TRY(cudaEventRecord(h->ev_in, st));
  CUDA_TRY(cudaStreamWaitEvent(S.cstream[AX_Z], h->ev_in, 0));
  if (h->wstage.ptr) {
    // AG_z on the copy engines (no SMs): stage Ŵ in symmetric memory, then
    // pull every rank's slice over NVLink into W_{j,i} in z order.
    cudaStream_t zs = S.cstream[AX_Z];
    const size_t bytes = S_el * elem_size(h->d.dtype);
    STATUS_TRY(fused_barrier(AX_Z, zs));  // peers are done reading my previous staging
    CUDA_TRY(cudaMemcpyAsync(h->wstage.ptr, W_hat, bytes, cudaMemcpyDeviceToDevice, zs));
    STATUS_TRY(fused_barrier(AX_Z, zs));  // every rank's Ŵ is staged
    std::vector<const void*> src(S.g[AX_Z]);
    for (int q = 0; q < S.g[AX_Z]; ++q) src[q] = q == S.c[AX_Z] ? W_hat : h->wpeer[q];
    CUDA_TRY(axonn::sym_gather_copy(src.data(), S.g[AX_Z], bytes, h->wbuf, zs));
    count_comm(0, S.g[AX_Z], S_el, h->d.dtype);
    CUDA_TRY(cudaEventRecord(h->ev_ag, zs));
    h->prefetched = true;
    return AXONN_OK;
  }
  NCCL_TRY(ncclAllGather(W_hat, h->wbuf, S_el, nccl_type(h->d.dtype), S.axis_comm[AX_Z],
                         S.cstream[AX_Z]));
  count_comm(0, S.g[AX_Z], S_el, h->d.dtype);
  CUDA_TRY(cudaEventRecord(h->ev_ag, S.cstream[AX_Z]));
  h->prefetched = true;
  return AXONN_OK;
}

// O_local holds Z = all-reduce(Ô): keep Z for the backward, O_local := GELU(Z)
axonn_status_t apply_act(axonn_fc* h, void* O_local, cudaStream_t st) {
  CUDA_TRY(axonn::gelu_forward_inplace(O_local, h->zbuf, h->geo.m_l * h->geo.n_l, S.num_sms, st));
  g_launches.fetch_add(1);
  return AXONN_OK;
}

}  // namespace

namespace axonn {
axonn_status_t rt_gemm(int op, int dtype, int64_t M, int64_t N, int64_t K, const void* A,
                       int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                       cudaStream_t st, const EpiTarget* epi, const SideSum* side) {
  return run_gemm(op, dtype, M, N, K, A, lda, B, ldb, C, ldc, st, epi, side);
}
axonn_status_t rt_fail(axonn_status_t s, const char* msg) { return fail(s, "%s", msg); }
void rt_count_launch() { g_launches.fetch_add(1); }
int rt_num_sms() { return S.num_sms; }
}  // namespace axonn

extern "C" {

const char* axonn_last_error(void) { return g_err.c_str(); }
int axonn_version(void) { return 200; }

axonn_status_t axonn_unique_id(unsigned char id[128]) {
  if (!id) return fail(AXONN_ERR_ARG, "NULL id");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  ncclUniqueId uid;
  NCCL_TRY(ncclGetUniqueId(&uid));
  std::memcpy(id, &uid, 128);
  return AXONN_OK;
}

axonn_status_t axonn_bootstrap(int world_rank, int world_size, const unsigned char* id,
                               int cuda_device) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (S.booted) return fail(AXONN_ERR_STATE, "already bootstrapped");
  if (world_size < 1 || world_rank < 0 || world_rank >= world_size || cuda_device < 0)
    return fail(AXONN_ERR_ARG, "bad rank/world/device (%d/%d/%d)", world_rank, world_size,
                cuda_device);
  if (world_size > 1 && !id) return fail(AXONN_ERR_ARG, "world_size > 1 needs an NCCL id");
  CUDA_TRY(cudaSetDevice(cuda_device));
  S.num_sms = 0;
  STATUS_TRY(ensure_device());
  if (world_size > 1) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    NCCL_TRY(ncclCommInitRankConfig(&S.world_comm, world_size, uid, world_rank, &cfg));
  }
  S.rank = world_rank;
  S.world = world_size;
  S.booted = true;
  return AXONN_OK;
}

axonn_status_t axonn_rank_to_coords(int rank, int gx, int gy, int gz, int gd, int coords[4]) {
  STATUS_TRY(check_grid_args(gx, gy, gz, gd));
  if (!coords) return fail(AXONN_ERR_ARG, "NULL coords");
  const int g[4] = {gx, gy, gz, gd};
  if (rank < 0 || rank >= gx * gy * gz * gd) return fail(AXONN_ERR_ARG, "rank out of range");
  int r = rank;
  for (int a = 0; a < 4; ++a) {
    coords[a] = r % g[a];
    r /= g[a];
  }
  return AXONN_OK;
}

axonn_status_t axonn_group_members(int rank, int gx, int gy, int gz, int gd, int axis,
                                   int* members) {
  int c[4];
  STATUS_TRY(axonn_rank_to_coords(rank, gx, gy, gz, gd, c));
  if (axis < 0 || axis > 3 || !members) return fail(AXONN_ERR_ARG, "bad axis or NULL members");
  const int g[4] = {gx, gy, gz, gd};
  for (int v = 0; v < g[axis]; ++v) {
    int cc[4] = {c[0], c[1], c[2], c[3]};
    cc[axis] = v;
    members[v] = coords_to_rank(g, cc);
  }
  return AXONN_OK;
}

axonn_status_t axonn_grid_init(int gx, int gy, int gz, int gd) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  STATUS_TRY(check_grid_args(gx, gy, gz, gd));
  const int G = gx * gy * gz * gd;
  if (S.grid) return fail(AXONN_ERR_STATE, "grid already initialised; call axonn_grid_finalize");
  if (!S.booted) {
    if (G != 1)
      return fail(AXONN_ERR_STATE, "axonn_bootstrap must precede a grid of %d ranks", G);
    S.rank = 0;  // single-GPU: bind to the current device, no communicator
    S.world = 1;
    S.num_sms = 0;
    STATUS_TRY(ensure_device());
    S.booted = true;
  }
  if (G != S.world)
    return fail(AXONN_ERR_CONFIG, "configuration error: gx*gy*gz*gd = %d != world size %d", G,
                S.world);
  const int g[4] = {gx, gy, gz, gd};
  std::memcpy(S.g, g, sizeof g);
  STATUS_TRY(axonn_rank_to_coords(S.rank, gx, gy, gz, gd, S.c));
  int lo = 0, hi = 0;
  CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  for (int a = 0; a < 4; ++a) {
    S.sym_why[a] = "axis of size 1: no collective";
    if (g[a] > 1) {
      int cc[4] = {S.c[0], S.c[1], S.c[2], S.c[3]};
      cc[a] = 0;
      const int color = coords_to_rank(g, cc);
      // NCCL kernels (the paths not fused below): NCCL's own CTA budget by
      // default; AXONN_NCCL_MAX_CTAS=n caps it (to fit beside a GEMM given
      // fewer SMs with axonn_set_gemm_sms).  Measured at G=4: capping at 8 costs
      // 0.6% on (1,1,2,2) and 2% on the all-NCCL (1,1,1,4) step.
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      const int max_ctas = env_int("AXONN_NCCL_MAX_CTAS", 0);
      if (max_ctas > 0) {
        cfg.maxCTAs = max_ctas;
        cfg.minCTAs = std::min(max_ctas, env_int("AXONN_NCCL_MIN_CTAS", 1));
        cfg.nvlsCTAs = max_ctas;
      }
      NCCL_TRY(ncclCommSplit(S.world_comm, color, S.c[a], &S.axis_comm[a], &cfg));
      // Symmetric memory for the fused GEMM + collective epilogues over NVLS
      // (2..8 ranks of one NVSwitch domain; AXONN_FUSED=0 disables, §4.3).
      S.sym_why[a].clear();
      if (g[a] > 8)
        S.sym_why[a] = "fused all-reduce implemented for up to 8 ranks";
      else if (env_int("AXONN_FUSED", 1) == 0)
        S.sym_why[a] = "disabled by AXONN_FUSED=0";
      else
        axonn::sym_axis_init(S.axis_comm[a], &S.sym[a], &S.sym_why[a]);
    }
    CUDA_TRY(cudaStreamCreateWithPriority(&S.cstream[a], cudaStreamNonBlocking, hi));
  }
  S.grid = true;
  return AXONN_OK;
}

axonn_status_t axonn_grid_coords(int* i, int* j, int* k, int* d) {
  if (!S.grid) return fail(AXONN_ERR_STATE, "no grid");
  if (!i || !j || !k || !d) return fail(AXONN_ERR_ARG, "NULL argument");
  *i = S.c[0];
  *j = S.c[1];
  *k = S.c[2];
  *d = S.c[3];
  return AXONN_OK;
}

axonn_status_t axonn_fc_destroy(axonn_fc_t h);

axonn_status_t axonn_grid_finalize(void) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!S.grid) return AXONN_OK;
  std::vector<axonn_fc*> hs(S.handles.begin(), S.handles.end());
  for (auto* h : hs) axonn_fc_destroy(h);
  for (int a = 0; a < 4; ++a) {
    if (S.cstream[a]) cudaStreamSynchronize(S.cstream[a]);
    axonn::sym_axis_destroy(&S.sym[a]);
    if (S.axis_comm[a]) ncclCommDestroy(S.axis_comm[a]);
    if (S.cstream[a]) cudaStreamDestroy(S.cstream[a]);
    S.axis_comm[a] = nullptr;
    S.cstream[a] = nullptr;
  }
  S.pending_grads.clear();
  if (S.flag_dev) cudaFree(S.flag_dev);
  S.flag_dev = nullptr;
  if (S.zstream) cudaStreamDestroy(S.zstream);
  if (S.zsrc) cudaFree(S.zsrc);
  S.zstream = nullptr;
  S.zsrc = nullptr;
  S.zsrc_bytes = 0;
  S.grid = false;
  return AXONN_OK;
}

axonn_status_t axonn_shard_geometry(const axonn_fc_desc_t* desc, int gx, int gy, int gz, int gd,
                                    int rank, axonn_geometry_t* out) {
  STATUS_TRY(check_grid_args(gx, gy, gz, gd));
  const int g[4] = {gx, gy, gz, gd};
  return geometry_of(desc, g, rank, out);
}

axonn_status_t axonn_fc_create(const axonn_fc_desc_t* desc, axonn_fc_t* out) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!desc || !out) return fail(AXONN_ERR_ARG, "NULL argument");
  if (!S.grid) return fail(AXONN_ERR_STATE, "axonn_grid_init must precede axonn_fc_create");
  axonn_geometry_t geo;
  STATUS_TRY(geometry_of(desc, S.g, S.rank, &geo));
  if (desc->dtype != AXONN_F32 && (geo.k_l % 8 || geo.n_l % 8))
    return fail(AXONN_ERR_SHAPE,
                "bf16 shards need k_l=%lld and n_l=%lld to be multiples of 8 (16-byte rows for TMA)",
                (long long)geo.k_l, (long long)geo.n_l);
  auto* h = new axonn_fc();
  h->d = *desc;
  if (h->d.chunks < 1) h->d.chunks = 1;
  h->geo = geo;
  h->ax_fwd = desc->transposed ? AX_X : AX_Y;
  h->ax_bwd = desc->transposed ? AX_Y : AX_X;
  const size_t wbytes = static_cast<size_t>(geo.k_l) * geo.n_l * elem_size(desc->dtype);
  const size_t gbytes = static_cast<size_t>(geo.k_l) * geo.n_l * elem_size(grad_dtype(desc->dtype));
  auto cleanup = [&](axonn_status_t s) {
    axonn_fc_destroy(h);
    return s;
  };
  S.handles.insert(h);
  if (desc->act != AXONN_ACT_NONE) {
    if (desc->dtype == AXONN_F32)
      return cleanup(fail(AXONN_ERR_UNSUPPORTED, "an activation needs bf16 activations"));
    const size_t zb = static_cast<size_t>(geo.m_l) * geo.n_l * 2;
    if (zb && (cudaMalloc(&h->zbuf, zb) != cudaSuccess || cudaMalloc(&h->dzbuf, zb) != cudaSuccess))
      return cleanup(fail(AXONN_ERR_CUDA, "cudaMalloc of %zu bytes failed", 2 * zb));
  }
  if (S.g[AX_Z] > 1 && wbytes) {
    if (cudaMalloc(&h->wbuf, wbytes) != cudaSuccess || cudaMalloc(&h->dwpart, gbytes) != cudaSuccess)
      return cleanup(fail(AXONN_ERR_CUDA, "cudaMalloc of %zu bytes failed", wbytes + gbytes));
  }
  for (cudaEvent_t* e : {&h->ev_in, &h->ev_ag, &h->ev_ar, &h->ev_dw, &h->ev_rs, &h->ev_grad,
                         &h->ev_rsdone, &h->ev_wdone})
    if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess)
      return cleanup(fail(AXONN_ERR_CUDA, "cudaEventCreate failed"));
  // Fused (NVLS) buffers.  A failure here is not fatal: the layer falls back
  // to NCCL collectives (still the GPU path), but only if EVERY rank does, so
  // the ranks agree (MIN over the world) before anything is used.  Local
  // allocations come first and are agreed on before any (collective) window
  // registration, so a rank that runs out of memory never leaves its peers
  // waiting inside a registration it will not make.
  std::string why;
  std::vector<SymReq> reqs;
  const int ges = static_cast<int>(elem_size(grad_dtype(desc->dtype)));
  if (desc->dtype != AXONN_F32) {
    // O and dI reduce bf16; dŴ in its gradient precision (fp32 for AXONN_BF16_GRADF32)
    fused_plan(&h->fo, h->ax_fwd, geo.m_l, geo.n_l, geo.k_l, 2, &reqs);
    fused_plan(&h->fi, h->ax_bwd, geo.m_l, geo.k_l, geo.n_l, 2, &reqs);
    if (S.g[AX_Z] == 1) fused_plan(&h->fw, AX_D, geo.k_l, geo.n_l, geo.m_l, ges, &reqs);
  }
  if (desc->dtype != AXONN_F32 && S.g[AX_Z] > 1 && S.sym[AX_Z].impl && geo.what_len > 0 &&
      geo.what_len % 8 == 0 && geo.m_l > 0) {
    // RS_z fused into the dW epilogue: owner of flat index f is f / S, its Ŵ slice (R4)
    h->fz.axis = AX_Z;
    h->fz.es = ges;
    h->fz.elems = static_cast<size_t>(geo.k_l * geo.n_l);
    h->fz.epi.mode = axonn::kScatter;
    reqs.push_back({AX_Z, h->fz.elems * ges, &h->fz.recv});
    reqs.push_back({AX_Z, static_cast<size_t>(geo.what_len) * 2, &h->wstage});
    // the data-parallel sum of dŴ fused behind it: the Z owner phase scatters
    // its reduced slice to the DATA owners (16-B units of what_len / Gd)
    const int Pd = S.g[AX_D];
    if (Pd > 1 && S.sym[AX_D].impl && geo.what_len % (static_cast<int64_t>(16 / ges) * Pd) == 0) {
      h->fd.axis = AX_D;
      h->fd.es = ges;
      h->fd.elems = static_cast<size_t>(geo.what_len);
      h->fd.epi.mode = axonn::kScatter;
      reqs.push_back({AX_D, h->fd.elems * ges, &h->fd.recv});
      reqs.push_back({AX_D, h->fd.elems * ges, &h->fd.out});
    }
  }
  bool ok = true;
  for (const SymReq& r : reqs) ok = ok && axonn::sym_mem_alloc(r.bytes, r.buf, &why);
  bool all_ok = ok;
  axonn_status_t st_agree = agree_all(&all_ok);
  if (st_agree != AXONN_OK) return cleanup(st_agree);
  if (all_ok) {
    // every rank registers every buffer, in the same order, even after a
    // failure (the calls are collective); the outcome is agreed again
    bool reg = true;
    for (const SymReq& r : reqs) {
      std::string w;
      if (!axonn::sym_register(&S.sym[r.axis], r.buf, &w) && reg) {
        reg = false;
        why = w;
      }
    }
    ok = reg && fused_bind(&h->fo, &why) && fused_bind(&h->fi, &why) && fused_bind(&h->fw, &why);
    if (ok && h->fz.epi.mode == axonn::kScatter) {
      const int P = S.g[AX_Z];
      unsigned long long peer[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      h->wpeer.resize(P);
      for (int q = 0; q < P && ok; ++q) {
        peer[q] = reinterpret_cast<unsigned long long>(axonn::sym_peer_ptr(&h->fz.recv, q));
        h->wpeer[q] = axonn::sym_peer_ptr(&h->wstage, q);
        if (!peer[q] || !h->wpeer[q]) {
          why = "peer address of a Z window unavailable";
          ok = false;
        }
      }
      if (ok) h->fz.epi = axonn::epi_scatter(P, S.c[AX_Z], geo.what_len, peer);
    }
    if (ok && h->fd.epi.mode == axonn::kScatter) ok = fused_bind(&h->fd, &why);
    all_ok = ok;
    st_agree = agree_all(&all_ok);
    if (st_agree != AXONN_OK) return cleanup(st_agree);
  }
  if (!all_ok) {
    for (axonn_fc::Fused* f : {&h->fo, &h->fi, &h->fw, &h->fz, &h->fd}) fused_reset(f);
    axonn::sym_free(&S.sym[AX_Z], &h->wstage);
    h->wpeer.clear();
    h->fused_why = ok ? "another rank could not allocate its fused buffers" : why;
    std::fprintf(stderr, "[axonn] rank %d: fused NVLS buffers unavailable (%s); this layer uses "
                 "NCCL collectives\n", S.rank, h->fused_why.c_str());
  }
  h->ev_chunk.resize(h->d.chunks + 1, nullptr);
  for (auto& e : h->ev_chunk)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return cleanup(fail(AXONN_ERR_CUDA, "cudaEventCreate failed"));
  *out = h;
  return AXONN_OK;
}

axonn_status_t axonn_fc_geometry(axonn_fc_t h, axonn_geometry_t* out) {
  if (!h || !out) return fail(AXONN_ERR_ARG, "NULL argument");
  *out = h->geo;
  return AXONN_OK;
}

axonn_status_t axonn_fc_output_buffer(axonn_fc_t h, int which, void** ptr) {
  if (!h || !ptr || which < 0 || which > 2) return fail(AXONN_ERR_ARG, "bad argument");
  const axonn_fc::Fused* f = which == 0 ? &h->fo : which == 1 ? &h->fi
                            : h->fd.epi.mode != axonn::kStore ? &h->fd : &h->fw;
  *ptr = f->epi.mode != axonn::kStore ? f->out.ptr : nullptr;
  return AXONN_OK;
}

axonn_status_t axonn_nvlink_probe(int axis, int64_t bytes, int mode, int ctas, int iters,
                                  double* gbps) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (axis < 0 || axis > 3 || bytes <= 0 || mode < 0 || mode > 6 || ctas < 1 || iters < 1 || !gbps)
    return fail(AXONN_ERR_ARG, "bad argument");
  if (!S.sym[axis].impl) return fail(AXONN_ERR_STATE, "axis %d has no symmetric memory: %s", axis,
                                     S.sym_why[axis].c_str());
  axonn::SymBuf b;
  std::string why;
  if (!axonn::sym_alloc(&S.sym[axis], static_cast<size_t>(bytes), &b, &why))
    return fail(AXONN_ERR_NCCL, "%s", why.c_str());
  float ms = 0.f;
  const int peer = (S.c[axis] + 1) % S.g[axis];
  cudaError_t e = axonn::sym_probe(&S.sym[axis], &b, mode, peer, ctas, iters, &ms);
  const double moved = static_cast<double>(b.bytes);
  axonn::sym_free(&S.sym[axis], &b);
  if (e != cudaSuccess) return fail(AXONN_ERR_CUDA, "probe: %s", cudaGetErrorString(e));
  *gbps = moved / (ms * 1e-3) / 1e9;
  return AXONN_OK;
}

axonn_status_t axonn_fused_mode(int P, int elem_bytes, int64_t rows, int64_t cols, int64_t kdim,
                                char* buf, int cap) {
  if (P < 1 || (elem_bytes != 2 && elem_bytes != 4) || rows < 0 || cols < 0 || kdim < 0 || !buf ||
      cap < 1)
    return fail(AXONN_ERR_ARG, "bad argument");
  // the same call fused_plan makes, with the same switches
  const int mode = axonn::fused_mode(P, elem_bytes, rows, cols, kdim,
                                     env_int("AXONN_RED_MIN_K", 8192),
                                     env_int("AXONN_EXCHANGE", 1) != 0,
                                     env_int("AXONN_PAIRSUM", 0) != 0, env_int("AXONN_XSUM", 0),
                                     env_int("AXONN_REDPAIR", 2));
  const char* name = mode == axonn::kRedPair    ? "red_add_pair"
                     : mode == axonn::kMcRed    ? "multimem_red"
                     : mode == axonn::kExchange ? "exchange"
                     : mode == axonn::kScatter  ? "scatter"
                     : mode == axonn::kXSum     ? "xsum"
                     : mode == axonn::kPairSum  ? "pair_sum"
                                                : "none";
  std::snprintf(buf, static_cast<size_t>(cap), "%s", name);
  return AXONN_OK;
}

axonn_status_t axonn_fused_status(int axis, char* buf, int cap) {
  if (axis < 0 || axis > 3 || !buf || cap < 1) return fail(AXONN_ERR_ARG, "bad argument");
  const std::string m = S.sym[axis].impl ? std::string("fused") : S.sym_why[axis];
  std::snprintf(buf, static_cast<size_t>(cap), "%s", m.c_str());
  return AXONN_OK;
}

axonn_status_t axonn_fc_prefetch(axonn_fc_t h, const void* W_hat, void* stream) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!h || (!W_hat && h->geo.what_len)) return fail(AXONN_ERR_ARG, "NULL argument");
  if (!S.grid) return fail(AXONN_ERR_STATE, "no grid");
  return issue_allgather(h, W_hat, as_stream(stream));
}

axonn_status_t axonn_fc_forward(axonn_fc_t h, const void* I_local, const void* W_hat,
                                void* O_local, void* stream) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!h) return fail(AXONN_ERR_ARG, "NULL handle");
  if (!S.grid) return fail(AXONN_ERR_STATE, "no grid");
  const axonn_geometry_t& g = h->geo;
  if ((!I_local && (g.m_l * g.k_l) != 0) || (!W_hat && g.what_len != 0) || (!O_local && (g.m_l * g.n_l) != 0))
    return fail(AXONN_ERR_ARG, "NULL tensor");
  STATUS_TRY(check_async_nccl());
  cudaStream_t st = as_stream(stream);
  // line 2: W_{j,i} = all-gather_z(W_hat)
  bool inline_ag = false;
  if (!h->prefetched) {
    inline_ag = S.g[AX_Z] > 1 && h->wstage.ptr && env_int("AXONN_AG_INLINE", 1) != 0;
    if (inline_ag)
      STATUS_TRY(gather_inline(h, W_hat, st));
    else
      STATUS_TRY(issue_allgather(h, W_hat, st));
  }
  h->prefetched = false;
  const void* W = S.g[AX_Z] > 1 ? h->wbuf : W_hat;
  if (S.g[AX_Z] > 1 && !inline_ag) CUDA_TRY(cudaStreamWaitEvent(st, h->ev_ag, 0));
  const int P = S.g[h->ax_fwd];
  const size_t es = elem_size(h->d.dtype);
  if (h->fo.epi.mode != axonn::kStore) {
    // line 3 + line 4 fused: the GEMM epilogue sends each bf16 tile of Ô
    // over NVLink (fused_setup); barriers order the buffer reuse.
    const size_t bytes = static_cast<size_t>(g.m_l * g.n_l) * es;
    STATUS_TRY(fused_pre(h->fo, st));
    STATUS_TRY(run_gemm(AXONN_OP_NN, act_dtype(h->d.dtype), g.m_l, g.n_l, g.k_l, I_local, g.k_l, W, g.n_l,
                        h->fo.out.ptr, g.n_l, st, &h->fo.epi));
    const bool act_fused = h->zbuf && h->fo.epi.mode == axonn::kExchange;
    STATUS_TRY(fused_post(h->fo, st, 0, act_fused ? h->zbuf : nullptr));
    count_comm(2, P, static_cast<size_t>(g.m_l * g.n_l), h->d.dtype);
    if (O_local != h->fo.out.ptr)
      CUDA_TRY(cudaMemcpyAsync(O_local, h->fo.out.ptr, bytes, cudaMemcpyDeviceToDevice, st));
    if (h->zbuf && !act_fused) STATUS_TRY(apply_act(h, O_local, st));
    h->I = I_local;
    h->W = W;
    h->have_fwd = true;
    return AXONN_OK;
  }
  // line 3 + line 4 over NCCL, pipelined over M-chunks when requested
  int chunks = (P > 1) ? h->d.chunks : 1;
  int64_t rows_per = (g.m_l + chunks - 1) / chunks;
  rows_per = (rows_per + 127) / 128 * 128;  // whole 128-row GEMM tiles per chunk
  if (rows_per <= 0) rows_per = 1;
  cudaStream_t cs = S.cstream[h->ax_fwd];
  int c = 0;
  for (int64_t r0 = 0; r0 < g.m_l || (g.m_l == 0 && c == 0); r0 += rows_per, ++c) {
    const int64_t rows = std::min<int64_t>(rows_per, g.m_l - r0);
    const char* Ic = static_cast<const char*>(I_local) + r0 * g.k_l * es;
    char* Oc = static_cast<char*>(O_local) + r0 * g.n_l * es;
    STATUS_TRY(run_gemm(AXONN_OP_NN, act_dtype(h->d.dtype), rows, g.n_l, g.k_l, Ic, g.k_l, W, g.n_l, Oc,
                        g.n_l, st));
    if (P > 1 && rows > 0) {
      cudaEvent_t ev = h->ev_chunk[std::min<size_t>(c, h->ev_chunk.size() - 1)];
      CUDA_TRY(cudaEventRecord(ev, st));
      CUDA_TRY(cudaStreamWaitEvent(cs, ev, 0));
      NCCL_TRY(ncclAllReduce(Oc, Oc, static_cast<size_t>(rows * g.n_l), nccl_type(h->d.dtype),
                             ncclSum, S.axis_comm[h->ax_fwd], cs));
      count_comm(2, P, static_cast<size_t>(rows * g.n_l), h->d.dtype);
    }
    if (g.m_l == 0) break;
  }
  if (P > 1) {
    CUDA_TRY(cudaEventRecord(h->ev_ar, cs));
    CUDA_TRY(cudaStreamWaitEvent(st, h->ev_ar, 0));
  }
  if (h->zbuf) STATUS_TRY(apply_act(h, O_local, st));
  // line 5: cache I_{k,j} and W_{j,i}
  h->I = I_local;
  h->W = W;
  h->have_fwd = true;
  return AXONN_OK;
}

axonn_status_t axonn_fc_backward(axonn_fc_t h, const void* dO_local, void* dI_local,
                                 void* dW_hat, void* stream) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!h) return fail(AXONN_ERR_ARG, "NULL handle");
  if (!S.grid) return fail(AXONN_ERR_STATE, "no grid");
  if (!h->have_fwd) return fail(AXONN_ERR_STATE, "axonn_fc_backward before axonn_fc_forward");
  const axonn_geometry_t& g = h->geo;
  if ((!dO_local && (g.m_l * g.n_l) != 0) || (!dI_local && (g.m_l * g.k_l) != 0) || (!dW_hat && g.what_len != 0))
    return fail(AXONN_ERR_ARG, "NULL tensor");
  STATUS_TRY(check_async_nccl());
  cudaStream_t st = as_stream(stream);
  const void* dO_caller = dO_local;  // another layer's output buffer, possibly
  if (h->zbuf && g.m_l != 0 && g.n_l != 0) {
    // dZ = dO ⊙ GELU'(Z) replaces dO in lines 11 and 13 (R18)
    CUDA_TRY(axonn::gelu_backward(dO_local, h->zbuf, h->dzbuf, g.m_l * g.n_l, S.num_sms, st));
    g_launches.fetch_add(1);
    dO_local = h->dzbuf;
  }
  const int dt = h->d.dtype;
  const ncclDataType_t nt = nccl_type(dt);
  const int gdt = grad_dtype(dt);             // dWpart / dŴ and their reductions
  const ncclDataType_t gnt = nccl_type(gdt);
  const int adt = act_dtype(dt);              // the dI product
  const int Pb = S.g[h->ax_bwd];
  cudaStream_t bs = S.cstream[h->ax_bwd];
  const bool rs = S.g[AX_Z] > 1;
  const bool fI = h->fi.epi.mode != axonn::kStore;  // dI all-reduce fused into the dI GEMM
  const bool fW = h->fw.epi.mode != axonn::kStore;  // data-parallel dŴ all-reduce fused into the dW GEMM
  const bool fZ = h->fz.epi.mode == axonn::kScatter;  // RS_z fused into the dW GEMM
  const bool fD = fZ && h->fd.epi.mode == axonn::kScatter;  // DP sum fused behind RS_z
  const size_t es = elem_size(dt);
  void* dst = fW ? h->fw.out.ptr : (rs && !fZ ? h->dwpart : dW_hat);
  const size_t S_el = static_cast<size_t>(g.what_len);
  cudaEvent_t last = nullptr;
  // line 11: dI^ = dO x W^T  (M = m_l, N = k_l, K = n_l)
  auto dI_gemm = [&]() -> axonn_status_t {
    return run_gemm(AXONN_OP_NT, adt, g.m_l, g.k_l, g.n_l, dO_local, g.n_l, h->W, g.n_l,
                    fI ? h->fi.out.ptr : dI_local, g.k_l, st, fI ? &h->fi.epi : nullptr);
  };
  // line 12's local sum inside line 13's GEMM (opt-in, AXONN_SIDESUM=1): a
  // 2-rank exchange of dÎ is summed by the dW GEMM's idle helper warps beside
  // its tiles (SideSum), so no barrier kernel and no pass over dI follow the
  // dW GEMM (measured: the GEMM slows by about what the pass cost)
  axonn::SideSum side;
  const bool side_on = fI && h->fi.epi.mode == axonn::kExchange && h->fi.epi.P == 2 &&
                       h->fi.side_arrive_peer && h->fi.par && env_int("AXONN_SIDESUM", 0) != 0 &&
                       g.k_l > 0 && g.n_l > 0 && g.m_l > 0 &&
                       !(fW && h->fw.epi.mode == axonn::kXSum);
  if (side_on) {
    char* c = static_cast<char*>(h->fi.ctrl.ptr);
    side.recv0 = h->fi.recv.ptr;
    side.recv1 = h->fi.recv2.ptr;
    side.out = h->fi.out.ptr;
    side.n16 = static_cast<long long>(h->fi.elems * h->fi.es / 16);
    side.par = h->fi.par;
    side.arrive_own = reinterpret_cast<int*>(c);
    side.arrive_peer = h->fi.side_arrive_peer;
    side.go = reinterpret_cast<int*>(c + 64);
    side.fin = reinterpret_cast<unsigned*>(c + 128);
  }
  // line 13: dW partial = I^T x dO  (M = k_l, N = n_l, K = m_l)
  auto dW_gemm = [&]() -> axonn_status_t {
    // the previous RS_z of this layer must be done with its source: the
    // fused one's slots on every rank (released by its final Z barrier), or
    // the NCCL one's read of dwpart (write-after-read race)
    if (rs) CUDA_TRY(wait_xcall(st, h->ev_rsdone));
    return run_gemm(AXONN_OP_TN, dt, g.k_l, g.n_l, g.m_l, h->I, g.k_l, dO_local, g.n_l, dst, g.n_l,
                    st, fW ? &h->fw.epi : (fZ ? &h->fz.epi : nullptr), side_on ? &side : nullptr);
  };
  // line 14 (ORS, waited in grads_sync) and the per-layer data-parallel sum
  auto grad_comm = [&]() -> axonn_status_t {
    cudaStream_t zs = S.cstream[AX_Z];
    if (rs) {
      CUDA_TRY(cudaEventRecord(h->ev_rs, st));
      CUDA_TRY(cudaStreamWaitEvent(zs, h->ev_rs, 0));
      // the previous data-parallel reduction of this layer is done with dŴ
      // (NCCL) or with the DATA receive slots (fused: its final DATA barrier
      // means every DATA owner finished reading them)
      CUDA_TRY(wait_xcall(zs, h->ev_wdone));
    }
    if (rs && fZ) {
      // fused RS_z, owner phase deferred on the Z stream (ORS): sum the Gz
      // slots in rank order into this rank's Ŵ gradient slice, or — fused
      // data-parallel sum — into the DATA owners' receive slots
      STATUS_TRY(fused_barrier(AX_Z, zs));  // every rank's scatter has landed
      axonn::OwnerOut o;
      if (fD) {
        o.mode = axonn::kOwnScatter;
        for (int q = 0; q < S.g[AX_D]; ++q) o.dst[q] = h->fd.epi.peer[q];
        o.me2 = h->fd.epi.me;
        o.slice2 = h->fd.epi.slice;
      } else {
        o.n_dst = 1;
        o.dst[0] = reinterpret_cast<unsigned long long>(dW_hat);
      }
      CUDA_TRY(axonn::sym_owner_reduce(h->fz.recv.ptr, h->fz.epi.slice, h->fz.epi.P,
                                       h->fz.es == 4, o, S.num_sms, zs));
      g_launches.fetch_add(1);
      STATUS_TRY(fused_barrier(AX_Z, zs));  // every owner is done with its slots
      CUDA_TRY(record_xcall(h->ev_rsdone, zs));
      count_comm(1, S.g[AX_Z], S_el, gdt);
      CUDA_TRY(cudaEventRecord(h->ev_grad, zs));
      last = h->ev_grad;
    } else if (rs) {
      NCCL_TRY(ncclReduceScatter(h->dwpart, dW_hat, S_el, gnt, ncclSum, S.axis_comm[AX_Z], zs));
      CUDA_TRY(record_xcall(h->ev_rsdone, zs));
      count_comm(1, S.g[AX_Z], S_el, gdt);
      CUDA_TRY(cudaEventRecord(h->ev_grad, zs));
      last = h->ev_grad;
    }
    if (S.g[AX_D] > 1) {
      cudaStream_t ds = S.cstream[AX_D];
      CUDA_TRY(cudaEventRecord(h->ev_rs, rs ? zs : st));
      CUDA_TRY(cudaStreamWaitEvent(ds, h->ev_rs, 0));
      if (fD) {
        // the DATA owner phase: barrier, sum the Gd slots, broadcast, barrier
        STATUS_TRY(fused_post(h->fd, ds, 1));
        if (dW_hat != h->fd.out.ptr)
          CUDA_TRY(cudaMemcpyAsync(dW_hat, h->fd.out.ptr, S_el * h->fd.es,
                                   cudaMemcpyDeviceToDevice, ds));
      } else {
        NCCL_TRY(ncclAllReduce(dW_hat, dW_hat, S_el, gnt, ncclSum, S.axis_comm[AX_D], ds));
      }
      count_comm(4, S.g[AX_D], S_el, gdt);
      CUDA_TRY(record_xcall(h->ev_wdone, ds));
      CUDA_TRY(cudaEventRecord(h->ev_grad, ds));
      last = h->ev_grad;
    }
    return AXONN_OK;
  };
  // fused outputs: buffers ready on every rank before any rank's epilogue writes
  if (fI) STATUS_TRY(fused_pre(h->fi, st));
  if (fW) {
    CUDA_TRY(wait_xcall(st, h->ev_wdone));  // previous deferred reduction done
    STATUS_TRY(fused_pre(h->fw, st));
  }
  if (Pb > 1 && !fI) {
    // line 11, then line 12 on the bwd-axis stream overlapped with line 13 (OAR)
    STATUS_TRY(dI_gemm());
    CUDA_TRY(cudaEventRecord(h->ev_dw, st));
    CUDA_TRY(cudaStreamWaitEvent(bs, h->ev_dw, 0));
    NCCL_TRY(ncclAllReduce(dI_local, dI_local, static_cast<size_t>(g.m_l * g.k_l), nt, ncclSum,
                           S.axis_comm[h->ax_bwd], bs));
    count_comm(3, Pb, static_cast<size_t>(g.m_l * g.k_l), dt);
    CUDA_TRY(cudaEventRecord(h->ev_ar, bs));
    STATUS_TRY(dW_gemm());
    if (!fW) STATUS_TRY(grad_comm());
  } else if (Pb > 1) {
    // line 12 fused into line 11; line 13 follows, its reduction overlaps nothing to wait on
    STATUS_TRY(dI_gemm());
    count_comm(3, Pb, static_cast<size_t>(g.m_l * g.k_l), dt);
    STATUS_TRY(dW_gemm());
    if (!fW) STATUS_TRY(grad_comm());
  } else {
    // no dI all-reduce to hide: compute dW first so its reduce-scatter /
    // data-parallel all-reduce overlaps the dI GEMM (same results)
    STATUS_TRY(dW_gemm());
    if (!fW) STATUS_TRY(grad_comm());
    STATUS_TRY(dI_gemm());
  }
  if (fW) count_comm(4, S.g[AX_D], S_el, gdt);
  // fused dI: every rank's reductions have landed after this (side_on: the
  // dW GEMM summed them)
  if (fI && !side_on) STATUS_TRY(fused_post(h->fi, st));
  if (fI && dI_local != h->fi.out.ptr)
    CUDA_TRY(cudaMemcpyAsync(dI_local, h->fi.out.ptr, static_cast<size_t>(g.m_l * g.k_l) * es,
                             cudaMemcpyDeviceToDevice, st));
  if (fW) {
    // the data-parallel reduction completes on the DATA stream, like the
    // paper's ORS: only axonn_grads_sync waits for it, so its barriers (which
    // absorb rank skew) and owner phase stay off this stream
    cudaStream_t ds = S.cstream[AX_D];
    CUDA_TRY(cudaEventRecord(h->ev_rs, st));
    CUDA_TRY(cudaStreamWaitEvent(ds, h->ev_rs, 0));
    STATUS_TRY(fused_post(h->fw, ds, 1));
    if (dW_hat != h->fw.out.ptr)
      CUDA_TRY(cudaMemcpyAsync(dW_hat, h->fw.out.ptr, S_el * h->fw.es, cudaMemcpyDeviceToDevice,
                               ds));
    CUDA_TRY(record_xcall(h->ev_wdone, ds));
    CUDA_TRY(cudaEventRecord(h->ev_grad, ds));
    last = h->ev_grad;
  }
  if (last) {
    bool seen = false;
    for (auto e : S.pending_grads) seen = seen || (e == last);
    if (!seen) S.pending_grads.push_back(last);
  }
  // dI must be complete in `stream` order when we return
  if (Pb > 1 && !fI) CUDA_TRY(cudaStreamWaitEvent(st, h->ev_ar, 0));
  // this backward was the last reader of its cached input and of dO: if
  // either is another layer's red.add output, zero it in the background
  STATUS_TRY(prezero_after(h->I, st));
  STATUS_TRY(prezero_after(dO_caller, st));
  h->have_fwd = false;
  return AXONN_OK;
}

axonn_status_t axonn_grads_sync(void* stream) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  cudaStream_t st = as_stream(stream);
  for (auto e : S.pending_grads) CUDA_TRY(cudaStreamWaitEvent(st, e, 0));
  S.pending_grads.clear();
  return AXONN_OK;
}

axonn_status_t axonn_fc_destroy(axonn_fc_t h) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!h) return AXONN_OK;
  if (!S.handles.count(h)) return fail(AXONN_ERR_ARG, "unknown handle");
  S.handles.erase(h);
  cudaDeviceSynchronize();
  for (cudaEvent_t e : {h->ev_in, h->ev_ag, h->ev_ar, h->ev_dw, h->ev_rs, h->ev_grad, h->ev_rsdone,
                        h->ev_wdone}) {
    if (!e) continue;
    for (size_t i = 0; i < S.pending_grads.size(); ++i)
      if (S.pending_grads[i] == e) S.pending_grads.erase(S.pending_grads.begin() + i--);
    cudaEventDestroy(e);
  }
  for (auto e : h->ev_chunk)
    if (e) cudaEventDestroy(e);
  if (h->wbuf) cudaFree(h->wbuf);
  if (h->dwpart) cudaFree(h->dwpart);
  if (h->zbuf) cudaFree(h->zbuf);
  if (h->dzbuf) cudaFree(h->dzbuf);
  for (axonn_fc::Fused* f : {&h->fo, &h->fi, &h->fw, &h->fz, &h->fd}) fused_reset(f);
  axonn::sym_free(&S.sym[AX_Z], &h->wstage);
  delete h;
  return AXONN_OK;
}

axonn_status_t axonn_gemm(int op, int dtype, int64_t M, int64_t N, int64_t K, const void* A,
                          int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                          void* stream) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (op < 0 || op > 2) return fail(AXONN_ERR_ARG, "op must be 0 (NN), 1 (NT) or 2 (TN)");
  if (!valid_dtype(dtype)) return fail(AXONN_ERR_ARG, "bad dtype");
  if (M < 0 || N < 0 || K < 0) return fail(AXONN_ERR_ARG, "negative dimension");
  if (M && N && (!C || (K && (!A || !B)))) return fail(AXONN_ERR_ARG, "NULL matrix");
  const int64_t a_cols = (op == AXONN_OP_TN) ? M : K;
  const int64_t b_cols = (op == AXONN_OP_NT) ? K : N;
  if ((K && M && lda < a_cols) || (K && N && ldb < b_cols) || (M && ldc < N))
    return fail(AXONN_ERR_ARG, "leading dimension smaller than the row length");
  return run_gemm(op, dtype, M, N, K, A, lda, B, ldb, C, ldc, as_stream(stream));
}

axonn_status_t axonn_loopback_step(const axonn_fc_desc_t* desc, int gx, int gy, int gz, int gd,
                                   const void* const* I_local, const void* const* W_hat,
                                   const void* const* dO_local, void* const* O_local,
                                   void* const* dI_local, void* const* dW_hat, int flags,
                                   void* stream, int* paths) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  STATUS_TRY(check_grid_args(gx, gy, gz, gd));
  if (!desc || !I_local || !W_hat || !dO_local || !O_local || !dI_local || !dW_hat)
    return fail(AXONN_ERR_ARG, "NULL argument");
  if (gx * gy * gz * gd > 64) return fail(AXONN_ERR_ARG, "loopback: at most 64 ranks");
  if (gx > 8 || gy > 8 || gz > 8 || gd > 8)
    return fail(AXONN_ERR_UNSUPPORTED, "loopback: fused collectives span at most 8 ranks per axis");
  if (!valid_dtype(desc->dtype)) return fail(AXONN_ERR_ARG, "bad dtype");
  STATUS_TRY(ensure_device());
  const int g[4] = {gx, gy, gz, gd};
  return axonn::loopback_step(desc, g, I_local, W_hat, dO_local, O_local, dI_local, dW_hat, flags,
                              as_stream(stream), paths);
}

axonn_status_t axonn_profile_enable(int enabled) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  S.profiling = enabled != 0;
  return AXONN_OK;
}

axonn_status_t axonn_profile_read(int64_t* launches, double* ms, double* flops) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!launches || !ms || !flops) return fail(AXONN_ERR_ARG, "NULL argument");
  *launches = 0;
  *ms = 0.0;
  *flops = 0.0;
  for (auto& p : S.prof) {
    CUDA_TRY(cudaEventSynchronize(p.stop));
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, p.start, p.stop));
    *ms += t;
    *flops += p.flops;
    *launches += 1;
    S.prof_free.push_back(p.start);
    S.prof_free.push_back(p.stop);
  }
  S.prof.clear();
  return AXONN_OK;
}

int64_t axonn_kernel_launches(void) { return g_launches.load(); }

axonn_status_t axonn_stream_k_items(int sk_tiles, int num_kb, int pair, int pairs, int* tile,
                                    int* role, int* kb0, int* kb1, int cap, int* n) {
  if (sk_tiles < 0 || num_kb < 1 || pairs < 1 || pair < 0 || pair >= pairs || cap < 0 || !n ||
      (cap > 0 && (!tile || !role || !kb0 || !kb1)))
    return fail(AXONN_ERR_ARG, "bad argument");
  // the kernel's decomposition needs every pair's range to span a tile
  if (static_cast<long long>(sk_tiles) < pairs)
    return fail(AXONN_ERR_ARG, "stream-K needs sk_tiles >= pairs");
  *n = axonn::gemm_stream_k_items(sk_tiles, num_kb, pair, pairs, tile, role, kb0, kb1, cap);
  return AXONN_OK;
}

int64_t axonn_stream_k_launches(void) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  return axonn::gemm_stream_k_launches();
}

axonn_status_t axonn_comm_bytes(int64_t out[5], int reset) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!out) return fail(AXONN_ERR_ARG, "NULL argument");
  for (int i = 0; i < 5; ++i) {
    out[i] = S.comm_bytes[i];
    if (reset) S.comm_bytes[i] = 0;
  }
  return AXONN_OK;
}

axonn_status_t axonn_set_gemm_sms(int sms) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  STATUS_TRY(ensure_device());
  S.gemm_sms = (sms <= 0 || sms > S.num_sms) ? S.num_sms : sms;
  return AXONN_OK;
}

axonn_status_t axonn_grid_select(const axonn_layer_t* layers, int n_layers, int G, int g_node,
                                 const axonn_bw_entry_t* table, int n_table, double beta_inter,
                                 int bytes_per_elem, int fixed_gd, axonn_grid_score_t* out,
                                 int cap, int* n_out) {
  return axonn_grid_select_mp(layers, n_layers, G, g_node, table, n_table, beta_inter,
                              bytes_per_elem, bytes_per_elem, fixed_gd, out, cap, n_out);
}

axonn_status_t axonn_grid_select_mp(const axonn_layer_t* layers, int n_layers, int G, int g_node,
                                    const axonn_bw_entry_t* table, int n_table, double beta_inter,
                                    int bytes_per_elem, int grad_bytes_per_elem, int fixed_gd,
                                    axonn_grid_score_t* out, int cap, int* n_out) {
  if ((!layers && n_layers) || n_layers < 0 || G < 1 || g_node < 1 || (!table && n_table) ||
      n_table < 0 || !(beta_inter > 0) || bytes_per_elem < 1 || grad_bytes_per_elem < 1 ||
      cap < 0 || (!out && cap) || !n_out)
    return fail(AXONN_ERR_ARG, "bad argument to axonn_grid_select");
  std::vector<axonn::Layer> ls;
  for (int i = 0; i < n_layers; ++i) {
    if (layers[i].m < 0 || layers[i].k < 0 || layers[i].n < 0)
      return fail(AXONN_ERR_ARG, "negative layer dimension");
    ls.push_back({layers[i].m, layers[i].k, layers[i].n, layers[i].transposed != 0});
  }
  std::vector<axonn::BwEntry> tb;
  for (int i = 0; i < n_table; ++i) {
    if (!(table[i].bytes_per_s > 0)) return fail(AXONN_ERR_ARG, "bandwidth must be > 0");
    tb.push_back({table[i].inner, table[i].size, table[i].bytes_per_s});
  }
  std::vector<axonn::Scored> ranked;
  std::string err;
  const int n = axonn::rank_configs(ls, G, g_node, tb, beta_inter, bytes_per_elem,
                                    grad_bytes_per_elem, fixed_gd, &ranked, &err);
  if (n < 0) return fail(AXONN_ERR_CONFIG, "configuration error: %s", err.c_str());
  *n_out = n;
  if (n == 0) return fail(AXONN_ERR_INFEASIBLE, "infeasible: no configuration of %d GPUs divides every layer", G);
  for (int i = 0; i < n && i < cap; ++i) {
    const auto& s = ranked[i];
    out[i] = {s.c.gx, s.c.gy, s.c.gz, s.c.gd, s.t.ag_z, s.t.rs_z,
              s.t.ar_y, s.t.ar_x, s.t.ar_d, s.t.comm};
  }
  return AXONN_OK;
}

}  // extern "C"
