/*
 * axonn.h — C ABI of libaxonn.so, the B200 (sm_100a) implementation of the
 * data-parallel hot path of AxoNN's 4D hybrid parallelism (arXiv 2502.08145):
 * the 3D parallel matrix multiply (3D PMM) of one transformer FC layer on a
 * Gx x Gy x Gz grid nested in Gd-way data parallelism.
 *
 * Citations "PAPER.md:N" are lines of the paper's LaTeX source; "Alg. 1" is
 * Algorithm 1.  DESIGN.md lists every reading (R1..R17)
 * taken where the paper is silent or ambiguous.
 *
 * Conventions for every call
 *   - Return value: AXONN_OK or an error status.  A thread-local message is
 *     available from axonn_last_error() until the next failing call.
 *   - Device pointers are caller-owned CUDA memory on the calling rank's
 *     device (cudaMalloc/torch allocations).  Host pointers are marked "host".
 *   - Device-side calls are stream-ordered on the `stream` argument (a
 *     cudaStream_t passed as void*; NULL = legacy default stream): they
 *     enqueue work and return without synchronising.  Asynchronous CUDA /
 *     NCCL failures surface as AXONN_ERR_CUDA / AXONN_ERR_NCCL on a later call.
 *   - Collective calls (forward, backward, prefetch, grads_sync) must be issued
 *     in the same order on every rank, on one stream per rank (or on streams
 *     the caller orders): their cross-rank barriers are per-axis sequences
 *     that must not run concurrently.  The library's own side streams (one
 *     per axis) are ordered internally.  CUDA-graph capture of such a
 *     sequence is supported (external event nodes order it across replays).
 *   - All matrices are row-major with an explicit leading dimension in
 *     elements; bf16 buffers hold IEEE bfloat16, f32 buffers IEEE binary32.
 *   - No call ever falls back to a CPU path: if the CUDA device or the
 *     sm_100a kernels are unavailable the call fails with AXONN_ERR_CUDA.
 */
#ifndef AXONN_H
#define AXONN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  AXONN_OK = 0,
  AXONN_ERR_ARG = 1,          /* NULL pointer, negative size, bad enum           */
  AXONN_ERR_CONFIG = 2,       /* grid factor product != world size, zero factor  */
  AXONN_ERR_SHAPE = 3,        /* divisibility failure; message names the axis    */
  AXONN_ERR_STATE = 4,        /* e.g. backward before forward, no grid           */
  AXONN_ERR_INFEASIBLE = 5,   /* grid_select found no configuration              */
  AXONN_ERR_CUDA = 6,         /* CUDA runtime/driver failure or no sm_100 device */
  AXONN_ERR_NCCL = 7,         /* NCCL failure (sync or async)                    */
  AXONN_ERR_UNSUPPORTED = 8   /* valid request this build does not implement    */
} axonn_status_t;

typedef enum {
  AXONN_BF16 = 0,             /* bf16 storage, fp32 accumulate on tcgen05 */
  AXONN_F32 = 1,              /* fp32 storage and SIMT fp32 arithmetic: test mode            */
  AXONN_BF16_GRADF32 = 2      /* bf16 operands, activations and W; the weight gradient dŴ is
                                 fp32 (the dW product's accumulator is stored unrounded) and
                                 RS_z / the data-parallel all-reduce sum fp32 (b = 4 in
                                 Eqs. 2, 5, reading R17), fused over
                                 NVLS like bf16 (scatter + fp32 owner phase) or NCCL fp32  */
} axonn_dtype_t;

/* Message of the last failing call on this thread ("" if none). Never NULL. */
const char* axonn_last_error(void);
/* ABI version, major*100 + minor. */
int axonn_version(void);

/* ======================================================================== */
/* Process bootstrap (one process per GPU).                                  */
/* ======================================================================== */

/* Fill `id` (host, 128 bytes) with a fresh NCCL unique id.  Call on world
 * rank 0 only; the caller broadcasts the bytes to every rank out of band
 * (torch.distributed).  Errors: AXONN_ERR_NCCL. */
axonn_status_t axonn_unique_id(unsigned char id[128]);

/* Bind this process to `cuda_device` and create the world communicator
 * (world_size ranks).  world_size == 1 creates no communicator and needs no
 * id (id may be NULL).  Errors: ARG, CUDA, NCCL; STATE if already bootstrapped. */
axonn_status_t axonn_bootstrap(int world_rank, int world_size, const unsigned char* id,
                               int cuda_device);

/* ======================================================================== */
/* The 4D virtual grid.                 */
/*   rank r <-> (i, j, k, d),  r = i + Gx*(j + Gy*(k + Gz*d))               */
/*   X innermost, then Y, then Z, data-parallel outermost */
/* ======================================================================== */

/* Create the four axis sub-communicators X, Y, Z, DATA (members ordered by
 * the axis coordinate) and this rank's streams.  Requires bootstrap.
 * Errors: CONFIG (gx*gy*gz*gd != world size, or a factor < 1), STATE, NCCL. */
axonn_status_t axonn_grid_init(int gx, int gy, int gz, int gd);
/* This rank's coordinates (host out-pointers). Errors: STATE (no grid). */
axonn_status_t axonn_grid_coords(int* i, int* j, int* k, int* d);
/* Destroy communicators, streams and every outstanding layer handle's
 * communication state.  Safe to call twice. */
axonn_status_t axonn_grid_finalize(void);

/* Pure host helpers (no device, no communicator): the rank <-> coordinate
 * bijection and the members of rank's group along `axis` (0=X,1=Y,2=Z,3=DATA),
 * written to `members` (host, capacity >= extent of that axis) in coordinate
 * order.  Errors: CONFIG, ARG. */
axonn_status_t axonn_rank_to_coords(int rank, int gx, int gy, int gz, int gd, int coords[4]);
axonn_status_t axonn_group_members(int rank, int gx, int gy, int gz, int gd, int axis,
                                   int* members);

/* ======================================================================== */
/* One FC layer, Algorithm 1.                             */
/* ======================================================================== */

typedef struct {
  int64_t m;          /* global tokens: rows of X over ALL data-parallel replicas */
  int64_t k;          /* input features (rows of W)                               */
  int64_t n;          /* output features (cols of W)                              */
  int transposed;     /* 1: X/Y roles swapped (reading R2)       */
  int dtype;          /* axonn_dtype_t                                            */
  int chunks;         /* forward AR pipelining: M-chunks of the local GEMM whose
                         all-reduce starts as each finishes (0/1 = unchunked).    */
  int act;            /* axonn_act_t applied to the layer's output (fc1 of a GPT
                         block: AXONN_ACT_GELU).  0 = none.                       */
} axonn_fc_desc_t;

/* Activation on a layer's output (reading R18):
 *   forward  Z = all-reduce(Ô) (Alg. 1 line 4), O_local = GELU(Z),
 *   backward dZ = dO_local ⊙ GELU'(Z) takes dO's place in lines 11 and 13,
 * with GELU(x) = x Φ(x) exactly (erf).  Z is rounded to bf16 where Alg. 1
 * rounds O (R8); the handle keeps Z for the backward.  bf16 layers only. */
typedef enum { AXONN_ACT_NONE = 0, AXONN_ACT_GELU = 1 } axonn_act_t;

/* Shard geometry of one rank (readings R1, R2, R4, R6):
 *   I_local  = X[row0 : row0+m_l, in_col0 : in_col0+k_l]         ([m_l][k_l])
 *   W_local  = W[in_col0 : +k_l, out_col0 : +n_l]                ([k_l][n_l])
 *   W_hat    = flat(W_local)[what_off : what_off+what_len]       (S elements)
 *   O_local  = O[row0 : +m_l, out_col0 : +n_l]                   ([m_l][n_l])
 * with m_l = m/(Gz*Gd), row0 = (d*Gz + k)*m_l; normal layer: k_l = k/Gy,
 * n_l = n/Gx, in_col0 = j*k_l, out_col0 = i*n_l; transposed layer: k_l = k/Gx,
 * n_l = n/Gy, in_col0 = i*k_l, out_col0 = j*n_l; S = k_l*n_l/Gz,
 * what_off = k*S. */
typedef struct {
  int64_t m_l, k_l, n_l, row0, in_col0, out_col0, what_off, what_len;
} axonn_geometry_t;

/* Pure host: geometry of `rank` on grid (gx,gy,gz,gd).  Errors: CONFIG, ARG,
 * SHAPE ("k=... not divisible by Gy=..."; no padding). */
axonn_status_t axonn_shard_geometry(const axonn_fc_desc_t* desc, int gx, int gy, int gz, int gd,
                                    int rank, axonn_geometry_t* out);

typedef struct axonn_fc* axonn_fc_t;

/* Create a layer handle on the current grid; validates divisibility and
 * allocates the handle-owned buffers (gathered W_{j,i} when Gz>1, the dW
 * partial when Gz>1, the symmetric buffers of the fused collectives).  bf16
 * layers also need k_l and n_l to be multiples of 8 (TMA rows are 16-byte
 * aligned); m_l is unrestricted.  Errors: ARG, STATE (no grid), SHAPE, CUDA,
 * NCCL. */
axonn_status_t axonn_fc_create(const axonn_fc_desc_t* desc, axonn_fc_t* out);
/* Geometry of this rank for handle `h` (host out). */
axonn_status_t axonn_fc_geometry(axonn_fc_t h, axonn_geometry_t* out);

/* Handle-owned output buffers of the fused GEMM + all-reduce path (B200
 * NVLS): which = 0 -> O_local, 1 -> dI_local, 2 -> dW_hat.  *ptr is NULL when
 * that output takes the NCCL path (fp32 mode, a row length
 * not a multiple of 8, or AXONN_FUSED=0).  Passing the returned pointer as the
 * output argument of axonn_fc_forward / axonn_fc_backward avoids the final
 * device-to-device copy; its contents are valid until the next call that
 * writes that output.  The buffer is read-only for the caller: when it is
 * passed on as another layer's I_local (dO_local), the library may zero it
 * in the background once that layer's backward, its last reader, has been
 * enqueued (the 2-rank red.add reduction's next use needs it zeroed).  A
 * buffer that feeds more than one layer needs AXONN_PREZERO=0.
 * Errors: ARG. */
axonn_status_t axonn_fc_output_buffer(axonn_fc_t h, int which, void** ptr);
/* The epilogue mode the multi-GPU path picks for a reduction of a rows x cols
 * output of a GEMM with contraction length kdim over P ranks with
 * elem_bytes-byte elements (2 bf16, 4 fp32), under the current AXONN_*
 * switches: "none" (not fused: P = 1, an empty output, rows not a whole number
 * of 16-B units; NCCL when P > 1), "red_add_pair", "multimem_red",
 * "exchange", "scatter", "xsum" or "pair_sum" (host buf).  Host only; no
 * grid needed.  Errors: ARG. */
axonn_status_t axonn_fused_mode(int P, int elem_bytes, int64_t rows, int64_t cols, int64_t kdim,
                                char* buf, int cap);
/* "fused" if collectives along `axis` (0=X,1=Y,2=Z,3=DATA) of the current grid
 * are fused into the GEMM epilogue over NVLS, else the reason (host buf). */
axonn_status_t axonn_fused_status(int axis, char* buf, int cap);

/* Diagnostics: bytes/s one rank moves over NVLink with one primitive on the
 * symmetric memory of `axis` (mode 0: multimem.red.add bf16, 1: multimem.st,
 * 2: plain 16-B stores to the next rank's copy, 3: multimem.ld_reduce,
 * 4: local stores, 5: red.add bf16 into the next rank's copy, 6: local
 * red.add bf16), `ctas` x 512 threads.  Collective over the axis. */
axonn_status_t axonn_nvlink_probe(int axis, int64_t bytes, int mode, int ctas, int iters,
                                  double* gbps);

/* OAG: start the Z all-gather of W_hat for the NEXT
 * forward of h now, on the communication stream (copy engines, no SMs), after
 * the work already enqueued on `stream`.  To overlap it with layer i's GEMM,
 * call prefetch(layer i+1) BEFORE forward(layer i).  Optional: a forward
 * that was not prefetched gathers inline on `stream` with every SM pulling
 * from the peers' staging copies (it would wait for the gather anyway). */
axonn_status_t axonn_fc_prefetch(axonn_fc_t h, const void* W_hat, void* stream);

/* Forward, Alg. 1 lines 1-7:
 *   W_{j,i} = all-gather_z(W_hat)            (line 2; skipped when Gz == 1)
 *   Ô       = I_local x W_{j,i}               (line 3; tcgen05 GEMM, fp32 acc)
 *   O_local = all-reduce_y(Ô)                 (line 4; over X if transposed)
 * I_local [m_l][k_l] (ld = k_l), W_hat [what_len], O_local [m_l][n_l]
 * (ld = n_l), all of desc.dtype.  O_local holds Ô rounded to the dtype
 * before the all-reduce (R8).  Line 5 caches I_local (caller keeps it alive
 * and unmodified until backward is enqueued) and W_{j,i} (handle-owned; when
 * Gz == 1 W_{j,i} IS W_hat, which must then also stay alive).
 * Errors: ARG, STATE (no grid), CUDA, NCCL. */
axonn_status_t axonn_fc_forward(axonn_fc_t h, const void* I_local, const void* W_hat,
                                void* O_local, void* stream);

/* Backward, Alg. 1 lines 9-15:
 *   dÎ      = dO_local x W_{j,i}^T           (line 11)
 *   dI      = all-reduce_x(dÎ)                (line 12; over Y if transposed),
 *             overlapped with line 13 (OAR)
 *   dWpart  = I_local^T x dO_local            (line 13)
 *   dW_hat  = reduce-scatter_z(dWpart)        (line 14), NOT waited here (ORS,
 *             PAPER.md:660-669): it completes at axonn_grads_sync
 *   if Gd > 1: dW_hat += all-reduce over DATA (sum, R9),
 *             issued right after this layer's reduce-scatter.
 * dO_local [m_l][n_l], dI_local [m_l][k_l], dW_hat [what_len] (fp32 when
 * desc.dtype is AXONN_BF16_GRADF32, else desc.dtype).  dI_local is
 * ready in `stream` order when this call returns; dW_hat only after
 * axonn_grads_sync(stream).  Errors: STATE (no forward since the last
 * backward), ARG, CUDA, NCCL. */
axonn_status_t axonn_fc_backward(axonn_fc_t h, const void* dO_local, void* dI_local,
                                 void* dW_hat, void* stream);

/* The single ORS / data-parallel wait point: makes `stream` wait for every
 * reduce-scatter and data-parallel all-reduce issued since the last call. */
axonn_status_t axonn_grads_sync(void* stream);

axonn_status_t axonn_fc_destroy(axonn_fc_t h);

/* ======================================================================== */
/* The three local products on the tensor cores (Alg. 1 lines 3, 11, 13),    */
/* exposed for kernel parity tests and the GEMM-only timing of bench.py.     */
/*   AXONN_OP_NN: C[M][N] = A[M][K]   x B[K][N]    (line 3:  I x W)           */
/*   AXONN_OP_NT: C[M][N] = A[M][K]   x B[N][K]^T  (line 11: dO x W^T)        */
/*   AXONN_OP_TN: C[M][N] = A[K][M]^T x B[K][N]    (line 13: I^T x dO)        */
/* Row-major, leading dimensions lda/ldb/ldc in elements (multiples of 8 for */
/* bf16, 16-byte aligned base pointers).  bf16: tcgen05.mma kind::f16 with   */
/* fp32 accumulation in TMEM, one RNE rounding to bf16 at the end.  f32: SIMT*/
/* fp32 FMA (test mode).  AXONN_BF16_GRADF32 (op TN only, else ARG): bf16   */
/* A and B on tcgen05, C fp32 = the unrounded TMEM accumulator (ldc % 4 == 0 */
/* for the TMA-store epilogue, any ldc otherwise).                           */
/* M, N, K >= 0 (K == 0 writes zeros).                                       */
/* ======================================================================== */
typedef enum { AXONN_OP_NN = 0, AXONN_OP_NT = 1, AXONN_OP_TN = 2 } axonn_op_t;

axonn_status_t axonn_gemm(int op, int dtype, int64_t M, int64_t N, int64_t K,
                          const void* A, int64_t lda, const void* B, int64_t ldb,
                          void* C, int64_t ldc, void* stream);

/* ======================================================================== */
/* Test support: the fused collectives of the multi-GPU path on ONE GPU.     */
/* ======================================================================== */
/* Runs Alg. 1 (forward, backward, RS_z and the data-parallel sum;           */
/* PAPER.md:375-390, 313-317) for EVERY rank of the grid (gx,gy,gz,gd) on    */
/* the current device, with the same device code that moves data between    */
/* ranks on NVLink: GEMM epilogues that multimem.red into a multicast buffer */
/* or scatter 16-B units into the owners' receive slots, the owner phase     */
/* that sums the slots in rank order and broadcasts (multimem.st, or plain   */
/* stores to the peer on 2-rank axes) or re-scatters to the DATA owners, and */
/* the Z all-gather by copy engines or SM pull.  Every rank's "symmetric"    */
/* buffers are allocated side by side on this device; stream order replaces  */
/* the cross-rank barriers; multicast uses a one-device multicast object     */
/* (its single copy is then copied to each member, as NVSwitch replicates).  */
/* Arrays hold one pointer per rank r = 0..G-1 (host arrays of device        */
/* pointers, laid out as for axonn_fc_forward/backward with rank r's shard   */
/* geometry: axonn_shard_geometry).  Device-synchronous: returns after the   */
/* step has finished.  `paths` (host, may be NULL) receives the                */
/* AXONN_LB_PATH_* bits of the fused paths that ran.  Only bf16 and          */
/* AXONN_BF16_GRADF32 (the fp32 test mode reduces through NCCL).            */
/* Errors: ARG, CONFIG, SHAPE, CUDA; UNSUPPORTED when a needed collective    */
/* would not be fused for this shape on the multi-GPU path (it would use     */
/* NCCL, which has no loopback) or an axis exceeds 8 ranks.                 */
/* ======================================================================== */
enum {
  AXONN_LB_RED_ALWAYS = 1,   /* 2-rank bf16 axes: multimem.red at any K          */
  AXONN_LB_RED_NEVER = 2,    /* never multimem.red: scatter + owner phase        */
  AXONN_LB_GATHER_PULL = 4,  /* AG_z by the SM pull kernel (else copy engines)   */
  AXONN_LB_EMULATE_MC = 8,   /* no multicast object: red.global.add / plain st   */
  AXONN_LB_NO_EXCHANGE = 16, /* 2-rank axes below the red threshold: scatter +
                                owner phase instead of the exchange of partials */
  AXONN_LB_PAIRSUM = 32,     /* 2-rank bf16 axes: the sum finished in the epilogue */
  AXONN_LB_REVERSE = 64,     /* run each phase's ranks in reverse order (the
                                pair-sum's second arriver is then rank 0)     */
  AXONN_LB_PAIRPULL = 128,   /* with AXONN_LB_PAIRSUM: each rank keeps its partial
                                in its own receive buffer and the second
                                arriver reads the peer's over NVLink (pull)   */
  AXONN_LB_XSUM = 256,       /* 2-rank bf16 axes at every K: the exchange summed
                                inside the GEMM (kXSum, AXONN_XSUM=1 on the
                                multi-GPU path; opt-in, measured slower)      */
  AXONN_LB_NO_REDPAIR = 1024, /* 2-rank bf16 axes below the multimem.red threshold:
                                 not unicast red.add into both ranks' outputs
                                 (kRedPair, the default there) but the exchange
                                 + local sum (AXONN_REDPAIR=0)                 */
  AXONN_LB_SIDESUM = 512     /* the backward's 2-rank exchange of dÎ summed by the
                                dW GEMM's helper warps instead of a separate
                                pass (AXONN_SIDESUM=1 on the multi-GPU path;
                                opt-in, measured no faster)                   */
};
enum {
  AXONN_LB_PATH_FWD_RED = 1, AXONN_LB_PATH_FWD_SCATTER = 2,
  AXONN_LB_PATH_BWD_RED = 4, AXONN_LB_PATH_BWD_SCATTER = 8,
  AXONN_LB_PATH_RS_Z = 16,
  AXONN_LB_PATH_DP_RED = 32, AXONN_LB_PATH_DP_SCATTER = 64,
  AXONN_LB_PATH_DP_AFTER_RS = 128,
  AXONN_LB_PATH_GATHER_COPY = 256, AXONN_LB_PATH_GATHER_PULL = 512,
  AXONN_LB_PATH_MULTICAST = 1024,  /* a real one-device multicast object was used */
  AXONN_LB_PATH_FWD_EXCHANGE = 2048, AXONN_LB_PATH_BWD_EXCHANGE = 4096,
  AXONN_LB_PATH_DP_EXCHANGE = 8192,
  AXONN_LB_PATH_FWD_PAIRSUM = 16384, AXONN_LB_PATH_BWD_PAIRSUM = 32768,
  AXONN_LB_PATH_DP_PAIRSUM = 65536,
  AXONN_LB_PATH_FWD_XSUM = 131072, AXONN_LB_PATH_BWD_XSUM = 262144,
  AXONN_LB_PATH_DP_XSUM = 524288,
  AXONN_LB_PATH_BWD_SIDESUM = 1048576,  /* dÎ's exchange summed inside the dW GEMM */
  AXONN_LB_PATH_FWD_REDPAIR = 2097152, AXONN_LB_PATH_BWD_REDPAIR = 4194304,
  AXONN_LB_PATH_DP_REDPAIR = 8388608
};
axonn_status_t axonn_loopback_step(const axonn_fc_desc_t* desc, int gx, int gy, int gz, int gd,
                                   const void* const* I_local, const void* const* W_hat,
                                   const void* const* dO_local, void* const* O_local,
                                   void* const* dI_local, void* const* dW_hat, int flags,
                                   void* stream, int* paths);

/* ======================================================================== */
/* Instrumentation: CUDA events around every GEMM launch on its launching    */
/* stream, and a count of every kernel this library launched.                */
/* ======================================================================== */
axonn_status_t axonn_profile_enable(int enabled);
/* Synchronises the recorded events; returns the number of GEMM launches, the
 * summed GEMM device time (ms) and summed algorithmic flops (2*M*N*K) since
 * the last reset, then resets. */
axonn_status_t axonn_profile_read(int64_t* gemm_launches, double* gemm_ms, double* gemm_flops);
/* Kernels launched by this library since load (GEMMs + helper kernels; NCCL
 * kernels excluded). */
int64_t axonn_kernel_launches(void);
/* GEMM launches since load that split their last, partial wave of tiles along
 * K (the stream-K tail of gemm_tc.cu: tiles that would leave CTA pairs idle
 * are shared by all pairs; a tile's two pieces are summed in fp32 in a fixed
 * order, so results are deterministic).  AXONN_SK=0 turns the split off. */
int64_t axonn_stream_k_launches(void);
/* Host-only view of that decomposition: the items CTA pair `pair` of `pairs`
 * processes, in order, when the first `sk_tiles` tiles (of `num_kb` 64-wide
 * K-blocks each) are split: tile index, role (0 whole tile, 1 HEAD = K-blocks
 * [0, h) whose fp32 partial goes to the finisher, 2 TAIL = [t0, num_kb) which
 * adds the HEAD's partial; at run time a TAIL whose HEAD pair has not started
 * takes the whole tile instead) and the K-block range [kb0, kb1).  Host
 * arrays of `cap`; *n = the count (may exceed cap).  Errors: ARG. */
axonn_status_t axonn_stream_k_items(int sk_tiles, int num_kb, int pair, int pairs, int* tile,
                                    int* role, int* kb0, int* kb1, int cap, int* n);
/* SM budget of the persistent GEMM grid (<= 0 or > #SMs: all SMs).  Leaving
 * SMs free lets NCCL kernels run beside the GEMM when collectives overlap. */
axonn_status_t axonn_set_gemm_sms(int sms);
/* Bytes this rank sends in ring collectives issued since the last reset,
 * computed from the element counts passed to NCCL with the ring formulas of
 * Eqs. 1-5 (all-gather (p-1)*count*b, reduce-scatter (p-1)*recvcount*b,
 * all-reduce 2(p-1)/p*count*b): out = {AG_z, RS_z, forward AR (Eq. 3 form),
 * backward dI AR (Eq. 4 form), data-parallel AR (Eq. 5)} (host). */
axonn_status_t axonn_comm_bytes(int64_t out[5], int reset);

/* ======================================================================== */
/* Performance model: Eqs. 1-6 per layer, summed over     */
/* layers, with per-level bandwidths from the Case-1 table*/
/* or Eq. 7, ranked ascending.         */
/* ======================================================================== */
typedef struct {
  int64_t m, k, n;    /* m = global tokens (all replicas) */
  int transposed;
} axonn_layer_t;

/* Case-1 database entry: groups of size G1 whose preceding hierarchy product
 * is G0 achieve `bytes_per_s`. */
typedef struct {
  int inner;          /* G0 = prod_{j<i} G_j */
  int size;           /* G1 = G_i            */
  double bytes_per_s;
} axonn_bw_entry_t;

/* One ranked configuration.  t_ar_y / t_ar_x are the Eq. 3 / Eq. 4 terms
 * (forward / backward-dI all-reduce) summed over layers after the transposed
 * layers' X<->Y swap. */
typedef struct {
  int gx, gy, gz, gd;
  double t_ag_z, t_rs_z, t_ar_y, t_ar_x, t_ar_data, t_comm;   /* seconds */
} axonn_grid_score_t;

/* Enumerate every (gx,gy,gz,gd) with product G (gd fixed when fixed_gd > 0),
 * drop those that do not divide every layer, score by Eq. 6 summed over
 * layers with b = bytes_per_elem, sort ascending on t_comm rounded to 12
 * significant digits, ties
 * broken lexicographically on (gx,gy,gz,gd) (reading R12), and write the
 * first min(cap, count) to `out` (host).  *n_out = total feasible count.
 * Errors: ARG, CONFIG (a needed Case-1 table entry is missing; the message
 * names (G0,G1)), INFEASIBLE (no configuration). */
axonn_status_t axonn_grid_select(const axonn_layer_t* layers, int n_layers, int G, int g_node,
                                 const axonn_bw_entry_t* table, int n_table, double beta_inter,
                                 int bytes_per_elem, int fixed_gd, axonn_grid_score_t* out,
                                 int cap, int* n_out);

/* Mixed precision (reading R17): as axonn_grid_select,
 * with b = bytes_per_elem in Eqs. 1, 3, 4 (weights and activations) and
 * b = grad_bytes_per_elem in Eqs. 2 and 5 (the gradient reductions; 4 for
 * layers created with AXONN_BF16_GRADF32).  axonn_grid_select(b) ==
 * axonn_grid_select_mp(b, b). */
axonn_status_t axonn_grid_select_mp(const axonn_layer_t* layers, int n_layers, int G, int g_node,
                                    const axonn_bw_entry_t* table, int n_table, double beta_inter,
                                    int bytes_per_elem, int grad_bytes_per_elem, int fixed_gd,
                                    axonn_grid_score_t* out, int cap, int* n_out);

#ifdef __cplusplus
}
#endif
#endif /* AXONN_H */
