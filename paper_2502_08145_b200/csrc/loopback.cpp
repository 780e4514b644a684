// loopback.cpp — axonn_loopback_step: every rank of a 4D grid on ONE GPU.
//
// Test support (include/axonn.h).  The multi-GPU path moves data between
// ranks with device code: GEMM epilogues that multimem.red into an NVLS
// multicast buffer or scatter 16-B units into the owner ranks' receive slots
// (gemm_tc.cu), owner phases that sum the slots and broadcast or re-scatter
// (sym.cu k_owner_reduce), and the Z all-gather by copy engines or an SM pull
// (sym.cu).  This file runs that same device code for all G ranks of a grid
// on one device, with each rank's "symmetric" buffers allocated side by side
// and its peers' addresses pointing at them, so that a single-GPU box can
// check AG_z, AR_y, AR_x, RS_z, the data-parallel sum and the transposed
// layer's axis swap against the oracle's per-rank results (SURVEY.md §8(a)
// a2, a4, a7, a9, a10, a11; Alg. 1 lines 2, 4, 12, 14, PAPER.md:375-390;
// PAPER.md:313-317).
//
// What differs from the multi-GPU path is only the orchestration:
//   * ranks run one after another on one stream, phase by phase, and stream
//     order takes the place of the cross-rank barriers (every rank's
//     epilogue writes of a phase precede every owner phase);
//   * NVLS multicast: one multicast object with this single device bound,
//     so multimem.red / multimem.st land in one physical copy per group (the
//     switch's view of it), which is then copied to each member's output —
//     what the switch's replication does on NVSwitch.  When the device has
//     no multicast support the epilogue uses red.global.add (kRedLocal) and
//     the owner phase plain stores instead (reported in `paths`).
// Mode selection (fused_mode), epilogue targets (epi_red / epi_scatter), the
// owner-phase outputs and the gather helpers are the multi-GPU path's own.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <array>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/axonn.h"
#include "act.h"
#include "gemm.h"
#include "runtime.h"
#include "sym.h"

namespace axonn {
namespace {

template <class F>
F drv(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

// One multicast object with this device as its only member, bound to one
// physical allocation mapped twice: `uc` (plain loads/stores) and `mc`
// (multimem.*).  real == false: plain memory, mc == uc (emulation).
struct McArena {
  bool real = false;
  char* uc = nullptr;
  char* mc = nullptr;
  size_t size = 0;
  bool vmm = false;  // uc/mc come from the driver's VMM calls (else cudaMalloc)
  CUmemGenericAllocationHandle mem = 0, mch = 0;
  int dev = 0;
  std::string why;

  ~McArena() { release(); }

  bool create(size_t bytes, bool allow_real) {
    size = bytes < 256 ? 256 : bytes;
    if (allow_real && create_real()) return true;
    release();
    real = false;
    size = bytes < 256 ? 256 : bytes;
    void* p = nullptr;
    if (cudaMalloc(&p, size) != cudaSuccess) return false;
    uc = mc = static_cast<char*>(p);
    return true;
  }

  bool create_real() {
    auto getattr = drv<PFN_cuDeviceGetAttribute_v2000>("cuDeviceGetAttribute");
    auto mcCreate = drv<PFN_cuMulticastCreate_v12010>("cuMulticastCreate");
    auto mcAdd = drv<PFN_cuMulticastAddDevice_v12010>("cuMulticastAddDevice");
    auto mcGran = drv<PFN_cuMulticastGetGranularity_v12010>("cuMulticastGetGranularity");
    auto mcBind = drv<PFN_cuMulticastBindMem_v12010>("cuMulticastBindMem");
    auto memCreate = drv<PFN_cuMemCreate_v10020>("cuMemCreate");
    auto memGran = drv<PFN_cuMemGetAllocationGranularity_v10020>("cuMemGetAllocationGranularity");
    auto reserve = drv<PFN_cuMemAddressReserve_v10020>("cuMemAddressReserve");
    auto map = drv<PFN_cuMemMap_v10020>("cuMemMap");
    auto access = drv<PFN_cuMemSetAccess_v10020>("cuMemSetAccess");
    if (!getattr || !mcCreate || !mcAdd || !mcGran || !mcBind || !memCreate || !memGran ||
        !reserve || !map || !access) {
      why = "driver entry points for multicast unavailable";
      return false;
    }
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    vmm = true;
    int sup = 0;
    if (getattr(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS || !sup) {
      why = "device reports no multicast support";
      return false;
    }
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof mp);
    mp.numDevices = 1;
    mp.size = size;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
    size_t g1 = 0, g2 = 0;
    if (mcGran(&g1, &mp, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS) {
      why = "cuMulticastGetGranularity failed";
      return false;
    }
    CUmemAllocationProp ap;
    std::memset(&ap, 0, sizeof ap);
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = dev;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_NONE;
    if (memGran(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS) {
      why = "cuMemGetAllocationGranularity failed";
      return false;
    }
    const size_t gran = g1 > g2 ? g1 : g2;
    size = (size + gran - 1) / gran * gran;
    mp.size = size;
    if (mcCreate(&mch, &mp) != CUDA_SUCCESS) {
      why = "cuMulticastCreate failed";
      mch = 0;
      return false;
    }
    if (mcAdd(mch, dev) != CUDA_SUCCESS) {
      why = "cuMulticastAddDevice failed";
      return false;
    }
    if (memCreate(&mem, size, &ap, 0) != CUDA_SUCCESS) {
      why = "cuMemCreate failed";
      mem = 0;
      return false;
    }
    if (mcBind(mch, 0, mem, 0, size, 0) != CUDA_SUCCESS) {
      why = "cuMulticastBindMem failed";
      return false;
    }
    CUdeviceptr a = 0, b = 0;
    CUmemAccessDesc ad;
    std::memset(&ad, 0, sizeof ad);
    ad.location = ap.location;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (reserve(&a, size, gran, 0, 0) != CUDA_SUCCESS) {
      why = "cuMemAddressReserve failed";
      return false;
    }
    uc = reinterpret_cast<char*>(a);
    if (map(a, size, 0, mem, 0) != CUDA_SUCCESS || access(a, size, &ad, 1) != CUDA_SUCCESS) {
      why = "mapping the unicast view failed";
      return false;
    }
    if (reserve(&b, size, gran, 0, 0) != CUDA_SUCCESS) {
      why = "cuMemAddressReserve failed";
      return false;
    }
    mc = reinterpret_cast<char*>(b);
    if (map(b, size, 0, mch, 0) != CUDA_SUCCESS || access(b, size, &ad, 1) != CUDA_SUCCESS) {
      why = "mapping the multicast view failed";
      return false;
    }
    real = true;
    return true;
  }

  void release() {
    if (!vmm) {
      if (uc) cudaFree(uc);
    } else {
      auto unmap = drv<PFN_cuMemUnmap_v10020>("cuMemUnmap");
      auto freeva = drv<PFN_cuMemAddressFree_v10020>("cuMemAddressFree");
      auto rel = drv<PFN_cuMemRelease_v10020>("cuMemRelease");
      auto unbind = drv<PFN_cuMulticastUnbind_v12010>("cuMulticastUnbind");
      cudaDeviceSynchronize();
      if (unmap && freeva) {
        if (mc) {
          unmap(reinterpret_cast<CUdeviceptr>(mc), size);
          freeva(reinterpret_cast<CUdeviceptr>(mc), size);
        }
        if (uc) {
          unmap(reinterpret_cast<CUdeviceptr>(uc), size);
          freeva(reinterpret_cast<CUdeviceptr>(uc), size);
        }
      }
      if (unbind && mch && mem) unbind(mch, dev, 0, size);
      if (rel) {
        if (mem) rel(mem);
        if (mch) rel(mch);
      }
    }
    uc = mc = nullptr;
    mem = mch = 0;
    real = vmm = false;
  }
};

size_t align256(size_t b) { return (b + 255) & ~static_cast<size_t>(255); }

struct Pool {  // plain device buffers of one step, freed together
  std::vector<void*> ptrs;
  void* get(size_t bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes < 16 ? 16 : bytes) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return p;
  }
  ~Pool() {
    for (void* p : ptrs) cudaFree(p);
  }
};

// One fused reduction of every rank's rows x cols output over `axis`.
struct LbOp {
  int axis = 0, P = 1, es = 2, mode = kStore;
  int64_t elems = 0;
  std::vector<char*> recv, out;  // per rank (scatter mode)
  std::vector<char*> recv2;      // per rank (exchange-sum mode): the second receive set
  std::vector<char*> ctrl;       // per rank (pair-sum mode): tickets, done, calls
  int64_t cols = 0;
  long long chunks = 0;
  std::map<int, size_t> region;  // group leader rank -> arena offset (red, or P >= 3 owner output)
};

}  // namespace

// Deliberately serial and plain: see the file comment.
axonn_status_t loopback_step(const axonn_fc_desc_t* d, const int g[4], const void* const* I,
                             const void* const* What, const void* const* dO, void* const* O,
                             void* const* dI, void* const* dW, int flags, cudaStream_t st,
                             int* paths) {
  const int G = g[0] * g[1] * g[2] * g[3];
  if (d->dtype == AXONN_F32)
    return rt_fail(AXONN_ERR_UNSUPPORTED, "loopback: the fp32 test mode reduces through NCCL only");
  const bool gf32 = d->dtype == AXONN_BF16_GRADF32;
  const int ges = gf32 ? 4 : 2;  // dŴ element bytes (reading R17)
  std::vector<axonn_geometry_t> geo(G);
  std::vector<std::array<int, 4>> cc(G);
  for (int r = 0; r < G; ++r) {
    axonn_status_t s = axonn_shard_geometry(d, g[0], g[1], g[2], g[3], r, &geo[r]);
    if (s != AXONN_OK) return s;
    int c4[4];
    axonn_rank_to_coords(r, g[0], g[1], g[2], g[3], c4);
    for (int a = 0; a < 4; ++a) cc[r][a] = c4[a];
  }
  for (int r = 0; r < G; ++r) {
    const axonn_geometry_t& q = geo[r];
    if ((q.m_l != 0 && (!I[r] || !dO[r] || !O[r] || !dI[r])) || (q.what_len && (!What[r] || !dW[r])))
      return rt_fail(AXONN_ERR_ARG, "loopback: NULL tensor");
    if (q.k_l % 8 || q.n_l % 8)
      return rt_fail(AXONN_ERR_SHAPE, "loopback: bf16 shards need k_l, n_l multiples of 8");
  }
  const axonn_geometry_t& g0 = geo[0];
  const int64_t m_l = g0.m_l, k_l = g0.k_l, n_l = g0.n_l, S = g0.what_len;
  const int ax_fwd = d->transposed ? 0 : 1, ax_bwd = d->transposed ? 1 : 0;
  int red_min_k = 8192;
  if (const char* v = std::getenv("AXONN_RED_MIN_K")) red_min_k = std::atoi(v);
  if (flags & AXONN_LB_RED_ALWAYS) red_min_k = 0;
  if (flags & AXONN_LB_RED_NEVER) red_min_k = INT_MAX;
  bool exchange2 = true;
  if (const char* v = std::getenv("AXONN_EXCHANGE")) exchange2 = std::atoi(v) != 0;
  if (flags & AXONN_LB_NO_EXCHANGE) exchange2 = false;
  bool pairsum2 = false;
  if (const char* v = std::getenv("AXONN_PAIRSUM")) pairsum2 = std::atoi(v) != 0;
  if (flags & AXONN_LB_PAIRSUM) pairsum2 = true;
  // pull: each rank's partial stays in its own receive buffer (AXONN_PAIRSUM=2)
  bool pairpull = false;
  if (const char* v = std::getenv("AXONN_PAIRSUM")) pairpull = std::atoi(v) == 2;
  if (flags & AXONN_LB_PAIRPULL) pairpull = true;
  // the in-GEMM exchange sum (kXSum, opt-in), as on the multi-GPU path (AXONN_XSUM)
  int xsum2 = 0;
  if (const char* v = std::getenv("AXONN_XSUM")) xsum2 = std::atoi(v);
  if (flags & AXONN_LB_XSUM) xsum2 = 1;
  // unicast reductions into both ranks' outputs (kRedPair), as on the
  // multi-GPU path (AXONN_REDPAIR)
  int redpair2 = 2;
  if (const char* v = std::getenv("AXONN_REDPAIR")) redpair2 = std::atoi(v);
  if (flags & AXONN_LB_NO_REDPAIR) redpair2 = 0;
  // dÎ's 2-rank exchange summed inside the dW GEMM (SideSum), as on the
  // multi-GPU path (AXONN_SIDESUM)
  bool sidesum = false;
  if (const char* v = std::getenv("AXONN_SIDESUM")) sidesum = std::atoi(v) != 0;
  if (flags & AXONN_LB_SIDESUM) sidesum = true;
  const bool reverse = (flags & AXONN_LB_REVERSE) != 0;
  auto members = [&](int r, int axis) {
    std::vector<int> m(g[axis]);
    axonn_group_members(r, g[0], g[1], g[2], g[3], axis, m.data());
    return m;
  };
  const int Pz = g[2], Pd = g[3];
  int p = 0;

  // ------------------------------------------------------------- planning
  LbOp fo, fi, fw, fz, fd;
  auto plan = [&](LbOp* op, int axis, int64_t rows, int64_t cols, int64_t kdim, int es,
                  const char* what) -> axonn_status_t {
    op->axis = axis;
    op->P = g[axis];
    op->es = es;
    op->elems = rows * cols;
    if (op->P == 1) return AXONN_OK;
    op->mode = fused_mode(op->P, es, rows, cols, kdim, red_min_k, exchange2, pairsum2, xsum2,
                          redpair2);
    op->cols = cols;
    op->chunks = ((rows + 31) / 32) * ((cols + 63) / 64);
    if (op->mode == kStore) {
      char buf[200];
      std::snprintf(buf, sizeof buf,
                    "loopback: %s over %d ranks is not fused for this shape (the multi-GPU path "
                    "would use NCCL)", what, op->P);
      return rt_fail(AXONN_ERR_UNSUPPORTED, buf);
    }
    return AXONN_OK;
  };
  axonn_status_t s;
  if ((s = plan(&fo, ax_fwd, m_l, n_l, k_l, 2, "the forward all-reduce")) != AXONN_OK) return s;
  if ((s = plan(&fi, ax_bwd, m_l, k_l, n_l, 2, "the backward all-reduce")) != AXONN_OK) return s;
  if (Pz == 1 && Pd > 1) {
    if ((s = plan(&fw, 3, k_l, n_l, m_l, ges, "the data-parallel all-reduce")) != AXONN_OK) return s;
  }
  if (Pz > 1) {
    if (S % 8 || m_l <= 0)
      return rt_fail(AXONN_ERR_UNSUPPORTED, "loopback: RS_z is not fused for this shape");
    fz.axis = 2;
    fz.P = Pz;
    fz.es = ges;
    fz.mode = kScatter;
    fz.elems = k_l * n_l;
    if (Pd > 1) {
      if (S % ((16 / ges) * Pd))
        return rt_fail(AXONN_ERR_UNSUPPORTED,
                       "loopback: the data-parallel sum behind RS_z is not fused for this shape");
      fd.axis = 3;
      fd.P = Pd;
      fd.es = ges;
      fd.mode = kScatter;
      fd.elems = S;
    }
  }

  // ------------------------------------------------------------- buffers
  Pool pool;
  McArena arena;
  size_t arena_bytes = 0;
  for (LbOp* op : {&fo, &fi, &fw, &fd}) {
    if (op->mode == kStore) continue;
    if (op->mode == kMcRed || op->P >= 3) {
      for (int r = 0; r < G; ++r) {
        const int lead = members(r, op->axis)[0];
        if (!op->region.count(lead)) {
          op->region[lead] = arena_bytes;
          arena_bytes += align256(static_cast<size_t>(op->elems) * op->es);
        }
      }
    }
    if (op->mode == kPairSum) {
      op->recv.resize(G);
      op->out.resize(G);
      op->ctrl.resize(G);
      for (int r = 0; r < G; ++r) {
        op->recv[r] = static_cast<char*>(pool.get(op->elems * op->es));
        op->out[r] = static_cast<char*>(pool.get(op->elems * op->es));
        op->ctrl[r] = static_cast<char*>(pool.get(pair_ctrl_bytes(op->chunks)));
        if (!op->recv[r] || !op->out[r] || !op->ctrl[r])
          return rt_fail(AXONN_ERR_CUDA, "loopback: cudaMalloc failed");
        if (cudaMemsetAsync(op->ctrl[r], 0, pair_ctrl_bytes(op->chunks), st) != cudaSuccess)
          return rt_fail(AXONN_ERR_CUDA, "loopback: memset failed");
      }
    }
    if (op->mode == kRedPair) {  // each rank's output, zeroed before the GEMMs
      op->out.resize(G);
      for (int r = 0; r < G; ++r)
        if (!(op->out[r] = static_cast<char*>(pool.get(op->elems * op->es))))
          return rt_fail(AXONN_ERR_CUDA, "loopback: cudaMalloc failed");
    }
    if (op->mode == kXSum) {  // two receive sets of 2 slots, output, control block
      const long long U = xsum_units(op->elems / op->cols, op->cols);
      op->recv.resize(G);
      op->recv2.resize(G);
      op->out.resize(G);
      op->ctrl.resize(G);
      for (int r = 0; r < G; ++r) {
        op->recv[r] = static_cast<char*>(pool.get(op->elems * op->es * 2));
        op->recv2[r] = static_cast<char*>(pool.get(op->elems * op->es * 2));
        op->out[r] = static_cast<char*>(pool.get(op->elems * op->es));
        op->ctrl[r] = static_cast<char*>(pool.get(xsum_ctrl_bytes(U)));
        if (!op->recv[r] || !op->recv2[r] || !op->out[r] || !op->ctrl[r])
          return rt_fail(AXONN_ERR_CUDA, "loopback: cudaMalloc failed");
        if (cudaMemsetAsync(op->ctrl[r], 0, xsum_ctrl_bytes(U), st) != cudaSuccess)
          return rt_fail(AXONN_ERR_CUDA, "loopback: memset failed");
      }
    }
    if (op->mode == kScatter || op->mode == kExchange) {
      // scatter: P slots of elems / P; exchange: P slots of elems (whole partials)
      const int64_t rbytes = op->elems * op->es * (op->mode == kExchange ? op->P : 1);
      op->recv.resize(G);
      op->out.resize(G, nullptr);
      for (int r = 0; r < G; ++r) {
        op->recv[r] = static_cast<char*>(pool.get(rbytes));
        if (op->P == 2) op->out[r] = static_cast<char*>(pool.get(op->elems * op->es));
        if (!op->recv[r] || (op->P == 2 && !op->out[r]))
          return rt_fail(AXONN_ERR_CUDA, "loopback: cudaMalloc failed");
      }
    }
  }
  // side sum of dÎ: per rank a parity counter and the go / finished words
  // (no cross-rank barrier here: stream order already completed every rank's dI GEMM)
  const bool side_on = sidesum && fi.mode == kExchange && fi.P == 2 && m_l > 0 && k_l > 0 &&
                       n_l > 0 && fw.mode != kXSum;
  std::vector<char*> side_ctrl(G, nullptr);
  if (side_on) {
    for (int r = 0; r < G; ++r) {
      side_ctrl[r] = static_cast<char*>(pool.get(256));
      if (!side_ctrl[r] || cudaMemsetAsync(side_ctrl[r], 0, 256, st) != cudaSuccess)
        return rt_fail(AXONN_ERR_CUDA, "loopback: cudaMalloc failed");
    }
  }
  if (fz.mode == kScatter) {
    fz.recv.resize(G);
    for (int r = 0; r < G; ++r)
      if (!(fz.recv[r] = static_cast<char*>(pool.get(fz.elems * ges))))
        return rt_fail(AXONN_ERR_CUDA, "loopback: cudaMalloc failed");
  }
  if (arena_bytes && !arena.create(arena_bytes, !(flags & AXONN_LB_EMULATE_MC)))
    return rt_fail(AXONN_ERR_CUDA, "loopback: multicast arena allocation failed");
  const bool real_mc = arena.real;
  if (real_mc) p |= AXONN_LB_PATH_MULTICAST;
  auto uc_of = [&](const LbOp& op, int r) {
    return arena.uc + op.region.at(members(r, op.axis)[0]);
  };
  auto mc_of = [&](const LbOp& op, int r) {
    return reinterpret_cast<unsigned long long>(arena.mc + op.region.at(members(r, op.axis)[0]));
  };
  // epilogue target of rank r for a fused op (kStore: plain output)
  auto target = [&](const LbOp& op, int r) {
    if (op.mode == kMcRed) {
      EpiTarget t = epi_red(mc_of(op, r));
      if (!real_mc) t.mode = kRedLocal;
      return t;
    }
    if (op.mode == kPairSum) {  // as fused_bind in axonn.cpp: rank 0's tickets are shared
      const std::vector<int> mem = members(r, op.axis);
      const int me = cc[r][op.axis], peer = mem[1 - me];
      EpiTarget t;
      t.mode = kPairSum;
      t.P = 2;
      t.me = me;
      t.slice = (op.cols + 63) / 64;
      t.mc = reinterpret_cast<unsigned long long>(op.ctrl[mem[0]]);
      const size_t done = pair_done_off(op.chunks);
      // push: our partial to the peer's receive buffer, the peer's read from
      // ours; pull: ours stays in our buffer, the peer's is read from its own
      t.peer[0] = reinterpret_cast<unsigned long long>(op.recv[pairpull ? peer : r]);
      t.peer[1] = reinterpret_cast<unsigned long long>(op.recv[pairpull ? r : peer]);
      t.peer[2] = reinterpret_cast<unsigned long long>(op.out[r]);
      t.peer[3] = reinterpret_cast<unsigned long long>(op.out[peer]);
      t.peer[4] = reinterpret_cast<unsigned long long>(op.ctrl[r] + done);
      t.peer[5] = reinterpret_cast<unsigned long long>(op.ctrl[peer] + done);
      return t;
    }
    if (op.mode == kRedPair) {  // as fused_bind in axonn.cpp
      const std::vector<int> mem = members(r, op.axis);
      EpiTarget t;
      t.mode = kRedPair;
      t.P = 2;
      t.me = cc[r][op.axis];
      t.mc = reinterpret_cast<unsigned long long>(op.out[r]);
      t.peer[0] = reinterpret_cast<unsigned long long>(op.out[mem[1 - t.me]]);
      return t;
    }
    if (op.mode == kXSum) {  // as fused_bind in axonn.cpp
      const std::vector<int> mem = members(r, op.axis);
      const int me = cc[r][op.axis];
      unsigned long long recv[2], alt[2];
      for (int q = 0; q < 2; ++q) {
        recv[q] = reinterpret_cast<unsigned long long>(op.recv[mem[q]]);
        alt[q] = reinterpret_cast<unsigned long long>(op.recv2[mem[q]]);
      }
      return epi_xsum(me, op.elems / op.cols, op.cols, recv, alt, op.out[r], op.ctrl[r],
                      op.ctrl[mem[1 - me]]);
    }
    if (op.mode == kScatter || op.mode == kExchange) {
      const std::vector<int> mem = members(r, op.axis);
      unsigned long long peer[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int q = 0; q < op.P; ++q) peer[q] = reinterpret_cast<unsigned long long>(op.recv[mem[q]]);
      if (op.mode == kExchange) return epi_exchange(op.P, cc[r][op.axis], op.elems, peer, nullptr, nullptr);
      return epi_scatter(op.P, cc[r][op.axis], op.elems / op.P, peer);
    }
    return EpiTarget();
  };
  // owner phase output of rank r for a scatter-mode op (its own + the peer's
  // copy on 2-rank axes, else the group's multicast copy)
  auto owner_out = [&](const LbOp& op, int r) {
    OwnerOut o;
    const int me = cc[r][op.axis];
    const size_t off = static_cast<size_t>(me) * (op.elems / op.P) * op.es;
    if (op.P == 2) {
      const int peer = members(r, op.axis)[1 - me];
      o.mode = kOwnPlain;
      o.n_dst = 2;
      o.dst[0] = reinterpret_cast<unsigned long long>(op.out[r] + off);
      o.dst[1] = reinterpret_cast<unsigned long long>(op.out[peer] + off);
    } else {
      o.mode = real_mc ? kOwnMc : kOwnPlain;
      o.n_dst = 1;
      o.dst[0] = mc_of(op, r) + off;
    }
    return o;
  };
  auto zero_regions = [&](const LbOp& op) -> axonn_status_t {
    if (op.mode == kRedPair) {
      for (int r = 0; r < G; ++r)
        if (cudaMemsetAsync(op.out[r], 0, op.elems * op.es, st) != cudaSuccess)
          return rt_fail(AXONN_ERR_CUDA, "loopback: memset failed");
      return AXONN_OK;
    }
    if (op.mode != kMcRed) return AXONN_OK;
    for (const auto& kv : op.region)
      if (cudaMemsetAsync(arena.uc + kv.second, 0, op.elems * op.es, st) != cudaSuccess)
        return rt_fail(AXONN_ERR_CUDA, "loopback: memset failed");
    return AXONN_OK;
  };
  // every rank's owner phase (scatter mode) or local sum (exchange mode);
  // act_z: the forward GeLU rides on the exchange's local sum (Z -> act_z[r])
  auto owner_phase = [&](const LbOp& op, const std::vector<void*>* act_z = nullptr) -> axonn_status_t {
    if (op.mode == kPairSum) {  // the epilogues finished the sums: each rank's completion wait
      for (int r = 0; r < G; ++r) {
        if (sym_pair_wait(op.ctrl[r] + pair_done_off(op.chunks), op.ctrl[r] + pair_calls_off(op.chunks),
                          static_cast<uint32_t>(op.chunks), st) != cudaSuccess)
          return rt_fail(AXONN_ERR_CUDA, "loopback: pair-sum wait launch failed");
        rt_count_launch();
      }
      return AXONN_OK;
    }
    if (op.mode == kXSum) {  // what the GEMMs left open (here: all of the first ranks')
      for (int r = 0; r < G; ++r) {
        if (sym_xsum_sweep(op.recv[r], op.recv2[r], op.out[r], op.ctrl[r], op.elems / op.cols,
                           op.cols, rt_num_sms(), st) != cudaSuccess)
          return rt_fail(AXONN_ERR_CUDA, "loopback: exchange-sum sweep launch failed");
        rt_count_launch();
      }
      return AXONN_OK;
    }
    if (op.mode == kExchange) {  // every rank sums its own P slots locally
      for (int r = 0; r < G; ++r) {
        OwnerOut o;
        o.n_dst = 1;
        o.local = 1;
        o.dst[0] = reinterpret_cast<unsigned long long>(op.out[r]);
        if (act_z) {
          o.dst[0] = reinterpret_cast<unsigned long long>((*act_z)[r]);
          o.act = 1;
          o.act_dst = reinterpret_cast<unsigned long long>(op.out[r]);
        }
        if (sym_owner_reduce(op.recv[r], op.elems, op.P, op.es == 4, o, rt_num_sms(), st) !=
            cudaSuccess)
          return rt_fail(AXONN_ERR_CUDA, "loopback: exchange sum launch failed");
        rt_count_launch();
      }
      return AXONN_OK;
    }
    if (op.mode != kScatter) return AXONN_OK;
    for (int r = 0; r < G; ++r) {
      if (sym_owner_reduce(op.recv[r], op.elems / op.P, op.P, op.es == 4, owner_out(op, r),
                           rt_num_sms(), st) != cudaSuccess)
        return rt_fail(AXONN_ERR_CUDA, "loopback: owner phase launch failed");
      rt_count_launch();
    }
    return AXONN_OK;
  };
  // the reduced result of rank r -> its caller buffer
  auto deliver = [&](const LbOp& op, int r, void* dst) -> axonn_status_t {
    const char* src =
        ((op.mode == kScatter || op.mode == kExchange || op.mode == kPairSum || op.mode == kXSum ||
          op.mode == kRedPair) &&
         op.P == 2)
            ? op.out[r]
            : uc_of(op, r);
    if (op.elems &&
        cudaMemcpyAsync(dst, src, op.elems * op.es, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return rt_fail(AXONN_ERR_CUDA, "loopback: copy failed");
    return AXONN_OK;
  };

  // ------------------------------------------------ line 2: AG_z (Eq. 1)
  std::vector<const void*> Wfull(G);
  if (Pz > 1) {
    std::vector<void*> stage(G), wbuf(G);
    for (int r = 0; r < G; ++r) {
      stage[r] = pool.get(S * 2);
      wbuf[r] = pool.get(k_l * n_l * 2);
      if (!stage[r] || !wbuf[r]) return rt_fail(AXONN_ERR_CUDA, "loopback: cudaMalloc failed");
      if (S && cudaMemcpyAsync(stage[r], What[r], S * 2, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return rt_fail(AXONN_ERR_CUDA, "loopback: staging copy failed");
    }
    const bool pull = (flags & AXONN_LB_GATHER_PULL) != 0;
    p |= pull ? AXONN_LB_PATH_GATHER_PULL : AXONN_LB_PATH_GATHER_COPY;
    for (int r = 0; r < G; ++r) {
      const std::vector<int> mem = members(r, 2);
      std::vector<const void*> src(Pz);
      for (int q = 0; q < Pz; ++q) src[q] = q == cc[r][2] ? What[r] : stage[mem[q]];
      cudaError_t e = pull ? sym_gather_pull(src.data(), Pz, S * 2, wbuf[r], rt_num_sms(), st)
                           : sym_gather_copy(src.data(), Pz, S * 2, wbuf[r], st);
      if (e != cudaSuccess) return rt_fail(AXONN_ERR_CUDA, "loopback: gather failed");
      if (pull) rt_count_launch();
      Wfull[r] = wbuf[r];
    }
  } else {
    for (int r = 0; r < G; ++r) Wfull[r] = What[r];
  }

  // activation (fc1's GeLU, reading R18): Z kept per rank, dZ formed per rank
  const bool act = d->act == AXONN_ACT_GELU;
  std::vector<void*> zbuf(G, nullptr), dzbuf(G, nullptr);
  if (act) {
    for (int r = 0; r < G; ++r) {
      zbuf[r] = pool.get(m_l * n_l * 2);
      dzbuf[r] = pool.get(m_l * n_l * 2);
      if (!zbuf[r] || !dzbuf[r]) return rt_fail(AXONN_ERR_CUDA, "loopback: cudaMalloc failed");
    }
  }

  // ------------------------------------------------ lines 3-4: Ô, AR (Eq. 3)
  if ((s = zero_regions(fo)) != AXONN_OK) return s;
  for (int rr = 0; rr < G; ++rr) {
    const int r = reverse ? G - 1 - rr : rr;
    const EpiTarget t = target(fo, r);
    if ((s = rt_gemm(AXONN_OP_NN, AXONN_BF16, m_l, n_l, k_l, I[r], k_l, Wfull[r], n_l,
                     fo.mode == kStore ? O[r] : nullptr, n_l, st,
                     fo.mode == kStore ? nullptr : &t)) != AXONN_OK)
      return s;
  }
  const bool act_fused = act && fo.mode == kExchange;
  if ((s = owner_phase(fo, act_fused ? &zbuf : nullptr)) != AXONN_OK) return s;
  if (fo.mode != kStore) {
    p |= fo.mode == kMcRed ? AXONN_LB_PATH_FWD_RED
         : fo.mode == kPairSum ? AXONN_LB_PATH_FWD_PAIRSUM
         : fo.mode == kXSum ? AXONN_LB_PATH_FWD_XSUM
         : fo.mode == kRedPair ? AXONN_LB_PATH_FWD_REDPAIR
         : fo.mode == kExchange ? AXONN_LB_PATH_FWD_EXCHANGE : AXONN_LB_PATH_FWD_SCATTER;
    for (int r = 0; r < G; ++r)
      if ((s = deliver(fo, r, O[r])) != AXONN_OK) return s;
  }
  if (act && !act_fused) {  // O holds Z: keep it, O := GELU(Z)
    for (int r = 0; r < G; ++r) {
      if (gelu_forward_inplace(O[r], zbuf[r], m_l * n_l, rt_num_sms(), st) != cudaSuccess)
        return rt_fail(AXONN_ERR_CUDA, "loopback: GeLU launch failed");
      rt_count_launch();
    }
  }
  // backward of the activation: dZ = dO ⊙ GELU'(Z) replaces dO in lines 11, 13
  std::vector<const void*> dOa(dO, dO + G);
  if (act) {
    for (int r = 0; r < G; ++r) {
      if (gelu_backward(dO[r], zbuf[r], dzbuf[r], m_l * n_l, rt_num_sms(), st) != cudaSuccess)
        return rt_fail(AXONN_ERR_CUDA, "loopback: dGeLU launch failed");
      rt_count_launch();
      dOa[r] = dzbuf[r];
    }
  }

  // ------------------------------------------------ lines 11-12: dÎ, AR (Eq. 4)
  if ((s = zero_regions(fi)) != AXONN_OK) return s;
  for (int rr = 0; rr < G; ++rr) {
    const int r = reverse ? G - 1 - rr : rr;
    const EpiTarget t = target(fi, r);
    if ((s = rt_gemm(AXONN_OP_NT, AXONN_BF16, m_l, k_l, n_l, dOa[r], n_l, Wfull[r], n_l,
                     fi.mode == kStore ? dI[r] : nullptr, k_l, st,
                     fi.mode == kStore ? nullptr : &t)) != AXONN_OK)
      return s;
  }
  if (!side_on && (s = owner_phase(fi)) != AXONN_OK) return s;
  if (fi.mode != kStore) {
    p |= fi.mode == kMcRed ? AXONN_LB_PATH_BWD_RED
         : fi.mode == kPairSum ? AXONN_LB_PATH_BWD_PAIRSUM
         : fi.mode == kXSum ? AXONN_LB_PATH_BWD_XSUM
         : fi.mode == kRedPair ? AXONN_LB_PATH_BWD_REDPAIR
         : fi.mode == kExchange ? AXONN_LB_PATH_BWD_EXCHANGE : AXONN_LB_PATH_BWD_SCATTER;
    if (!side_on)
      for (int r = 0; r < G; ++r)
        if ((s = deliver(fi, r, dI[r])) != AXONN_OK) return s;
  }

  // ------------------------------------------------ line 13: dW partial
  if ((s = zero_regions(fw)) != AXONN_OK) return s;
  for (int rr = 0; rr < G; ++rr) {
    const int r = reverse ? G - 1 - rr : rr;
    EpiTarget t;
    const EpiTarget* tp = nullptr;
    if (fz.mode == kScatter) {
      const std::vector<int> mem = members(r, 2);
      unsigned long long peer[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int q = 0; q < Pz; ++q) peer[q] = reinterpret_cast<unsigned long long>(fz.recv[mem[q]]);
      t = epi_scatter(Pz, cc[r][2], S, peer);
      tp = &t;
    } else if (fw.mode != kStore) {
      t = target(fw, r);
      tp = &t;
    }
    SideSum side;
    if (side_on) {  // rank r's dW GEMM sums rank r's exchange slots of dÎ
      side.recv0 = fi.recv[r];
      side.recv1 = fi.recv[r];
      side.out = fi.out[r];
      side.n16 = fi.elems * fi.es / 16;
      side.par = reinterpret_cast<int*>(side_ctrl[r]);
      side.go = reinterpret_cast<int*>(side_ctrl[r] + 64);
      side.fin = reinterpret_cast<unsigned*>(side_ctrl[r] + 128);
    }
    if ((s = rt_gemm(AXONN_OP_TN, d->dtype, k_l, n_l, m_l, I[r], k_l, dOa[r], n_l,
                     tp ? nullptr : dW[r], n_l, st, tp, side_on ? &side : nullptr)) != AXONN_OK)
      return s;
  }
  if (side_on) {
    p |= AXONN_LB_PATH_BWD_SIDESUM;
    for (int r = 0; r < G; ++r)
      if ((s = deliver(fi, r, dI[r])) != AXONN_OK) return s;
  }
  // ------------------------------------------------ line 14: RS_z (Eq. 2)
  if (fz.mode == kScatter) {
    p |= AXONN_LB_PATH_RS_Z;
    for (int r = 0; r < G; ++r) {
      OwnerOut o;
      if (fd.mode == kScatter) {  // straight into the DATA owners' slots
        const std::vector<int> mem = members(r, 3);
        o.mode = kOwnScatter;
        for (int q = 0; q < Pd; ++q) o.dst[q] = reinterpret_cast<unsigned long long>(fd.recv[mem[q]]);
        o.me2 = cc[r][3];
        o.slice2 = S / Pd;
      } else {
        o.n_dst = 1;
        o.dst[0] = reinterpret_cast<unsigned long long>(dW[r]);
      }
      if (sym_owner_reduce(fz.recv[r], S, Pz, gf32, o, rt_num_sms(), st) != cudaSuccess)
        return rt_fail(AXONN_ERR_CUDA, "loopback: RS_z owner phase launch failed");
      rt_count_launch();
    }
  }
  // ------------------------------------------------ data-parallel sum (Eq. 5)
  if (fw.mode != kStore) {
    if ((s = owner_phase(fw)) != AXONN_OK) return s;
    p |= fw.mode == kMcRed ? AXONN_LB_PATH_DP_RED
         : fw.mode == kPairSum ? AXONN_LB_PATH_DP_PAIRSUM
         : fw.mode == kXSum ? AXONN_LB_PATH_DP_XSUM
         : fw.mode == kRedPair ? AXONN_LB_PATH_DP_REDPAIR
         : fw.mode == kExchange ? AXONN_LB_PATH_DP_EXCHANGE : AXONN_LB_PATH_DP_SCATTER;
    for (int r = 0; r < G; ++r)
      if ((s = deliver(fw, r, dW[r])) != AXONN_OK) return s;
  }
  if (fd.mode == kScatter) {
    if ((s = owner_phase(fd)) != AXONN_OK) return s;
    p |= AXONN_LB_PATH_DP_AFTER_RS;
    for (int r = 0; r < G; ++r)
      if ((s = deliver(fd, r, dW[r])) != AXONN_OK) return s;
  }
  if (cudaStreamSynchronize(st) != cudaSuccess)
    return rt_fail(AXONN_ERR_CUDA, "loopback: step failed on the device");
  if (paths) *paths = p;
  return AXONN_OK;
}

}  // namespace axonn
