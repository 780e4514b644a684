"""Python binding of libaxonn.so (include/axonn.h) — argument marshalling only.

Every function here has the name of the C entry point it calls and does no
arithmetic of the method: shapes, pointers and streams are passed through
ctypes; every step of the hot path runs in the library's CUDA kernels and
NCCL calls.  Importing this module fails loudly if the library has not been
built (``python paper_2502_08145_b200/build.py``); there is no fallback.

torch is used only for device memory, streams and torch.distributed
bootstrap, and is imported lazily so the pure-host calls work without it.
"""
from __future__ import annotations

import ctypes
import os
from collections import namedtuple
from ctypes import (POINTER, Structure, byref, c_char_p, c_double, c_int, c_int64, c_ubyte,
                    c_void_p)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libaxonn.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2502_08145_b200/build.py`")
_lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)

# ---------------------------------------------------------------- constants
AXONN_OK, AXONN_ERR_ARG, AXONN_ERR_CONFIG, AXONN_ERR_SHAPE, AXONN_ERR_STATE = 0, 1, 2, 3, 4
AXONN_ERR_INFEASIBLE, AXONN_ERR_CUDA, AXONN_ERR_NCCL, AXONN_ERR_UNSUPPORTED = 5, 6, 7, 8
AXONN_BF16, AXONN_F32, AXONN_BF16_GRADF32 = 0, 1, 2
AXONN_OP_NN, AXONN_OP_NT, AXONN_OP_TN = 0, 1, 2
AXONN_ACT_NONE, AXONN_ACT_GELU = 0, 1
AXIS = {"x": 0, "y": 1, "z": 2, "d": 3}
AXONN_LB_RED_ALWAYS, AXONN_LB_RED_NEVER, AXONN_LB_GATHER_PULL, AXONN_LB_EMULATE_MC = 1, 2, 4, 8
AXONN_LB_NO_EXCHANGE, AXONN_LB_PAIRSUM, AXONN_LB_REVERSE, AXONN_LB_PAIRPULL = 16, 32, 64, 128
AXONN_LB_XSUM, AXONN_LB_SIDESUM, AXONN_LB_NO_REDPAIR = 256, 512, 1024
LB_PATHS = {"fwd_red": 1, "fwd_scatter": 2, "bwd_red": 4, "bwd_scatter": 8, "rs_z": 16,
            "dp_red": 32, "dp_scatter": 64, "dp_after_rs": 128, "gather_copy": 256,
            "gather_pull": 512, "multicast": 1024, "fwd_exchange": 2048, "bwd_exchange": 4096,
            "dp_exchange": 8192, "fwd_pairsum": 16384, "bwd_pairsum": 32768,
            "dp_pairsum": 65536, "fwd_xsum": 131072, "bwd_xsum": 262144, "dp_xsum": 524288,
            "bwd_sidesum": 1048576, "fwd_redpair": 2097152, "bwd_redpair": 4194304,
            "dp_redpair": 8388608}
_STATUS_NAMES = {0: "OK", 1: "ARG", 2: "CONFIG", 3: "SHAPE", 4: "STATE", 5: "INFEASIBLE",
                 6: "CUDA", 7: "NCCL", 8: "UNSUPPORTED"}


class AxonnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"AXONN_ERR_{_STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


# ---------------------------------------------------------------- structs
class FcDesc(Structure):
    _fields_ = [("m", c_int64), ("k", c_int64), ("n", c_int64), ("transposed", c_int),
                ("dtype", c_int), ("chunks", c_int), ("act", c_int)]


class GeometryT(Structure):
    _fields_ = [(f, c_int64) for f in
                ("m_l", "k_l", "n_l", "row0", "in_col0", "out_col0", "what_off", "what_len")]


class LayerT(Structure):
    _fields_ = [("m", c_int64), ("k", c_int64), ("n", c_int64), ("transposed", c_int)]


class BwEntry(Structure):
    _fields_ = [("inner", c_int), ("size", c_int), ("bytes_per_s", c_double)]


class GridScore(Structure):
    _fields_ = [("gx", c_int), ("gy", c_int), ("gz", c_int), ("gd", c_int),
                ("t_ag_z", c_double), ("t_rs_z", c_double), ("t_ar_y", c_double),
                ("t_ar_x", c_double), ("t_ar_data", c_double), ("t_comm", c_double)]


Geometry = namedtuple("Geometry", [f for f, _ in GeometryT._fields_])

# ---------------------------------------------------------------- prototypes
_S = c_int  # axonn_status_t
_PROTOS = {
    "axonn_last_error": (c_char_p, []),
    "axonn_version": (c_int, []),
    "axonn_unique_id": (_S, [POINTER(c_ubyte)]),
    "axonn_bootstrap": (_S, [c_int, c_int, POINTER(c_ubyte), c_int]),
    "axonn_grid_init": (_S, [c_int, c_int, c_int, c_int]),
    "axonn_grid_coords": (_S, [POINTER(c_int)] * 4),
    "axonn_grid_finalize": (_S, []),
    "axonn_rank_to_coords": (_S, [c_int, c_int, c_int, c_int, c_int, POINTER(c_int)]),
    "axonn_group_members": (_S, [c_int, c_int, c_int, c_int, c_int, c_int, POINTER(c_int)]),
    "axonn_shard_geometry": (_S, [POINTER(FcDesc), c_int, c_int, c_int, c_int, c_int,
                                  POINTER(GeometryT)]),
    "axonn_fc_create": (_S, [POINTER(FcDesc), POINTER(c_void_p)]),
    "axonn_fc_geometry": (_S, [c_void_p, POINTER(GeometryT)]),
    "axonn_fc_prefetch": (_S, [c_void_p, c_void_p, c_void_p]),
    "axonn_fc_output_buffer": (_S, [c_void_p, c_int, POINTER(c_void_p)]),
    "axonn_fused_status": (_S, [c_int, c_char_p, c_int]),
    "axonn_fused_mode": (_S, [c_int, c_int, c_int64, c_int64, c_int64, c_char_p, c_int]),
    "axonn_nvlink_probe": (_S, [c_int, c_int64, c_int, c_int, c_int, POINTER(c_double)]),
    "axonn_fc_forward": (_S, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "axonn_fc_backward": (_S, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "axonn_grads_sync": (_S, [c_void_p]),
    "axonn_fc_destroy": (_S, [c_void_p]),
    "axonn_gemm": (_S, [c_int, c_int, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                        c_int64, c_void_p, c_int64, c_void_p]),
    "axonn_loopback_step": (_S, [POINTER(FcDesc), c_int, c_int, c_int, c_int, POINTER(c_void_p),
                                 POINTER(c_void_p), POINTER(c_void_p), POINTER(c_void_p),
                                 POINTER(c_void_p), POINTER(c_void_p), c_int, c_void_p,
                                 POINTER(c_int)]),
    "axonn_profile_enable": (_S, [c_int]),
    "axonn_profile_read": (_S, [POINTER(c_int64), POINTER(c_double), POINTER(c_double)]),
    "axonn_kernel_launches": (c_int64, []),
    "axonn_stream_k_launches": (c_int64, []),
    "axonn_stream_k_items": (_S, [c_int, c_int, c_int, c_int, POINTER(c_int), POINTER(c_int),
                                  POINTER(c_int), POINTER(c_int), c_int, POINTER(c_int)]),
    "axonn_set_gemm_sms": (_S, [c_int]),
    "axonn_comm_bytes": (_S, [POINTER(c_int64), c_int]),
    "axonn_grid_select": (_S, [POINTER(LayerT), c_int, c_int, c_int, POINTER(BwEntry), c_int,
                               c_double, c_int, c_int, POINTER(GridScore), c_int, POINTER(c_int)]),
    "axonn_grid_select_mp": (_S, [POINTER(LayerT), c_int, c_int, c_int, POINTER(BwEntry), c_int,
                                  c_double, c_int, c_int, c_int, POINTER(GridScore), c_int,
                                  POINTER(c_int)]),
}
for _name, (_res, _args) in _PROTOS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_PROTOS)


def _check(status: int) -> None:
    if status != AXONN_OK:
        raise AxonnError(status, _lib.axonn_last_error().decode())


def _stream_ptr(stream):
    """cudaStream_t of a torch stream / raw int / None (= torch current stream)."""
    if stream is None:
        import torch
        return c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return c_void_p(stream)
    return c_void_p(stream.cuda_stream)


def _ptr(t):
    """Device pointer of a torch tensor (or an int address)."""
    if t is None:
        return c_void_p(0)
    if isinstance(t, int):
        return c_void_p(t)
    return c_void_p(t.data_ptr())


# ---------------------------------------------------------------- API
def axonn_last_error() -> str:
    return _lib.axonn_last_error().decode()


def axonn_version() -> int:
    return _lib.axonn_version()


def axonn_unique_id() -> bytes:
    buf = (c_ubyte * 128)()
    _check(_lib.axonn_unique_id(buf))
    return bytes(buf)


def axonn_bootstrap(world_rank: int, world_size: int, uid: bytes | None, cuda_device: int) -> None:
    arr = (c_ubyte * 128).from_buffer_copy(uid) if uid else None
    _check(_lib.axonn_bootstrap(world_rank, world_size, arr, cuda_device))


def axonn_grid_init(gx: int, gy: int, gz: int, gd: int) -> None:
    _check(_lib.axonn_grid_init(gx, gy, gz, gd))


def axonn_grid_coords():
    v = [c_int() for _ in range(4)]
    _check(_lib.axonn_grid_coords(*[byref(x) for x in v]))
    return tuple(x.value for x in v)


def axonn_grid_finalize() -> None:
    _check(_lib.axonn_grid_finalize())


def axonn_rank_to_coords(rank: int, cfg):
    out = (c_int * 4)()
    _check(_lib.axonn_rank_to_coords(rank, *cfg, out))
    return tuple(out)


def axonn_group_members(rank: int, cfg, axis):
    a = AXIS[axis] if isinstance(axis, str) else int(axis)
    out = (c_int * cfg[a])()
    _check(_lib.axonn_group_members(rank, *cfg, a, out))
    return tuple(out)


def _desc(m, k, n, transposed=False, dtype=AXONN_BF16, chunks=1, act=AXONN_ACT_NONE):
    return FcDesc(m, k, n, int(bool(transposed)), dtype, chunks, act)


def axonn_shard_geometry(m, k, n, cfg, rank, transposed=False, dtype=AXONN_BF16) -> Geometry:
    g = GeometryT()
    d = _desc(m, k, n, transposed, dtype)
    _check(_lib.axonn_shard_geometry(byref(d), *cfg, rank, byref(g)))
    return Geometry(*[getattr(g, f) for f in Geometry._fields])


def axonn_fc_create(m, k, n, transposed=False, dtype=AXONN_BF16, chunks=1,
                    act=AXONN_ACT_NONE) -> int:
    h = c_void_p()
    d = _desc(m, k, n, transposed, dtype, chunks, act)
    _check(_lib.axonn_fc_create(byref(d), byref(h)))
    return h.value


def axonn_fc_geometry(h) -> Geometry:
    g = GeometryT()
    _check(_lib.axonn_fc_geometry(c_void_p(h), byref(g)))
    return Geometry(*[getattr(g, f) for f in Geometry._fields])


def axonn_fc_output_buffer(h, which: int):
    """Device address of the handle-owned fused output buffer (0=O, 1=dI, 2=dŴ) or None."""
    p = c_void_p()
    _check(_lib.axonn_fc_output_buffer(c_void_p(h), which, byref(p)))
    return p.value


def axonn_nvlink_probe(axis, nbytes, mode, ctas=148, iters=10) -> float:
    a = AXIS[axis] if isinstance(axis, str) else int(axis)
    v = c_double()
    _check(_lib.axonn_nvlink_probe(a, nbytes, mode, ctas, iters, byref(v)))
    return v.value


def axonn_fused_status(axis) -> str:
    a = AXIS[axis] if isinstance(axis, str) else int(axis)
    buf = ctypes.create_string_buffer(256)
    _check(_lib.axonn_fused_status(a, buf, 256))
    return buf.value.decode()


def axonn_fused_mode(P, elem_bytes, rows, cols, kdim) -> str:
    """The epilogue mode the multi-GPU path picks for this reduction (host only)."""
    buf = ctypes.create_string_buffer(64)
    _check(_lib.axonn_fused_mode(P, elem_bytes, rows, cols, kdim, buf, 64))
    return buf.value.decode()


def axonn_fc_prefetch(h, W_hat, stream=None) -> None:
    _check(_lib.axonn_fc_prefetch(c_void_p(h), _ptr(W_hat), _stream_ptr(stream)))


def axonn_fc_forward(h, I_local, W_hat, O_local, stream=None) -> None:
    _check(_lib.axonn_fc_forward(c_void_p(h), _ptr(I_local), _ptr(W_hat), _ptr(O_local),
                                 _stream_ptr(stream)))


def axonn_fc_backward(h, dO_local, dI_local, dW_hat, stream=None) -> None:
    _check(_lib.axonn_fc_backward(c_void_p(h), _ptr(dO_local), _ptr(dI_local), _ptr(dW_hat),
                                  _stream_ptr(stream)))


def axonn_grads_sync(stream=None) -> None:
    _check(_lib.axonn_grads_sync(_stream_ptr(stream)))


def axonn_fc_destroy(h) -> None:
    _check(_lib.axonn_fc_destroy(c_void_p(h)))


def axonn_gemm(op, dtype, M, N, K, A, lda, B, ldb, C, ldc, stream=None) -> None:
    _check(_lib.axonn_gemm(op, dtype, M, N, K, _ptr(A), lda, _ptr(B), ldb, _ptr(C), ldc,
                           _stream_ptr(stream)))


def axonn_loopback_step(m, k, n, cfg, I, W_hat, dO, O, dI, dW, transposed=False,
                        dtype=AXONN_BF16, flags=0, stream=None, act=AXONN_ACT_NONE) -> set:
    """Alg. 1 for every rank of grid ``cfg`` on this GPU (include/axonn.h, test
    support).  I, W_hat, dO, O, dI, dW: per-rank lists of tensors (rank order).
    Returns the names of the fused paths that ran (LB_PATHS)."""
    G = cfg[0] * cfg[1] * cfg[2] * cfg[3]
    arrs = []
    for lst in (I, W_hat, dO, O, dI, dW):
        if len(lst) != G:
            raise ValueError(f"need {G} per-rank tensors, got {len(lst)}")
        arrs.append((c_void_p * G)(*[_ptr(t).value or 0 for t in lst]))
    d = _desc(m, k, n, transposed, dtype, 1, act)
    paths = c_int()
    _check(_lib.axonn_loopback_step(byref(d), *cfg, *arrs, flags, _stream_ptr(stream),
                                    byref(paths)))
    return {name for name, bit in LB_PATHS.items() if paths.value & bit}


def axonn_profile_enable(enabled: bool = True) -> None:
    _check(_lib.axonn_profile_enable(int(bool(enabled))))


def axonn_profile_read():
    n, ms, fl = c_int64(), c_double(), c_double()
    _check(_lib.axonn_profile_read(byref(n), byref(ms), byref(fl)))
    return n.value, ms.value, fl.value


def axonn_kernel_launches() -> int:
    return _lib.axonn_kernel_launches()


def axonn_stream_k_launches() -> int:
    return _lib.axonn_stream_k_launches()


def axonn_stream_k_items(sk_tiles, num_kb, pair, pairs) -> list:
    """The stream-K items of CTA pair `pair` (host-only; include/axonn.h):
    a list of (tile, role, kb0, kb1), role 0 whole tile, 1 HEAD, 2 TAIL."""
    cap = 16
    arrs = [(c_int * cap)() for _ in range(4)]
    n = c_int()
    _check(_lib.axonn_stream_k_items(sk_tiles, num_kb, pair, pairs, *arrs, cap, byref(n)))
    return [tuple(a[i] for a in arrs) for i in range(min(n.value, cap))]


def axonn_set_gemm_sms(sms: int) -> None:
    _check(_lib.axonn_set_gemm_sms(sms))


def axonn_comm_bytes(reset: bool = False) -> dict:
    out = (c_int64 * 5)()
    _check(_lib.axonn_comm_bytes(out, int(bool(reset))))
    return dict(zip(("ag_z", "rs_z", "ar_fwd", "ar_bwd", "ar_d"), list(out)))


def axonn_grid_select(layers, G, g_node, table, beta_inter, bytes_per_elem=2, fixed_gd=0,
                      cap=None, grad_bytes_per_elem=None):
    """layers: iterable of (m, k, n, transposed); table: {(G0, G1): bytes/s}.

    Returns the ranked list of dicts (gx, gy, gz, gd, t_ag_z, ..., t_comm).
    grad_bytes_per_elem (default: bytes_per_elem) is b of Eqs. 2 and 5
    (axonn_grid_select_mp)."""
    layers = list(layers)
    L = (LayerT * max(1, len(layers)))(*[LayerT(m, k, n, int(bool(t))) for m, k, n, t in layers])
    items = sorted(table.items())
    T = (BwEntry * max(1, len(items)))(*[BwEntry(a, b, v) for (a, b), v in items])
    cap = 4096 if cap is None else cap
    out = (GridScore * max(1, cap))()
    n = c_int()
    if grad_bytes_per_elem is None:
        _check(_lib.axonn_grid_select(L, len(layers), G, g_node, T, len(items), beta_inter,
                                      bytes_per_elem, fixed_gd, out, cap, byref(n)))
    else:
        _check(_lib.axonn_grid_select_mp(L, len(layers), G, g_node, T, len(items), beta_inter,
                                         bytes_per_elem, grad_bytes_per_elem, fixed_gd, out, cap,
                                         byref(n)))
    return [{f: getattr(out[i], f) for f, _ in GridScore._fields_} for i in range(min(cap, n.value))]


def axonn_grid_select_mp(layers, G, g_node, table, beta_inter, bytes_per_elem=2,
                         grad_bytes_per_elem=4, fixed_gd=0, cap=None):
    """axonn_grid_select with b = grad_bytes_per_elem in Eqs. 2 and 5."""
    return axonn_grid_select(layers, G, g_node, table, beta_inter, bytes_per_elem, fixed_gd, cap,
                             grad_bytes_per_elem=grad_bytes_per_elem)


# ---------------------------------------------------------------- helpers
def bootstrap_from_torch_distributed(device: int | None = None) -> None:
    """Bootstrap with the world of an initialised torch.distributed group.

    Rank 0 draws the NCCL id; it is broadcast with torch.distributed (the
    plumbing), then every rank calls axonn_bootstrap."""
    import torch
    import torch.distributed as dist
    if device is None:
        device = torch.cuda.current_device()
    rank, world = dist.get_rank(), dist.get_world_size()
    obj = [axonn_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    axonn_bootstrap(rank, world, obj[0], device)


def gemm(op, A, B, C, stream=None) -> None:
    """axonn_gemm on torch tensors (row-major, contiguous rows)."""
    import torch
    if C.dtype == torch.float32:
        dtype = AXONN_BF16_GRADF32 if A.dtype == torch.bfloat16 else AXONN_F32
    else:
        dtype = AXONN_BF16
    M, N = C.shape
    K = A.shape[0] if op == AXONN_OP_TN else A.shape[1]
    axonn_gemm(op, dtype, M, N, K, A, A.stride(0), B, B.stride(0), C, C.stride(0), stream)
