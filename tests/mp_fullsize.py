"""Full-size multi-GPU parity, run under torchrun (one process per GPU).

The launch configurations bench.py times for N > 1: the GPT-5B block
(BASELINE.json C2 shapes, 16384 tokens per GPU, global m = 16384 N) on the grid
the performance model ranks first, and the tensor-parallel proxies of
BASELINE C3/C4/C5 (20B/40B/80B layers on (2,2,1,1), (2,1,1,2), (1,2,2,1),
(1,1,2,2)), default (fused NVLS) collectives, outputs in the handle-owned
buffers.  Every rank checks 1024 sampled entries of each of
its output shards (O, dI, dŴ of all four layers) against exact fp64 dot
products of the seeded global inputs (oracle.fc.dot_entries), to the
north_star tolerance: |gpu - ref| <= 2e-2 * max|ref| over the sample.
Prints FULLSIZE_OK on success.
"""
import ctypes
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2502_08145_b200 as ax  # noqa: E402
import synthdata  # noqa: E402
from bench import block_layers  # noqa: E402
from oracle import fc  # noqa: E402


def to_dev(a32):
    bits = synthdata.bf16_bits(a32).view(np.int16)
    return torch.from_numpy(np.ascontiguousarray(bits)).view(torch.bfloat16).cuda()


def read(ptr_or_t, shape):
    if isinstance(ptr_or_t, torch.Tensor):
        return ptr_or_t.float().cpu().numpy().astype(np.float64).reshape(shape)
    n = int(np.prod(shape))
    t = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    ctypes.CDLL("libcudart.so.12").cudaMemcpy(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(ptr_or_t),
                                              ctypes.c_size_t(2 * n), 3)
    return t.float().cpu().numpy().astype(np.float64).reshape(shape)


def cases(world):
    """(label, h, global m, grid, layer indices).  The first is bench.py's
    data-parallel default; the rest are the tensor-parallel proxies of
    BASELINE C3/C4/C5, where the fused epilogues run with
    K >= 8192 on 2-rank axes (512x256 tiles, multimem.red)."""
    layers = block_layers(4096, 16384 * world)
    tb = {(g0, g1): 1.0e11 for g0 in range(1, 9) for g1 in range(2, 9) if g0 * g1 <= 8}
    best = ax.axonn_grid_select(layers, world, 8, tb, 1.0e11, 2, 0, cap=1)[0]
    out = [("5B-model-top1", 4096, 16384 * world,
            (best["gx"], best["gy"], best["gz"], best["gd"]), (0, 1, 2, 3))]
    if world == 2:
        out += [("20B-tp", 7168, 8192, (2, 1, 1, 1), (0, 1, 2, 3)),
                ("20B-tpY", 7168, 8192, (1, 2, 1, 1), (1, 3))]
    elif world == 4:
        out += [("20B-C3proxy", 7168, 8192, (2, 2, 1, 1), (0, 1, 2, 3)),
                ("40B-C5proxy", 9216, 16384, (2, 1, 1, 2), (0, 3)),
                ("80B-C4aproxy", 12288, 16384, (1, 2, 2, 1), (1,)),
                ("80B-C4bproxy", 12288, 16384, (2, 2, 1, 1), (1,)),
                ("20B-Z-DP", 7168, 16384, (1, 1, 2, 2), (0, 1))]
    return out


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ax.bootstrap_from_torch_distributed(local)
    rng = np.random.default_rng(1234 + rank)
    ar = np.arange(1024)

    def sampled(A, B, rows, cols):   # exact fp64 dot products of the samples only
        return fc.dot_entries(A[rows, :], B[:, cols], ar, ar)

    for label, hid, mglob, cfg, which in cases(world):
        ax.axonn_grid_init(*cfg)
        layers = block_layers(hid, mglob)
        s = torch.cuda.current_stream()
        for li in which:
            m, k, n, t = layers[li]
            X, W, dY = synthdata.layer_tensors(m, k, n, 100 + li)
            h = ax.axonn_fc_create(m, k, n, t, ax.AXONN_BF16, 4)
            g = ax.axonn_fc_geometry(h)
            I = to_dev(X[g.row0:g.row0 + g.m_l, g.in_col0:g.in_col0 + g.k_l])
            Wl = np.ascontiguousarray(W[g.in_col0:g.in_col0 + g.k_l, g.out_col0:g.out_col0 + g.n_l])
            What = to_dev(Wl.reshape(1, -1)[:, g.what_off:g.what_off + g.what_len]).reshape(-1)
            del Wl
            dO = to_dev(dY[g.row0:g.row0 + g.m_l, g.out_col0:g.out_col0 + g.n_l])
            outs = []
            for which_o, shape in ((0, (g.m_l, g.n_l)), (1, (g.m_l, g.k_l)), (2, (g.what_len,))):
                p = ax.axonn_fc_output_buffer(h, which_o)
                outs.append(p if p else torch.empty(shape, dtype=torch.bfloat16, device="cuda"))
            ax.axonn_fc_prefetch(h, What, s)
            ax.axonn_fc_forward(h, I, What, outs[0], s)
            ax.axonn_fc_backward(h, dO, outs[1], outs[2], s)
            ax.axonn_grads_sync(s)
            torch.cuda.synchronize()
            O = read(outs[0], (g.m_l, g.n_l))
            dI = read(outs[1], (g.m_l, g.k_l))
            dW = read(outs[2], (g.what_len,))
            # O = X W, dI = dY W^T, dW = X^T dY (all rows of all replicas)
            r = rng.integers(0, g.m_l, 1024)
            c = rng.integers(0, g.n_l, 1024)
            ref = sampled(X, W, g.row0 + r, g.out_col0 + c)
            e_o = np.max(np.abs(O[r, c] - ref)) / np.max(np.abs(ref))
            c2 = rng.integers(0, g.k_l, 1024)
            ref = sampled(dY, W.T, g.row0 + r, g.in_col0 + c2)
            e_i = np.max(np.abs(dI[r, c2] - ref)) / np.max(np.abs(ref))
            f = rng.integers(0, g.what_len, 1024) + g.what_off
            wr, wc = f // g.n_l, f % g.n_l
            ref = sampled(X.T, dY, g.in_col0 + wr, g.out_col0 + wc)
            e_w = np.max(np.abs(dW[f - g.what_off] - ref)) / np.max(np.abs(ref))
            print(f"rank {rank} {label} layer {li} ({m}x{k}x{n} T={t}) grid {cfg}: normwise "
                  f"O {e_o:.2e} dI {e_i:.2e} dW {e_w:.2e}", flush=True)
            assert max(e_o, e_i, e_w) <= 2e-2, f"{label} layer {li} rank {rank} out of tolerance"
            ax.axonn_fc_destroy(h)
            del X, W, dY, O, dI, dW, I, What, dO, outs
        ax.axonn_grid_finalize()
        torch.cuda.empty_cache()
        dist.barrier()
    if rank == 0:
        print("FULLSIZE_OK", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
