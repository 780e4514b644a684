"""Multi-rank parity worker, run under torchrun (one process per GPU).

For every factorisation (Gx, Gy, Gz, Gd) of the world size and several layer
shapes (normal and transposed, ragged 128-row tiles), each rank slices its
shards of the seeded global tensors with the library's own geometry, runs
axonn_fc_forward / axonn_fc_backward / axonn_grads_sync, and rank 0 reassembles
the global O, dI, dW and compares them with the unsharded oracle (oracle.fc):
  * fp32 test mode, integer inputs: bit-exact (all partial sums < 2^24, NCCL
    fp32 sums of integers are exact) — covers every collective and offset;
  * bf16, uniform inputs: normwise error <= 2e-2;
  * members of every all-reduce group hold bit-identical copies;
  * the bytes the library hands to NCCL equal Eqs. 1-5 exactly;
  * AXONN_BF16_GRADF32 (reading R17), integer inputs: dŴ (fp32 GEMM output,
    fp32 RS_z / data-parallel sums) bit-exact, bytes = Eqs. 1-5 with b = 4 in
    Eqs. 2 and 5.
Prints MP_OK on success; any failure raises (non-zero exit).
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2502_08145_b200 as ax  # noqa: E402
import synthdata  # noqa: E402
from oracle import fc, grid as ogrid, perf_model as pm  # noqa: E402


def dev(a32, dtype):
    if dtype == torch.bfloat16:
        bits = synthdata.bf16_bits(a32).view(np.int16)
        return torch.from_numpy(np.ascontiguousarray(bits)).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(a32, dtype=np.float32)).cuda()


def host(t):
    return t.float().cpu().numpy().astype(np.float64)


def run_case(cfg, m, k, n, transposed, kind, dtype, chunks, rank, world, zero_copy=False,
             grad_f32=False):
    X, W, dY = synthdata.layer_tensors(m, k, n, 7, kind=kind)
    dt = ax.AXONN_F32 if dtype == torch.float32 else ax.AXONN_BF16
    if grad_f32:
        dt = ax.AXONN_BF16_GRADF32
    gdtype = torch.float32 if grad_f32 else dtype
    h = ax.axonn_fc_create(m, k, n, transposed, dt, chunks)
    g = ax.axonn_fc_geometry(h)
    I = dev(X[g.row0:g.row0 + g.m_l, g.in_col0:g.in_col0 + g.k_l], dtype)
    Wl = W[g.in_col0:g.in_col0 + g.k_l, g.out_col0:g.out_col0 + g.n_l]
    What = dev(np.ascontiguousarray(Wl).reshape(1, -1)[:, g.what_off:g.what_off + g.what_len],
               dtype).reshape(-1)
    dO = dev(dY[g.row0:g.row0 + g.m_l, g.out_col0:g.out_col0 + g.n_l], dtype)
    O = torch.full((g.m_l, g.n_l), float("nan"), dtype=dtype, device="cuda")
    dI = torch.full((g.m_l, g.k_l), float("nan"), dtype=dtype, device="cuda")
    dW = torch.full((g.what_len,), float("nan"), dtype=gdtype, device="cuda")
    fused = [ax.axonn_fc_output_buffer(h, w) for w in range(3)]
    outs = [O, dI, dW]
    if zero_copy:   # write straight into the handle-owned symmetric buffers
        for w in range(3):
            if fused[w]:
                outs[w] = fused[w]
    ax.axonn_comm_bytes(reset=True)
    s = torch.cuda.current_stream()
    ax.axonn_fc_prefetch(h, What, s)           # OAG path
    ax.axonn_fc_forward(h, I, What, outs[0], s)
    ax.axonn_fc_backward(h, dO, outs[1], outs[2], s)
    ax.axonn_grads_sync(s)
    torch.cuda.synchronize()
    sent = ax.axonn_comm_bytes(reset=True)
    for w, shape in ((0, O.shape), (1, dI.shape), (2, dW.shape)):
        if zero_copy and fused[w]:   # read the symmetric buffer back into the tensor
            n_el = int(np.prod(shape))
            src = torch.empty(n_el, dtype=gdtype if w == 2 else dtype, device="cuda")
            import ctypes
            ctypes.CDLL("libcudart.so.12").cudaMemcpy(ctypes.c_void_p(src.data_ptr()),
                                                      ctypes.c_void_p(fused[w]),
                                                      ctypes.c_size_t(n_el * src.element_size()), 3)
            (O, dI, dW)[w].copy_(src.view(shape))
    ax.axonn_fc_destroy(h)
    mine = (tuple(g), host(O), host(dI), host(dW), sent, [f is not None for f in fused])
    allv = [None] * world
    dist.all_gather_object(allv, mine)
    if rank != 0:
        return
    O_ref, dI_ref, dW_ref = fc.fc_layer(X, W, dY)
    Og = np.full((m, n), np.nan)
    dIg = np.full((m, k), np.nan)
    dWg = np.full((k, n), np.nan)
    L = pm.Layer(m, k, n, transposed)
    eq = pm.layer_bytes(L, cfg, b=4 if dt == ax.AXONN_F32 else 2,
                        b_grad=2 if dt == ax.AXONN_BF16 else 4)
    tag = (f"cfg={cfg} shape={(m, k, n)} T={transposed} {kind}/{dtype}"
           f"{'/gradf32' if grad_f32 else ''} chunks={chunks}")
    for r, (gg, o, di, dw, snt, _) in enumerate(allv):
        gg = ax.Geometry(*gg)
        for dst, val, r0, c0 in ((Og, o, gg.row0, gg.out_col0), (dIg, di, gg.row0, gg.in_col0)):
            blk = dst[r0:r0 + val.shape[0], c0:c0 + val.shape[1]]
            if not np.all(np.isnan(blk)):
                assert np.array_equal(blk, val), f"replicas differ: {tag} rank {r}"
            dst[r0:r0 + val.shape[0], c0:c0 + val.shape[1]] = val
        wb = dWg[gg.in_col0:gg.in_col0 + gg.k_l, gg.out_col0:gg.out_col0 + gg.n_l].reshape(-1).copy()
        seg = wb[gg.what_off:gg.what_off + gg.what_len]
        if not np.all(np.isnan(seg)):
            assert np.array_equal(seg, dw), f"dW replicas differ: {tag} rank {r}"
        wb[gg.what_off:gg.what_off + gg.what_len] = dw
        dWg[gg.in_col0:gg.in_col0 + gg.k_l, gg.out_col0:gg.out_col0 + gg.n_l] = wb.reshape(gg.k_l, gg.n_l)
        # bytes handed to NCCL == Eqs. 1-5 (exact)
        want = {"ag_z": eq["ag_z"], "rs_z": eq["rs_z"], "ar_fwd": eq["ar_y"], "ar_bwd": eq["ar_x"],
                "ar_d": eq["ar_d"]}
        if chunks == 1:
            for key, v in want.items():
                assert snt[key] == v, f"bytes {key}: {snt} != Eq. {want} ({tag})"
    for name, got, ref in (("O", Og, O_ref), ("dI", dIg, dI_ref), ("dW", dWg, dW_ref)):
        assert not np.isnan(got).any(), f"{name} not fully covered: {tag}"
        if kind == "int" and (dtype == torch.float32 or (grad_f32 and name == "dW")):
            assert np.array_equal(got, ref), f"{name} not bit-exact: {tag}"
        else:
            err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
            assert err <= 2e-2, f"{name} normwise {err}: {tag}"
    nf = sum(allv[0][5])
    print(f"ok {tag} fused_outputs={nf}", flush=True)
    return Og, dIg, dWg


def run_chain(cfg, kind, dtype, rank):
    """A normal layer feeding a transposed one, through the
    ABI with no redistribution: layer 2's I_local IS layer 1's O_local buffer,
    layer 1's dO_local IS layer 2's dI_local.  Each rank checks its own shards
    against the composed fp64 network (fp32 + integers: bit-exact, all sums
    < 2^24; bf16: normwise <= 2e-2 per shard)."""
    m, k, hdim, n = 256, 128, 256, 128
    X = synthdata.tensor((m, k), 301, kind=kind)
    W1 = synthdata.tensor((k, hdim), 302, kind=kind)
    W2 = synthdata.tensor((hdim, n), 303, kind=kind)
    dY = synthdata.tensor((m, n), 304, kind=kind)
    dt = ax.AXONN_F32 if dtype == torch.float32 else ax.AXONN_BF16
    h1 = ax.axonn_fc_create(m, k, hdim, False, dt)
    h2 = ax.axonn_fc_create(m, hdim, n, True, dt)
    g1, g2 = ax.axonn_fc_geometry(h1), ax.axonn_fc_geometry(h2)
    assert (g1.m_l, g1.row0, g1.n_l, g1.out_col0) == (g2.m_l, g2.row0, g2.k_l, g2.in_col0)

    def what(W, g):
        Wl = np.ascontiguousarray(W[g.in_col0:g.in_col0 + g.k_l, g.out_col0:g.out_col0 + g.n_l])
        return dev(Wl.reshape(1, -1)[:, g.what_off:g.what_off + g.what_len], dtype).reshape(-1)

    I1 = dev(X[g1.row0:g1.row0 + g1.m_l, g1.in_col0:g1.in_col0 + g1.k_l], dtype)
    dO2 = dev(dY[g2.row0:g2.row0 + g2.m_l, g2.out_col0:g2.out_col0 + g2.n_l], dtype)
    Wh1, Wh2 = what(W1, g1), what(W2, g2)
    O1 = torch.empty((g1.m_l, g1.n_l), dtype=dtype, device="cuda")
    O2 = torch.empty((g2.m_l, g2.n_l), dtype=dtype, device="cuda")
    dI2 = torch.empty((g2.m_l, g2.k_l), dtype=dtype, device="cuda")
    dI1 = torch.empty((g1.m_l, g1.k_l), dtype=dtype, device="cuda")
    dW1 = torch.empty((g1.what_len,), dtype=dtype, device="cuda")
    dW2 = torch.empty((g2.what_len,), dtype=dtype, device="cuda")
    s = torch.cuda.current_stream()
    ax.axonn_fc_forward(h1, I1, Wh1, O1, s)
    ax.axonn_fc_forward(h2, O1, Wh2, O2, s)          # chained: no redistribution
    ax.axonn_fc_backward(h2, dO2, dI2, dW2, s)
    ax.axonn_fc_backward(h1, dI2, dI1, dW1, s)       # chained
    ax.axonn_grads_sync(s)
    torch.cuda.synchronize()
    ax.axonn_fc_destroy(h1)
    ax.axonn_fc_destroy(h2)
    # composed network, fp64 (oracle.fc)
    rO1 = fc.fc_forward(X, W1)
    rO2 = fc.fc_forward(rO1, W2)
    rdO1 = fc.fc_backward_input(dY, W2)
    rdW2 = fc.fc_backward_weight(rO1, dY)
    rdX = fc.fc_backward_input(rdO1, W1)
    rdW1 = fc.fc_backward_weight(X, rdO1)

    def flat_slice(R, g):
        return np.ascontiguousarray(R[g.in_col0:g.in_col0 + g.k_l, g.out_col0:g.out_col0 + g.n_l]
                                    ).reshape(-1)[g.what_off:g.what_off + g.what_len]

    checks = (("O2", host(O2), rO2[g2.row0:g2.row0 + g2.m_l, g2.out_col0:g2.out_col0 + g2.n_l]),
              ("dX", host(dI1), rdX[g1.row0:g1.row0 + g1.m_l, g1.in_col0:g1.in_col0 + g1.k_l]),
              ("dW1", host(dW1), flat_slice(rdW1, g1)), ("dW2", host(dW2), flat_slice(rdW2, g2)))
    for name, got, ref in checks:
        if kind == "int" and dtype == torch.float32:
            assert np.array_equal(got, ref), f"chain {name} not bit-exact cfg={cfg} rank {rank}"
        else:
            err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
            assert err <= 2e-2, f"chain {name} normwise {err} cfg={cfg} rank {rank}"
    if rank == 0:
        print(f"ok chain N->T cfg={cfg} {kind}/{dtype}", flush=True)


def run_chain_zero_copy(cfg, rank, steps=3):
    """The chained pair of run_chain through the handle-owned output buffers
    (layer 2's I_local IS layer 1's output buffer, layer 1's dO_local IS layer
    2's dI buffer), for several steps: a reduction buffer that the library
    zeroes in the background after its last reader (2-rank red.add outputs)
    must give every step the same bits, within tolerance of the oracle."""
    from bench import copy_raw
    m, k, hdim, n = 256, 128, 256, 128
    X = synthdata.tensor((m, k), 311)
    W1 = synthdata.tensor((k, hdim), 312)
    W2 = synthdata.tensor((hdim, n), 313)
    dY = synthdata.tensor((m, n), 314)
    bf = torch.bfloat16
    h1 = ax.axonn_fc_create(m, k, hdim, False, ax.AXONN_BF16)
    h2 = ax.axonn_fc_create(m, hdim, n, True, ax.AXONN_BF16)
    g1, g2 = ax.axonn_fc_geometry(h1), ax.axonn_fc_geometry(h2)

    def what(W, g):
        Wl = np.ascontiguousarray(W[g.in_col0:g.in_col0 + g.k_l, g.out_col0:g.out_col0 + g.n_l])
        return dev(Wl.reshape(1, -1)[:, g.what_off:g.what_off + g.what_len], bf).reshape(-1)

    I1 = dev(X[g1.row0:g1.row0 + g1.m_l, g1.in_col0:g1.in_col0 + g1.k_l], bf)
    dO2 = dev(dY[g2.row0:g2.row0 + g2.m_l, g2.out_col0:g2.out_col0 + g2.n_l], bf)
    Wh1, Wh2 = what(W1, g1), what(W2, g2)
    O1 = ax.axonn_fc_output_buffer(h1, 0) or torch.empty((g1.m_l, g1.n_l), dtype=bf, device="cuda")
    dI2 = ax.axonn_fc_output_buffer(h2, 1) or torch.empty((g2.m_l, g2.k_l), dtype=bf, device="cuda")
    O2 = torch.empty((g2.m_l, g2.n_l), dtype=bf, device="cuda")
    dI1 = torch.empty((g1.m_l, g1.k_l), dtype=bf, device="cuda")
    dW1 = torch.empty((g1.what_len,), dtype=bf, device="cuda")
    dW2 = torch.empty((g2.what_len,), dtype=bf, device="cuda")
    s = torch.cuda.current_stream()
    outs = []
    for _ in range(steps):
        ax.axonn_fc_forward(h1, I1, Wh1, O1, s)
        ax.axonn_fc_forward(h2, O1, Wh2, O2, s)
        ax.axonn_fc_backward(h2, dO2, dI2, dW2, s)
        ax.axonn_fc_backward(h1, dI2, dI1, dW1, s)
        ax.axonn_grads_sync(s)
        O1c = torch.empty((g1.m_l, g1.n_l), dtype=bf, device="cuda")
        copy_raw(O1c.data_ptr(), O1 if isinstance(O1, int) else O1.data_ptr(), 2 * O1c.numel(), s)
        torch.cuda.synchronize()
        outs.append([host(t) for t in (O1c, O2, dI1, dW1, dW2)])
    ax.axonn_fc_destroy(h1)
    ax.axonn_fc_destroy(h2)
    for st in outs[1:]:
        for name, a, b in zip(("O1", "O2", "dX", "dW1", "dW2"), outs[0], st):
            assert np.array_equal(a, b), f"zero-copy chain: step differs in {name} cfg={cfg} rank {rank}"
    rO1 = fc.fc_forward(X, W1)
    rO2 = fc.fc_forward(rO1, W2)
    rdX = fc.fc_backward_input(fc.fc_backward_input(dY, W2), W1)
    for name, got, ref in (("O2", outs[0][1], rO2[g2.row0:g2.row0 + g2.m_l, g2.out_col0:g2.out_col0 + g2.n_l]),
                           ("dX", outs[0][2], rdX[g1.row0:g1.row0 + g1.m_l, g1.in_col0:g1.in_col0 + g1.k_l])):
        err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
        assert err <= 2e-2, f"zero-copy chain {name} normwise {err} cfg={cfg} rank {rank}"
    if rank == 0:
        print(f"ok zero-copy chain x{steps} cfg={cfg}", flush=True)


def run_graph(cfg, rank):
    """One layer step (OAG prefetch, forward, backward, grads_sync) captured in a
    CUDA graph — NCCL calls, device-side barriers, copy-engine gathers and the
    library's cross-stream forks included — must reproduce the eager outputs
    bit for bit on every replay."""
    m, k, n = 256, 512, 1024
    X, W, dY = synthdata.layer_tensors(m, k, n, 11)
    h = ax.axonn_fc_create(m, k, n, False, ax.AXONN_BF16)
    g = ax.axonn_fc_geometry(h)
    I = dev(X[g.row0:g.row0 + g.m_l, g.in_col0:g.in_col0 + g.k_l], torch.bfloat16)
    Wl = np.ascontiguousarray(W[g.in_col0:g.in_col0 + g.k_l, g.out_col0:g.out_col0 + g.n_l])
    What = dev(Wl.reshape(1, -1)[:, g.what_off:g.what_off + g.what_len], torch.bfloat16).reshape(-1)
    dO = dev(dY[g.row0:g.row0 + g.m_l, g.out_col0:g.out_col0 + g.n_l], torch.bfloat16)
    outs = [torch.empty((g.m_l, g.n_l), dtype=torch.bfloat16, device="cuda"),
            torch.empty((g.m_l, g.k_l), dtype=torch.bfloat16, device="cuda"),
            torch.empty((g.what_len,), dtype=torch.bfloat16, device="cuda")]

    def step(s):
        ax.axonn_fc_prefetch(h, What, s)
        ax.axonn_fc_forward(h, I, What, outs[0], s)
        ax.axonn_fc_backward(h, dO, outs[1], outs[2], s)
        ax.axonn_grads_sync(s)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step(s)
    torch.cuda.synchronize()
    eager = [o.clone() for o in outs]
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s, capture_error_mode="thread_local"):
        step(s)
    for rep in range(2):
        for o in outs:
            o.fill_(float("nan"))
        dist.barrier()
        graph.replay()
        torch.cuda.synchronize()
        for name, a, b in zip(("O", "dI", "dW"), outs, eager):
            assert torch.equal(a.view(torch.int16), b.view(torch.int16)), \
                f"graph replay {rep} {name} differs at cfg={cfg} rank {rank}"
    del graph
    ax.axonn_fc_destroy(h)
    if rank == 0:
        print(f"ok graph replay cfg={cfg}", flush=True)


def run_empty(cfg, rank):
    """m = 0 on every grid: no tokens -> O, dI empty; dŴ = 0 exactly."""
    k, n = 128, 256
    h = ax.axonn_fc_create(0, k, n, False, ax.AXONN_BF16)
    g = ax.axonn_fc_geometry(h)
    e = lambda *sh: torch.empty(sh, dtype=torch.bfloat16, device="cuda")  # noqa: E731
    What = torch.ones((max(g.what_len, 1),), dtype=torch.bfloat16, device="cuda")
    dW = torch.full((g.what_len,), float("nan"), dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.current_stream()
    ax.axonn_fc_forward(h, e(0, g.k_l), What, e(0, g.n_l), s)
    ax.axonn_fc_backward(h, e(0, g.n_l), e(0, g.k_l), dW, s)
    ax.axonn_grads_sync(s)
    torch.cuda.synchronize()
    assert torch.count_nonzero(dW).item() == 0 and not torch.isnan(dW).any(), f"m=0 cfg={cfg}"
    ax.axonn_fc_destroy(h)


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ax.bootstrap_from_torch_distributed(local)
    shapes = [(256, 512, 1024), (384, 192, 320)]
    for cfg in ogrid.enumerate_configs(world):
        results = {}
        # "xsum": 2-rank axes exchange partials and sum them inside the GEMM
        # (the default); "red": 2-rank axes reduce with multimem.red; "exchange": 2-rank axes
        # exchange whole partials and sum locally; "scatter": 2-rank axes use
        # the scatter + owner phase; "0": NCCL collectives (AXONN_FUSED=0)
        for fused in ("xsum", "red", "redpair", "exchange", "exchange_side", "pairsum", "pairpull",
                      "scatter", "0"):
            os.environ["AXONN_FUSED"] = "0" if fused == "0" else "1"
            os.environ["AXONN_RED_MIN_K"] = "0" if fused == "red" else str(1 << 30)
            os.environ["AXONN_EXCHANGE"] = "0" if fused == "scatter" else "1"
            os.environ["AXONN_PAIRSUM"] = {"pairsum": "1", "pairpull": "2"}.get(fused, "0")
            os.environ["AXONN_XSUM"] = "1" if fused == "xsum" else "0"
            # "redpair": unicast red.add at every K (the default uses it below the red threshold)
            os.environ["AXONN_REDPAIR"] = "1" if fused == "redpair" else "0"
            # the backward's exchange of dÎ summed by the dW GEMM's helper warps, or by a pass
            os.environ["AXONN_SIDESUM"] = "1" if fused == "exchange_side" else "0"
            ax.axonn_grid_init(*cfg)
            if fused == "red" and rank == 0:
                print(f"cfg={cfg} fused status:",
                      {a: ax.axonn_fused_status(a) for a in "xyzd"}, flush=True)
            for (m, k, n) in shapes:
                for transposed in (False, True):
                    if not pm.feasible(pm.Layer(m, k, n, transposed), cfg):
                        continue
                    if fused == "0":
                        run_case(cfg, m, k, n, transposed, "int", torch.float32, 1, rank, world)
                    results[(fused, m, k, n, transposed)] = run_case(
                        cfg, m, k, n, transposed, "uniform", torch.bfloat16, 1, rank, world)
                    if fused in ("red", "0"):
                        # fp32 gradients: fused (scatter + fp32 owner phase) or NCCL fp32
                        # RS_z / AR_data beside bf16 AR_x/y; integer dŴ bit-exact either way
                        run_case(cfg, m, k, n, transposed, "int", torch.bfloat16, 1, rank, world,
                                 grad_f32=True)
                    if fused == "red":
                        zc = run_case(cfg, m, k, n, transposed, "uniform", torch.bfloat16, 1, rank,
                                      world, zero_copy=True)
                        if rank == 0:
                            for a, b in zip(zc, results[(fused, m, k, n, transposed)]):
                                assert np.array_equal(a, b), f"zero-copy differs {cfg}"
            run_chain(cfg, "uniform", torch.bfloat16, rank)
            if fused in ("exchange", "redpair", "red"):
                run_chain_zero_copy(cfg, rank)
            if fused in ("xsum", "red", "redpair", "exchange", "pairsum", "pairpull", "0"):
                run_graph(cfg, rank)
                run_empty(cfg, rank)
            if fused == "0":
                run_chain(cfg, "int", torch.float32, rank)
                run_case(cfg, 512, 256, 512, False, "int", torch.float32, 3, rank, world)
                run_case(cfg, 512, 256, 512, False, "uniform", torch.bfloat16, 3, rank, world)
            ax.axonn_grid_finalize()
        if rank == 0:
            # fused (NVLS) vs NCCL: bit-identical when every axis has <= 2 ranks
            # (both compute RNE(a + b)); with 4-rank axes the fused owner phase
            # rounds once where NCCL's ring rounds per hop -> compare to tolerance
            exact = max(cfg) <= 2
            for key, val in results.items():
                if key[0] == "0":
                    continue
                ref = results[("0",) + key[1:]]
                for name, a, b in zip(("O", "dI", "dW"), val, ref):
                    if exact:
                        assert np.array_equal(a, b), f"fused != NCCL for {name} at {cfg} {key}"
                    else:
                        err = np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30)
                        assert err <= 2e-2, f"fused vs NCCL {name} {err} at {cfg} {key}"
            print(f"fused vs nccl {'bit-exact' if exact else 'within 2e-2'} cfg={cfg}", flush=True)
    dist.barrier()
    if rank == 0:
        print("MP_OK", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
