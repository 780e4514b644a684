"""Where does a fused forward's time go?  (torchrun, 2 GPUs, grid 2,1,1,1)
Times the transposed proj layer's axonn_fc_forward: whole call (CUDA events) vs
its GEMM alone (axonn_profile events around the library's GEMM launch)."""
import os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_08145_b200 as ax
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
ax.bootstrap_from_torch_distributed(local)
m, k, n = int(os.environ.get("PM", 32768)), 4096, 4096
for mode, env in (("red", "0"), ("scatter", str(1 << 30)), ("red", "0"), ("scatter", str(1 << 30))):
    os.environ["AXONN_RED_MIN_K"] = env
    ax.axonn_grid_init(2, 1, 1, 1)
    h = ax.axonn_fc_create(m, k, n, True, ax.AXONN_BF16, 1)
    g = ax.axonn_fc_geometry(h)
    I = torch.empty(g.m_l, g.k_l, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    W = torch.empty(g.what_len, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    O = ax.axonn_fc_output_buffer(h, 0)
    s = torch.cuda.current_stream()
    for _ in range(3):
        ax.axonn_fc_forward(h, I, W, O, s)
    torch.cuda.synchronize(); dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ax.axonn_profile_read(); ax.axonn_profile_enable(True)
    e0.record(s)
    for _ in range(20):
        ax.axonn_fc_forward(h, I, W, O, s)
    e1.record(s)
    torch.cuda.synchronize()
    ax.axonn_profile_enable(False)
    nl, gms, _ = ax.axonn_profile_read()
    tot = e0.elapsed_time(e1) / 20
    gemm = torch.empty(g.k_l, g.n_l, dtype=torch.bfloat16, device="cuda")
    C = torch.empty(g.m_l, g.n_l, dtype=torch.bfloat16, device="cuda")
    e0.record(s)
    for _ in range(20):
        ax.axonn_gemm(0, 0, g.m_l, g.n_l, g.k_l, I, g.k_l, gemm, g.n_l, C, g.n_l, s)
    e1.record(s); torch.cuda.synchronize()
    plain = e0.elapsed_time(e1) / 20
    if dist.get_rank() == 0:
        print(f"{mode:8s} m_l={g.m_l} k_l={g.k_l} n_l={g.n_l}: forward {tot:.3f} ms, its GEMM {gms / nl:.3f} ms, "
              f"plain GEMM {plain:.3f} ms, rest {tot - gms / nl:.3f} ms", flush=True)
    ax.axonn_fc_destroy(h)
    ax.axonn_grid_finalize()
dist.destroy_process_group()
