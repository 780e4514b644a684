"""Small workload for compute-sanitizer memcheck: every local-product op on
ragged shapes (1-CTA and CTA-pair kernels, TMA-store and per-thread
epilogues) and Alg. 1 fwd/bwd at G=1."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_08145_b200 as ax
bf = torch.bfloat16
for (M, N, K) in ((296, 520, 200), (136, 264, 72), (512, 512, 256)):
    for op in (0, 1, 2):
        a_shape = (K, M) if op == 2 else (M, K)
        b_shape = (N, K) if op == 1 else (K, N)
        A = torch.empty(a_shape, dtype=bf, device="cuda").uniform_(-1, 1)
        B = torch.empty(b_shape, dtype=bf, device="cuda").uniform_(-1, 1)
        C = torch.empty(M, N, dtype=bf, device="cuda")
        ax.axonn_gemm(op, 0, M, N, K, A, A.stride(0), B, B.stride(0), C, N)
        Cf = torch.empty(M, N, dtype=torch.float32, device="cuda")
        ax.axonn_gemm(op, 1, M, N, K, A.float(), A.stride(0), B.float(), B.stride(0), Cf, N)
ax.axonn_grid_init(1, 1, 1, 1)
h = ax.axonn_fc_create(384, 256, 520)
I = torch.empty(384, 256, dtype=bf, device="cuda").uniform_(-1, 1)
W = torch.empty(256 * 520, dtype=bf, device="cuda").uniform_(-1, 1)
dO = torch.empty(384, 520, dtype=bf, device="cuda").uniform_(-1, 1)
O, dI, dW = torch.empty(384, 520, dtype=bf, device="cuda"), torch.empty(384, 256, dtype=bf, device="cuda"), torch.empty(256 * 520, dtype=bf, device="cuda")
ax.axonn_fc_forward(h, I, W, O)
ax.axonn_fc_backward(h, dO, dI, dW)
ax.axonn_grads_sync()
torch.cuda.synchronize()
ax.axonn_fc_destroy(h)
ax.axonn_grid_finalize()
print("SANITIZE_WORKLOAD_DONE")
