"""Run one local product a few times (for ncu / quick timing).
    python tools/gemm_one.py OP M N K [reps]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_08145_b200 as ax
op, M, N, K = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
bf = torch.bfloat16
a_shape = (K, M) if op == 2 else (M, K)
b_shape = (N, K) if op == 1 else (K, N)
A = torch.empty(a_shape, dtype=bf, device="cuda").uniform_(-1, 1)
B = torch.empty(b_shape, dtype=bf, device="cuda").uniform_(-1, 1)
C = torch.empty(M, N, dtype=bf, device="cuda")
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(reps):
    if i == reps - 1:
        e0.record(s)
    ax.axonn_gemm(op, 0, M, N, K, A, A.stride(0), B, B.stride(0), C, N, s)
e1.record(s)
torch.cuda.synchronize()
print(f"op={op} {M}x{N}x{K}: {e0.elapsed_time(e1):.3f} ms, {2*M*N*K/e0.elapsed_time(e1)/1e9:.1f} TF/s")
