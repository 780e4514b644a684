"""NVLink primitive throughput on a 2-rank axis (run under torchrun, 2 GPUs)."""
import os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_08145_b200 as ax
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
ax.bootstrap_from_torch_distributed(local)
ax.axonn_grid_init(2, 1, 1, 1)
names = {0: "multimem.red.add.bf16x8", 1: "multimem.st.v4", 2: "st.global peer", 3: "multimem.ld_reduce",
         4: "local st", 5: "red.add.bf16x8 peer", 6: "red.add.bf16x8 local"}
for mode in (4, 6, 2, 5, 1, 0, 3):
    for ctas in (16, 148):
        g = ax.axonn_nvlink_probe("x", 256 << 20, mode, ctas, 10)
        if dist.get_rank() == 0:
            print(f"{names[mode]:28s} ctas={ctas:4d}: {g:8.1f} GB/s", flush=True)
ax.axonn_grid_finalize()
dist.destroy_process_group()
