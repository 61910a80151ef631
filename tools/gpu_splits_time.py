"""Tuning: cost of the distributed split search (NCCL, one rank, interior diagonals)."""
import os, sys, time
import torch
import torch.distributed as dist
sys.path.insert(0, '.')  # run from the repo root
from paper_2005_12648_b200.dist import global_splits
from paper_2005_12648_b200.workloads import config_input_device
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29641")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
k0, p0, m = config_input_device(2, seed=1, log_len=29)
N = k0.numel()
for nd in (3, 9):
    diags = [N * i // (nd - 1) for i in range(nd)]
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        s = global_splits(k0, diags, m)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{nd} diagonals: {dt*1e3:.2f} ms")
dist.destroy_process_group()
