"""NCCL all_to_all_single bus bandwidth on this box (reference point for the fused peer-store exchange).
torchrun --nproc-per-node N scripts/nccl_a2a_bench.py"""
import os
import torch
import torch.distributed as dist

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank))))
for mb in (8, 32, 64, 128):
    n = mb * 2 ** 20 // 2
    x = torch.randn(n, device="cuda").bfloat16()
    y = torch.empty_like(x)
    for _ in range(5):
        dist.all_to_all_single(y, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dist.all_to_all_single(y, x)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 20], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    bus = (mb * 2 ** 20) * (world - 1) / world / (ms / 1e3) / 1e9
    if rank == 0:
        print(f"NCCL all_to_all {mb} MiB/GPU world {world}: {ms * 1e3:.1f} us, bus {bus:.1f} GB/s", flush=True)
dist.destroy_process_group()
