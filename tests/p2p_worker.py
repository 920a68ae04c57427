"""torchrun worker of tests/test_gpu_ep.py::test_p2p_sweep_multi_gpu: the NVLink sweep feeding the
measured-topology pipeline, fitted and smoothed on every rank."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_09915_b200 import ops  # noqa: E402
from paper_2302_09915_b200.layer import nccl_unique_id  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    ndev = torch.cuda.device_count()
    shared = os.environ.get("TAMOE_EP_BOOTSTRAP") == "store" or ndev < world
    torch.cuda.set_device(local % ndev)
    sizes = (4.0, 32.0, 128.0)
    if shared:  # NCCL-free bootstrap over gloo (ranks may share a GPU)
        dist.init_process_group("gloo")
        samples = ops.p2p_sweep_store(world, rank, sizes, reps=3, warmup=1)
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        samples = ops.p2p_sweep(obj[0], world, rank, sizes, reps=3, warmup=1)
    assert len(samples) == world * world * len(sizes) * 3
    assert all(us > 0 for (_, _, _, us) in samples)
    a, b = ops.fit_profile(samples, world)
    a, b = ops.fill_partial_profile(a, b, [world])
    assert np.all(np.isfinite(a)) and np.all(a >= 0) and np.all(b > 0)
    off = b[~np.eye(world, dtype=bool)]
    distinct = ndev >= world  # every rank on its own GPU: off-diagonal pairs are real NVLink transfers
    if distinct:
        # NVLink peer stores cost more per MB than a local HBM copy
        assert np.mean(np.diag(b)) < off.mean(), (np.diag(b), off)
        assert 0.5 < off.mean() < 20.0, off  # us/MB: 50 GB/s .. 2 TB/s
    else:
        assert 0.01 < off.mean() < 20.0, off  # shared GPU: every pair is a device-local copy
    # every rank sees the same matrix
    t = torch.tensor(b, device="cpu" if shared else "cuda")
    ref = t.clone()
    dist.broadcast(ref, 0)
    assert torch.equal(t, ref)
    c_hat, _, bh = ops.solve_target_tree([world], a, b, 64, 1, 16384)
    np.testing.assert_allclose(c_hat.sum(1), 16384)
    dist.barrier()
    if rank == 0:
        print("P2P_SWEEP_OK bootstrap=%s world=%d devices=%d beta_self=%.3f beta_peer=%.3f us/MB"
              % ("store" if shared else "nccl", world, min(ndev, world), np.mean(np.diag(b)), off.mean()),
              flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
