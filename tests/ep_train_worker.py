"""Expert-parallel train() (torchrun --nproc-per-node W tests/ep_train_worker.py [kind] [cap]): every rank trains
its own process (gate replica, S tokens) and its E = N / W experts through tamoe_layer_train; rank 0 compares the
report with the reference's own train() (compiled from its sources, oracle/_ref) at P = W processes on identical
bf16-representable data (trainer.cpp:183-452): per-step task / aux losses (bf16 tolerance, as
tests/test_gpu_train.py), dropped rates, dispatch, the alpha-beta comm estimate (exactly the model of the same
counts) and a measured exchange time for every step.  Fewer GPUs than ranks: the NCCL-free bootstrap over gloo."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def bf(a):
    return torch.tensor(np.asarray(a), dtype=torch.float32).bfloat16().double().numpy()


def main():
    kind = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    cap = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    ndev = torch.cuda.device_count()
    shared = os.environ.get("TAMOE_EP_BOOTSTRAP") == "store" or ndev < world
    dev = local % ndev
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo" if shared else "nccl", **({} if shared else {"device_id": torch.device("cuda", dev)}))
    import oracle
    from paper_2302_09915_b200 import ops
    from paper_2302_09915_b200.layer import LayerConfig, TAMoELayer, nccl_unique_id
    from paper_2302_09915_b200.train import LossKind, TrainConfig, train_layer

    P, S, d, dout, N, k, steps, lr = world, 256, 256, 128, 8 * world // 2, 2, 10, 0.05
    E = N // P
    R = oracle.ref()
    x, y, _, _ = R.gen_synthetic(3, P, S, d, dout, N=N, k=k, clusters=4)
    x, y = bf(x), bf(y)
    rng = np.random.default_rng(3)
    gates = bf(rng.normal(size=(P, d, N)) * 0.01)
    experts = bf(rng.normal(size=(N, d, dout)) / np.sqrt(d))
    beta = np.array([[0.1 if i == j else (1.0 if i // 2 == j // 2 else 4.0) for j in range(P)] for i in range(P)])
    c_hat = ops.target_closed_form(beta, N, k, S) if kind in (1, 2) else None

    nid = None
    if not shared:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    cfg = LayerConfig(P=1, S=S, d=d, d_out=dout, N=N, k=k, f=0, act=0, cap_mode=cap, capacity_factor=1.25,
                      aux_kind=kind, need_dx=False, world_size=world, rank=rank)
    layer = TAMoELayer(cfg, c_hat, nccl_id=nid)
    params = dict(wg=TAMoELayer.gates_from_reference(gates[rank:rank + 1], cfg.n_pad),
                  w1=TAMoELayer.linear_from_reference(experts[rank * E:(rank + 1) * E]))
    xt = torch.tensor(x[rank], dtype=torch.float32).bfloat16().cuda()
    yt = torch.tensor(y[rank], dtype=torch.float32).bfloat16().cuda()
    tc = TrainConfig(P=P, S=S, d=d, d_out=dout, N=N, k=k, lr=lr, steps=steps,
                     capacity=ops.CapacityPolicy(ops.CapacityMode(cap), 1.25), alpha_hat=np.zeros((P, P)),
                     beta_hat=beta)
    rep = train_layer(layer, params, xt, yt, tc, kind=LossKind(kind), c_hat=c_hat)
    # the report is identical on every rank
    t = torch.tensor(np.concatenate([rep.task_loss, rep.aux_loss, rep.initial_dispatch.ravel()]),
                     device="cpu" if shared else "cuda")
    ref0 = t.clone()
    dist.broadcast(ref0, 0)
    assert torch.equal(t, ref0), "ranks disagree on the report"
    if rank == 0:
        ref = R.train(x, y, gates, experts, kind=kind, cap_mode=cap, cf=1.25, c_hat=c_hat, lr=lr, steps=steps, k=k)
        print("task", rep.task_loss, ref["task_loss"], "\naux", rep.aux_loss, ref["aux_loss"], "\ndropped",
              rep.dropped_rate, ref["dropped_rate"], "\ndispatch0", rep.initial_dispatch, ref["initial_dispatch"],
              "\ncomm", rep.comm_us, rep.comm_measured_us, flush=True)
        np.testing.assert_allclose(rep.task_loss, ref["task_loss"], rtol=3e-2)
        np.testing.assert_allclose(rep.aux_loss, ref["aux_loss"], rtol=5e-2, atol=1e-6)
        np.testing.assert_allclose(rep.dropped_rate, ref["dropped_rate"], atol=0.02)
        np.testing.assert_allclose(rep.initial_dispatch, ref["initial_dispatch"], atol=0.01 * S * k)
        assert rep.task_loss[-1] < rep.task_loss[0]
        # alpha-beta model of this step's dispatch matrix (comm_cost.cpp:24-55) next to the measured exchange
        pay = ops.device_payload_tokens(rep.initial_dispatch)
        rounds = 1 if cap in (1, 3) else 0
        want = (beta * (pay * (d * 4 / 1e6))).max() + rounds * 0.0
        assert abs(rep.comm_us[0] - want) <= 1e-9 * want, (rep.comm_us[0], want)
        assert np.all(rep.comm_measured_us > 0)
        print(f"EP_TRAIN_OK world={world} kind={kind} cap={cap} task {rep.task_loss[0]:.5f}->{rep.task_loss[-1]:.5f} "
              f"(ref {ref['task_loss'][0]:.5f}->{ref['task_loss'][-1]:.5f}) comm model {np.mean(rep.comm_us):.2f} us, "
              f"measured {np.mean(rep.comm_measured_us):.2f} us", flush=True)
    dist.barrier()
    del layer
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
