"""Expert-parallel parity on W ranks (torchrun --nproc-per-node W tests/ep_worker.py [case] [steps]).
With fewer GPUs than ranks (or TAMOE_EP_BOOTSTRAP=store) the ranks bootstrap over gloo and share devices
round-robin -- the same kernels, peer stores and device barriers, several ranks per GPU.

Every rank owns one logical process (its gate replica and S tokens) and E = N/W experts; the
layer exchanges tokens, expert outputs and gradients over NCCL.  Rank 0 gathers losses and
gradients and compares them with the oracle's P=W multi-process step (trainer.cpp:371-482)
on identical bf16-representable inputs: routing bit-exact (audited near-ties), values and
gradients within bf16 rel 2e-2."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {
    "ffn_prop": dict(S=512, d=256, dout=256, f=512, k=2, cap=3, kind=1, need_dx=True),
    "linear_none": dict(S=384, d=256, dout=256, f=0, k=1, cap=0, kind=0, need_dx=True),
    "ffn_local": dict(S=1000, d=512, dout=256, f=256, k=1, cap=2, kind=1, need_dx=True),
    # global capacity across ranks (gate.cpp:157-164): one cap per expert over every rank's picks
    # (cf 0.5: about half of the picks are dropped, so the cross-rank selection order is exercised)
    "ffn_global": dict(S=512, d=256, dout=256, f=512, k=2, cap=1, kind=0, need_dx=True, cf=0.5),
    # C5 link-throttle emulation on every cross-rank link (each payload store issued 3x): same results
    "ffn_prop_throttled": dict(S=512, d=256, dout=256, f=512, k=2, cap=3, kind=1, need_dx=True, throttle=3),
}


def bf(a):
    return torch.tensor(np.asarray(a), dtype=torch.float32).bfloat16().double().numpy()


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def main():
    case = sys.argv[1] if len(sys.argv) > 1 else "ffn_prop"
    # optional second argument: number of steps; > 2 turns the run into a determinism stress loop (every
    # step's losses and gradients must be bitwise identical to the first step's: same inputs, same weights)
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    c = CASES[case]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    ndev = torch.cuda.device_count()
    # store bootstrap (no NCCL): the workspace handles go over gloo, so several ranks may share one GPU
    shared = os.environ.get("TAMOE_EP_BOOTSTRAP") == "store" or ndev < world
    dev = local % ndev
    torch.cuda.set_device(dev)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    import oracle
    from paper_2302_09915_b200 import ops
    from paper_2302_09915_b200.layer import LayerConfig, TAMoELayer, nccl_unique_id

    S, d, dout, f, k = c["S"], c["d"], c["dout"], c["f"], c["k"]
    if c.get("throttle"):
        ops.set_link_emulation(1, c["throttle"])
    N = 8 * world
    E = N // world
    P = world
    rng = np.random.default_rng(7)
    x = bf(rng.normal(size=(P, S, d)))
    y = bf(rng.normal(size=(P, S, dout)) * 0.5)
    gates = bf(rng.normal(size=(P, d, N)) * 0.05)
    if f == 0:
        U = bf(rng.normal(size=(N, d, dout)) / np.sqrt(d))
        W1 = W2 = None
    else:
        U = None
        W1 = bf(rng.normal(size=(N, d, f)) / np.sqrt(d))
        W2 = bf(rng.normal(size=(N, f, dout)) / np.sqrt(f))
    beta = np.array([[0.1 if i == j else (1.0 if i // 2 == j // 2 else 4.0) for j in range(P)] for i in range(P)])
    c_hat = ops.target_closed_form(beta, N, k, S)

    obj = [None]
    if not shared:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
    cfg = LayerConfig(P=1, S=S, d=d, d_out=dout, N=N, k=k, f=f, act=1, cap_mode=c["cap"], capacity_factor=c.get("cf", 1.25),
                      aux_kind=c["kind"], need_dx=c["need_dx"], world_size=world, rank=rank)
    layer = TAMoELayer(cfg, c_hat, nccl_id=obj[0])
    lo, hi = rank * E, (rank + 1) * E
    params = dict(wg=TAMoELayer.gates_from_reference(gates[rank:rank + 1], cfg.n_pad))
    if f == 0:
        params["w1"] = TAMoELayer.linear_from_reference(U[lo:hi])
    else:
        params["w1"] = torch.tensor(W1[lo:hi], dtype=torch.float32).transpose(1, 2).contiguous().bfloat16().cuda()
        params["w2"] = torch.tensor(W2[lo:hi], dtype=torch.float32).transpose(1, 2).contiguous().bfloat16().cuda()
    xt = torch.tensor(x[rank], dtype=torch.float32).bfloat16().cuda()
    yt = torch.tensor(y[rank], dtype=torch.float32).bfloat16().cuda()
    first = None
    for it in range(steps):  # the second step re-uses every buffer (graph replay from then on)
        layer.step(xt, yt, params)
        if steps > 2:
            cur = [layer.losses, layer.dwg, layer.dw1] + ([layer.dw2] if f else []) + ([layer.dx] if c["need_dx"] else [])
            if first is None:
                first = [t.clone() for t in cur]
            else:
                for a, b in zip(first, cur):
                    assert torch.equal(a, b), f"rank {rank}: step {it} differs from step 0 (non-deterministic)"
    layer.status()
    torch.cuda.synchronize()

    def gather(t):
        if shared:  # gloo: CPU tensors
            t = t.contiguous().cpu()
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t.contiguous())
        return [o.cpu() for o in out]

    losses = gather(layer.losses)
    dwg = gather(layer.dwg)
    dw1 = gather(layer.dw1)
    dw2 = gather(layer.dw2) if f else None
    dx = gather(layer.dx) if c["need_dx"] else None
    idx = gather(torch.from_numpy(layer.read(ops.R_IDX, (1, S, k))).cuda())
    kept = gather(torch.from_numpy(layer.read(ops.R_KEPT, (1, S, k))).cuda())
    a2a = layer.a2a_bytes()
    if rank == 0:
        pen = np.stack([ops.penalty_weights(c_hat[i]) for i in range(P)])
        o = oracle.orc().layer_step(x, y, gates, U=U, W1=W1, W2=W2, k=k, cap_mode=c["cap"], cf=c.get("cf", 1.25), c_hat=c_hat,
                                    aux_kind=c["kind"], penalties=pen, act=1, want_dx=c["need_dx"])
        gi = np.concatenate([t.numpy() for t in idx])
        mism = int((gi != o["expert"]).sum())
        assert mism <= max(1, gi.size // 2000), f"routing mismatches {mism}"
        if mism == 0:
            assert np.array_equal(np.concatenate([t.numpy() for t in kept]), o["kept"])
        task = sum(float(t[0]) for t in losses)
        aux = sum(float(t[1]) for t in losses)
        assert abs(task - o["task_loss"]) <= 2e-2 * abs(o["task_loss"]), (task, o["task_loss"])
        assert abs(aux - o["aux_loss"]) <= 1e-3 * abs(o["aux_loss"]), (aux, o["aux_loss"])
        g = np.stack([t.numpy()[0, :N, :].T for t in dwg])
        assert rel(g, o["gate_grads"]) < 2e-2, rel(g, o["gate_grads"])
        w1 = np.concatenate([t.float().numpy() for t in dw1]).transpose(0, 2, 1)
        if f == 0:
            assert rel(w1, o["grad_u"]) < 2e-2, rel(w1, o["grad_u"])
        else:
            assert rel(w1, o["grad_w1"]) < 2e-2, rel(w1, o["grad_w1"])
            w2 = np.concatenate([t.float().numpy() for t in dw2]).transpose(0, 2, 1)
            assert rel(w2, o["grad_w2"]) < 2e-2, rel(w2, o["grad_w2"])
        if dx is not None:
            gx = np.stack([t.float().numpy() for t in dx])
            assert rel(gx, o["dx"]) < 2e-2, rel(gx, o["dx"])
        print(f"EP_PARITY_OK case={case} world={world} devices={min(ndev, world)} "
              f"bootstrap={'store' if shared else 'nccl'} steps={steps} task={task:.6f} "
              f"oracle={o['task_loss']:.6f} aux={aux:.6f} a2a_bytes_rank0={a2a} routing_mismatch={mism}",
              flush=True)
    dist.barrier()
    del layer  # teardown barrier: every rank unmaps its peers before any workspace is freed
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
