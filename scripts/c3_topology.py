#!/usr/bin/env python
"""BASELINE C3 / C5: topology-aware vs even dispatch on a MEASURED
P2P matrix, plus the alpha-beta model (comm_cost.cpp:24-55) validated against the measured exchange.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
      scripts/c3_topology.py [--tokens 16384[,32768,...]] [--levels 8] [--cross-throttle 1] [--out file.jsonl]

1. NVLink sweep (`tamoe_p2p_sweep`, every ordered pair incl. self, 1-128 MB x 5 reps) -> TransferSample rows
   -> fit_profile -> fill_partial_profile(tree) -> smooth_profile -> closed form c_hat (Eq. 8).
   `--levels 2,2 --cross-throttle 4` is the C5 emulation: `tamoe_set_link_emulation(group, 4)` really
   throttles every cross-group link -- each payload store to a peer in another group (the sweep's copies,
   dispatch, expert-output return, dO, dX return) is issued 4 times, so the link delivers 1/4 of its
   bandwidth -- and the sweep MEASURES those slow links; c_hat comes from the measured profile.
   (`--posthoc` instead scales the cross-group samples before fitting and leaves the transfers alone.)
   `--tokens` takes a comma list (C5 sweeps 4k-64k tokens/GPU); one JSON line per size.
2. The C2 layer (d=1024, ffn=4096, 64 experts, top-1, GELU, bf16, dX on) with expert parallelism, twice:
   even      : local capacity (cf 1.25), balance loss, no gate bias;
   topo-aware: proportional capacity from c_hat (cf 1.25), topo loss.
   Both runs route through a per-rank gate bias on a constant input feature, calibrated on the actual
   gate logits so the top-1 routing shares match the target (c_hat row / uniform): the routing a
   converged topo / balance loss produces, with (almost) no capacity drops in
   either run so the comparison moves the same work.
3. Per mode: tokens/s, step time, dispatch phase, off-rank bytes, dropped slots, and the alpha-beta
   prediction of the dispatch exchange for the dispatch matrix that actually happened.
Rank 0 prints one JSON line (and writes --out).
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", default="16384")
    ap.add_argument("--posthoc", action="store_true", help="scale cross-group samples instead of throttling links")
    ap.add_argument("--levels", default=None, help="symmetric tree, e.g. 8 or 2,4 (default: one switch)")
    ap.add_argument("--cross-throttle", type=float, default=1.0)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--samples-csv", default=None)
    args = ap.parse_args()

    import torch
    import torch.distributed as dist
    from paper_2302_09915_b200 import ops
    from paper_2302_09915_b200.layer import LayerConfig, TAMoELayer, LOSS_BALANCE, LOSS_TOPO, ACT_GELU, \
        nccl_unique_id

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    ndev = torch.cuda.device_count()
    # more ranks than GPUs (e.g. C5's 2 x 4 tree on a 4-GPU lease): the NCCL-free bootstrap over gloo, ranks
    # sharing GPUs round-robin -- the pipeline runs end to end, the timings are not per-GPU numbers
    shared = ndev < world
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    cdev = torch.device("cpu") if shared else dev  # device of the torch.distributed collectives

    def bcast_id():
        if shared:
            return None  # TAMoELayer all-gathers the workspace handles over the default (gloo) group
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    levels = [int(v) for v in args.levels.split(",")] if args.levels else [world]
    assert int(np.prod(levels)) == world, "levels must multiply to the world size"
    N, k, d, f = 64, 1, 1024, 4096
    token_list = [int(v) for v in args.tokens.split(",")]
    group_size = levels[-1]
    emulate = args.cross_throttle != 1.0 and not args.posthoc
    if emulate:
        ops.set_link_emulation(group_size, int(round(args.cross_throttle)))

    # ---- 1. measured profile -> c_hat
    sizes = (1.0, 4.0, 16.0, 64.0, 128.0)  # >= L2 at the top: the self link is a real HBM copy
    if shared:
        samples = ops.p2p_sweep_store(world, rank, sizes, reps=args.reps, warmup=2)
    else:
        samples = ops.p2p_sweep(bcast_id(), world, rank, sizes, reps=args.reps, warmup=2)
    post = args.cross_throttle if args.posthoc else 1.0
    thr = [(i, j, mb, us * (post if (i // group_size != j // group_size) else 1.0))
           for (i, j, mb, us) in samples]
    if rank == 0 and args.samples_csv:
        ops.save_samples_csv(args.samples_csv, thr)
    alpha, beta = ops.fit_profile(thr, world)
    alpha, beta = ops.fill_partial_profile(alpha, beta, levels)
    for S in token_list:
        run_size(args, ops, torch, dist, dev, rank, world, levels, emulate, sizes, alpha, beta, bcast_id,
                 N, k, S, d, f, LayerConfig, TAMoELayer, LOSS_BALANCE, LOSS_TOPO, ACT_GELU, cdev, shared)
    dist.barrier()
    dist.destroy_process_group()


def run_size(args, ops, torch, dist, dev, rank, world, levels, emulate, sizes, alpha, beta, bcast_id,
             N, k, S, d, f, LayerConfig, TAMoELayer, LOSS_BALANCE, LOSS_TOPO, ACT_GELU, cdev, shared):
    c_topo, a_hat, b_hat = ops.solve_target_tree(levels, alpha, beta, N, k, S)
    c_even = ops.target_closed_form(np.ones((world, world)), N, k, S)

    # ---- 2. the layer, even vs topology-aware
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    x = torch.randn(S, d, generator=g, device=dev)
    x[:, d - 1] = 1.0  # constant feature carrying the per-rank gate bias
    x = x.bfloat16()
    y = (torch.randn(S, d, generator=g, device=dev) * 0.5).bfloat16()
    def calibrate_bias(wg_rows, target, iters=200):
        """Per-expert logit bias such that argmax(x.Wg^T + bias) hits `target` shares on this rank's tokens
        (damped multiplicative updates; the bias is applied in bf16 exactly as the gate will see it)."""
        base = (x[:, :d - 1].float() @ wg_rows[:, :d - 1].float().T)  # [S x N] logits without the bias column
        tgt = torch.tensor(target / target.sum(), dtype=torch.float32, device=dev)
        b = torch.log(tgt)
        for _ in range(iters):
            frac = torch.bincount((base + b.bfloat16().float()).argmax(1), minlength=N).float() / base.shape[0]
            b = b + torch.clamp(torch.log(tgt + 1e-4) - torch.log(frac + 1e-4), -0.25, 0.25) * 0.5
        frac = torch.bincount((base + b.bfloat16().float()).argmax(1), minlength=N).float() / base.shape[0]
        calib_err[0] = max(calib_err[0], float((frac - tgt).abs().max() / tgt.max()))
        return b

    calib_err = [0.0]

    results = {}
    for mode in ("even", "topo"):
        topo = mode == "topo"
        c_hat = c_topo if topo else c_even
        cfg = LayerConfig(P=1, S=S, d=d, d_out=d, N=N, k=k, f=f, act=ACT_GELU, cap_mode=3 if topo else 2,
                          capacity_factor=1.25, aux_kind=LOSS_TOPO if topo else LOSS_BALANCE, need_dx=True,
                          world_size=world, rank=rank)
        layer = TAMoELayer(cfg, c_hat, nccl_id=bcast_id())
        params = layer.init_params(seed=1 + rank)
        params["wg"][0, :N, d - 1] = calibrate_bias(params["wg"][0, :N], c_hat[rank]).bfloat16()
        for _ in range(args.warmup):
            layer.step(x, y, params)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            layer.step(x, y, params)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        layer.enable_timing(True)
        for _ in range(5):
            layer.step(x, y, params)
        torch.cuda.synchronize()
        phases, _ = layer.timing()
        layer.enable_timing(False)
        nbytes = layer.a2a_bytes()
        counts = layer.read(ops.R_COUNTS, (1, N)).astype(np.float64)
        dropped = layer.read(ops.R_DROPPED, (1, N)).sum()
        allc = torch.tensor(counts, device=cdev)
        gathered = [torch.zeros_like(allc) for _ in range(world)]
        dist.all_gather(gathered, allc)
        cmat = torch.cat(gathered, 0).cpu().numpy()  # [P x N] kept tokens: the dispatch matrix that happened
        pred = ops.exchange_cost(a_hat, b_hat, cmat, d=d, b=2, extra_alpha_rounds=1)
        disp = phases.get("a2a_dispatch", 0.0) * 1e3
        results[mode] = {
            "tokens_per_s": world * S / (ms / 1e3), "ms_per_step": ms,
            "dispatch_phase_us": disp, "combine_phase_us": phases.get("combine_loss", 0.0) * 1e3,
            "offrank_dispatch_bytes_rank0": nbytes[0],
            "local_fraction_rank0": float(counts[0, rank * (N // world):(rank + 1) * (N // world)].sum() / max(counts.sum(), 1)),
            "dropped_slots_rank0": int(dropped), "kept_slots_rank0": int(counts.sum()),
            "alpha_beta_predicted_exchange_us": pred["total_estimate_us"],
            "alpha_beta_bottleneck_us": pred["bottleneck_us"],
            "losses": layer.losses.cpu().tolist(),
            "routing_share_max_rel_err_vs_target": calib_err[0],
        }
        dist.barrier()  # nobody frees its peer-mapped workspace while a peer may still touch it
        del layer
        torch.cuda.synchronize()
        dist.barrier()

    if rank == 0:
        out = {"config": {"workload": "C5 emulation" if args.cross_throttle != 1.0 else "C3",
                          "ranks": world, "gpus": min(world, torch.cuda.device_count()),
                          "ranks_share_gpus": shared, "tokens_per_rank": S, "levels": levels, "cross_throttle": args.cross_throttle,
                          "throttle_mode": ("links throttled (every cross-group payload store issued "
                                            f"{int(round(args.cross_throttle))}x), profile measured on them")
                          if emulate else ("post-hoc sample scaling" if args.cross_throttle != 1.0 else "none"),
                          "layer": "C2: d=1024 ffn=4096 64 experts top-1 bf16 GELU dX on", "capacity_factor": 1.25},
               "profile": {"sizes_mb": list(sizes), "reps": args.reps,
                           "alpha_us": alpha.tolist(), "beta_us_per_mb": beta.tolist(),
                           "beta_hat": b_hat.tolist(), "c_hat_row0": c_topo[0].tolist()},
               "even": results["even"], "topo": results["topo"],
               "speedup_topo_vs_even": results["even"]["ms_per_step"] / results["topo"]["ms_per_step"]}
        line = json.dumps(out)
        print(line, flush=True)
        if args.out:
            with open(args.out, "a") as fh:
                fh.write(line + "\n")
    dist.barrier()


if __name__ == "__main__":
    main()
