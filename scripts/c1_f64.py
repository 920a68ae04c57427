#!/usr/bin/env python
"""BASELINE config 1 (the reference's CPU layer: d=512, 8 experts, top-2, 4096 tokens, RE-1 [2,2] topology,
topo loss + proportional capacity 1.25) in the reference's own precision on the device (tamoe_layer_step_f64).
Prints one JSON line.  The comparison with the reference's own train() (compiled from its sources) is test
infrastructure and lives in tests/test_gpu_layer_f64.py::test_c1_trajectory_vs_reference_train.

  python scripts/c1_f64.py [--reps 20]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    from paper_2302_09915_b200 import ops
    P, S, d, dout, N, k = 4, 1024, 512, 512, 8, 2
    rng = np.random.default_rng(0)
    x = rng.normal(size=(P, S, d))
    y = rng.normal(size=(P, S, dout)) * 0.5
    gates = rng.normal(size=(P, d, N)) * 0.05
    U = rng.normal(size=(N, d, dout)) / np.sqrt(d)
    beta = np.array([[0.1 if i == j else (1.0 if i // 2 == j // 2 else 4.0) for j in range(P)] for i in range(P)])
    c_hat = ops.target_closed_form(beta, N, k, S)
    pen = np.stack([ops.penalty_weights(c_hat[i]) for i in range(P)])
    pol = ops.CapacityPolicy(ops.CapacityMode.local_proportional, 1.25)
    dev = torch.device("cuda", 0)
    xt, yt, gt, ut = (torch.tensor(a, dtype=torch.float64, device=dev) for a in (x, y, gates, U))
    router = None
    for _ in range(3):
        o = ops.layer_step_f64(xt, yt, gt, ut, k, pol, c_hat, 1, 1.0, pen, router)
        router = o["router"]
    torch.cuda.synchronize()
    times = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        o = ops.layer_step_f64(xt, yt, gt, ut, k, pol, c_hat, 1, 1.0, pen, router)
        times.append(time.perf_counter() - t0)  # the step synchronises (losses returned to the host)
    gpu_ms = float(np.median(times) * 1e3)
    line = {"config": "C1: d=512 d_out=512 N=8 top-2 P=4 x S=1024 fp64 linear experts, topo loss, proportional cf 1.25",
            "gpu_step_ms": gpu_ms, "gpu_tokens_per_s": P * S / (gpu_ms / 1e3),
            "task_loss": o["task_loss"], "aux_loss": o["aux_loss"]}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
