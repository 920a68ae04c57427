"""Generate tests/golden/*.npz from the reference compiled from its own sources
(oracle/_ref/libtadref.so, built by `make ref` in the builder container).

The fixtures travel with the repo so GPU-box tests can check parity without
/root/reference.  Re-run: python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def re1_beta():
    return np.array([[0.1 if i == j else (1.0 if i // 2 == j // 2 else 4.0) for j in range(4)] for i in range(4)])


def main():
    R = oracle.ref()
    # ---- routing: logits -> softmax_rows -> topk_route, every capacity mode, k in {1,2}
    rng = np.random.default_rng(2302)
    cases = {}
    for mode in range(4):
        for k in (1, 2):
            P, S, N = 4, 48, 8
            logits = rng.normal(size=(P, S, N)).astype(np.float32).astype(np.float64)
            logits[:, 7] = logits[:, 6]
            probs = np.stack([R.softmax_rows(l) for l in logits])
            c_hat = R.target_closed_form(re1_beta(), N, k, S)
            r = R.topk_route(probs, k, mode, 1.25, c_hat)
            tag = f"route_m{mode}_k{k}"
            cases[tag + "_logits"] = logits
            cases[tag + "_probs"] = probs
            cases[tag + "_c_hat"] = c_hat
            for key, v in r.items():
                cases[f"{tag}_{key}"] = v
    np.savez_compressed(os.path.join(OUT, "routing.npz"), **cases)

    # ---- topology inputs
    topo = {}
    topo["re1_beta"] = re1_beta()
    topo["re1_c_hat_k1_S120"] = R.target_closed_form(re1_beta(), 4, 1, 120)
    topo["re1_c_hat_k2_S1024_N8"] = R.target_closed_form(re1_beta(), 8, 2, 1024)
    topo["re1_penalty_sum"] = R.penalty_weights(topo["re1_c_hat_k1_S120"][0], 0)
    topo["re1_penalty_softmax"] = R.penalty_weights(topo["re1_c_hat_k1_S120"][0], 1)
    vals = rng.uniform(0, 30, size=(20, 7))
    topo["lrr_values"] = vals
    topo["lrr_targets"] = np.array([int(v.sum()) + t for v, t in zip(vals, rng.integers(-3, 4, 20))])
    topo["lrr_out"] = np.stack([R.largest_remainder_round(v, t) for v, t in zip(vals, topo["lrr_targets"])])
    np.savez_compressed(os.path.join(OUT, "topology.npz"), **topo)

    # ---- layer: reference train() trajectory on the C1-like RE-1 parity shape (reduced)
    layer = {}
    P, S, d, dout, N, k = 4, 128, 64, 32, 8, 2
    x, y, _, _ = R.gen_synthetic(11, P, S, d, dout, N, k, noise_std=0.1, map_spread=0.5)
    gates = np.stack([0.01 * R.rng_normal(R.derive_seed(11, 2000 + i), d * N).reshape(d, N) for i in range(P)])
    U = np.stack([R.rng_normal(R.derive_seed(11, 3000 + e), d * dout).reshape(d, dout) / np.sqrt(d)
                  for e in range(N)])
    c_hat = R.target_closed_form(re1_beta(), N, k, S)
    for kind in (0, 1):
        for cap in (0, 3):
            if kind == 0 and cap == 3:
                continue  # reference withholds c_hat from balance routing -> ValidationError (trainer.cpp:250)
            rep = R.train(x, y, gates, U, kind=kind, cap_mode=cap, cf=1.25, c_hat=c_hat, lr=0.1, steps=3, k=k)
            tag = f"train_kind{kind}_cap{cap}"
            layer[tag + "_task_loss"] = rep["task_loss"]
            layer[tag + "_aux_loss"] = rep["aux_loss"]
            layer[tag + "_initial_dispatch"] = rep["initial_dispatch"]
    layer.update(x=x, y=y, gates=gates, U=U, c_hat=c_hat, dims=np.array([P, S, d, dout, N, k]))
    np.savez_compressed(os.path.join(OUT, "layer.npz"), **layer)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
