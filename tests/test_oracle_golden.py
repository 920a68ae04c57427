"""The C restatement reproduces the committed golden fixtures (generated from the
compiled reference by tests/golden/make_golden.py).  Runs without oracle/_ref."""
import os

import numpy as np
import pytest

import oracle

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def O():
    return oracle.orc()


def test_routing_fixtures(O):
    z = np.load(os.path.join(G, "routing.npz"))
    for mode in range(4):
        for k in (1, 2):
            tag = f"route_m{mode}_k{k}"
            probs = np.stack([O.softmax_rows(l) for l in z[tag + "_logits"]])
            assert np.array_equal(probs, z[tag + "_probs"])
            r = O.topk_route(probs, k, mode, 1.25, z[tag + "_c_hat"])
            for key in ("expert", "gate", "score", "kept", "counts", "dropped", "mean_probs"):
                assert np.array_equal(r[key], z[f"{tag}_{key}"]), (tag, key)


def test_topology_fixtures(O):
    z = np.load(os.path.join(G, "topology.npz"))
    assert np.array_equal(O.target_closed_form(z["re1_beta"], 4, 1, 120), z["re1_c_hat_k1_S120"])
    assert np.array_equal(O.target_closed_form(z["re1_beta"], 8, 2, 1024), z["re1_c_hat_k2_S1024_N8"])
    assert np.array_equal(O.penalty_weights(z["re1_c_hat_k1_S120"][0], 0), z["re1_penalty_sum"])
    assert np.array_equal(O.penalty_weights(z["re1_c_hat_k1_S120"][0], 1), z["re1_penalty_softmax"])
    for v, t, o in zip(z["lrr_values"], z["lrr_targets"], z["lrr_out"]):
        assert np.array_equal(O.largest_remainder_round(v, t), o)


@pytest.mark.parametrize("kind,cap", [(0, 0), (1, 0), (1, 3)])
def test_layer_trajectory_fixture(O, kind, cap):
    z = np.load(os.path.join(G, "layer.npz"))
    P, S, d, dout, N, k = (int(v) for v in z["dims"])
    x, y, g, u, c_hat = z["x"], z["y"], z["gates"].copy(), z["U"].copy(), z["c_hat"]
    pen = np.stack([O.penalty_weights(c_hat[i]) for i in range(P)])
    tag = f"train_kind{kind}_cap{cap}"
    for s in range(len(z[tag + "_task_loss"])):
        o = O.layer_step(x, y, g, U=u, k=k, cap_mode=cap, cf=1.25, c_hat=c_hat, aux_kind=kind, penalties=pen)
        assert o["task_loss"] == z[tag + "_task_loss"][s]
        assert o["aux_loss"] == z[tag + "_aux_loss"][s]
        if s == 0:
            assert np.array_equal(o["counts"].astype(float), z[tag + "_initial_dispatch"])
        g -= 0.1 * o["gate_grads"]
        u -= 0.1 * o["grad_u"]
