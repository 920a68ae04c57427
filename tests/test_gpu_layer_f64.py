"""BASELINE config 1 in the reference's own precision on the device: tamoe_layer_step_f64 (fp64, linear experts,
the inline step of train(), trainer.cpp:246-356) against
  * the reference itself (train(), compiled from its sources into oracle/_ref): per-step task / aux loss
    trajectories with SGD in between (the gradients feed every later step), and
  * the C restatement (oracle/tamoe_oracle.c, layer_step): routing arrays, y_hat, gate and expert gradients.
Compulsory quota routing (aux kind 2, apply_compulsory_quota trainer.cpp:121-169) is pinned by the trajectories.

The device follows the reference's summation order without FMA, so everything downstream of the softmax agrees
to the last few ulp (CUDA's exp may differ from glibc's by one ulp): tolerance rel 1e-12, far inside the north
star's fp32 rel 1e-4.  Routing (expert indices, kept flags, counts) is compared bit for bit."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-12


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def re1_beta(P):
    return np.array([[0.1 if i == j else (1.0 if i // 2 == j // 2 else 4.0) for j in range(P)] for i in range(P)])


def inputs(P, S, d, dout, N, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(P, S, d))
    y = rng.normal(size=(P, S, dout)) * 0.5
    gates = rng.normal(size=(P, d, N)) * 0.05
    U = rng.normal(size=(N, d, dout)) / np.sqrt(d)
    return x, y, gates, U


def run(P, S, d, dout, N, k, cap, kind, cf=1.25, seed=0, sparse_x=False):
    from paper_2302_09915_b200 import ops
    x, y, gates, U = inputs(P, S, d, dout, N, seed)
    if sparse_x:  # the reference skips x_r == 0 terms (trainer.cpp:286, 312)
        x[:, :, ::3] = 0.0
    c_hat = ops.target_closed_form(re1_beta(P), N, k, S) if P > 1 else np.full((1, N), float(S * k) / N)
    pen = np.stack([ops.penalty_weights(c_hat[i]) for i in range(P)])
    pol = ops.CapacityPolicy(ops.CapacityMode(cap), cf)
    got = ops.layer_step_f64(x, y, gates, U, k, pol, c_hat if (cap == 3 or kind == 2) else None, kind, 1.0,
                             pen if kind == 1 else None)
    o = oracle.orc().layer_step(x, y, gates, U=U, k=k, cap_mode=cap, cf=cf, c_hat=c_hat, aux_kind=kind,
                                penalties=pen, act=0, want_dx=False)
    return got, o, (x, y, gates, U, c_hat, pen)


def check(got, o, P, S, N, k):
    from paper_2302_09915_b200 import ops
    r = got["router"]
    assert np.array_equal(r.read(ops.R_IDX), o["expert"])
    assert np.array_equal(r.read(ops.R_KEPT), o["kept"])
    assert np.array_equal(r.read(ops.R_COUNTS), o["counts"])
    assert rel(got["probs"].cpu().numpy(), o["probs"]) < TOL
    assert got["task_loss"] == pytest.approx(o["task_loss"], rel=TOL)
    assert got["aux_loss"] == pytest.approx(o["aux_loss"], rel=TOL, abs=1e-300)
    assert rel(got["y_hat"].cpu().numpy(), o["y_hat"]) < TOL
    assert rel(got["gate_grads"].cpu().numpy(), o["gate_grads"]) < TOL
    assert rel(got["expert_grads"].cpu().numpy(), o["grad_u"]) < TOL


def test_c1_reference_config_vs_restatement():
    """BASELINE C1: d = d_out = 512, 8 experts, top-2, 4096 tokens (P=4 x S=1024, RE-1 [2,2] topology),
    topo loss with proportional capacity 1.25."""
    P, S, d, dout, N, k = 4, 1024, 512, 512, 8, 2
    got, o, _ = run(P, S, d, dout, N, k, cap=3, kind=1)
    check(got, o, P, S, N, k)
    assert o["kept"].sum() < P * S * k  # the capacity really drops picks at this shape


@pytest.mark.parametrize("P,S,d,dout,N,k,cap,kind,sparse", [
    (1, 300, 64, 48, 8, 1, 0, 0, False),    # top-1, no capacity, balance, ragged S
    (2, 257, 96, 80, 4, 2, 2, 1, True),     # local capacity, topo, zero inputs skipped
    (4, 128, 64, 64, 16, 4, 1, 0, False),   # top-4, global capacity
    (2, 64, 32, 32, 8, 8, 3, 1, False),     # k = N = 8 (every expert picked)
])
def test_layer_step_f64_cases(P, S, d, dout, N, k, cap, kind, sparse):
    got, o, _ = run(P, S, d, dout, N, k, cap, kind, sparse_x=sparse)
    check(got, o, P, S, N, k)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("kind,cap,k", [(1, 3, 2), (0, 0, 2), (0, 2, 1), (2, 2, 1)])
def test_c1_trajectory_vs_reference_train(kind, cap, k):
    """The reference's own train() (compiled from its sources) vs train_f64 on the device, C1 shape: the SGD
    updates make every step depend on all of the previous step's gradients."""
    from paper_2302_09915_b200 import ops
    P, S, d, dout, N, steps, lr = 4, 1024, 512, 512, 8, 3, 0.05
    x, y, gates, U = inputs(P, S, d, dout, N, seed=5)
    c_hat = ops.target_closed_form(re1_beta(P), N, k, S)
    pen = np.stack([ops.penalty_weights(c_hat[i]) for i in range(P)])
    ref = oracle.ref().train(x, y, gates, U, kind=kind, cap_mode=cap, cf=1.25,
                             c_hat=c_hat if kind != 0 else None, lr=lr, steps=steps, k=k)
    got = ops.train_f64(x, y, gates, U, k, steps, lr, ops.CapacityPolicy(ops.CapacityMode(cap), 1.25),
                        c_hat if kind != 0 else None, kind, 1.0, pen if kind == 1 else None)
    np.testing.assert_allclose(got["task_loss"], ref["task_loss"], rtol=1e-11)
    np.testing.assert_allclose(got["aux_loss"], ref["aux_loss"], rtol=1e-11)
    assert got["task_loss"][-1] < got["task_loss"][0]


def test_layer_step_f64_validation():
    from paper_2302_09915_b200 import ops, _lib
    x, y, gates, U = inputs(1, 32, 16, 16, 4)
    with pytest.raises(_lib.ValidationError):
        ops.layer_step_f64(x, y, gates, U, 1, aux_kind=2)  # compulsory without a target pattern
    with pytest.raises(_lib.ValidationError):
        ops.layer_step_f64(x, y, gates, U, 2, c_hat=np.ones((1, 4)), aux_kind=2)  # compulsory is top-1 only
    with pytest.raises(_lib.ValidationError):
        ops.layer_step_f64(x, y, gates, U, 1, aux_kind=3)
    with pytest.raises(_lib.ValidationError):
        ops.layer_step_f64(x, y, gates, U, 1, aux_kind=1)  # topo without penalties
    bad = gates.copy()
    bad[0, 0, 0] = np.inf
    with pytest.raises(_lib.ValidationError, match="non-finite"):
        ops.layer_step_f64(x, y, bad, U, 1)
    with pytest.raises(_lib.ValidationError):
        ops.layer_step_f64(x, y, gates, U, 5)  # k > N
