"""GPU-backed train() against the reference's own train() (trainer.cpp:183-452, compiled
from its sources into oracle/_ref) on identical bf16-representable data and initial weights: the per-step
task / aux loss trajectories, dropped rates and dispatch matrices of the report.

Tolerance: the device computes in bf16 with fp32 accumulation and fp32 master weights, the reference in fp64,
so trajectories agree to bf16 level (task loss rel 3e-2 per step, aux loss rel 5e-2), not bitwise."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")]


def bf(a):
    return torch.tensor(np.asarray(a), dtype=torch.float32).bfloat16().double().numpy()


def setup(P, S, d, dout, N, k, seed=3):
    R = oracle.ref()
    x, y, _, _ = R.gen_synthetic(seed, P, S, d, dout, N=N, k=k, clusters=4)
    rng = np.random.default_rng(seed)
    gates = bf(rng.normal(size=(P, d, N)) * 0.01)
    experts = bf(rng.normal(size=(N, d, dout)) / np.sqrt(d))
    return R, bf(x), bf(y), gates, experts


@pytest.mark.parametrize("kind,cap,switch,k", [(0, 0, None, 2), (1, 3, None, 2), (1, 2, 3, 2), (2, 0, None, 1)])
def test_train_matches_reference_trajectory(kind, cap, switch, k):
    from paper_2302_09915_b200 import ops
    from paper_2302_09915_b200.train import TrainConfig, LossKind, train
    P, S, d, dout, N, steps, lr = 4, 256, 256, 128, 8, 12, 0.05
    R, x, y, gates, experts = setup(P, S, d, dout, N, k)
    beta = np.array([[0.1 if i == j else (1.0 if i // 2 == j // 2 else 4.0) for j in range(P)] for i in range(P)])
    c_hat = ops.target_closed_form(beta, N, k, S) if kind in (1, 2) else None
    ref = R.train(x, y, gates, experts, kind=kind, cap_mode=cap, cf=1.25, c_hat=c_hat, lr=lr, steps=steps, k=k,
                  switch_step=switch)
    cfg = TrainConfig(P=P, S=S, d=d, d_out=dout, N=N, k=k, lr=lr, steps=steps, switch_step=switch,
                      capacity=ops.CapacityPolicy(ops.CapacityMode(cap), 1.25), report_window=100,
                      alpha_hat=np.zeros((P, P)), beta_hat=beta)
    rep = train(cfg, x, y, gates, experts, kind=LossKind(kind), c_hat=c_hat)
    np.testing.assert_allclose(rep.task_loss, ref["task_loss"], rtol=3e-2)
    np.testing.assert_allclose(rep.aux_loss, ref["aux_loss"], rtol=5e-2, atol=1e-6)
    np.testing.assert_allclose(rep.dropped_rate, ref["dropped_rate"], atol=0.02)
    np.testing.assert_allclose(rep.initial_dispatch, ref["initial_dispatch"], atol=0.01 * S * k)
    np.testing.assert_allclose(rep.final_dispatch.sum(1), ref["final_dispatch"].sum(1), rtol=0.02)
    assert rep.task_loss[-1] < rep.task_loss[0]  # it trains
    # report bookkeeping (trainer.cpp:374-452)
    assert rep.final_task_loss == pytest.approx(rep.task_loss.mean())  # window = min(100, steps)
    pay = ops.device_payload_tokens(rep.initial_dispatch)
    assert rep.comm_us[0] == pytest.approx((beta * pay * d * 4 / 1e6).max() + (0 if cap in (0, 2) else 0.0))
    if c_hat is not None:
        assert len(rep.tv_rows) == P and 0.0 <= rep.tv_final_mean <= 1.0


def test_train_validation():
    from paper_2302_09915_b200 import ops
    from paper_2302_09915_b200.train import TrainConfig, LossKind, train
    P, S, d, dout, N, k = 2, 128, 256, 128, 4, 1
    _, x, y, gates, experts = setup(P, S, d, dout, N, k)
    cfg = TrainConfig(P=P, S=S, d=d, d_out=dout, N=N, k=k, steps=1)
    with pytest.raises(ops.ValidationError):  # topo needs c_hat (trainer.cpp:189-190)
        train(cfg, x, y, gates, experts, kind=LossKind.topo)
    with pytest.raises(ops.ValidationError):  # balance withholds c_hat: proportional capacity throws
        train(TrainConfig(P=P, S=S, d=d, d_out=dout, N=N, k=k, steps=1,
                          capacity=ops.CapacityPolicy(ops.CapacityMode.local_proportional, 1.25)),
              x, y, gates, experts, kind=LossKind.balance, c_hat=np.ones((P, N)))
