"""Whole-layer parity: the device step (gate, routing, experts, combine, MSE, aux loss,
backward) against the oracle's restatement of trainer.cpp:371-482 on identical
(bf16-representable) inputs.  Tolerance: bf16 rel 2e-2 (north star) on values and
gradients (relative L2); routing bit-exact except audited near-ties."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

TOL = 2e-2


def bf(a):
    return torch.tensor(np.asarray(a), dtype=torch.float32).bfloat16().double().numpy()


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def re1_beta(P):
    return np.array([[0.1 if i == j else (1.0 if i // 2 == j // 2 else 4.0) for j in range(P)] for i in range(P)])


def run_case(P, S, d, dout, N, k, f, cap, kind, need_dx, seed=0, cf=1.25, hot_expert=None):
    from paper_2302_09915_b200 import ops
    from paper_2302_09915_b200.layer import LayerConfig, TAMoELayer
    O = oracle.orc()
    rng = np.random.default_rng(seed)
    x = bf(rng.normal(size=(P, S, d)))
    y = bf(rng.normal(size=(P, S, dout)) * 0.5)
    gates = bf(rng.normal(size=(P, d, N)) * 0.05)
    if hot_expert is not None:  # every token's top choice is `hot_expert` (extreme imbalance)
        x[:, :, 0] = 1.0
        gates[:, 0, :] = 0.0
        gates[:, 0, hot_expert] = 8.0
    if f == 0:
        U = bf(rng.normal(size=(N, d, dout)) / np.sqrt(d))
        W1 = W2 = None
    else:
        U = None
        W1 = bf(rng.normal(size=(N, d, f)) / np.sqrt(d))
        W2 = bf(rng.normal(size=(N, f, dout)) / np.sqrt(f))
    c_hat = ops.target_closed_form(re1_beta(P), N, k, S) if P > 1 else rng.uniform(0.5, 3.0, size=(1, N))
    pen = np.stack([ops.penalty_weights(c_hat[i]) for i in range(P)])

    cfg = LayerConfig(P=P, S=S, d=d, d_out=dout, N=N, k=k, f=f, act=1, cap_mode=cap, capacity_factor=cf,
                      aux_kind=kind, need_dx=need_dx)
    layer = TAMoELayer(cfg, c_hat)
    params = dict(wg=TAMoELayer.gates_from_reference(gates, cfg.n_pad))
    if f == 0:
        params["w1"] = TAMoELayer.linear_from_reference(U)
    else:
        params["w1"] = torch.tensor(W1, dtype=torch.float32).transpose(1, 2).contiguous().bfloat16().cuda()
        params["w2"] = torch.tensor(W2, dtype=torch.float32).transpose(1, 2).contiguous().bfloat16().cuda()
    xt = torch.tensor(x.reshape(P * S, d), dtype=torch.float32).bfloat16().cuda()
    yt = torch.tensor(y.reshape(P * S, dout), dtype=torch.float32).bfloat16().cuda()
    yh = torch.zeros(P * S, dout, dtype=torch.bfloat16, device="cuda")
    layer.step(xt, yt, params, y_hat=yh)
    torch.cuda.synchronize()
    o = O.layer_step(x, y, gates, U=U, W1=W1, W2=W2, k=k, cap_mode=cap, cf=cf, c_hat=c_hat, aux_kind=kind,
                     penalties=pen, act=1, want_dx=need_dx)
    return layer, o, dict(yh=yh, x=x, args=(xt, yt, params, yh))


def check(layer, o, extra, P, S, N, k, f, need_dx):
    from paper_2302_09915_b200 import ops
    idx = layer.read(ops.R_IDX, (P, S, k))
    mism = np.argwhere(idx != o["expert"])
    assert len(mism) <= max(1, idx.size // 2000), f"{len(mism)} routing mismatches"
    for (i, s, j) in mism:
        pr = np.sort(o["probs"][i, s])[::-1]
        assert abs(pr[j] - pr[j + 1]) < 1e-5, (i, s, j, pr[:3])
    if len(mism) == 0:
        assert np.array_equal(layer.read(ops.R_KEPT, (P, S, k)), o["kept"])
        assert np.array_equal(layer.read(ops.R_COUNTS, (P, N)), o["counts"])
    losses = layer.losses.cpu().numpy()
    assert abs(losses[0] - o["task_loss"]) <= TOL * abs(o["task_loss"])
    assert abs(losses[1] - o["aux_loss"]) <= 1e-3 * abs(o["aux_loss"]) + 1e-12
    assert rel(extra["yh"].float().cpu().numpy().reshape(o["y_hat"].shape), o["y_hat"]) < TOL
    dwg = layer.dwg.cpu().numpy()[:, :N, :].transpose(0, 2, 1)
    assert rel(dwg, o["gate_grads"]) < TOL
    if f == 0:
        assert rel(layer.dw1.float().cpu().numpy().transpose(0, 2, 1), o["grad_u"]) < TOL
    else:
        assert rel(layer.dw1.float().cpu().numpy().transpose(0, 2, 1), o["grad_w1"]) < TOL
        assert rel(layer.dw2.float().cpu().numpy().transpose(0, 2, 1), o["grad_w2"]) < TOL
    if need_dx:
        assert rel(layer.dx.float().cpu().numpy().reshape(o["dx"].shape), o["dx"]) < TOL


@pytest.mark.parametrize("P,S,d,dout,N,k,f,cap,kind,need_dx", [
    (1, 512, 256, 128, 8, 1, 0, 0, 0, True),     # linear expert, top-1, no capacity
    (4, 128, 256, 256, 8, 2, 0, 3, 1, False),   # RE-1 style: topo loss + proportional capacity
    (2, 256, 256, 128, 4, 2, 0, 2, 1, True),    # local capacity
    (1, 384, 256, 128, 8, 2, 512, 0, 0, True),  # FFN expert (GELU), top-2
    (1, 1000, 512, 256, 16, 1, 256, 1, 1, True),  # FFN, global capacity, ragged S
    (2, 208, 256, 128, 16, 4, 256, 2, 1, True),   # top-4 (runtime-k combine / dX paths), local capacity, ragged
])
def test_layer_step_parity(P, S, d, dout, N, k, f, cap, kind, need_dx):
    layer, o, extra = run_case(P, S, d, dout, N, k, f, cap, kind, need_dx)
    check(layer, o, extra, P, S, N, k, f, need_dx)


def test_layer_c1_reference_config():
    """BASELINE config 1: d = d_out = 512, 8 experts, top-2, 4096 tokens (P=4 x S=1024, RE-1 [2,2]
    topology), linear experts, topo loss with proportional capacity 1.25."""
    P, S, d, dout, N, k = 4, 1024, 512, 512, 8, 2
    layer, o, extra = run_case(P, S, d, dout, N, k, 0, 3, 1, False)
    check(layer, o, extra, P, S, N, k, 0, False)


def test_layer_validation_errors():
    from paper_2302_09915_b200 import ops
    from paper_2302_09915_b200.layer import LayerConfig, TAMoELayer
    with pytest.raises(ops.ValidationError):  # reference: balance routing withholds c_hat (trainer.cpp:250)
        TAMoELayer(LayerConfig(P=1, S=128, d=256, d_out=128, N=8, cap_mode=3, aux_kind=0), np.ones((1, 8)))
    with pytest.raises(ops.ValidationError):
        TAMoELayer(LayerConfig(P=1, S=128, d=256, d_out=128, N=8, k=9))
    with pytest.raises(ops.ValidationError):
        TAMoELayer(LayerConfig(P=1, S=128, d=256, d_out=128, N=8, aux_kind=1), None)


def test_layer_c4_expert_shape_reduced():
    """BASELINE config 4 expert shape (d=4096, f=16384, top-2, capacity factor 1.25, local proportional
    capacities from a 2-level topology) reduced so the fp64 oracle fits and finishes: 4 experts (each
    2 x 4096 x 16384), P=2 logical processes x S=16 tokens."""
    P, S, d, dout, N, k, f = 2, 16, 4096, 4096, 4, 2, 16384
    layer, o, extra = run_case(P, S, d, dout, N, k, f, 3, 1, True, seed=4)
    check(layer, o, extra, P, S, N, k, f, True)


def test_layer_graph_replay_bitwise():
    """Steps after the first replay a captured CUDA graph of the whole step; they must reproduce the eager
    step bit for bit, also after a buffer pointer changes (re-capture) and when switching back (cache)."""
    P, S, d, dout, N, k, f = 1, 384, 256, 128, 8, 2, 512
    layer, o, extra = run_case(P, S, d, dout, N, k, f, 0, 1, True)
    snap = lambda: [layer.losses.cpu().clone(), layer.dwg.cpu().clone(), layer.dw1.float().cpu().clone(),
                    layer.dw2.float().cpu().clone(), layer.dx.float().cpu().clone(), extra["yh"].float().cpu().clone()]
    ref = snap()
    x, y, params, yh = extra["args"]
    for it in range(3):
        yh2 = yh if it != 1 else torch.zeros_like(yh)
        layer.step(x, y, params, y_hat=yh2)
        torch.cuda.synchronize()
        got = snap()
        got[5] = yh2.float().cpu()
        for a, b in zip(ref, got):
            assert torch.equal(a, b)


def compulsory_restated(probs, score, c_hat, S):
    """trainer.cpp:121-169 restated (test-only): quotas by LRR of the c_hat row share; tokens by (top-1 score
    desc, token asc) claim their best expert (probability desc, expert asc) with quota left."""
    P, _, N = probs.shape
    O = oracle.orc()
    out = np.zeros((P, S), np.int64)
    for i in range(P):
        share = c_hat[i] / c_hat[i].sum() * S
        quota = O.largest_remainder_round(share, S).astype(np.int64)
        order = sorted(range(S), key=lambda s: (-score[i, s], s))
        for s in order:
            for e in sorted(range(N), key=lambda e: (-probs[i, s, e], e)):
                if quota[e] > 0:
                    quota[e] -= 1
                    out[i, s] = e
                    break
    return out


def test_layer_compulsory_quota_routing():
    """Compulsory-quota ablation (aux kind 2): device claims == the restated greedy on the device's own
    probabilities (softmax of the stored logits in fp64); every token kept; counts equal the quotas."""
    from paper_2302_09915_b200 import ops
    from paper_2302_09915_b200.layer import LayerConfig, TAMoELayer
    P, S, d, dout, N = 2, 384, 256, 128, 8
    rng = np.random.default_rng(5)
    beta = np.array([[0.1, 4.0], [4.0, 0.1]])
    c_hat = ops.target_closed_form(beta, N, 1, S)
    cfg = LayerConfig(P=P, S=S, d=d, d_out=dout, N=N, k=1, f=0, act=0, cap_mode=0, aux_kind=2, need_dx=False)
    layer = TAMoELayer(cfg, c_hat)
    params = layer.init_params(seed=3, gate_std=0.05)
    x = torch.tensor(rng.normal(size=(P * S, d)), dtype=torch.float32).bfloat16().cuda()
    y = torch.tensor(rng.normal(size=(P * S, dout)), dtype=torch.float32).bfloat16().cuda()
    layer.step(x, y, params)
    torch.cuda.synchronize()
    logits = layer.read(ops.R_LOGITS, (P, S, N)).astype(np.float64)
    z = np.exp(logits - logits.max(-1, keepdims=True))
    probs = z / z.sum(-1, keepdims=True)
    score = probs.max(-1)
    want = compulsory_restated(probs, score, c_hat, S)
    got = layer.read(ops.R_IDX, (P, S, 1))[..., 0]
    mism = np.argwhere(got != want)
    assert len(mism) <= max(2, want.size // 500), f"{len(mism)} claim mismatches"
    assert np.all(layer.read(ops.R_KEPT, (P, S, 1)) == 1)
    O = oracle.orc()
    quotas = np.stack([O.largest_remainder_round(c_hat[i] / c_hat[i].sum() * S, S) for i in range(P)])
    np.testing.assert_array_equal(layer.read(ops.R_COUNTS, (P, N)), quotas)
    with pytest.raises(ops.ValidationError):  # top-1 only (trainer.cpp:124)
        TAMoELayer(LayerConfig(P=P, S=S, d=d, d_out=dout, N=N, k=2, aux_kind=2), c_hat)


def test_layer_graph_falls_back_when_buffers_change():
    """A caller handing new buffers every step would make every step a capture: after a few such misses the
    layer runs eagerly; results stay bit-identical."""
    P, S, d, dout, N, k, f = 1, 256, 256, 128, 8, 1, 256
    layer, o, extra = run_case(P, S, d, dout, N, k, f, 0, 1, True)
    x, y, params, yh = extra["args"]
    ref = layer.losses.cpu().clone()
    for _ in range(14):
        yh2 = torch.zeros_like(yh)  # a fresh y_hat buffer each step
        layer.step(x, y, params, y_hat=yh2)
        torch.cuda.synchronize()
        assert torch.equal(layer.losses.cpu(), ref)
        assert torch.equal(yh2, yh)


@pytest.mark.parametrize("P,S,d,dout,N,k,f,cap,kind,need_dx", [
    (1, 1, 256, 128, 8, 1, 256, 0, 0, True),       # a single token
    (3, 48, 256, 128, 12, 2, 0, 3, 1, True),       # tiny multi-process (S % 128 != 0), proportional capacity
    (1, 300, 256, 128, 256, 8, 256, 2, 1, True),   # the device maxima: N = 256 experts, top-8
])
def test_layer_edge_shapes(P, S, d, dout, N, k, f, cap, kind, need_dx):
    layer, o, extra = run_case(P, S, d, dout, N, k, f, cap, kind, need_dx, seed=3)
    check(layer, o, extra, P, S, N, k, f, need_dx)


@pytest.mark.parametrize("cap,cf", [(0, 1.0), (2, 1.25), (1, 0.05)])
def test_layer_all_tokens_on_one_expert(cap, cf):
    """Extreme imbalance: every token's top-1 is expert 5 -- one full expert segment, the rest empty (no
    capacity), or almost everything dropped (local / tiny global capacity)."""
    P, S, d, dout, N, k, f = 2, 640, 256, 128, 8, 2, 256
    layer, o, extra = run_case(P, S, d, dout, N, k, f, cap, 1, True, seed=5, cf=cf, hot_expert=5)
    assert (o["expert"][:, :, 0] == 5).all()
    check(layer, o, extra, P, S, N, k, f, True)


@pytest.mark.parametrize("k,bad,N", [(1, float("inf"), 8), (2, float("nan"), 8), (1, float("nan"), 64),
                                     (2, float("-inf"), 48)])
def test_layer_non_finite_logit_raises(k, bad, N):
    """gate.cpp:16-17 throws ValidationError("non-finite gate logit").  The stream-ordered step reports it
    deferred: tamoe_layer_status (and the next step, once the bad step completed) returns status 2 through
    the C ABI and the Python mirror raises ValidationError.  The bad row is routed in range (no fault) and
    poisons the step's losses with NaN; a later clean step is unaffected."""
    import ctypes
    from paper_2302_09915_b200 import _lib, ops
    from paper_2302_09915_b200.layer import LayerConfig, TAMoELayer
    P, S, d, dout, f = 1, 256, 256, 128, 256
    cfg = LayerConfig(P=P, S=S, d=d, d_out=dout, N=N, k=k, f=f, act=1, cap_mode=2, aux_kind=0, need_dx=True)
    layer = TAMoELayer(cfg)
    params = layer.init_params(seed=2)
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(S, d, generator=g, device="cuda").bfloat16()
    y = torch.randn(S, dout, generator=g, device="cuda").bfloat16()
    layer.step(x, y, params)
    layer.status()  # clean
    clean = layer.losses.cpu().clone()
    xb = x.clone()
    xb[37, 5] = bad
    layer.step(xb, y, params)
    torch.cuda.synchronize()
    assert _lib.lib.tamoe_layer_status(layer._h) == 2  # C ABI: status 2 = ValidationError
    assert b"non-finite gate logit" in _lib.lib.tamoe_last_error()
    assert not np.isfinite(layer.losses.cpu().numpy()).all()  # poisoned, not silently finite
    idx = layer.read(ops.R_IDX, (S, k))
    assert idx.min() >= 0 and idx.max() < N and list(idx[37]) == list(range(k))
    # the next step reports a completed bad step before running
    layer.step(xb, y, params)
    torch.cuda.synchronize()
    with pytest.raises(ops.ValidationError, match="non-finite gate logit"):
        layer.step(x, y, params)
    layer.step(x, y, params)
    layer.status()
    assert torch.equal(layer.losses.cpu(), clean)
