"""Pins the C restatement (oracle/tamoe_oracle.c) against the reference compiled
from its own sources (oracle/_ref) and against the reference's own known-answer
tests (test_gate.cpp, test_optimizer.cpp).  CPU only."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (make ref)")


@pytest.fixture(scope="module")
def O():
    return oracle.orc()


@pytest.fixture(scope="module")
def R():
    return oracle.ref()


def stream(R, seed, *shapes, scale=1.0):
    """Consecutive tad::Rng normal() draws, like test_gate.cpp:14-18 random_matrix on one rng."""
    n = sum(int(np.prod(s)) for s in shapes)
    v = R.rng_normal(seed, n) * 1.0
    out, o = [], 0
    for s in shapes:
        m = int(np.prod(s))
        out.append(v[o:o + m].reshape(s) * scale)
        o += m
    return out


def test_softmax_and_gate_bitwise(O, R):
    for seed in range(1, 6):
        x, w = stream(R, seed, (37, 13), (13, 7))
        assert np.array_equal(O.gate_forward(x, w), R.gate_forward(x, w))
        lg = x @ w * 17.0
        assert np.array_equal(O.softmax_rows(lg), R.softmax_rows(lg))


def test_softmax_rejects_nonfinite(O, R):
    lg = np.array([[0.0, np.inf]])
    for impl in (O, R):
        with pytest.raises(oracle.OracleError):
            impl.softmax_rows(lg)


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("P", [1, 3, 4])
def test_topk_route_bitwise(O, R, mode, k, P):
    rng = np.random.default_rng(100 * mode + 10 * k + P)
    S, N = 29, 8
    logits = rng.normal(size=(P, S, N))
    logits[:, 3] = logits[:, 2]           # duplicate tokens -> exact score ties across tokens
    logits[:, 5, 1] = logits[:, 5, 4]     # exact tie inside a row -> lower index wins
    probs = np.stack([R.softmax_rows(l) for l in logits])
    c_hat = rng.uniform(0.5, 3.0, size=(P, N))
    for cf in (0.6, 1.0, 1.25):
        a = O.topk_route(probs, k, mode, cf, c_hat)
        b = R.topk_route(probs, k, mode, cf, c_hat)
        for key in a:
            assert np.array_equal(a[key], b[key]), (key, cf)


def test_lrr_kat_and_random(O, R):
    # test_gate.cpp:81-88
    col = np.array([104.348, 10.435, 2.609, 2.609])
    w = 144.0 * col / col.sum()
    assert list(O.largest_remainder_round(w, 144)) == [125, 13, 3, 3]
    rng = np.random.default_rng(7)
    for _ in range(200):
        n = int(rng.integers(1, 12))
        v = rng.uniform(0, 50, n) * (rng.uniform(size=n) > 0.2)
        t = int(rng.integers(0, 400))
        assert np.array_equal(O.largest_remainder_round(v, t), R.largest_remainder_round(v, t))


def test_penalty_kats(O, R):
    # test_gate.cpp:196-232
    for impl in (O, R):
        np.testing.assert_allclose(impl.penalty_weights(np.full(8, 30.0)), 1 / 8, rtol=1e-12)
        p = impl.penalty_weights([104.3478260869565, 10.43478260869565, 2.608695652173913, 2.608695652173913])
        np.testing.assert_allclose(p, np.array([0.1, 1, 4, 4]) / 9.1, rtol=1e-5)
        for norm in (0, 1):
            p = impl.penalty_weights([50.0, 10.0, 3.0, 1.0], norm)
            assert np.all(np.diff(p) > 0)
        with pytest.raises(oracle.OracleError):
            impl.penalty_weights([1.0, 0.0])
    rng = np.random.default_rng(3)
    for _ in range(50):
        c = rng.uniform(0.1, 100, 16)
        for norm in (0, 1):
            for t in (0.0, 0.3):
                assert np.array_equal(O.penalty_weights(c, norm, t), R.penalty_weights(c, norm, t))


def test_closed_form_re1(O, R):
    # test_optimizer.cpp:60-74 (RE-1: beta diag .1, intra 1, inter 4; k=1, S=120, N=P=4)
    beta = np.array([[0.1 if i == j else (1.0 if i // 2 == j // 2 else 4.0) for j in range(4)] for i in range(4)])
    a = O.target_closed_form(beta, 4, 1, 120)
    b = R.target_closed_form(beta, 4, 1, 120)
    assert np.array_equal(a, b)
    np.testing.assert_allclose(a[0], [104.3478, 10.4348, 2.6087, 2.6087], rtol=1e-5)
    np.testing.assert_allclose(a.sum(1), 120.0)


def test_losses_and_grads_bitwise(O, R):
    for seed in range(1, 9):  # test_gate.cpp:269-312 instance shapes
        x, w = stream(R, seed, (16, 8), (8, 4))
        w = w * 0.5
        c_hat = R.rng_uniform(seed + 1000, 4, 0.5, 40.0)
        p = R.penalty_weights(c_hat)
        probs = R.gate_forward(x, w)
        r = R.topk_route(probs, 1)
        cnt, mp = r["counts"][0], r["mean_probs"][0]
        assert O.loss_topo(cnt, mp, p, 1, 16) == R.loss_topo(cnt, mp, p, 1, 16)
        assert O.loss_balance(cnt, mp, 16) == R.loss_balance(cnt, mp, 16)
        g_ref = R.grad_loss_topo(x, probs, cnt, mp, p, 1)
        g_orc = O.grad_aux(x, probs, O.topo_coefficients(cnt, p, 1, 16))
        assert np.array_equal(g_ref, g_orc)
        g_ref = R.grad_loss_balance(x, probs, cnt, mp)
        g_orc = O.grad_aux(x, probs, O.balance_coefficients(cnt, 16))
        assert np.array_equal(g_ref, g_orc)


def _re1_beta():
    return np.array([[0.1 if i == j else (1.0 if i // 2 == j // 2 else 4.0) for j in range(4)] for i in range(4)])


@pytest.mark.parametrize("kind,cap,k", [(0, 0, 1), (1, 0, 1), (1, 3, 2), (0, 1, 2), (1, 2, 1)])
def test_layer_step_matches_reference_train(O, R, kind, cap, k):
    """orc_layer_step + SGD reproduces the reference train() loss trajectory bit for bit
    (trainer.cpp:371-416), which pins the forward, routing, aux loss and every gradient."""
    P, S, d, dout, N = 4, 40, 8, 4, 4
    x, y, _, _ = R.gen_synthetic(3, P, S, d, dout, N, k, noise_std=0.5, map_spread=0.05)
    gates = np.stack([0.01 * R.rng_normal(R.derive_seed(3, 2000 + i), d * N).reshape(d, N) for i in range(P)])
    U = np.stack([R.rng_normal(R.derive_seed(3, 3000 + e), d * dout).reshape(d, dout) / np.sqrt(d)
                  for e in range(N)])
    c_hat = R.target_closed_form(_re1_beta(), N, k, S)
    pen = np.stack([R.penalty_weights(c_hat[i]) for i in range(P)])
    lr, steps = 0.2, 4
    rep = R.train(x, y, gates, U, kind=kind, cap_mode=cap, cf=1.0, c_hat=c_hat, lr=lr, steps=steps, k=k)
    g, u = gates.copy(), U.copy()
    for s in range(steps):
        o = O.layer_step(x, y, g, U=u, k=k, cap_mode=cap, cf=1.0, c_hat=c_hat, aux_kind=kind, penalties=pen)
        assert o["task_loss"] == rep["task_loss"][s], s
        assert o["aux_loss"] == rep["aux_loss"][s], s
        if s == 0:
            assert np.array_equal(o["counts"].astype(float), rep["initial_dispatch"])
        for i in range(P):
            g[i] = g[i] - lr * o["gate_grads"][i]
        for e in range(N):
            u[e] = u[e] - lr * o["grad_u"][e]


def test_ffn_extension_finite_differences(O):
    """The FFN expert and dX are extensions without a reference counterpart: check them with
    central differences of the oracle's own loss (SURVEY §8(c) 'parity-unpinned' items)."""
    rng = np.random.default_rng(5)
    P, S, d, dout, N, f, k = 2, 6, 5, 3, 4, 7, 2
    x = rng.normal(size=(P, S, d))
    y = rng.normal(size=(P, S, dout))
    gates = rng.normal(size=(P, d, N)) * 0.3
    W1 = rng.normal(size=(N, d, f)) * 0.5
    W2 = rng.normal(size=(N, f, dout)) * 0.5

    def loss(W1_, W2_, x_):
        o = O.layer_step(x_, y, gates, W1=W1_, W2=W2_, k=k, aux_weight=0.0, act=1)
        return o["task_loss"]

    o = O.layer_step(x, y, gates, W1=W1, W2=W2, k=k, aux_weight=0.0, act=1, want_dx=True)
    h = 1e-6
    for arr, grad in ((W1, o["grad_w1"]), (W2, o["grad_w2"])):
        idx = [tuple(rng.integers(0, s) for s in arr.shape) for _ in range(6)]
        for ix in idx:
            a = arr.copy(); a[ix] += h
            b = arr.copy(); b[ix] -= h
            fd = (loss(a if arr is W1 else W1, a if arr is W2 else W2, x) -
                  loss(b if arr is W1 else W1, b if arr is W2 else W2, x)) / (2 * h)
            assert abs(fd - grad[ix]) < 1e-6 * max(1.0, abs(fd)), (ix, fd, grad[ix])
    # dx: the expert path only (the gate term's FD would also move the routing weights' probs,
    # which the layer differentiates through softmax; aux off, routing held by tiny h)
    for _ in range(6):
        ix = tuple(rng.integers(0, s) for s in x.shape)
        a = x.copy(); a[ix] += h
        b = x.copy(); b[ix] -= h
        fd = (loss(W1, W2, a) - loss(W1, W2, b)) / (2 * h)
        assert abs(fd - o["dx"][ix]) < 1e-5 * max(1.0, abs(fd)), (ix, fd, o["dx"][ix])
