"""The fp64 value-semantics gate operators (tamoe_softmax_rows_f64 / tamoe_gate_forward_f64 /
tamoe_grad_aux_loss_f64) against the reference, and the reference's OWN unit suite (proj/tests, 68 cases)
linked with gate.cpp replaced by the B200 drop-in shim integration/tad_gate_b200.cpp (oracle/ref.mk
`suite_b200`): every gate, routing and aux-loss call of that suite -- including the ones inside the
reference's train() -- runs on the GPU through the C ABI."""
import os
import subprocess

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "oracle", "_ref", "unit_tests_b200")
SUITE_TRAIN = os.path.join(ROOT, "oracle", "_ref", "unit_tests_b200_train")


def _ops():
    from paper_2302_09915_b200 import ops
    return ops


def _ref():
    return oracle.ref() if oracle.ref_available() else oracle.orc()


@pytest.mark.parametrize("S,d,N", [(5, 4, 3), (32, 8, 6), (1024, 512, 8), (333, 100, 64)])
def test_gate_forward_f64_matches_reference(S, d, N):
    ops = _ops()
    rng = np.random.default_rng(S + d + N)
    x = rng.normal(size=(S, d))
    x[rng.random(size=(S, d)) < 0.1] = 0.0  # exercise the reference's zero skip
    W = rng.normal(size=(d, N)) * 0.5
    got = ops.gate_forward_f64(x, W).cpu().numpy()
    want = _ref().gate_forward(x, W)
    # bit-identical logits; exp may differ by an ulp between CUDA and glibc
    np.testing.assert_allclose(got, want, rtol=4e-16 * N, atol=0)
    np.testing.assert_allclose(got.sum(1), 1.0, rtol=1e-12)


def test_softmax_rows_f64_and_nonfinite():
    ops = _ops()
    rng = np.random.default_rng(3)
    z = rng.normal(size=(257, 64)) * 30
    np.testing.assert_allclose(ops.softmax_rows(z).cpu().numpy(), _ref().softmax_rows(z), rtol=1e-14, atol=1e-300)
    z[100, 7] = np.inf
    with pytest.raises(ops.ValidationError):
        ops.softmax_rows(z)
    with pytest.raises(ops.ValidationError):
        ops.gate_forward_f64(np.full((4, 2), np.nan), np.ones((2, 3)))


@pytest.mark.parametrize("S,d,N", [(16, 8, 4), (1024, 512, 8), (300, 64, 64)])
def test_grad_aux_loss_f64_bit_exact(S, d, N):
    """dz = p (coeff - <coeff, p>), x^T dz in the reference's order: identical bits on identical inputs."""
    ops = _ops()
    O = oracle.orc()
    rng = np.random.default_rng(S * N)
    x = rng.normal(size=(S, d))
    probs = O.softmax_rows(rng.normal(size=(S, N)))
    counts = rng.integers(0, S, N)
    pen = ops.penalty_weights(rng.uniform(0.5, 40, N))
    res = ops.RoutingResult(None, None, None, None, counts.astype(np.int64), np.zeros(N, np.int64),
                            probs.mean(0), [])
    coeff = ops.topo_coefficients(res, pen, N, 4, S)
    got = ops.grad_aux_loss(x, probs, coeff).cpu().numpy()
    assert np.array_equal(got, O.grad_aux(x, probs, coeff))
    if oracle.ref_available():
        want = oracle.ref().grad_loss_topo(x, probs, counts, probs.mean(0), pen, 4)
        assert np.array_equal(ops.grad_loss_topo(x, probs, res, pen, N, 4, S).cpu().numpy(), want)


def test_reference_unit_suite_on_the_b200_gate():
    if not os.path.exists(SUITE):
        pytest.skip("oracle/_ref/unit_tests_b200 not built (make -f oracle/ref.mk suite_b200, needs /root/reference)")
    r = subprocess.run([SUITE], capture_output=True, text=True, timeout=600, cwd=ROOT)
    summary = [ln for ln in r.stdout.splitlines() if "[doctest-shim]" in ln]
    assert summary, r.stdout[-2000:] + r.stderr[-4000:]
    print(summary[0])
    assert r.returncode == 0, summary[0] + "\n" + r.stderr[-6000:]
    assert "failed: 0 " in summary[0]


def test_reference_unit_suite_with_train_step_on_the_b200():
    """The reference's 68-case suite with gate.cpp AND train()'s inline layer step replaced: every train() call of
    test_trainer.cpp / test_report_io.cpp runs its whole step (gate, routing, experts, combine, backward, SGD) on
    the GPU in fp64 through tamoe_train_f64 (integration/tad_train_b200.cpp)."""
    if not os.path.exists(SUITE_TRAIN):
        pytest.skip("oracle/_ref/unit_tests_b200_train not built (make -f oracle/ref.mk suite_b200_train)")
    r = subprocess.run([SUITE_TRAIN], capture_output=True, text=True, timeout=900, cwd=ROOT)
    summary = [ln for ln in r.stdout.splitlines() if "[doctest-shim]" in ln]
    assert summary, r.stdout[-2000:] + r.stderr[-4000:]
    print(summary[0])
    assert r.returncode == 0, summary[0] + "\n" + r.stdout[-4000:] + r.stderr[-6000:]
    assert "failed: 0 " in summary[0]
