"""C-ABI boundary on the CPU: the library loads without a GPU, exports every symbol
include/tamoe.h declares, and its host-side topology inputs (c_hat, penalties,
capacities, payloads) are bit-identical to the oracle / reference."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "tamoe.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(tamoe_\w+)\s*\(", text, re.M)))


def test_library_loads_and_exports_header_symbols():
    from paper_2302_09915_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 20, syms
    missing = [s for s in syms if not hasattr(_lib.lib, s)]
    assert not missing, missing
    assert _lib.lib.tamoe_version() >= 1


def test_no_cpu_fallback_without_library(tmp_path, monkeypatch):
    """The product path refuses to run without the CUDA library (no silent fallback)."""
    import paper_2302_09915_b200._lib as L
    monkeypatch.setattr(L, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        L._load()  # (no reload afterwards: it would redefine the exception classes other modules hold)


def re1_beta(P=4):
    return np.array([[0.1 if i == j else (1.0 if i // 2 == j // 2 else 4.0) for j in range(P)] for i in range(P)])


def test_host_inputs_match_oracle():
    from paper_2302_09915_b200 import ops
    O = oracle.orc()
    for P, N, k, S in [(4, 4, 1, 120), (4, 8, 2, 1024), (8, 64, 1, 16384), (2, 8, 2, 256)]:
        beta = re1_beta(P) if P % 2 == 0 else np.ones((P, P))
        c = ops.target_closed_form(beta, N, k, S)
        assert np.array_equal(c, O.target_closed_form(beta, N, k, S))
        np.testing.assert_allclose(c.sum(1), k * S)
        for i in range(P):
            for norm in (0, 1):
                assert np.array_equal(ops.penalty_weights(c[i], ops.PenaltyNorm(norm)), O.penalty_weights(c[i], norm))
    rng = np.random.default_rng(0)
    for _ in range(100):
        n = int(rng.integers(1, 10))
        v = rng.uniform(0, 40, n)
        t = int(v.sum()) + int(rng.integers(-2, 3))
        assert np.array_equal(ops.largest_remainder_round(v, t), O.largest_remainder_round(v, t))


def test_capacity_caps_follow_reference_rules():
    """gate.cpp:151-180: global floor(C+1e-9); local floor(C/P+1e-9); proportional LRR of C c_hat/col."""
    from paper_2302_09915_b200 import ops
    O = oracle.orc()
    P, N, k, S = 4, 8, 2, 1024
    c_hat = ops.target_closed_form(re1_beta(), N, k, S)
    C = 1.25 * k * S * P / N
    g = ops.capacity_caps(ops.CapacityPolicy(ops.CapacityMode.global_, 1.25), k, S, N, P, c_hat)
    assert np.all(g == int(np.floor(C + 1e-9)))
    loc = ops.capacity_caps(ops.CapacityPolicy(ops.CapacityMode.local, 1.25), k, S, N, P, c_hat)
    assert np.all(loc == int(np.floor(C / P + 1e-9)))
    pr = ops.capacity_caps(ops.CapacityPolicy(ops.CapacityMode.local_proportional, 1.25), k, S, N, P, c_hat)
    for e in range(N):
        w = c_hat[:, e] * C / c_hat[:, e].sum()
        assert np.array_equal(pr[:, e], O.largest_remainder_round(w, int(np.floor(C + 1e-9))))
    none = ops.capacity_caps(ops.CapacityPolicy(), k, S, N, P)
    assert np.all(none == np.iinfo(np.int64).max)


def test_validation_status_codes():
    from paper_2302_09915_b200 import ops
    with pytest.raises(ops.ValidationError):
        ops.penalty_weights([1.0, 0.0])
    with pytest.raises(ops.ValidationError):
        ops.capacity_caps(ops.CapacityPolicy(ops.CapacityMode.local_proportional, 1.0), 1, 16, 4, 2, None)
    with pytest.raises(ops.ValidationError):
        ops.target_closed_form(np.ones((3, 3)), 4, 1, 16)  # N % P != 0
    with pytest.raises(ops.ValidationError):
        ops.target_closed_form(np.zeros((2, 2)), 4, 1, 16)  # beta must be > 0
    with pytest.raises(ops.ValidationError):
        ops.capacity_caps(ops.CapacityPolicy(), 5, 16, 4, 1)  # k > N
    from paper_2302_09915_b200 import _lib
    assert _lib.lib.tamoe_penalty_weights(None, 0, 0, ctypes.c_double(0.0), None) == 2
    assert b"empty" in _lib.lib.tamoe_last_error()


def test_device_payload_tokens():
    from paper_2302_09915_b200 import ops
    counts = np.arange(32, dtype=np.float64).reshape(4, 8)
    pay = ops.device_payload_tokens(counts)
    for i in range(4):
        for j in range(4):
            assert pay[i, j] == counts[i, 2 * j:2 * j + 2].sum()


def test_aux_losses_and_coefficients_match_oracle():
    """loss_balance / loss_topo / *_coefficients (gate.cpp:209-214, 248-255, 273-287) through the C ABI are
    bit-identical to the oracle restatement (itself pinned to the compiled reference in test_oracle_ref)."""
    from paper_2302_09915_b200 import ops
    O = oracle.orc()
    rng = np.random.default_rng(7)
    for N, P, S in [(4, 4, 24), (8, 2, 1024), (64, 8, 16384), (6, 1, 30)]:
        counts = rng.integers(0, S, N).astype(np.int64)
        mean = rng.dirichlet(np.ones(N))
        pen = ops.penalty_weights(rng.uniform(0.5, 40.0, N))
        res = ops.RoutingResult(None, None, None, None, counts, np.zeros(N, np.int64), mean, [])
        assert ops.loss_balance(res, S) == O.loss_balance(counts, mean, S)
        assert ops.loss_topo(res, pen, N, P, S) == O.loss_topo(counts, mean, pen, P, S)
        assert np.array_equal(ops.topo_coefficients(res, pen, N, P, S), O.topo_coefficients(counts, pen, P, S))
        assert np.array_equal(ops.balance_coefficients(res, S), O.balance_coefficients(counts, S))
        if oracle.ref_available():
            R = oracle.ref()
            assert ops.loss_balance(res, S) == R.loss_balance(counts, mean, S)
            assert ops.loss_topo(res, pen, N, P, S) == R.loss_topo(counts, mean, pen, P, S)
    with pytest.raises(ops.ValidationError):
        ops.loss_topo(ops.RoutingResult(None, None, None, None, np.zeros(4, np.int64), None, np.zeros(4), []),
                      np.ones(3), 4, 1, 8)


def test_link_emulation_validation():
    from paper_2302_09915_b200 import ops
    ops.set_link_emulation(2, 4)
    ops.set_link_emulation(0, 1)  # off again
    with pytest.raises(ops.ValidationError):
        ops.set_link_emulation(2, 0)
    with pytest.raises(ops.ValidationError):
        ops.set_link_emulation(-1, 2)


def test_reference_precision_entry_points_validate_before_touching_the_device():
    """tamoe_layer_step_f64 / tamoe_train_f64 (BASELINE C1 in fp64, the drop-in train()) reject malformed calls
    with status 2 on the host, as the reference throws ValidationError (no GPU needed for these checks)."""
    from paper_2302_09915_b200 import _lib
    L = _lib.lib
    L.tamoe_layer_step_f64.restype = ctypes.c_int
    assert L.tamoe_layer_step_f64(None, 4, 4, None, None, None, None, None, None, 0, ctypes.c_double(1.0), 0,
                                  None, None, None, None, None, None, None) == 2
    assert b"null router" in L.tamoe_last_error()
    L.tamoe_train_f64.restype = ctypes.c_int
    assert L.tamoe_train_f64(None, None, None, None, None, None, None, None, None) == 2
    assert b"null argument" in L.tamoe_last_error()
