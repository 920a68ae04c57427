"""Measured-topology pipeline on the host: fit_profile, fill_partial_profile,
smooth_profile, device_groups, exchange_cost and the closed-form target on the smoothed profile.

Pinned two ways: the reference's own known-answer cases (test_commcost.cpp, test_profile.cpp) restated
below with their file:line, and bit-exact randomized parity against the reference compiled from its
sources (oracle/_ref, skipped when it is not built)."""
import numpy as np
import pytest

import oracle
from paper_2302_09915_b200 import ops

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


# ---------------------------------------------------------------- reference known-answer cases
def test_fit_profile_table1_pairs():
    # test_commcost.cpp:169-179 (the paper's Table 1 two-point fits)
    a, b = ops.fit_profile([(0, 1, 32.0, 758.0), (0, 1, 64.0, 1492.0)], 2)
    assert a[0, 1] == pytest.approx(24.0) and b[0, 1] == pytest.approx(22.9375)
    a, b = ops.fit_profile([(0, 1, 32.0, 5609.0), (0, 1, 16.0, 2835.0)], 2)
    assert a[0, 1] == pytest.approx(61.0) and b[0, 1] == pytest.approx(173.375)
    assert np.isnan(a[1, 0]) and np.isnan(b[0, 0])  # unobserved pairs stay NaN


def test_fit_profile_origin_single_size_and_errors():
    # test_commcost.cpp:181-212
    a, b = ops.fit_profile([(1, 0, 2.0, 10.0), (1, 0, 8.0, 40.0)], 2)
    assert a[1, 0] == pytest.approx(0.0) and b[1, 0] == pytest.approx(5.0)
    a, b = ops.fit_profile([(0, 1, 32.0, 758.0)], 2)
    assert a[0, 1] == 0.0 and b[0, 1] == pytest.approx(758.0 / 32.0)
    with pytest.raises(ops.ValidationError):
        ops.fit_profile([(0, 1, 1.0, 10.0), (0, 1, 2.0, 1.0)], 2)  # negative beta
    with pytest.raises(ops.ValidationError):
        ops.fit_profile([(0, 1, 0.0, 10.0)], 2)  # sizes must be positive
    rng = np.random.default_rng(21)
    for _ in range(20):  # noiseless recovery within 1e-9
        al, be = rng.uniform(0, 100), rng.uniform(0.01, 50)
        a, b = ops.fit_profile([(0, 1, s, al + be * s) for s in (1.0, 2.0, 7.5, 32.0)], 2)
        assert abs(a[0, 1] - al) <= 1e-9 * max(1.0, al) and abs(b[0, 1] - be) <= 1e-9 * be


def _example_raw_22():
    # test_profile.cpp:17-34: intra 0.9 / 1.1, inter 3.8 / 4.0 / 4.2 / 4.0, diagonal 0.1
    beta = np.full((4, 4), 0.1)
    for i, j, v in [(0, 1, 0.9), (2, 3, 1.1), (0, 2, 3.8), (0, 3, 4.0), (1, 2, 4.2), (1, 3, 4.0)]:
        beta[i, j] = beta[j, i] = v
    return np.zeros((4, 4)), beta


def test_smooth_profile_level_means():
    # test_profile.cpp:38-49
    a, b = _example_raw_22()
    ah, bh, la, lb = ops.smooth_profile([2, 2], a, b)
    assert list(lb) == pytest.approx([1.0, 4.0])
    assert bh[0, 1] == pytest.approx(1.0) and bh[1, 3] == pytest.approx(4.0) and bh[0, 0] == pytest.approx(0.1)
    assert np.all(ah == 0.0)


def test_smooth_profile_hierarchical_constant_and_idempotent():
    # test_profile.cpp:51-111
    beta = np.array([[0.5 if i == j else (1.5 if i // 2 == j // 2 else 6.0) for j in range(4)] for i in range(4)])
    ah, bh, _, _ = ops.smooth_profile([2, 2], np.full((4, 4), 2.0), beta)
    np.testing.assert_allclose(bh, beta)
    np.testing.assert_allclose(ah, 2.0)
    rng = np.random.default_rng(3)
    b = rng.uniform(0.5, 8.0, (8, 8))
    np.fill_diagonal(b, 0.3)
    _, b1, _, _ = ops.smooth_profile([2, 4], np.zeros((8, 8)), b)
    _, b2, _, _ = ops.smooth_profile([2, 4], np.zeros((8, 8)), b1)
    np.testing.assert_allclose(b1, b2, rtol=1e-14)
    np.testing.assert_allclose(b1, b1.T, rtol=1e-14)
    with pytest.raises(ops.ValidationError):
        ops.smooth_profile([2, 3], np.zeros((4, 4)), np.ones((4, 4)))  # levels do not match P


def test_fill_partial_profile_symmetry_level_average_diagonal():
    # test_profile.cpp:172-197 (load_profile_csv fills through fill_partial_profile)
    nan = np.nan
    a = np.full((4, 4), nan)
    b = np.full((4, 4), nan)
    for (i, j, v) in [(0, 1, 1.0), (0, 2, 3.8), (0, 3, 4.2), (0, 0, 0.1)]:
        a[i, j], b[i, j] = 0.0, v
    ao, bo = ops.fill_partial_profile(a, b, [2, 2])
    assert bo[1, 0] == pytest.approx(1.0)  # symmetry
    assert bo[2, 3] == pytest.approx(1.0)  # level average
    assert bo[1, 2] == pytest.approx(4.0)  # level average of 3.8 / 4.2
    assert bo[1, 1] == pytest.approx(0.1)  # diagonal from the measured mean
    assert ao[3, 1] == 0.0
    b = np.full((3, 3), 8.0)
    np.fill_diagonal(b, nan)
    _, bo = ops.fill_partial_profile(np.zeros((3, 3)), b)
    assert bo[0, 0] == pytest.approx(0.8) and bo[2, 2] == pytest.approx(0.8)
    with pytest.raises(ops.ValidationError):
        ops.fill_partial_profile(np.full((2, 2), nan), np.full((2, 2), nan))


def test_exchange_cost_fields():
    # test_commcost.cpp:38-117: zero payload costs alpha, size-exchange rounds add max alpha
    P, N = 2, 4
    alpha = np.array([[1.0, 5.0], [5.0, 1.0]])
    beta = np.array([[0.1, 2.0], [2.0, 0.1]])
    c = np.zeros((P, N))
    r = ops.exchange_cost(alpha, beta, c, d=1024, b=2, extra_alpha_rounds=1)
    np.testing.assert_allclose(r["pair_cost_us"], alpha)
    assert r["size_exchange_us"] == 5.0 and r["total_estimate_us"] == r["bottleneck_us"] + 5.0
    c = np.array([[100.0, 100.0, 50.0, 50.0], [10.0, 10.0, 200.0, 200.0]])
    r = ops.exchange_cost(alpha, beta, c, d=1024, b=2)
    mb = 1024 * 2 / 1e6
    assert r["pair_cost_us"][0, 1] == pytest.approx(5.0 + 2.0 * 100 * mb)
    assert r["total_bytes"] == pytest.approx(c.sum() * 1024 * 2)


# ---------------------------------------------------------------- bit-exact parity with the reference
TREES = [[4], [2, 2], [2, 4], [4, 2], [2, 2, 2], [8]]


@needs_ref
def test_fit_profile_matches_reference():
    R = oracle.ref()
    rng = np.random.default_rng(7)
    for trial in range(10):
        P = int(rng.integers(2, 9))
        samples = []
        for i in range(P):
            for j in range(P):
                if rng.uniform() < 0.3:
                    continue  # unmeasured pair
                al, be = rng.uniform(0, 30), rng.uniform(0.2, 20)
                sizes = [4.0] if rng.uniform() < 0.2 else list(rng.choice([0.5, 1, 2, 4, 8, 16], 4, replace=False))
                for s in sizes:
                    samples.append((i, j, float(s), al + be * s + rng.normal(0, 0.3)))
        rng.shuffle(samples)
        if not samples:
            continue
        try:
            ra, rb = R.fit_profile(samples, P)
        except oracle.OracleError:
            with pytest.raises(ops.ValidationError):
                ops.fit_profile(samples, P)
            continue
        a, b = ops.fit_profile(samples, P)
        np.testing.assert_array_equal(a, ra)
        np.testing.assert_array_equal(b, rb)


@needs_ref
@pytest.mark.parametrize("levels", [None] + TREES)
def test_fill_and_smooth_match_reference(levels):
    R = oracle.ref()
    rng = np.random.default_rng(11)
    P = int(np.prod(levels)) if levels else 6
    for trial in range(8):
        a = rng.uniform(0, 20, (P, P))
        b = rng.uniform(0.2, 10, (P, P))
        mask = rng.uniform(size=(P, P)) < 0.4
        a[mask] = np.nan
        b[mask] = np.nan
        ao, bo = ops.fill_partial_profile(a, b, levels)
        rao, rbo = R.fill_partial_profile(a, b, levels)
        np.testing.assert_array_equal(ao, rao)
        np.testing.assert_array_equal(bo, rbo)
        if levels:
            ah, bh, _, _ = ops.smooth_profile(levels, ao, bo)
            rah, rbh = R.smooth_profile(levels, ao, bo)
            np.testing.assert_array_equal(ah, rah)
            np.testing.assert_array_equal(bh, rbh)


@needs_ref
def test_exchange_cost_matches_reference():
    R = oracle.ref()
    rng = np.random.default_rng(5)
    for P, N in [(2, 8), (4, 8), (8, 64)]:
        a = rng.uniform(0, 20, (P, P))
        b = rng.uniform(0.2, 10, (P, P))
        c = rng.uniform(0, 500, (P, N))
        for rounds in (0, 1):
            mine = ops.exchange_cost(a, b, c, d=1024, b=2, extra_alpha_rounds=rounds)
            ref = R.exchange_cost(a, b, c, 1024, 2, rounds)
            np.testing.assert_array_equal(mine["pair_cost_us"], ref["pair_cost_us"])
            for key in ("bottleneck_us", "total_bytes", "size_exchange_us", "total_estimate_us"):
                assert mine[key] == ref[key]


@needs_ref
def test_measured_pipeline_end_to_end_matches_reference():
    """samples -> fit -> fill (tree) -> smooth -> closed form, ours vs the reference, on a synthetic
    [2,4] machine with a self-cheap diagonal and throttled cross-group links (the C5 emulation)."""
    R = oracle.ref()
    rng = np.random.default_rng(9)
    levels, P, N, k, S = [2, 4], 8, 64, 1, 16384
    true_b = np.array([[0.35 if i == j else (1.6 if i // 4 == j // 4 else 6.4) for j in range(P)] for i in range(P)])
    samples = [(i, j, s, 2.0 + true_b[i, j] * s * rng.uniform(0.97, 1.03))
               for i in range(P) for j in range(P) for s in (0.5, 1.0, 2.0, 4.0, 8.0) if (i + j) % 5 != 3]
    a, b = ops.fit_profile(samples, P)
    ra, rb = R.fit_profile(samples, P)
    np.testing.assert_array_equal(b, rb)
    a, b = ops.fill_partial_profile(a, b, levels)
    ra, rb = R.fill_partial_profile(ra, rb, levels)
    np.testing.assert_array_equal(b, rb)
    c_hat, ah, bh = ops.solve_target_tree(levels, a, b, N, k, S)
    rah, rbh = R.smooth_profile(levels, ra, rb)
    np.testing.assert_array_equal(bh, rbh)
    np.testing.assert_array_equal(c_hat, R.target_closed_form(rbh, N, k, S))
    # rows sum to k*S and favour the cheap links
    np.testing.assert_allclose(c_hat.sum(1), k * S)
    assert c_hat[0, 0] > c_hat[0, 8] > c_hat[0, 63]
