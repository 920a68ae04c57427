"""Device routing parity against the oracle (bit-exact: expert indices, kept flags,
per-rank counts and the permutation order; values within the stated tolerance)."""
import os

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _ops():
    from paper_2302_09915_b200 import ops
    return ops


def oracle_order(r, P, S, k, N):
    """Kept picks per expert in reference bucket order (process, token, slot)."""
    order = [[] for _ in range(N)]
    for i in range(P):
        for s in range(S):
            for j in range(k):
                if r["kept"][i, s, j]:
                    order[r["expert"][i, s, j]].append((i * S + s) * k + j)
    return [np.array(o, dtype=np.int64) for o in order]


def check_same(gpu, orc, P, S, k, N):
    ops = _ops()
    idx, gate, score, kept = gpu.read(ops.R_IDX), gpu.read(ops.R_GATE), gpu.read(ops.R_SCORE), gpu.read(ops.R_KEPT)
    assert np.array_equal(idx, orc["expert"])
    assert np.array_equal(score, orc["score"])          # same fp64 inputs -> identical bits
    np.testing.assert_allclose(gate, orc["gate"], rtol=1e-6)
    assert np.array_equal(gpu.read(ops.R_GATE64), orc["gate"])  # fp64 gate_value: same expression, same bits
    assert np.array_equal(kept, orc["kept"])
    assert np.array_equal(gpu.read(ops.R_COUNTS), orc["counts"])
    assert np.array_equal(gpu.read(ops.R_DROPPED), orc["dropped"])
    np.testing.assert_allclose(gpu.read(ops.R_MEAN_PROBS), orc["mean_probs"], rtol=1e-12, atol=1e-15)
    for e, (a, b) in enumerate(zip(gpu.expert_order(), oracle_order(orc, P, S, k, N))):
        assert np.array_equal(a, b), e


@pytest.mark.parametrize("P,S,N,k", [(1, 300, 8, 1), (4, 129, 8, 2), (3, 40, 4, 2), (2, 1000, 64, 2), (1, 64, 16, 8)])
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_route_probs_bit_exact(P, S, N, k, mode):
    ops = _ops()
    O = oracle.orc()
    rng = np.random.default_rng(P * 1000 + S + N + k + mode)
    logits = rng.normal(size=(P, S, N))
    logits[:, 1] = logits[:, 0]             # duplicate tokens: exact cross-token score ties
    logits[:, 2, 3 % N] = logits[:, 2, 0]   # in-row tie: lower index wins
    probs = np.stack([O.softmax_rows(l) for l in logits])
    c_hat = rng.uniform(0.5, 3.0, size=(P, N))
    for cf in (0.5, 1.0, 1.25):
        pol = ops.CapacityPolicy(ops.CapacityMode(mode), cf)
        caps = ops.capacity_caps(pol, k, S, N, P, c_hat)
        r = ops.Router(P, S, N, k)
        r.route_probs(torch.from_numpy(probs).cuda(), pol, caps)
        check_same(r, O.topk_route(probs, k, mode, cf, c_hat), P, S, k, N)


def test_route_golden_fixtures():
    ops = _ops()
    z = np.load(os.path.join(G, "routing.npz"))
    for mode in range(4):
        for k in (1, 2):
            tag = f"route_m{mode}_k{k}"
            probs = z[tag + "_probs"]
            P, S, N = probs.shape
            pol = ops.CapacityPolicy(ops.CapacityMode(mode), 1.25)
            caps = ops.capacity_caps(pol, k, S, N, P, z[tag + "_c_hat"])
            r = ops.Router(P, S, N, k)
            r.route_probs(torch.from_numpy(probs).cuda(), pol, caps)
            ref = {key: z[f"{tag}_{key}"] for key in ("expert", "gate", "score", "kept", "counts", "dropped",
                                                        "mean_probs")}
            check_same(r, ref, P, S, k, N)


@pytest.mark.parametrize("P,S,d,N,k,mode", [(1, 1000, 256, 64, 1, 0), (4, 256, 512, 8, 2, 3), (2, 300, 128, 16, 2, 2),
                                            (1, 16384, 1024, 64, 1, 0)])
def test_gate_route_from_identical_logits(P, S, d, N, k, mode):
    """tcgen05 gate: logits vs torch fp32; routing from the GPU's own logits == oracle routing fed the same
    logits (softmax_rows -> topk_route), bit for bit except audited near-ties."""
    ops = _ops()
    O = oracle.orc()
    torch.manual_seed(0)
    x = torch.randn(P * S, d, device="cuda").bfloat16()
    npd = ops.n_pad(N)
    wg = torch.zeros(P, npd, d, device="cuda", dtype=torch.bfloat16)
    wg[:, :N] = (torch.randn(P, N, d, device="cuda") * 0.05).bfloat16()
    c_hat = np.random.default_rng(1).uniform(0.5, 3, size=(P, N))
    pol = ops.CapacityPolicy(ops.CapacityMode(mode), 1.25)
    caps = ops.capacity_caps(pol, k, S, N, P, c_hat)
    r = ops.Router(P, S, N, k)
    logits, probs = r.route_gate(x, wg, pol, caps, want_probs=True)
    torch.cuda.synchronize()
    ref_logits = torch.stack([x[i * S:(i + 1) * S].float() @ wg[i, :N].float().t() for i in range(P)]).reshape(P * S, N)
    assert (logits - ref_logits).abs().max().item() < 1e-3 * max(1.0, ref_logits.abs().max().item())
    lg = logits.double().cpu().numpy().reshape(P, S, N)
    oprobs = np.stack([O.softmax_rows(l) for l in lg])
    gp = probs.cpu().numpy().reshape(P, S, N)
    np.testing.assert_allclose(gp, oprobs, rtol=1e-14, atol=1e-300)
    orc = O.topk_route(oprobs, k, mode, 1.25, c_hat)
    idx = r.read(ops.R_IDX)
    mism = np.argwhere(idx != orc["expert"])
    for (i, s, j) in mism:  # only allowed where the oracle's probabilities are within a few ulps
        pr = np.sort(oprobs[i, s])[::-1]
        assert abs(pr[j] - pr[j + 1]) <= 4 * np.spacing(pr[j]), (i, s, j)
    if len(mism) == 0:
        assert np.array_equal(r.read(ops.R_KEPT), orc["kept"])
        assert np.array_equal(r.read(ops.R_COUNTS), orc["counts"])
        for e, (a, b) in enumerate(zip(r.expert_order(), oracle_order(orc, P, S, k, N))):
            assert np.array_equal(a, b), e


@pytest.mark.parametrize("P,S,d,N,k,mode", [(1, 16384, 1024, 64, 1, 0), (4, 256, 512, 8, 2, 3), (2, 300, 128, 16, 2, 2),
                                            (1, 2048, 4096, 64, 2, 3), (1, 200, 256, 48, 8, 1), (3, 129, 256, 32, 1, 2)])
def test_fused_gate_routing_bit_exact(P, S, d, N, k, mode):
    """The one-launch gate (N <= 64: routing in the tcgen05 GEMM epilogue, no probabilities output) against the
    oracle fed the kernel's own fp32 logits: expert indices, fp64 scores and gate values, kept flags, counts,
    mean probabilities and the permutation order -- bit for bit (mean probabilities to 1e-12), except audited
    near-ties (probabilities within a few ulps).  Includes C2 (T=16,384, d=1,024, N=64, top-1) and C4's gate
    (d=4,096, N=64, top-2, proportional capacity) and in-row exact ties."""
    ops = _ops()
    O = oracle.orc()
    torch.manual_seed(P * 7 + S + N)
    x = torch.randn(P * S, d, device="cuda").bfloat16()
    npd = ops.n_pad(N)
    wg = torch.zeros(P, npd, d, device="cuda", dtype=torch.bfloat16)
    wg[:, :N] = (torch.randn(P, N, d, device="cuda") * 0.05).bfloat16()
    if N >= 8:  # identical weight rows 3 and 5: exact in-row logit ties (the lower expert wins)
        wg[:, 5] = wg[:, 3]
    c_hat = np.random.default_rng(2).uniform(0.5, 3, size=(P, N))
    pol = ops.CapacityPolicy(ops.CapacityMode(mode), 1.25)
    caps = ops.capacity_caps(pol, k, S, N, P, c_hat)
    r = ops.Router(P, S, N, k)
    logits, probs = r.route_gate(x, wg, pol, caps, want_probs=False)
    torch.cuda.synchronize()
    lg = logits.double().cpu().numpy().reshape(P, S, N)
    oprobs = np.stack([O.softmax_rows(l) for l in lg])
    orc = O.topk_route(oprobs, k, mode, 1.25, c_hat)
    idx = r.read(ops.R_IDX)
    mism = np.argwhere(idx != orc["expert"])
    for (i, s_, j) in mism:
        pr = np.sort(oprobs[i, s_])[::-1]
        assert abs(pr[j] - pr[j + 1]) <= 4 * np.spacing(pr[j]), (i, s_, j)
    assert len(mism) <= 2
    if len(mism) == 0:
        # the device's fp64 exp is within 1 ulp of glibc's (the oracle's): scores / gate values to 1e-14
        np.testing.assert_allclose(r.read(ops.R_SCORE), orc["score"], rtol=1e-14, atol=0)
        np.testing.assert_allclose(r.read(ops.R_GATE64), orc["gate"], rtol=1e-14, atol=0)
        assert np.array_equal(r.read(ops.R_KEPT), orc["kept"])
        assert np.array_equal(r.read(ops.R_COUNTS), orc["counts"])
        assert np.array_equal(r.read(ops.R_DROPPED), orc["dropped"])
        for e, (a, b) in enumerate(zip(r.expert_order(), oracle_order(orc, P, S, k, N))):
            assert np.array_equal(a, b), e
    np.testing.assert_allclose(r.read(ops.R_MEAN_PROBS), orc["mean_probs"], rtol=1e-12, atol=1e-15)


def test_gate_rejects_nonfinite():
    ops = _ops()
    x = torch.zeros(128, 64, device="cuda", dtype=torch.bfloat16)
    x[3, 5] = float("inf")
    wg = torch.ones(1, 16, 64, device="cuda", dtype=torch.bfloat16)
    r = ops.Router(1, 128, 8, 1)
    with pytest.raises(ops.ValidationError):
        r.route_gate(x, wg, ops.CapacityPolicy(), np.full((1, 8), 10 ** 9, np.int64))


@pytest.mark.parametrize("P,S,N,k,mode", [(1, 500, 8, 2, 0), (4, 128, 8, 2, 3), (2, 77, 64, 1, 2)])
def test_permute_rows(P, S, N, k, mode):
    ops = _ops()
    O = oracle.orc()
    rng = np.random.default_rng(5)
    probs = np.stack([O.softmax_rows(l) for l in rng.normal(size=(P, S, N))])
    c_hat = rng.uniform(0.5, 3.0, size=(P, N))
    pol = ops.CapacityPolicy(ops.CapacityMode(mode), 1.0)
    caps = ops.capacity_caps(pol, k, S, N, P, c_hat)
    r = ops.Router(P, S, N, k)
    r.route_probs(torch.from_numpy(probs).cuda(), pol, caps)
    d = 64
    x = torch.randn(P * S, d, device="cuda").bfloat16()
    r_max = P * S * k + 16 * N
    xp = r.permute(x, r_max)
    torch.cuda.synchronize()
    seg_start, seg_rows = r.read(ops.R_SEG_START), r.read(ops.R_SEG_ROWS)
    pos = r.read(ops.R_POS).reshape(-1)
    order = r.expert_order()
    xs = x.cpu()
    xpc = xp.cpu()
    for e in range(N):
        assert seg_rows[e] % 16 == 0 and seg_rows[e] >= len(order[e])
        for j, pick in enumerate(order[e]):
            row = seg_start[e] + j
            assert pos[pick] == row
            assert torch.equal(xpc[row], xs[pick // k])
        for row in range(seg_start[e] + len(order[e]), seg_start[e] + seg_rows[e]):
            assert torch.all(xpc[row] == 0)
    assert np.all(pos[r.read(ops.R_KEPT).reshape(-1) == 0] == -1)
