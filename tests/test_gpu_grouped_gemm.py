"""Grouped expert GEMMs (tcgen05) vs a plain PyTorch fp32 reference."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _segments(counts, dev):
    rows = [((c + 15) // 16) * 16 for c in counts]
    start = np.concatenate([[0], np.cumsum(rows)[:-1]]).astype(np.int32)
    R = int(sum(rows))
    return (torch.tensor(start, dtype=torch.int32, device=dev), torch.tensor(rows, dtype=torch.int32, device=dev),
            start, rows, R)


def _tokens(counts, start, R, K, dev, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    t = torch.zeros(R, K, dtype=torch.bfloat16)
    for s, c in zip(start, counts):
        t[s:s + c] = torch.randn(c, K, generator=g).to(torch.bfloat16)
    return t.to(dev)


def _rel(a, b):
    return (a.float() - b.float()).norm().item() / max(b.float().norm().item(), 1e-30)


@pytest.mark.parametrize("counts,M,K", [([5, 0, 300, 17, 256], 256, 128), ([1000], 128, 64), ([33, 64, 1, 270], 384, 256),
                                        ([16, 48, 272, 511, 0, 700], 512, 192)])
def test_grouped_fwd(dev, counts, M, K):
    from paper_2302_09915_b200 import _lib
    G = len(counts)
    ss, sr, start, rows, R = _segments(counts, dev)
    x = _tokens(counts, start, R, K, dev, 1)
    w = (torch.randn(G, M, K, device=dev) / K ** 0.5).to(torch.bfloat16)
    out = torch.full((R, M), float("nan"), dtype=torch.bfloat16, device=dev)
    pre = torch.full((R, M), float("nan"), dtype=torch.bfloat16, device=dev)
    _lib.call("tamoe_grouped_fwd", x.data_ptr(), w.data_ptr(), G, M, K, R, ss.data_ptr(), sr.data_ptr(),
              out.data_ptr(), pre.data_ptr(), 1, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for g in range(G):
        s, r = start[g], rows[g]
        ref = x[s:s + r].float() @ w[g].float().t()
        refd = ref.clone().requires_grad_(True)
        torch.nn.functional.gelu(refd, approximate="tanh").sum().backward()
        assert _rel(pre[s:s + r], refd.grad) < 1e-2, g   # stored gelu'(pre-activation)
        assert _rel(out[s:s + r], torch.nn.functional.gelu(ref, approximate="tanh")) < 1e-2, g


@pytest.mark.parametrize("counts,M,K", [([5, 0, 300, 17, 256], 256, 128), ([33, 64, 1, 270], 128, 192),
                                        ([16, 48, 272, 511, 0, 700], 512, 256)])
def test_grouped_dgrad(dev, counts, M, K):
    from paper_2302_09915_b200 import _lib
    G = len(counts)
    ss, sr, start, rows, R = _segments(counts, dev)
    dy = _tokens(counts, start, R, K, dev, 2)
    w = (torch.randn(G, K, M, device=dev) / K ** 0.5).to(torch.bfloat16)  # stored K x M
    deriv = torch.randn(R, M, device=dev).to(torch.bfloat16)  # act'(pre-activation) as grouped_fwd stores it
    out = torch.full((R, M), float("nan"), dtype=torch.bfloat16, device=dev)
    _lib.call("tamoe_grouped_dgrad", dy.data_ptr(), w.data_ptr(), G, M, K, R, ss.data_ptr(), sr.data_ptr(),
              out.data_ptr(), deriv.data_ptr(), 2, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for g in range(G):
        s, r = start[g], rows[g]
        ref = (dy[s:s + r].float() @ w[g].float()) * deriv[s:s + r].float()
        assert _rel(out[s:s + r], ref) < 1e-2, g


@pytest.mark.parametrize("counts,M,N", [([5, 0, 300, 17, 256], 128, 256), ([1000, 3], 256, 512),
                                        ([16, 0, 272, 48], 512, 256)])
def test_grouped_wgrad(dev, counts, M, N):
    from paper_2302_09915_b200 import _lib
    G = len(counts)
    ss, sr, start, rows, R = _segments(counts, dev)
    a = _tokens(counts, start, R, M, dev, 3)
    b = _tokens(counts, start, R, N, dev, 4)
    out = torch.full((G, M, N), float("nan"), dtype=torch.bfloat16, device=dev)
    _lib.call("tamoe_grouped_wgrad", a.data_ptr(), b.data_ptr(), G, M, N, R, ss.data_ptr(), sr.data_ptr(),
              out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for g in range(G):
        s, r = start[g], rows[g]
        ref = a[s:s + r].float().t() @ b[s:s + r].float()
        if r == 0:
            assert torch.all(out[g] == 0)
        else:
            assert _rel(out[g], ref) < 1e-2, g
