"""Microbenchmark of the tcgen05 grouped GEMM engine vs cuBLAS (torch.matmul) on dense and grouped shapes."""
import sys
import os
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_09915_b200 import _lib  # noqa: E402


def segs(counts):
    rows = [((c + 15) // 16) * 16 for c in counts]
    start = np.concatenate([[0], np.cumsum(rows)[:-1]]).astype(np.int32)
    return (torch.tensor(start, dtype=torch.int32, device="cuda"), torch.tensor(rows, dtype=torch.int32, device="cuda"),
            int(sum(rows)))


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def run(name, counts, M, K, mode="fwd", act=0, store_deriv=False):
    G = len(counts)
    ss, sr, R = segs(counts)
    x = torch.randn(R, K, device="cuda").bfloat16()
    st = torch.cuda.current_stream().cuda_stream
    if mode == "fwd":
        w = torch.randn(G, M, K, device="cuda").bfloat16()
        out = torch.empty(R, M, device="cuda", dtype=torch.bfloat16)
        pre = torch.empty(R, M, device="cuda", dtype=torch.bfloat16) if store_deriv else None
        fn = lambda: _lib.call("tamoe_grouped_fwd", x.data_ptr(), w.data_ptr(), G, M, K, R, ss.data_ptr(),
                               sr.data_ptr(), out.data_ptr(), pre.data_ptr() if pre is not None else None, act, st)
        flops = 2.0 * sum(counts) * M * K
    elif mode == "dgrad":
        w = torch.randn(G, K, M, device="cuda").bfloat16()
        out = torch.empty(R, M, device="cuda", dtype=torch.bfloat16)
        fn = lambda: _lib.call("tamoe_grouped_dgrad", x.data_ptr(), w.data_ptr(), G, M, K, R, ss.data_ptr(),
                               sr.data_ptr(), out.data_ptr(), None, 0, st)
        flops = 2.0 * sum(counts) * M * K
    else:  # wgrad: M x N=K over rows
        a = torch.randn(R, M, device="cuda").bfloat16()
        out = torch.empty(G, M, K, device="cuda", dtype=torch.bfloat16)
        fn = lambda: _lib.call("tamoe_grouped_wgrad", a.data_ptr(), x.data_ptr(), G, M, K, R, ss.data_ptr(),
                               sr.data_ptr(), out.data_ptr(), st)
        flops = 2.0 * sum(counts) * M * K
    ms = timeit(fn)
    # cuBLAS reference: dense equivalent with the same total rows
    A = torch.randn(sum(counts), K, device="cuda").bfloat16()
    B = torch.randn(K, M, device="cuda").bfloat16()
    ms_cb = timeit(lambda: torch.matmul(A, B))
    print(f"{name:34s} {mode:5s} G={G:3d} rows={sum(counts):6d} M={M:5d} K={K:5d}: ours {ms*1e3:8.1f} us "
          f"{flops/ms/1e9:7.1f} TF/s | cuBLAS dense {ms_cb*1e3:8.1f} us {flops/ms_cb/1e9:7.1f} TF/s", flush=True)


def c2_counts():
    """Per-expert token counts of one real C2 layer step (bench.py's inputs and initial weights)."""
    from paper_2302_09915_b200 import ops
    from paper_2302_09915_b200.layer import LayerConfig, TAMoELayer, LOSS_TOPO, ACT_GELU
    cfg = LayerConfig(P=1, S=16384, d=1024, d_out=1024, N=64, k=1, f=4096, act=ACT_GELU, cap_mode=0,
                      aux_kind=LOSS_TOPO, need_dx=True)
    layer = TAMoELayer(cfg, ops.target_closed_form([[1.0]], 64, 1, 16384))
    params = layer.init_params(seed=1)
    g = torch.Generator(device="cuda").manual_seed(100)
    x = torch.randn(16384, 1024, generator=g, device="cuda").bfloat16()
    y = (torch.randn(16384, 1024, generator=g, device="cuda") * 0.5).bfloat16()
    layer.step(x, y, params)
    torch.cuda.synchronize()
    c = [int(v) for v in layer.read(ops.R_COUNTS, (1, 64))[0]]
    del layer
    return c


if __name__ == "__main__":
    rng = np.random.default_rng(0)
    if "--c2" in sys.argv:
        real = c2_counts()
        print("C2 routed counts: min", min(real), "max", max(real), "std", float(np.std(real)), flush=True)
        run("C2 routed fwd1 plain", real, 4096, 1024)
        run("C2 routed fwd1 gelu", real, 4096, 1024, act=1)
        run("C2 routed fwd1 gelu+deriv", real, 4096, 1024, act=1, store_deriv=True)
        if "--act-only" in sys.argv:
            sys.exit(0)
        for nm, cnt in (("uniform 256", [256] * 64), ("C2 routed", real)):
            run(nm + " fwd1", cnt, 4096, 1024)
            run(nm + " fwd2", cnt, 1024, 4096)
            run(nm + " dgrad2", cnt, 4096, 1024, "dgrad")
            run(nm + " dgrad1", cnt, 1024, 4096, "dgrad")
            run(nm + " wgrad2", cnt, 1024, 4096, "wgrad")
            run(nm + " wgrad1", cnt, 4096, 1024, "wgrad")
        sys.exit(0)
    if "--c4" in sys.argv:
        c4 = [int(min(c, 640)) for c in rng.multinomial(32768, [1 / 64] * 64)]
        print("C4 counts: min", min(c4), "max", max(c4), "sum", sum(c4), flush=True)
        run("C4 fwd1", c4, 16384, 4096)
        run("C4 fwd2", c4, 4096, 16384)
        run("C4 dgrad2", c4, 16384, 4096, "dgrad")
        run("C4 dgrad1", c4, 4096, 16384, "dgrad")
        run("C4 wgrad2", c4, 4096, 16384, "wgrad")
        run("C4 wgrad1", c4, 16384, 4096, "wgrad")
        sys.exit(0)
    bal = list(rng.multinomial(16384, [1 / 64] * 64))
    run("dense 16384 rows", [16384], 4096, 1024)
    run("dense 16384 rows", [16384], 1024, 4096)
    run("dense 65536 rows", [65536], 4096, 4096)
    run("64 experts x ~256 (C2 fwd1)", bal, 4096, 1024)
    run("64 experts x ~256 (C2 fwd2)", bal, 1024, 4096)
    run("64 experts x ~256 (C2 dgrad1)", bal, 1024, 4096, "dgrad")
    run("64 experts x ~256 (C2 wgrad1)", bal, 4096, 1024, "wgrad")
    run("8 experts x ~2048 (C2 ep8 fwd1)", list(rng.multinomial(16384, [1 / 8] * 8)), 4096, 1024)
    run("8 experts x ~2048 (C2 ep8 fwd2)", list(rng.multinomial(16384, [1 / 8] * 8)), 1024, 4096)
    run("8 experts x ~2048 (C2 ep8 wgrad)", list(rng.multinomial(16384, [1 / 8] * 8)), 4096, 1024, "wgrad")
