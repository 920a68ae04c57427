"""Expert-parallel host logic on the CPU with world_size-2/4 gloo process groups.

Each rank routes its own process' tokens (oracle topk_route over all processes -- the
reference's multi-process semantics), packs its kept picks in (expert, token) order,
exchanges counts and payload rows with all_to_all, and lays the received rows out with
the library's C++ receive plan (tamoe_ep_plan).  The resulting expert-major layout must
equal the reference bucket order: per expert, ascending (process, token) -- the order
the device kernels and the NCCL exchange reproduce on the GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, k, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_2302_09915_b200 import ops
        from paper_2302_09915_b200.layer import ep_plan
        O = oracle.orc()
        S, N = 96, 8 * world
        E = N // world
        rng = np.random.default_rng(123)  # identical inputs on every rank
        probs = np.stack([O.softmax_rows(l) for l in rng.normal(size=(world, S, N))])
        beta = np.full((world, world), 2.0) + np.eye(world) * -1.5
        c_hat = ops.target_closed_form(beta, N, k, S)
        r = O.topk_route(probs, k, mode, 1.0, c_hat)
        # this rank's kept picks, packed in (expert, token, slot) order = destination-rank-major
        mine = [(r["expert"][rank, s, j], s, j) for s in range(S) for j in range(k) if r["kept"][rank, s, j]]
        mine.sort()
        send_counts = np.zeros(N, np.int64)
        for e, _, _ in mine:
            send_counts[e] += 1
        assert np.array_equal(send_counts, r["counts"][rank])
        payload = torch.tensor([rank * 100000 + s * k + j for _, s, j in mine], dtype=torch.int64)
        # counts all-to-all: E counts to every rank
        recv = torch.zeros(world * E, dtype=torch.int64)
        dist.all_to_all_single(recv, torch.tensor(send_counts, dtype=torch.int64))
        recv = recv.numpy().reshape(world, E)
        seg_start, seg_rows, recv_off = ep_plan(recv)
        # payload all-to-all (one block per destination rank), then place per (source, expert)
        in_split = [int(send_counts[j * E:(j + 1) * E].sum()) for j in range(world)]
        out_split = [int(recv[i].sum()) for i in range(world)]
        got = torch.empty(sum(out_split), dtype=torch.int64)
        dist.all_to_all_single(got, payload, output_split_sizes=out_split, input_split_sizes=in_split)
        got = got.numpy()
        layout = np.full(int(seg_start[-1] + seg_rows[-1]), -1, np.int64)
        o = 0
        for i in range(world):
            for e in range(E):
                c = recv[i, e]
                layout[recv_off[i, e]:recv_off[i, e] + c] = got[o:o + c]
                o += c
        # expected: reference bucket order of each local expert
        for e in range(E):
            ge = rank * E + e
            exp = [i * 100000 + s * k + j for i in range(world) for s in range(S) for j in range(k)
                   if r["kept"][i, s, j] and r["expert"][i, s, j] == ge]
            seg = layout[seg_start[e]:seg_start[e] + seg_rows[e]]
            assert seg_rows[e] % 16 == 0 and seg_rows[e] >= len(exp)
            assert list(seg[:len(exp)]) == exp, (rank, e)
            assert np.all(seg[len(exp):] == -1)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as ex:  # noqa: BLE001
        errq.put(f"rank {rank}: {type(ex).__name__}: {ex}")
        raise


@pytest.mark.parametrize("world,mode,k", [(2, 0, 1), (2, 3, 2), (4, 2, 2), (4, 3, 1)])
def test_ep_exchange_layout_gloo(world, mode, k):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    mp.start_processes(_worker, args=(world, _free_port(), mode, k, errq), nprocs=world, join=True,
                       start_method="spawn")
    assert errq.empty(), errq.get()
