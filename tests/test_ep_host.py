"""Expert-parallel host logic on the CPU with world_size-2/4/8 gloo process groups.

Each rank routes its own process' tokens (oracle topk_route over all processes -- the
reference's multi-process semantics), packs its kept picks in (expert, token) order with
16-row padded expert segments, exchanges counts and payload rows (gloo all_to_all stands in
for the NVLink peer stores), and places every source's rows at the offsets of the library's
C++ receive plan (tamoe_ep_plan, the host twin of the device plan kernel).  Each local expert's
receive segment must hold the reference bucket order: ascending (process, token)."""
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
        # sender layout: this rank's kept picks in (expert, token, slot) order, every expert segment padded
        # to 16 rows (-1 = pad); the rows for destination j form one contiguous block
        send_counts = r["counts"][rank].astype(np.int64)
        blocks = []
        for j in range(world):
            blk = []
            for e in range(j * E, (j + 1) * E):
                rows = [rank * 100000 + s * k + jj for s in range(S) for jj in range(k)
                        if r["kept"][rank, s, jj] and r["expert"][rank, s, jj] == e]
                assert len(rows) == send_counts[e]
                blk += rows + [-1] * ((-len(rows)) % 16)
            blocks.append(blk)
        payload = torch.tensor(sum(blocks, []), dtype=torch.int64)
        # counts all-to-all: E counts to every rank
        recv = torch.zeros(world * E, dtype=torch.int64)
        dist.all_to_all_single(recv, torch.tensor(send_counts, dtype=torch.int64))
        recv = recv.numpy().reshape(world, E)
        seg_start, seg_rows, src_off = ep_plan(recv)
        # payload all-to-all (one block per peer: the sender's padded segments of the peer's experts)
        in_split = [len(b) for b in blocks]
        out_split = [int(sum((c + 15) // 16 * 16 for c in recv[i])) for i in range(world)]
        got = torch.empty(sum(out_split), dtype=torch.int64)
        dist.all_to_all_single(got, payload, output_split_sizes=out_split, input_split_sizes=in_split)
        got = got.numpy()
        layout = np.full(int(seg_start[-1] + seg_rows[-1]), -2, np.int64)
        o = 0
        for i in range(world):
            for e in range(E):
                rows = (recv[i, e] + 15) // 16 * 16
                layout[src_off[i, e]:src_off[i, e] + rows] = got[o:o + rows]
                o += rows
        assert np.all(layout != -2)  # the plan tiles the receive buffer exactly
        # each local expert: per source, its picks in token order then padding; in source order this is the
        # reference bucket order (process, token)
        for e in range(E):
            ge = rank * E + e
            seg = layout[seg_start[e]:seg_start[e] + seg_rows[e]]
            order = [v for v in seg if v >= 0]
            ref = [i * 100000 + s * k + j for i in range(world) for s in range(S) for j in range(k)
                   if r["kept"][i, s, j] and r["expert"][i, s, j] == ge]
            assert order == ref, (rank, e)
            for i in range(world):
                c = recv[i, e]
                blk = layout[src_off[i, e]:src_off[i, e] + (c + 15) // 16 * 16]
                assert np.all(blk[c:] == -1) and np.all(blk[:c] >= 0)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as ex:  # noqa: BLE001
        errq.put(f"rank {rank}: {type(ex).__name__}: {ex}")
        raise


@pytest.mark.parametrize("world,mode,k", [(2, 0, 1), (2, 3, 2), (4, 2, 2), (4, 3, 1), (8, 3, 1), (8, 2, 2)])
def test_ep_exchange_layout_gloo(world, mode, k):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    mp.start_processes(_worker, args=(world, _free_port(), mode, k, errq), nprocs=world, join=True,
                       start_method="spawn")
    assert errq.empty(), errq.get()
