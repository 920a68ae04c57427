"""Expert parallelism on the GPU box, never skipped.

* >= 2 GPUs: one rank per GPU, NCCL bootstrap (world = min(GPUs, 4)).
* 1 GPU: the ranks share the device -- the NCCL-free bootstrap (tamoe_layer_create_ep_begin /
  tamoe_layer_ep_connect, handles all-gathered over gloo) runs the same kernels, peer stores and device
  barriers with several ranks per GPU.  World 4 and 8 run that way on any box (8 ranks = 2 per GPU on a
  4-GPU lease), and a 500-step loop checks that every step is bitwise identical (device barrier without
  per-thread fences, csrc/ep_plan.cu).
Host-side logic is covered on the CPU by tests/test_ep_host.py (gloo)."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(script, world, args=(), store=False, timeout=600):
    env = dict(os.environ)
    if store:
        env["TAMOE_EP_BOOTSTRAP"] = "store"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", script), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-4000:]
    return r.stdout


CASES = ["ffn_prop", "linear_none", "ffn_local", "ffn_global", "ffn_prop_throttled"]


@pytest.mark.parametrize("case", CASES)
def test_ep_parity(case):
    """One rank per GPU over NCCL when the box has >= 2 GPUs, else 2 ranks sharing the GPU."""
    n = torch.cuda.device_count()
    world = min(n, 4) if n >= 2 else 2
    out = _run("ep_worker.py", world, [case])
    assert "EP_PARITY_OK" in out, out[-2000:]


@pytest.mark.parametrize("case", ["ffn_prop", "ffn_global", "linear_none"])
def test_ep_parity_world4_store_bootstrap(case):
    """World 4 through the NCCL-free bootstrap on whatever GPUs the box has (ranks share devices)."""
    out = _run("ep_worker.py", 4, [case], store=True)
    assert "EP_PARITY_OK" in out and "bootstrap=store" in out, out[-2000:]


def test_ep_parity_world8_shared():
    """8 ranks (BASELINE C2-C5 name 8 GPUs): 64 experts, 8 per rank, parity vs the oracle's P=8 step."""
    out = _run("ep_worker.py", 8, ["ffn_prop"], store=True, timeout=900)
    assert "EP_PARITY_OK" in out and "world=8" in out, out[-2000:]


def test_ep_stress_500_steps_bitwise():
    """500 replays of the EP step (device barriers, peer stores) -- every step bitwise identical."""
    out = _run("ep_worker.py", 2, ["ffn_prop", "500"], store=True, timeout=900)
    assert "EP_PARITY_OK" in out and "steps=500" in out, out[-2000:]


def test_p2p_sweep():
    """Sweep -> fit_profile -> fill -> closed form (§8(f) row 1): NCCL bootstrap on >= 2 GPUs, the store
    bootstrap with 2 ranks on one GPU otherwise (then every "link" is a local HBM copy)."""
    n = torch.cuda.device_count()
    world = min(n, 4) if n >= 2 else 2
    out = _run("p2p_worker.py", world)
    assert "P2P_SWEEP_OK" in out, out[-2000:]


def test_p2p_sweep_store_bootstrap():
    out = _run("p2p_worker.py", 2, store=True)
    assert "P2P_SWEEP_OK" in out and "bootstrap=store" in out, out[-2000:]


@pytest.mark.parametrize("kind,cap", [(1, 3), (0, 2)])
def test_ep_train_matches_reference(kind, cap):
    """Expert-parallel train() (tamoe_layer_train) at world 2 vs the reference's train() at P = 2: loss
    trajectories, dispatch, and per-step modelled vs measured exchange (§8(f) rows 2 and 4)."""
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    n = torch.cuda.device_count()
    world = 2
    out = _run("ep_train_worker.py", world, [str(kind), str(cap)], store=n < world)
    assert "EP_TRAIN_OK" in out, out[-2000:]
