#!/usr/bin/env python
"""TA-MoE layer benchmark (BASELINE.json metric: MoE-layer tokens/sec).

One step = one MoE-layer forward + task/aux loss + backward over T tokens per GPU
(trainer.cpp:371-482 on the device): tcgen05 gate, routing, permute, expert FFN
(grouped tcgen05), combine + MSE, expert dgrad/wgrad, gate backward incl. dX.
Workload at N=1: BASELINE config 2 (GPT-MoE d=1024, ffn=4096, 64 experts, top-1,
16384 tokens/GPU, bf16), synthetic data, random-init weights.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N (one rank per GPU, NCCL).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer tokens/sec (fwd+bwd)"
A2A_CEILING_GBS = 587.0  # best concurrent 4-GPU all-to-all measured on this pool (scripts/p2p_bench.cu)
C2 = dict(S=16384, d=1024, d_out=1024, f=4096, N=64, k=1)
# BASELINE configs timed by bench.py: c2 (default, the headline) and c4 (large layer, proportional capacity)
CONFIGS = {
    "c2": dict(C2, cap=0, cf=1.0, name="C2: GPT-MoE layer d_model=1024 ffn=4096 64 experts top-1",
               extra="capacity none"),
    "c4": dict(S=16384, d=4096, d_out=4096, f=16384, N=64, k=2, cap=3, cf=1.25,
               name="C4: large MoE layer d_model=4096 ffn=16384 64 experts top-2",
               extra="local proportional capacity cf 1.25"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--tokens", type=int, default=None, help="tokens per GPU (default: the config's)")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return dict(hbm=j["hbm_gbs"], bf16=j["bf16_tflops"], bf16_sus=j.get("bf16_tflops_sustained", j["bf16_tflops"]),
                    source="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, source="fallback")


def bind_to_gpu_numa(cuda_index):
    """Pin this process to the CPUs NVML reports as local to the GPU, so the pinned host buffers of the e2e leg
    are first-touched on the GPU's NUMA node (with 4-8 ranks on one host, remote-node buffers halve H2D).
    Returns the CPU count bound to, or None when NVML / the affinity call is unavailable."""
    try:
        import pynvml as nv
        import torch
        nv.nvmlInit()
        pr = torch.cuda.get_device_properties(cuda_index)
        h = nv.nvmlDeviceGetHandleByPciBusId(
            f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0")
        ncpu = os.cpu_count() or 1
        words = nv.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (int(m) >> b) & 1}
        cpus &= set(os.sched_getaffinity(0))
        if not cpus:
            return None
        os.sched_setaffinity(0, cpus)
        return len(cpus)
    except Exception:
        return None


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled DURING the timed region through NVML every ~1 ms
    (nvidia-smi -lms needs ~1 s to produce its first line; a timed region is tens of ms).  The device is
    matched to the CUDA ordinal by PCI bus id."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, cuda_index, period_s=0.001):
        self.idx = cuda_index
        self.period = period_s
        self.rows = []
        self.err = None
        self.h = None
        self.nv = None
        self.stop = threading.Event()
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            self.nv = nv
            try:
                pr = torch.cuda.get_device_properties(cuda_index)
                bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
                self.h = nv.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = nv.nvmlDeviceGetHandleByIndex(cuda_index)
            self.max_sm = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception as e:  # no NVML: reported, not fatal
            self.err = f"nvml unavailable: {e}"

    def sample_now(self):
        """One synchronous sample from the launching thread (taken while queued steps still run on the GPU), so a
        short timed region has samples even when the sampler thread is starved of the GIL."""
        if self.h is None:
            return True
        nv = self.nv
        reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        try:
            self.rows.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM), reasons(self.h)))
            return True
        except Exception as e:
            self.err = str(e)
            return False

    def _sample(self):
        while not self.stop.is_set():
            if not self.sample_now():
                return
            time.sleep(self.period)

    def __enter__(self):
        if self.h is not None:
            self.t = threading.Thread(target=self._sample, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.h is not None:
            self.stop.set()
            self.t.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no samples"]}
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for _, m in self.rows for n, bit in self.REASONS.items() if m & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(self.max_sm), "reasons": reasons,
                "samples": len(self.rows), "source": "nvml, 1 ms period, timed region only"}


class NvlinkCounters:
    """NVLink data-payload byte counters of this GPU (NVML field values NVLINK_THROUGHPUT_DATA_TX / _RX, per link,
    cumulative KiB), read around the timed region: hardware evidence for the exchange's off-rank bytes, without a
    profiler on the multi-rank run."""

    def __init__(self, cuda_index, links=18):
        self.h = None
        self.err = None
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            self.nv = nv
            pr = torch.cuda.get_device_properties(cuda_index)
            self.h = nv.nvmlDeviceGetHandleByPciBusId(
                f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0")
            self.fields = [(f, l) for l in range(links)
                           for f in (nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX)]
            self.read()
        except Exception as e:  # noqa: BLE001
            self.h, self.err = None, f"nvml nvlink counters unavailable: {e}"

    def read(self):
        """(tx_bytes, rx_bytes) summed over the links."""
        if self.h is None:
            return None
        vals = self.nv.nvmlDeviceGetFieldValues(self.h, self.fields)
        tx = rx = 0
        for i, v in enumerate(vals):
            if v.nvmlReturn != 0:
                continue
            x = v.value.ullVal * 1024
            if i % 2 == 0:
                tx += x
            else:
                rx += x
        return tx, rx


# ------------------------------------------------------------------------------------------ CPU baseline
def host_threads(bytes_per_thread=1.6e9):
    """The host cores this process may use (up to 64), bounded by memory: each concurrent reference train() at the C2
    shape holds ~1.6 GB (its copies of the 64 fp64 expert maps and their gradients), and the arm must not drive
    the box out of memory -- at most 40 % of MemAvailable / the cgroup headroom."""
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    avail = None
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    avail = int(ln.split()[1]) * 1024
    except OSError:
        pass
    try:
        with open("/sys/fs/cgroup/memory.max") as f:
            lim = f.read().strip()
        if lim != "max":
            with open("/sys/fs/cgroup/memory.current") as f:
                head = int(lim) - int(f.read().strip())
            avail = head if avail is None else min(avail, head)
    except (OSError, ValueError):
        pass
    if avail is None:
        return min(ncpu, 16)
    # capped at 64 threads so the arm's K-step run stays within a few minutes on many-core hosts
    return max(1, min(ncpu, 64, int(0.4 * avail / bytes_per_thread)))


REF_TOKENS_PER_THREAD = 2048  # per-step fixed cost of the reference's train() (~0.6 s: 64 fp64 expert-gradient
# allocations, trainer.cpp:258, and SGD over 64 M doubles, trainer.cpp:414-416) is < 10 % of a 2,048-token step,
# so the measured rate is within 10 % of the reference's large-S per-token asymptote


def reference_cpu(tokens_per_thread=REF_TOKENS_PER_THREAD, threads=None, steps=1, seed=0, warm=True):
    """The reference's own train() step (compiled from its sources, oracle/_ref) at the C2 router/expert
    shape (d=1024, N=64, top-1; the reference expert is a linear d->d map, trainer.cpp:284-289),
    run concurrently on `threads` host threads (the reference is single-threaded).  Falls back to the
    C restatement (oracle port) when oracle/_ref is absent."""
    import numpy as np
    import oracle
    threads = threads or host_threads()
    d, N, k = C2["d"], C2["N"], C2["k"]
    rng = np.random.default_rng(seed)
    U = rng.normal(size=(N, d, d)) / np.sqrt(d)
    kind = "reference" if oracle.ref_available() else "port"
    datas = []
    for t in range(threads):
        x = rng.normal(size=(1, tokens_per_thread, d))
        y = rng.normal(size=(1, tokens_per_thread, d)) * 0.5
        g = rng.normal(size=(1, d, N)) * 0.02
        datas.append((x, y, g))

    if kind == "reference":
        R = oracle.ref()

        def one(i, out, nsteps):
            x, y, g = datas[i]
            out[i] = R.train(x, y, g, U, kind=0, lr=0.0, steps=nsteps, k=k)["seconds"]
    else:
        Orc = oracle.orc()

        def one(i, out, nsteps):
            x, y, g = datas[i]
            t0 = time.perf_counter()
            for _ in range(nsteps):
                Orc.layer_step(x, y, g, U=U, k=k)
            out[i] = time.perf_counter() - t0

    def run(nsteps):
        out = [0.0] * threads
        ths = [threading.Thread(target=one, args=(i, out, nsteps)) for i in range(threads)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        return out

    # keep the reference's large matrices in the malloc heap instead of fresh mmaps per call, so page
    # faults (setup) do not swamp the step cost; then one warm-up round
    try:
        import ctypes
        libc = ctypes.CDLL("libc.so.6")
        libc.mallopt(-3, 1 << 30)  # M_MMAP_THRESHOLD
        libc.mallopt(-1, 1 << 34)  # M_TRIM_THRESHOLD
    except OSError:
        pass
    if warm:
        run(1)
    # per-thread cost of one step = train(steps=2) - train(steps=1): setup (weight copies) cancels
    wall = []
    for _ in range(steps):
        t1 = run(1)
        t2 = run(2)
        wall.append(max(max(b - a for a, b in zip(t1, t2)), 1e-9))
    per_step = statistics.median(wall)
    tok = threads * tokens_per_thread
    return dict(value=tok / per_step, unit="tokens/s", cores=threads, kind=kind,
                sample=f"{threads} concurrent threads x {tokens_per_thread} tokens "
                       f"(d=1024, N=64, top-1, reference linear expert d->d, fp64); per-step time = "
                       f"train(steps=2) - train(steps=1) per thread, slowest thread, median of {steps}; "
                       f"{tokens_per_thread} tokens per thread keep the per-step fixed cost (expert-gradient "
                       f"allocation + SGD over 64 M doubles) below 10 % of the step")


def workload_config(S, world, name="c2"):
    """The `config` object of both arms (same workload, metric and unit)."""
    c = CONFIGS[name]
    wgb = 2 * 2 * c["N"] * c["d"] * c["f"] / 1e9
    return {"workload": f"{c['name']} {S} tokens/GPU, GELU FFN experts, topo aux loss, {c['extra']}, dX on",
            "tokens_per_gpu": S, "global_tokens": world * S,
            "parallelism": f"ep{world} (expert parallel, {c['N'] // world} experts per GPU, "
                           "all-to-all as NVLink peer stores fused into the kernels)" if world > 1
            else f"single GPU, {c['N']} local experts",
            "l2": f"working set > L2 ({wgb:.2f} GB expert weights + activations per step)"}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    # median of 3 (train(2) - train(1) at 2,048 tokens per thread): about two minutes whatever --steps says
    r = reference_cpu(steps=3)
    line = {"metric": METRIC, "value": r["value"], "unit": r["unit"], "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.tokens or CONFIGS[args.config]["S"], world, args.config),
            "cpu_baseline": {"value": r["value"], "unit": r["unit"], "cores": r["cores"], "kind": r["kind"],
                             "sample": r["sample"]},
            "e2e": {"value": r["value"], "unit": r["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


# ------------------------------------------------------------------------------------------ our arm
_REAL_STDOUT = None


def hold_stdout():
    """Native libraries (NCCL's version banner, CUDA / driver messages) write to fd 1 directly; the contract is
    ONE JSON line on stdout, so fd 1 points at stderr until emit() restores it for that line."""
    global _REAL_STDOUT
    sys.stdout.flush()
    _REAL_STDOUT = os.dup(1)
    os.dup2(2, 1)


def emit(line):
    sys.stdout.flush()
    if _REAL_STDOUT is not None:
        os.dup2(_REAL_STDOUT, 1)
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    hold_stdout()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    import torch.distributed as dist

    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # stdout carries exactly one JSON line: NCCL's own log lines (e.g. NCCL_DEBUG=VERSION) go to stderr
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    from paper_2302_09915_b200 import ops
    from paper_2302_09915_b200.layer import LayerConfig, TAMoELayer, LOSS_TOPO, ACT_GELU, nccl_unique_id

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    W = CONFIGS[args.config]
    S = args.tokens or W["S"]
    cfg = LayerConfig(P=1, S=S, d=W["d"], d_out=W["d_out"], N=W["N"], k=W["k"], f=W["f"], act=ACT_GELU,
                      cap_mode=W["cap"], capacity_factor=W["cf"], aux_kind=LOSS_TOPO, need_dx=True,
                      world_size=world, rank=rank)
    # homogeneous NVSwitch profile: every off-diagonal beta equal, so c_hat is the even pattern
    beta = [[1.0] * world for _ in range(world)]
    c_hat = ops.target_closed_form(beta, W["N"], W["k"], S)
    nccl_id = None
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    layer = TAMoELayer(cfg, c_hat, nccl_id=nccl_id)
    params = layer.init_params(seed=1 + rank)
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    x = torch.randn(S, cfg.d, generator=g, device=dev).bfloat16()
    y = (torch.randn(S, cfg.d_out, generator=g, device=dev) * 0.5).bfloat16()
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    # ---------------- device-timed region (inputs resident in HBM)
    for _ in range(args.warmup):
        layer.step(x, y, params)
    torch.cuda.synchronize()
    # NVML set-up and events before the barrier: any host work between the barrier and the first timed launch
    # on one rank is time the other ranks' GPUs spend in the step's device barrier (max over ranks)
    clk = ClockSampler(local)
    nvl = NvlinkCounters(local) if world > 1 else None
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with clk:
        # one untimed step enqueued ahead of ev0: its device barriers re-align the ranks' GPUs after any host skew
        layer.step(x, y, params)
        ev0.record(stream)
        for _ in range(args.steps):
            layer.step(x, y, params)
        ev1.record(stream)
        clk.sample_now()  # after ev1 is enqueued: an NVML call between launches stalls this rank's stream
        torch.cuda.synchronize()
    barrier()
    nvl0 = nvl1 = None
    if nvl is not None:
        # NVLink byte counters over a separate, untimed run of the same steps (an NVML read between the barrier and
        # the timed launches would bill host skew to the ranks waiting in the step's device barriers)
        torch.cuda.synchronize()
        nvl0 = nvl.read()
        for _ in range(args.steps):
            layer.step(x, y, params)
        torch.cuda.synchronize()
        nvl1 = nvl.read()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    clocks = clk.summary()
    if world > 1:  # every rank sampled its own GPU: union of reasons, per-rank medians
        allc = [None] * world
        dist.all_gather_object(allc, clocks)
        clocks = dict(clocks)
        clocks["reasons"] = sorted({r for c in allc for r in c["reasons"]})
        clocks["per_rank_sm_mhz"] = [c["sm_mhz"] for c in allc]
    # phase breakdown: separate eager steps with CUDA events between launches (not part of `value`)
    layer.enable_timing(True)
    for _ in range(max(3, min(args.steps, 10))):
        layer.step(x, y, params)
    torch.cuda.synchronize()
    phases, tsteps = layer.timing()
    layer.enable_timing(False)
    a2a = None
    if world > 1:
        # off-rank payload bytes per step: dispatch stores, combine loads, dO stores, dX loads (all NVLink
        # peer-memory accesses inside the compute kernels; NCCL only for counts + barriers)
        nbytes = layer.a2a_bytes()
        disp_ms = phases.get("a2a_dispatch", 0.0)  # fused permute + dispatch kernel + barrier
        comb_ms = phases.get("combine_loss", 0.0) + phases.get("a2a_barrier_combine", 0.0)  # dO stores
        a2a = {"offrank_bytes_per_step": {"dispatch": nbytes[0], "o_return": nbytes[1], "dO_stores": nbytes[2],
                                          "dx_return": nbytes[3]},
               "dispatch_ms": disp_ms, "combine_ms": comb_ms,
               "dispatch_bus_gbs": nbytes[0] / (disp_ms / 1e3) / 1e9 if disp_ms > 0 else 0.0,
               "combine_bus_gbs": nbytes[2] / (comb_ms / 1e3) / 1e9 if comb_ms > 0 else 0.0,
               "peak_gbs": 900.0, "measured_peer_peak_gbs": 698.0, "measured_a2a_gbs": A2A_CEILING_GBS,
               "note": "all payload moves as NVLink peer stores fused into compute kernels: dispatch (permute kernel "
                       "-> owner's layout), O return (owner's fwd2 epilogue -> home rank), dO (combine kernel -> "
                       "owner), dX return (owner's dgrad1 epilogue -> home rank); bus GB/s = off-rank bytes / phase "
                       "time (CUDA events, incl. the phase's device barrier); peaks: NVLink 5 nominal 900 GB/s per "
                       "direction; measured on this pool (profiles/r01_p2p_bench.txt): single pair 698 GB/s, best "
                       "4-GPU all-to-all of any engine (SM stores, TMA bulk, pulls, copy engines) 587 GB/s per GPU"}
        for kk in ("dispatch", "combine"):
            a2a[kk + "_frac_of_nvlink_peak"] = a2a[kk + "_bus_gbs"] / 900.0
            a2a[kk + "_frac_of_measured_a2a"] = a2a[kk + "_bus_gbs"] / A2A_CEILING_GBS
        ok = bool(nvl0 and nvl1)
        tx = (nvl1[0] - nvl0[0]) / args.steps if ok else -1.0
        rx = (nvl1[1] - nvl0[1]) / args.steps if ok else -1.0
        txm, rxm = max_over_ranks(tx), max_over_ranks(rx)  # collective on every rank
        if txm > 0:
            algo = float(sum(nbytes))
            a2a["nvlink_counters"] = {
                "source": "NVML NVLINK_THROUGHPUT_DATA_TX/RX field values, all links, read around an untimed "
                          "repeat of the timed steps (payload bytes; max over ranks)",
                "tx_bytes_per_step": txm, "rx_bytes_per_step": rxm,
                "algorithmic_offrank_bytes_per_step": algo,
                "tx_over_algorithmic": txm / algo if algo else None,
                "tx_gbs_over_step": txm / (ms / 1e3) / 1e9}
        else:
            a2a["nvlink_counters"] = {"unavailable": (nvl.err if nvl and nvl.err else
                                                      "NVLink throughput counters not exposed on this box (NVML "
                                                      "field values stay 0, nvidia-smi nvlink -gt d: N/A); see "
                                                      "profiles/ for the ncu nvltx/nvlrx byte counters")}
    losses = layer.losses.cpu().tolist()
    value = world * S / (ms / 1e3)

    # ---------------- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # every rank's pinned host buffers on its GPU's NUMA node (first touch after binding); the CPU-baseline
        # leg afterwards gets all host cores back
        all_cpus = os.sched_getaffinity(0)
        numa_cpus = bind_to_gpu_numa(local)
        xh = x.cpu().pin_memory()
        yh = y.cpu().pin_memory()
        lh = torch.zeros(2, dtype=torch.float64).pin_memory()
        xb = [torch.empty_like(x), torch.empty_like(x)]
        yb = [torch.empty_like(y), torch.empty_like(y)]
        copy = torch.cuda.Stream(device=dev)
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        done = [torch.cuda.Event(), torch.cuda.Event()]

        def prefetch(i):
            b = i % 2
            copy.wait_event(done[b])
            with torch.cuda.stream(copy):
                xb[b].copy_(xh, non_blocking=True)
                yb[b].copy_(yh, non_blocking=True)
            ready[b].record(copy)

        for e in done:
            e.record(stream)
        for i in range(args.warmup):
            prefetch(i)
            stream.wait_event(ready[i % 2])
            layer.step(xb[i % 2], yb[i % 2], params)
            done[i % 2].record(stream)
            lh.copy_(layer.losses, non_blocking=True)
        torch.cuda.synchronize()
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        prefetch(0)
        for i in range(args.steps):
            if i + 1 < args.steps:
                prefetch(i + 1)
            stream.wait_event(ready[i % 2])
            layer.step(xb[i % 2], yb[i % 2], params)
            done[i % 2].record(stream)
            lh.copy_(layer.losses, non_blocking=True)
        t1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = max_over_ranks(t0.elapsed_time(t1) / args.steps)
        h2d = int(x.numel() * 2 + y.numel() * 2)
        # the host link's own roofline: the same pinned H2D copies alone, timed on the copy stream
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        barrier()
        c0.record(copy)
        for i in range(5):
            with torch.cuda.stream(copy):
                xb[i % 2].copy_(xh, non_blocking=True)
                yb[i % 2].copy_(yh, non_blocking=True)
        c1.record(copy)
        torch.cuda.synchronize()
        barrier()
        h2d_ms = max_over_ranks(c0.elapsed_time(c1) / 5)
        h2d_gbs = h2d / (ems / 1e3) / 1e9
        h2d_peak = h2d / (h2d_ms / 1e3) / 1e9
        e2e = {"value": world * S / (ems / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 16,
               "ms_per_step": ems, "note": "pinned host x,y copied H2D every step on a copy stream "
                                           "(double-buffered, overlapping the previous step), losses read back "
                                           "D2H every step; bound = max(device step, H2D copy)",
               "h2d_gbs": h2d_gbs, "h2d_alone_gbs": h2d_peak, "h2d_frac_of_alone": h2d_gbs / h2d_peak,
               "h2d_alone_ms_per_step": h2d_ms, "host_numa_cpus": numa_cpus}
        try:
            os.sched_setaffinity(0, all_cpus)
        except OSError:
            pass

    # ---------------- roofline of the dominant kernel family (expert grouped GEMMs, tcgen05)
    # Per launch: FLOPs 2*R*d*f and ALGORITHMIC bytes = this GPU's expert weights (E = N/world experts, read for
    # fwd/dgrad, dW written for wgrad) + the token-row operands / outputs, R = T*k rows (every rank routes T*k
    # picks, so a rank receives T*k rows on average).  bound = whichever roofline time is larger.
    pk = peaks()
    T = S
    R = T * cfg.k
    E_loc = cfg.N // world
    wb = 2.0 * E_loc * cfg.d * cfg.f
    rows = {"fwd1": R * (cfg.d + 2 * cfg.f), "fwd2": R * (cfg.f + cfg.d_out), "dgrad2": R * (cfg.d_out + 2 * cfg.f),
            "wgrad2": R * (cfg.d_out + cfg.f), "wgrad1": R * (cfg.f + cfg.d), "dgrad1": R * (cfg.f + cfg.d)}
    bytes_per_launch = sum(wb + 2.0 * v for v in rows.values()) / len(rows)
    flop_per_launch = 2.0 * R * cfg.d * cfg.f
    gemm_names = [n for n in phases if n.startswith("expert_")]
    gemm_ms = sum(phases[n] for n in gemm_names)
    # six GEMMs per step whether they run as six launches or chained (fwd1+fwd2 and dgrad2+dgrad1 share a launch)
    avg_s = gemm_ms / len(rows) / 1e3
    tflops = flop_per_launch / avg_s / 1e12 if avg_s > 0 else 0.0
    gbs = bytes_per_launch / avg_s / 1e9 if avg_s > 0 else 0.0
    t_hbm = bytes_per_launch / (pk["hbm"] * 1e9)
    t_tc = flop_per_launch / (pk["bf16_sus"] * 1e12)
    hbm_bound = t_hbm > t_tc
    chained = any(n in phases for n in ("expert_fwd12", "expert_dgrad21"))
    roof = {"kernel": "expert grouped GEMMs (tcgen05; fwd1, fwd2, dgrad2, wgrad2, wgrad1, dgrad1" +
                      (" -- fwd1+fwd2 and dgrad2+dgrad1 as chained persistent launches, TAMOE_CHAIN=1)" if chained
                       else ": six persistent launches per step)"),
            "bound": "hbm" if hbm_bound else "tensor",
            "achieved": gbs if hbm_bound else tflops,
            "peak": pk["hbm"] if hbm_bound else pk["bf16_sus"],
            "unit": "GB/s" if hbm_bound else "TFLOP/s",
            "frac": (gbs / pk["hbm"]) if hbm_bound else (tflops / pk["bf16_sus"]),
            "peak_kind": f"{pk['source']} " + ("HBM copy bandwidth" if hbm_bound else "bf16 sustained"),
            "traffic": None,
            "algorithmic_bytes_per_launch": bytes_per_launch, "flop_per_launch": flop_per_launch,
            "arithmetic_intensity_flop_per_byte": flop_per_launch / bytes_per_launch,
            "ridge_flop_per_byte": pk["bf16_sus"] * 1e12 / (pk["hbm"] * 1e9),
            "avg_gemm_ms": avg_s * 1e3, "tensor_tflops": tflops, "tensor_frac_burst": tflops / pk["bf16"],
            "tensor_frac_sustained": tflops / pk["bf16_sus"],
            "hbm_gbs": gbs, "hbm_frac": gbs / pk["hbm"],
            "note": "launch durations from CUDA events on the step stream around each GEMM (eager phase steps); "
                    "rows = nominal T*k (picks dropped by capacity not subtracted, pad rows not added)"}
    # the newest committed ncu --set full capture of the same step (scripts/profile_round.sh -> ncu_summary.py)
    import glob
    caps = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_gemm_traffic.json")))
    prof_traffic = caps[-1] if caps else ""
    if prof_traffic and world == 1:
        with open(prof_traffic) as f:
            roof["traffic"] = json.load(f).get("traffic_bytes_per_launch")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config == "c2":
        try:
            cpu = reference_cpu(steps=1, warm=False)  # ~30 s of host work
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (randn tokens/targets, random-init weights)",
                "config": workload_config(S, world, args.config),
                "roofline": roof, "all_to_all": a2a, "phases_ms": phases, "timed_steps_for_phases": tsteps,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": layer.launches_per_step() * args.steps,
                "clocks": clocks, "losses_last_step": losses}
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
