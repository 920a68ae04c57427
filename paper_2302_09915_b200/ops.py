"""Python mirror of the reference operator API (namespace tad, gate.hpp:22-97,
solver.hpp target_closed_form, dispatch.hpp device_payload_tokens), executed by
libtamoe.so.  Host-side topology inputs run the library's C++ (fp64, bit-identical
to the reference); routing runs the sm_100a kernels.

Names, argument meaning and error behaviour follow the reference: malformed
inputs raise ValidationError (tad::ValidationError).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import IntEnum

import numpy as np
import torch

from . import _lib
from ._lib import ValidationError, TamoeError  # noqa: F401

_D = ctypes.POINTER(ctypes.c_double)
_L = ctypes.POINTER(ctypes.c_longlong)


class CapacityMode(IntEnum):  # gate.hpp:40
    none = 0
    global_ = 1
    local = 2
    local_proportional = 3


class PenaltyNorm(IntEnum):  # gate.hpp:74
    sum_norm = 0
    softmax = 1


def capacity_mode_from_string(s: str) -> CapacityMode:  # gate.cpp:34-40
    table = {"none": 0, "global": 1, "local": 2, "proportional": 3, "local_proportional": 3}
    if s not in table:
        raise ValidationError(f"unknown capacity mode: {s}")
    return CapacityMode(table[s])


@dataclass
class CapacityPolicy:  # gate.hpp:42-49
    mode: CapacityMode = CapacityMode.none
    capacity_factor: float = 1.0

    def expert_capacity(self, k: int, S: int, N: int, P: int) -> float:
        return self.capacity_factor * float(k) * S * P / N


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ----------------------------------------------------------------------------- host-side inputs
def largest_remainder_round(values, target: int) -> np.ndarray:
    v = _f64(values)
    out = np.zeros(len(v), dtype=np.int64)
    _lib.call("tamoe_largest_remainder_round", v.ctypes.data_as(_D), len(v), int(target), out.ctypes.data_as(_L))
    return out


def penalty_weights(c_hat_row, norm: PenaltyNorm = PenaltyNorm.sum_norm, temperature: float = 0.0) -> np.ndarray:
    c = _f64(c_hat_row)
    p = np.zeros(len(c))
    _lib.call("tamoe_penalty_weights", c.ctypes.data_as(_D), len(c), int(norm), float(temperature),
              p.ctypes.data_as(_D))
    return p


def target_closed_form(beta_hat, N: int, k: int, S: int) -> np.ndarray:
    b = _f64(beta_hat)
    P = b.shape[0]
    out = np.zeros((P, N))
    _lib.call("tamoe_target_closed_form", b.ctypes.data_as(_D), P, N, k, S, out.ctypes.data_as(_D))
    return out


# ------------------------------------------------------------------ measured-topology pipeline (§8(f) row 1)
DEFAULT_SELF_BETA_FLOOR = 0.1  # us/MB, profile.hpp:8


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _levels(levels):
    if levels is None:
        return None, 0
    lv = _i32(levels)
    return lv, int(lv.size)


def fit_profile(samples, P: int):
    """fit_profile (comm_cost.cpp:57-104).  samples: iterable of (src, dst, message_mb, time_us) rows (the
    reference's TransferSample / samples CSV).  Returns (alpha, beta) P x P, NaN for unmeasured pairs."""
    arr = np.asarray(list(samples), dtype=np.float64).reshape(-1, 4)
    src, dst = _i32(arr[:, 0]), _i32(arr[:, 1])
    mb, us = _f64(arr[:, 2]), _f64(arr[:, 3])
    alpha, beta = np.zeros((P, P)), np.zeros((P, P))
    _lib.call("tamoe_fit_profile", src.ctypes.data_as(_lib._I), dst.ctypes.data_as(_lib._I), mb.ctypes.data_as(_D),
              us.ctypes.data_as(_D), int(arr.shape[0]), P, alpha.ctypes.data_as(_D), beta.ctypes.data_as(_D))
    return alpha, beta


def fill_partial_profile(alpha, beta, levels=None, self_beta_floor=DEFAULT_SELF_BETA_FLOOR):
    """fill_partial_profile (profile.cpp:164-233); levels = symmetric tree level vector (root first) or None."""
    a, b = _f64(alpha), _f64(beta)
    P = a.shape[0]
    lv, nl = _levels(levels)
    ao, bo = np.zeros((P, P)), np.zeros((P, P))
    _lib.call("tamoe_fill_partial_profile", a.ctypes.data_as(_D), b.ctypes.data_as(_D), P,
              lv.ctypes.data_as(_lib._I) if lv is not None else None, nl, float(self_beta_floor),
              ao.ctypes.data_as(_D), bo.ctypes.data_as(_D))
    return ao, bo


def smooth_profile(levels, alpha, beta, self_beta_floor=DEFAULT_SELF_BETA_FLOOR):
    """smooth_profile (profile.cpp:46-98) over a symmetric tree -> (alpha_hat, beta_hat, level_alpha, level_beta)."""
    a, b = _f64(alpha), _f64(beta)
    P = a.shape[0]
    lv, nl = _levels(levels)
    ah, bh = np.zeros((P, P)), np.zeros((P, P))
    la, lb = np.full(nl, np.nan), np.full(nl, np.nan)
    _lib.call("tamoe_smooth_profile", lv.ctypes.data_as(_lib._I), nl, a.ctypes.data_as(_D), b.ctypes.data_as(_D), P,
              float(self_beta_floor), ah.ctypes.data_as(_D), bh.ctypes.data_as(_D), la.ctypes.data_as(_D),
              lb.ctypes.data_as(_D))
    keep = ~np.isnan(la)
    return ah, bh, la[keep], lb[keep]


def exchange_cost(alpha, beta, c, d: int, b: int = 2, extra_alpha_rounds: int = 0) -> dict:
    """exchange_cost (comm_cost.cpp:24-55): alpha-beta cost of one exchange of dispatch matrix c [P x N]."""
    a, bb, cc = _f64(alpha), _f64(beta), _f64(c)
    P, N = cc.shape
    pc, summ = np.zeros((P, P)), np.zeros(4)
    _lib.call("tamoe_exchange_cost", a.ctypes.data_as(_D), bb.ctypes.data_as(_D), cc.ctypes.data_as(_D), P, N, d, b,
              extra_alpha_rounds, pc.ctypes.data_as(_D), summ.ctypes.data_as(_D))
    return dict(pair_cost_us=pc, bottleneck_us=summ[0], total_bytes=summ[1], size_exchange_us=summ[2],
                total_estimate_us=summ[3])


def p2p_sweep(nccl_id: bytes, world: int, rank: int, sizes_mb=(1.0, 4.0, 16.0, 64.0, 128.0), reps: int = 5,
              warmup: int = 2):
    """Measured transfers between every ordered pair of the `world` GPUs (collective; call on every rank with
    the same arguments after torch.cuda.set_device).  Returns TransferSample rows (src, dst, message_mb,
    time_us) -- the samples CSV of the reference (profile_io.hpp:8-13)."""
    sz = _f64(list(sizes_mb))
    out = np.zeros((world, world, sz.size, reps))
    idb = ctypes.create_string_buffer(bytes(nccl_id), 128)
    _lib.call("tamoe_p2p_sweep", idb, world, rank, sz.ctypes.data_as(_D), int(sz.size), reps, warmup,
              out.ctypes.data_as(_D))
    return [(i, j, float(sz[s]), float(out[i, j, s, r])) for i in range(world) for j in range(world)
            for s in range(sz.size) for r in range(reps)]


def allgather_blobs(blob: bytes, group=None) -> bytes:
    """All-gather every rank's 128-byte expert-parallel blob over torch.distributed (any backend; gloo needs
    no GPU and lets several ranks share one device) -> world x 128 bytes in rank order."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(blob), group=group)
    assert all(len(b) == 128 for b in out)
    return b"".join(out)


def p2p_sweep_store(world: int, rank: int, sizes_mb=(1.0, 4.0, 16.0, 64.0, 128.0), reps: int = 5,
                    warmup: int = 2, group=None):
    """p2p_sweep with the NCCL-free bootstrap: the probe buffers' IPC handles are exchanged over
    torch.distributed (gloo works; ranks may share a device) and the per-rank rows summed the same way."""
    import torch
    import torch.distributed as dist
    sz = _f64(list(sizes_mb))
    h = ctypes.c_void_p()
    blob = ctypes.create_string_buffer(128)
    _lib.call("tamoe_p2p_probe_create", world, rank, float(sz.max()), ctypes.byref(h), blob)
    try:
        allb = ctypes.create_string_buffer(allgather_blobs(blob.raw, group), 128 * world)
        _lib.call("tamoe_p2p_probe_connect", h, allb, world)
        out = np.zeros((world, world, sz.size, reps))
        _lib.call("tamoe_p2p_probe_sweep", h, sz.ctypes.data_as(_D), int(sz.size), reps, warmup,
                  out.ctypes.data_as(_D))
    finally:
        _lib.call("tamoe_p2p_probe_destroy", h)
    t = torch.from_numpy(out)
    dist.all_reduce(t, group=group)  # every entry was written by exactly one rank
    out = t.numpy()
    return [(i, j, float(sz[s]), float(out[i, j, s, r])) for i in range(world) for j in range(world)
            for s in range(sz.size) for r in range(reps)]


def set_link_emulation(group_size: int, repeat: int) -> None:
    """Emulated heterogeneous topology (BASELINE C5): links between ranks in different groups of `group_size`
    consecutive ranks carry every payload store `repeat` times (1/repeat of the bandwidth).  (0, 1) = off."""
    _lib.call("tamoe_set_link_emulation", int(group_size), int(repeat))


def solve_target_tree(levels, alpha, beta, N: int, k: int, S: int, self_beta_floor=DEFAULT_SELF_BETA_FLOOR):
    """solve_target for a symmetric tree (solver.cpp:119-150, closed-form branch): smooth, then Eq. 8 on
    beta_hat.  Returns (c_hat [P x N], alpha_hat, beta_hat)."""
    ah, bh, _, _ = smooth_profile(levels, alpha, beta, self_beta_floor)
    return target_closed_form(bh, N, k, S), ah, bh


def load_samples_csv(path):
    """Samples CSV of the reference (profile_io.cpp: header src,dst,message_mb,time_us)."""
    with open(path) as f:
        head = f.readline().strip()
        if head != "src,dst,message_mb,time_us":
            raise ValidationError(f"expected CSV header 'src,dst,message_mb,time_us', got '{head}'")
        rows = [tuple(float(v) for v in line.split(",")) for line in f if line.strip()]
    return rows


def save_samples_csv(path, samples):
    with open(path, "w") as f:
        f.write("src,dst,message_mb,time_us\n")
        for s, d, mb, us in samples:
            f.write(f"{int(s)},{int(d)},{mb:.12g},{us:.12g}\n")


def capacity_caps(policy: CapacityPolicy, k: int, S: int, N: int, P: int, c_hat=None) -> np.ndarray:
    ch = _f64(c_hat) if c_hat is not None else None
    caps = np.zeros((P, N), dtype=np.int64)
    _lib.call("tamoe_capacity_caps", int(policy.mode), float(policy.capacity_factor), k, S, N, P,
              ch.ctypes.data_as(_D) if ch is not None else None, caps.ctypes.data_as(_L))
    return caps


def device_payload_tokens(counts) -> np.ndarray:
    c = _f64(counts)
    P, N = c.shape
    out = np.zeros((P, P))
    _lib.call("tamoe_device_payload_tokens", c.ctypes.data_as(_D), P, N, out.ctypes.data_as(_D))
    return out


# ----------------------------------------------------------------------------- device router
R_IDX, R_GATE, R_SCORE, R_KEPT, R_POS, R_COUNTS, R_DROPPED, R_MEAN_PROBS, R_SEG_START, R_SEG_ROWS, R_CLIST, \
    R_LIST_START, R_BAD, R_LOGITS, R_GATE64 = range(15)

_R_DTYPES = {R_IDX: np.int32, R_GATE: np.float32, R_SCORE: np.float64, R_KEPT: np.uint8, R_POS: np.int32,
             R_COUNTS: np.int32, R_DROPPED: np.int32, R_MEAN_PROBS: np.float64, R_SEG_START: np.int32,
             R_SEG_ROWS: np.int32, R_CLIST: np.int32, R_LIST_START: np.int32, R_BAD: np.int32,
             R_LOGITS: np.float32, R_GATE64: np.float64}


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def n_pad(N: int) -> int:
    return (N + 15) // 16 * 16


class Router:
    """Device routing for P processes x S tokens, N experts, top-k (topk_route, gate.cpp:91-202)."""

    def __init__(self, P: int, S: int, N: int, k: int):
        self.P, self.S, self.N, self.k = P, S, N, k
        h = ctypes.c_void_p()
        _lib.lib.tamoe_router_create.argtypes = [ctypes.c_int] * 4 + [ctypes.POINTER(ctypes.c_void_p)]
        _lib.call("tamoe_router_create", P, S, N, k, ctypes.byref(h))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.lib.tamoe_router_destroy(self._h)
            self._h = None

    def _shape(self, what):
        picks = self.P * self.S * self.k
        pn = self.P * self.N
        return {R_IDX: (self.P, self.S, self.k), R_GATE: (self.P, self.S, self.k), R_SCORE: (self.P, self.S, self.k),
                R_GATE64: (self.P, self.S, self.k),
                R_KEPT: (self.P, self.S, self.k), R_POS: (self.P, self.S, self.k), R_COUNTS: (self.P, self.N),
                R_DROPPED: (self.P, self.N), R_MEAN_PROBS: (self.P, self.N), R_SEG_START: (self.N,),
                R_SEG_ROWS: (self.N,), R_CLIST: (picks,), R_LIST_START: (self.N,), R_BAD: (1,)}[what] if what != R_LOGITS \
            else (self.P, self.S, self.N)

    def read(self, what) -> np.ndarray:
        out = np.zeros(self._shape(what), dtype=_R_DTYPES[what])
        self._read_fn(what, out)
        return out

    def _read_fn(self, what, out):
        _lib.call("tamoe_router_read", self._h, what, out.ctypes.data_as(ctypes.c_void_p), out.nbytes, _stream())

    def route_probs(self, probs: torch.Tensor, policy: CapacityPolicy, caps: np.ndarray):
        assert probs.dtype == torch.float64 and probs.is_cuda and probs.is_contiguous()
        c = np.ascontiguousarray(caps, np.int64)
        _lib.call("tamoe_router_route_probs", self._h, ctypes.c_void_p(probs.data_ptr()), int(policy.mode),
                  c.ctypes.data_as(_L), _stream())

    def route_gate(self, x: torch.Tensor, wg: torch.Tensor, policy: CapacityPolicy, caps: np.ndarray,
                   want_probs=False):
        """x bf16 [P*S, d]; wg bf16 [P, n_pad, d].  Returns (logits fp32, probs fp64 or None) on device."""
        d = x.shape[1]
        logits = torch.empty(self.P * self.S, self.N, dtype=torch.float32, device=x.device)
        probs = torch.empty(self.P * self.S, self.N, dtype=torch.float64, device=x.device) if want_probs else None
        c = np.ascontiguousarray(caps, np.int64)
        _lib.call("tamoe_router_route_gate", self._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(wg.data_ptr()),
                  wg.shape[1], d, ctypes.c_void_p(logits.data_ptr()),
                  ctypes.c_void_p(probs.data_ptr()) if probs is not None else None, int(policy.mode),
                  c.ctypes.data_as(_L), _stream())
        return logits, probs

    def permute(self, x: torch.Tensor, r_max: int) -> torch.Tensor:
        xp = torch.full((r_max, x.shape[1]), float("nan"), dtype=x.dtype, device=x.device)
        _lib.call("tamoe_router_permute", self._h, ctypes.c_void_p(x.data_ptr()), x.shape[1],
                  ctypes.c_void_p(xp.data_ptr()), r_max, _stream())
        return xp

    def expert_order(self) -> list:
        """Kept picks per expert in buffer order: list of arrays of pick ids (token*k + slot)."""
        clist, ls, cnt = self.read(R_CLIST), self.read(R_LIST_START), self.read(R_COUNTS).sum(0)
        return [clist[ls[e]:ls[e] + cnt[e]] for e in range(self.N)]


for _name, _args in {
    "tamoe_router_destroy": [ctypes.c_void_p],
    "tamoe_router_route_probs": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, _L, ctypes.c_void_p],
    "tamoe_router_route_gate": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, _L, ctypes.c_void_p],
    "tamoe_router_permute": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                             ctypes.c_void_p],
    "tamoe_router_read": [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p],
    "tamoe_softmax_rows_f64": [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p],
    "tamoe_gate_forward_f64": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.c_void_p, ctypes.c_void_p],
    "tamoe_grad_aux_loss_f64": [ctypes.c_void_p, ctypes.c_void_p, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                ctypes.c_void_p, ctypes.c_void_p],
    "tamoe_loss_balance": [_L, _D, ctypes.c_int, ctypes.c_int, _D],
    "tamoe_loss_topo": [_L, _D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D],
    "tamoe_aux_coefficients": [ctypes.c_int, _L, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D],
}.items():
    getattr(_lib.lib, _name).argtypes = _args
    getattr(_lib.lib, _name).restype = ctypes.c_int


def gate_forward(x: torch.Tensor, W: torch.Tensor):
    """gate_forward (gate.cpp:30-32) on the device: softmax(x W) in fp64 from tcgen05 fp32 logits.
    x [S, d] (any float dtype, rounded to bf16), W [d, N] (reference layout).  Returns fp64 probs [S, N]."""
    S, d = x.shape
    N = W.shape[1]
    dp = (d + 63) // 64 * 64
    np_ = n_pad(N)
    xb = torch.zeros(S, dp, dtype=torch.bfloat16, device="cuda")
    xb[:, :d] = x.to("cuda", torch.bfloat16)
    wg = torch.zeros(1, np_, dp, dtype=torch.bfloat16, device="cuda")
    wg[0, :N, :d] = W.to("cuda").t().to(torch.bfloat16)
    r = Router(1, S, N, 1)
    caps = np.full((1, N), np.iinfo(np.int64).max, dtype=np.int64)
    _, probs = r.route_gate(xb, wg, CapacityPolicy(), caps, want_probs=True)
    return probs


@dataclass
class RoutingResult:  # gate.hpp:32-38, arrays instead of nested vectors
    expert: np.ndarray
    gate_value: np.ndarray
    score: np.ndarray
    kept: np.ndarray
    counts: np.ndarray
    dropped: np.ndarray
    mean_probs: np.ndarray
    order: list  # kept picks per expert in dispatch order


def topk_route(probs, k: int, policy: CapacityPolicy = CapacityPolicy(), c_hat=None):
    """topk_route (gate.cpp:91-202): probs [P, S, N] (or [S, N]) fp64 -> list of per-process RoutingResult
    (a single RoutingResult for 2-D input, like the single-process wrapper gate.cpp:204-207)."""
    single = False
    p = torch.as_tensor(probs, dtype=torch.float64)
    if p.dim() == 2:
        p = p[None]
        single = True
    P, S, N = p.shape
    if k < 1 or k > N:
        raise ValidationError("k must be in [1, N]")
    if policy.mode == CapacityMode.local_proportional and c_hat is None:
        raise ValidationError("local_proportional capacity requires a target pattern")
    caps = capacity_caps(policy, k, S, N, P, c_hat)
    r = Router(P, S, N, k)
    r.route_probs(p.to("cuda").contiguous(), policy, caps)
    idx, gate, score, kept = r.read(R_IDX), r.read(R_GATE64), r.read(R_SCORE), r.read(R_KEPT)
    counts, dropped, mp = r.read(R_COUNTS), r.read(R_DROPPED), r.read(R_MEAN_PROBS)
    order = r.expert_order()
    res = [RoutingResult(idx[i], gate[i], score[i], kept[i].astype(bool), counts[i].astype(np.int64),
                         dropped[i].astype(np.int64), mp[i], order) for i in range(P)]
    return res[0] if single else res


def _cll(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong))


def _cd(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def loss_balance(result: RoutingResult, S: int) -> float:  # gate.cpp:209-214
    c, cp = _cll(result.counts)
    m, mp = _cd(result.mean_probs)
    out = ctypes.c_double()
    _lib.call("tamoe_loss_balance", cp, mp, c.shape[0], S, ctypes.byref(out))
    return out.value


def loss_topo(result: RoutingResult, penalty, N: int, P: int, S: int) -> float:  # gate.cpp:248-255
    pen, pp = _cd(penalty)
    if pen.shape[0] != result.counts.shape[0]:
        raise ValidationError("penalty row size does not match expert count")
    c, cp = _cll(result.counts)
    m, mp = _cd(result.mean_probs)
    out = ctypes.c_double()
    _lib.call("tamoe_loss_topo", cp, mp, pp, c.shape[0], N, P, S, ctypes.byref(out))
    return out.value


def balance_coefficients(result: RoutingResult, S: int) -> np.ndarray:  # gate.cpp:273-278
    c, cp = _cll(result.counts)
    out, op = _cd(np.zeros(c.shape[0]))
    _lib.call("tamoe_aux_coefficients", 0, cp, None, c.shape[0], 0, 0, S, op)
    return out


def topo_coefficients(result: RoutingResult, penalty, N: int, P: int, S: int) -> np.ndarray:  # gate.cpp:280-287
    c, cp = _cll(result.counts)
    pen, pp = _cd(penalty)
    if pen.shape[0] < c.shape[0]:
        raise ValidationError("penalty row size does not match expert count")
    out, op = _cd(np.zeros(c.shape[0]))
    _lib.call("tamoe_aux_coefficients", 1, cp, pp, c.shape[0], N, P, S, op)
    return out


def softmax_rows(logits) -> torch.Tensor:
    """softmax_rows (gate.cpp:12-28) on the device in fp64, the reference's order.  Returns fp64 [S, N] (cuda)."""
    z = torch.as_tensor(logits, dtype=torch.float64).to("cuda").contiguous()
    out = torch.empty_like(z)
    _lib.call("tamoe_softmax_rows_f64", ctypes.c_void_p(z.data_ptr()), z.shape[0], z.shape[1],
              ctypes.c_void_p(out.data_ptr()), _stream())
    return out


def gate_forward_f64(x, W) -> torch.Tensor:
    """gate_forward (gate.cpp:30-32) with the reference's fp64 semantics: bit-identical x W on the device,
    then softmax_rows.  x [S, d], W [d, N] -> fp64 [S, N] (cuda)."""
    xd = torch.as_tensor(x, dtype=torch.float64).to("cuda").contiguous()
    wd = torch.as_tensor(W, dtype=torch.float64).to("cuda").contiguous()
    if xd.shape[1] != wd.shape[0]:
        raise ValidationError("gate_forward: x columns must match W rows")
    out = torch.empty(xd.shape[0], wd.shape[1], dtype=torch.float64, device="cuda")
    _lib.call("tamoe_gate_forward_f64", ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(wd.data_ptr()), xd.shape[0],
              xd.shape[1], wd.shape[1], ctypes.c_void_p(out.data_ptr()), _stream())
    return out


def grad_aux_loss(x, probs, coeff) -> torch.Tensor:
    """grad_aux_loss (gate.cpp:257-271) on the device in fp64: x^T (p (coeff - <coeff, p>)), [d, N]."""
    xd = torch.as_tensor(x, dtype=torch.float64).to("cuda").contiguous()
    pd = torch.as_tensor(probs, dtype=torch.float64).to("cuda").contiguous()
    c, cp = _cd(coeff)
    out = torch.empty(xd.shape[1], pd.shape[1], dtype=torch.float64, device="cuda")
    _lib.call("tamoe_grad_aux_loss_f64", ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(pd.data_ptr()), cp,
              pd.shape[0], xd.shape[1], pd.shape[1], ctypes.c_void_p(out.data_ptr()), _stream())
    return out


def grad_loss_balance(x, probs, result: RoutingResult, S: int) -> torch.Tensor:  # gate.cpp:289-291
    return grad_aux_loss(x, probs, balance_coefficients(result, S))


def grad_loss_topo(x, probs, result: RoutingResult, penalty, N: int, P: int, S: int) -> torch.Tensor:  # :293-296
    return grad_aux_loss(x, probs, topo_coefficients(result, penalty, N, P, S))


# ----------------------------------------------------------------------------- reference-precision layer step
_lib.lib.tamoe_layer_step_f64.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 4 + \
    [_D, _D, ctypes.c_int, ctypes.c_double, ctypes.c_int, _L] + [ctypes.c_void_p] * 4 + [_D, ctypes.c_void_p]
_lib.lib.tamoe_layer_step_f64.restype = ctypes.c_int


def layer_step_f64(x, y, gates, experts, k: int, policy: CapacityPolicy = CapacityPolicy(), c_hat=None,
                   aux_kind: int = 0, aux_weight: float = 1.0, penalties=None, router: Router = None):
    """One step of the reference's MoE layer in its own precision (BASELINE config 1: fp64, linear experts) on
    the device -- the inline step of train() (trainer.cpp:246-356).  x [P, S, d], y [P, S, d_out],
    gates [P, d, N] (GateState::W), experts [N, d, d_out] (U_e); numpy or torch (moved to the GPU as fp64).
    aux_kind 0 balance / 1 topo (penalties [P, N] = penalty_weights of each c_hat row) / 2 compulsory quota
    routing (top-1, quotas from c_hat, balance loss).  Returns a dict with
    task_loss / aux_loss (TrainReport), gate_grads [P, d, N], expert_grads [N, d, d_out], probs [P, S, N],
    y_hat [P, S, d_out] (device fp64 tensors) and the router (routing arrays via Router.read)."""
    dev = torch.device("cuda", torch.cuda.current_device())

    def dt(a):
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a))
        return t.to(device=dev, dtype=torch.float64).contiguous()

    x, y, gates, experts = dt(x), dt(y), dt(gates), dt(experts)
    P, S, d = x.shape
    d_out = y.shape[2]
    N = gates.shape[2]
    if router is None or (router.P, router.S, router.N, router.k) != (P, S, N, k):
        router = Router(P, S, N, k)
    # the reference withholds c_hat from balance routing (trainer.cpp:250)
    caps = capacity_caps(policy, k, S, N, P, c_hat if aux_kind != 0 else None)
    pen = _f64(penalties) if penalties is not None else None
    ch = _f64(c_hat) if (c_hat is not None and aux_kind == 2) else None
    probs = torch.empty(P, S, N, dtype=torch.float64, device=dev)
    gg = torch.empty(P, d, N, dtype=torch.float64, device=dev)
    eg = torch.empty(N, d, d_out, dtype=torch.float64, device=dev)
    yh = torch.empty(P, S, d_out, dtype=torch.float64, device=dev)
    losses = np.zeros(2)
    _lib.call("tamoe_layer_step_f64", router._h, d, d_out, ctypes.c_void_p(x.data_ptr()),
              ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(gates.data_ptr()), ctypes.c_void_p(experts.data_ptr()),
              pen.ctypes.data_as(_D) if pen is not None else None, ch.ctypes.data_as(_D) if ch is not None else None,
              int(aux_kind), float(aux_weight),
              int(policy.mode), caps.ctypes.data_as(_L), ctypes.c_void_p(probs.data_ptr()),
              ctypes.c_void_p(gg.data_ptr()), ctypes.c_void_p(eg.data_ptr()), ctypes.c_void_p(yh.data_ptr()),
              losses.ctypes.data_as(_D), _stream())
    return dict(task_loss=float(losses[0]), aux_loss=float(losses[1]), gate_grads=gg, expert_grads=eg, probs=probs,
                y_hat=yh, router=router)


def train_f64(x, y, gates, experts, k: int, steps: int, lr: float, policy: CapacityPolicy = CapacityPolicy(),
              c_hat=None, aux_kind: int = 0, aux_weight: float = 1.0, penalties=None):
    """train()'s step loop (trainer.cpp:245-416) around layer_step_f64: per step the layer step, then the
    synchronized SGD update in the reference's rounding (W -= lr * grad, product rounded first).  Returns the
    task / aux loss trajectories and the final weights (device fp64)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.as_tensor(np.asarray(gates) if not isinstance(gates, torch.Tensor) else gates).to(dev, torch.float64).clone()
    U = torch.as_tensor(np.asarray(experts) if not isinstance(experts, torch.Tensor) else experts).to(dev, torch.float64).clone()
    task, aux = [], []
    router = None
    for _ in range(steps):
        o = layer_step_f64(x, y, g, U, k, policy, c_hat, aux_kind, aux_weight, penalties, router)
        router = o["router"]
        task.append(o["task_loss"])
        aux.append(o["aux_loss"])
        g.sub_(o["gate_grads"] * lr)
        U.sub_(o["expert_grads"] * lr)
    return dict(task_loss=np.array(task), aux_loss=np.array(aux), gates=g, experts=U)
