"""GPU-backed train() -- the reference's experiment entry point (trainer.hpp:45-106, trainer.cpp:183-452) on
the device layer.

    rep = train(TrainConfig(P=4, S=1024, d=512, d_out=512, N=8, k=2, steps=100, lr=0.05,
                            capacity=ops.CapacityPolicy(ops.CapacityMode.local_proportional, 1.25)),
                x, y, gates, experts, kind=LossKind.topo, c_hat=c_hat)

x [P][S][d], y [P][S][d_out] and the initial weights (reference layouts: gates [P][d][N], linear experts
[N][d][d_out], or FFN (W1 [N][d][f], W2 [N][f][d_out])) are host arrays; they are rounded to bf16 once,
trained on the GPU (fp32 master weights, plain SGD in the reference's order) and the trained weights come
back in the same layouts.  The report has the reference's TrainReport fields.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional

import numpy as np
import torch

from . import _lib, ops
from .layer import _Cfg, ACT_NONE, ACT_GELU, n_pad


class LossKind(IntEnum):
    balance = 0
    topo = 1
    compulsory = 2


class _Opts(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("steps", ctypes.c_int), ("lr", ctypes.c_double),
                ("has_switch", ctypes.c_int), ("switch_step", ctypes.c_int), ("report_window", ctypes.c_int),
                ("bytes_per_element", ctypes.c_double), ("alpha_hat", ctypes.c_void_p),
                ("beta_hat", ctypes.c_void_p), ("intra_groups", ctypes.c_void_p)]


class _Report(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("task_loss", "aux_loss", "comm_us", "dropped_rate",
                                               "initial_dispatch", "final_dispatch", "tv_rows")] + \
               [("summary", ctypes.c_double * 9), ("comm_measured_us", ctypes.c_void_p)]


_lib.lib.tamoe_train.argtypes = [ctypes.POINTER(_Cfg), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_Opts),
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.POINTER(_Report), ctypes.c_void_p]
_lib.lib.tamoe_train.restype = ctypes.c_int
_lib.lib.tamoe_layer_train.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_Opts),
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.POINTER(_Report), ctypes.c_void_p]
_lib.lib.tamoe_layer_train.restype = ctypes.c_int


@dataclass
class TrainConfig:
    """TrainConfig (trainer.hpp:47-68) + ModelDims (trainer.hpp:12-20); f > 0 selects GELU FFN experts."""
    P: int
    S: int
    d: int
    d_out: int
    N: int
    k: int = 1
    f: int = 0
    lr: float = 0.05
    steps: int = 2000
    aux_weight: float = 1.0
    norm: ops.PenaltyNorm = ops.PenaltyNorm.sum_norm
    temperature: float = 0.0
    capacity: ops.CapacityPolicy = field(default_factory=ops.CapacityPolicy)
    switch_step: Optional[int] = None
    report_window: int = 100
    bytes_per_element: float = 4.0
    alpha_hat: Optional[np.ndarray] = None
    beta_hat: Optional[np.ndarray] = None
    intra_groups: Optional[list] = None  # per device: the devices of its innermost group


@dataclass
class TrainReport:
    """TrainReport (trainer.hpp:75-99)."""
    loss: LossKind
    task_loss: np.ndarray
    aux_loss: np.ndarray
    comm_us: np.ndarray
    dropped_rate: np.ndarray
    initial_dispatch: np.ndarray
    final_dispatch: np.ndarray
    tv_rows: np.ndarray
    tv_initial_mean: float
    tv_final_mean: float
    col_balance_max_dev: float
    min_expert_load: float
    intra_share: float
    final_task_loss: float
    final_aux_loss: float
    final_comm_us: float
    dropped_total_rate: float
    weights: dict
    comm_measured_us: np.ndarray = None  # per step: the measured exchange (CUDA events, max over ranks)


def _dptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def train(cfg: TrainConfig, x, y, gates, experts=None, W1=None, W2=None, kind: LossKind = LossKind.balance,
          c_hat=None, device="cuda") -> TrainReport:
    P, S, d, dout, N, k, f = cfg.P, cfg.S, cfg.d, cfg.d_out, cfg.N, cfg.k, cfg.f
    dev = torch.device(device)
    xt = torch.as_tensor(np.asarray(x, np.float32).reshape(P * S, d)).bfloat16().to(dev)
    yt = torch.as_tensor(np.asarray(y, np.float32).reshape(P * S, dout)).bfloat16().to(dev)
    np_ = n_pad(N)
    wg = torch.zeros(P, np_, d, dtype=torch.bfloat16)
    wg[:, :N] = torch.as_tensor(np.asarray(gates, np.float32)).transpose(1, 2).bfloat16()
    wg = wg.to(dev).contiguous()
    if f == 0:
        w1 = torch.as_tensor(np.asarray(experts, np.float32)).transpose(1, 2).contiguous().bfloat16().to(dev)
        w2 = None
    else:
        w1 = torch.as_tensor(np.asarray(W1, np.float32)).transpose(1, 2).contiguous().bfloat16().to(dev)
        w2 = torch.as_tensor(np.asarray(W2, np.float32)).transpose(1, 2).contiguous().bfloat16().to(dev)
    c = _Cfg(P, S, d, dout, N, k, f, ACT_NONE if f == 0 else ACT_GELU, int(cfg.capacity.mode),
             float(cfg.capacity.capacity_factor), int(kind == LossKind.topo), float(cfg.aux_weight), int(cfg.norm),
             float(cfg.temperature), 0, 1, 0)
    o, arrs, d0, d1, tv, r = _opts_report(cfg, kind, P)
    ch = np.ascontiguousarray(c_hat, np.float64) if c_hat is not None else None
    s = torch.cuda.current_stream(dev)
    _lib.check(_lib.lib.tamoe_train(ctypes.byref(c), ch.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
                                    if ch is not None else None, ctypes.byref(o), xt.data_ptr(), yt.data_ptr(),
                                    wg.data_ptr(), w1.data_ptr(), w2.data_ptr() if w2 is not None else None,
                                    ctypes.byref(r), ctypes.c_void_p(s.cuda_stream)))
    sm = list(r.summary)
    weights = dict(gates=wg[:, :N].float().transpose(1, 2).cpu().numpy())
    if f == 0:
        weights["experts"] = w1.float().transpose(1, 2).cpu().numpy()
    else:
        weights["W1"] = w1.float().transpose(1, 2).cpu().numpy()
        weights["W2"] = w2.float().transpose(1, 2).cpu().numpy()
    return TrainReport(kind, arrs["task_loss"], arrs["aux_loss"], arrs["comm_us"], arrs["dropped_rate"], d0, d1,
                       tv if c_hat is not None else np.zeros(0), *sm, weights=weights,
                       comm_measured_us=arrs["comm_measured_us"])


def _opts_report(cfg: "TrainConfig", kind, P: int):
    """ctypes options + report buffers for P (global) processes."""
    N = cfg.N
    ah = np.ascontiguousarray(cfg.alpha_hat, np.float64) if cfg.alpha_hat is not None else None
    bh = np.ascontiguousarray(cfg.beta_hat, np.float64) if cfg.beta_hat is not None else None
    ig = None
    if cfg.intra_groups is not None:
        ig = np.zeros((P, P), np.int32)
        for i, members in enumerate(cfg.intra_groups):
            ig[i, list(members)] = 1
    o = _Opts(int(kind), cfg.steps, cfg.lr, int(cfg.switch_step is not None),
              int(cfg.switch_step) if cfg.switch_step is not None else 0, cfg.report_window, cfg.bytes_per_element,
              _dptr(ah), _dptr(bh), _dptr(ig))
    o._keep = (ah, bh, ig)  # the arrays must outlive the call
    arrs = {n: np.zeros(cfg.steps) for n in ("task_loss", "aux_loss", "comm_us", "dropped_rate", "comm_measured_us")}
    d0, d1, tv = np.zeros((P, N)), np.zeros((P, N)), np.zeros(P)
    r = _Report(*[_dptr(arrs[n]) for n in ("task_loss", "aux_loss", "comm_us", "dropped_rate")], _dptr(d0), _dptr(d1),
                _dptr(tv), (ctypes.c_double * 9)(), _dptr(arrs["comm_measured_us"]))
    return o, arrs, d0, d1, tv, r


def train_layer(layer, params: dict, x: torch.Tensor, y: torch.Tensor, cfg: "TrainConfig",
                kind: LossKind = LossKind.balance, c_hat=None) -> TrainReport:
    """train() on an existing TAMoELayer -- the expert-parallel training loop: every rank calls it with its own
    process' x / y (device bf16), its gate replica and its local experts (params, updated in place) and the same
    cfg / c_hat [P_global, N]; the report covers all processes and is identical on every rank
    (tamoe_layer_train)."""
    lc = layer.cfg
    Pg = lc.P * lc.world_size
    o, arrs, d0, d1, tv, r = _opts_report(cfg, kind, Pg)
    ch = np.ascontiguousarray(c_hat, np.float64) if c_hat is not None else None
    s = torch.cuda.current_stream(x.device)
    w2 = params.get("w2")
    _lib.check(_lib.lib.tamoe_layer_train(layer._h, ch.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
                                          if ch is not None else None, ctypes.byref(o), x.data_ptr(), y.data_ptr(),
                                          params["wg"].data_ptr(), params["w1"].data_ptr(),
                                          w2.data_ptr() if w2 is not None else None, ctypes.byref(r),
                                          ctypes.c_void_p(s.cuda_stream)))
    sm = list(r.summary)
    return TrainReport(kind, arrs["task_loss"], arrs["aux_loss"], arrs["comm_us"], arrs["dropped_rate"], d0, d1,
                       tv if c_hat is not None else np.zeros(0), *sm, weights=params,
                       comm_measured_us=arrs["comm_measured_us"])
