"""TAMoELayer: the reference's MoE layer step (trainer.cpp:243-356) on the B200
through libtamoe.so.  Torch is used only to own device memory and streams.

Weight layouts (device, bf16):
  wg  [P, n_pad, d]       gate weights, reference W_i (d x N) transposed, pad rows zero
  w1  linear: [E, d_out, d] (U_e^T);  FFN: [E, f, d]
  w2  FFN: [E, d_out, f]
Reference-layout converters are provided for the parity tests.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .ops import CapacityMode, PenaltyNorm, n_pad, _R_DTYPES, R_LOGITS  # noqa: F401

ACT_NONE, ACT_GELU, ACT_RELU = 0, 1, 2
LOSS_BALANCE, LOSS_TOPO = 0, 1


class _Cfg(ctypes.Structure):
    _fields_ = [("P", ctypes.c_int), ("S", ctypes.c_int), ("d", ctypes.c_int), ("d_out", ctypes.c_int),
                ("N", ctypes.c_int), ("k", ctypes.c_int), ("f", ctypes.c_int), ("act", ctypes.c_int),
                ("cap_mode", ctypes.c_int), ("capacity_factor", ctypes.c_double), ("aux_kind", ctypes.c_int),
                ("aux_weight", ctypes.c_double), ("penalty_norm", ctypes.c_int), ("temperature", ctypes.c_double),
                ("need_dx", ctypes.c_int), ("world_size", ctypes.c_int), ("rank", ctypes.c_int)]


class _IO(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("x", "y", "wg", "w1", "w2", "dwg", "dw1", "dw2", "dx", "y_hat",
                                               "losses")]


_lib.lib.tamoe_layer_create.argtypes = [ctypes.POINTER(_Cfg), ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_void_p)]
_lib.lib.tamoe_layer_destroy.argtypes = [ctypes.c_void_p]
_lib.lib.tamoe_layer_step.argtypes = [ctypes.c_void_p, ctypes.POINTER(_IO), ctypes.c_void_p]
_lib.lib.tamoe_layer_read.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong,
                                      ctypes.c_void_p]
_lib.lib.tamoe_layer_create_ep.argtypes = [ctypes.POINTER(_Cfg), ctypes.POINTER(ctypes.c_double), ctypes.c_char_p,
                                           ctypes.POINTER(ctypes.c_void_p)]
_lib.lib.tamoe_nccl_unique_id.argtypes = [ctypes.c_void_p]
_lib.lib.tamoe_layer_a2a_bytes.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong)]
_lib.lib.tamoe_ep_plan.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_longlong),
                                   ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                   ctypes.POINTER(ctypes.c_longlong)]
_lib.lib.tamoe_layer_launches_per_step.argtypes = [ctypes.c_void_p]
_lib.lib.tamoe_layer_enable_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
_lib.lib.tamoe_layer_timing.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_char_p),
                                        ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                        ctypes.POINTER(ctypes.c_int)]
_lib.lib.tamoe_layer_status.argtypes = [ctypes.c_void_p]
_lib.lib.tamoe_layer_create_ep_begin.argtypes = [ctypes.POINTER(_Cfg), ctypes.POINTER(ctypes.c_double),
                                                 ctypes.POINTER(ctypes.c_void_p), ctypes.c_void_p]
_lib.lib.tamoe_layer_ep_connect.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
_lib.lib.tamoe_layer_create_ep_begin.restype = ctypes.c_int
_lib.lib.tamoe_layer_ep_connect.restype = ctypes.c_int
for _n in ("tamoe_layer_status", "tamoe_layer_create", "tamoe_layer_destroy", "tamoe_layer_step", "tamoe_layer_read",
           "tamoe_layer_launches_per_step", "tamoe_layer_enable_timing", "tamoe_layer_timing", "tamoe_layer_create_ep",
           "tamoe_nccl_unique_id", "tamoe_layer_a2a_bytes", "tamoe_ep_plan"):
    getattr(_lib.lib, _n).restype = ctypes.c_int


@dataclass
class LayerConfig:
    P: int
    S: int
    d: int
    d_out: int
    N: int
    k: int = 1
    f: int = 0
    act: int = ACT_GELU
    cap_mode: int = 0
    capacity_factor: float = 1.0
    aux_kind: int = LOSS_BALANCE
    aux_weight: float = 1.0
    penalty_norm: int = 0
    temperature: float = 0.0
    need_dx: bool = False
    world_size: int = 1
    rank: int = 0

    @property
    def n_pad(self):
        return n_pad(self.N)

    @property
    def experts_local(self):
        return self.N // self.world_size


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for tamoe_layer_create_ep (broadcast it to every rank)."""
    buf = ctypes.create_string_buffer(128)
    _lib.check(_lib.lib.tamoe_nccl_unique_id(buf))
    return buf.raw


def ep_plan(recv):
    """Receive plan for recv[P, E] rows per (source rank, local expert): the segment of each local expert
    (seg_start, seg_rows [E]; expert-major, one 16-row padded block per source in rank order) and where each
    source's rows for it start (src_off [P, E]) -- the host twin of the device plan kernel."""
    r = np.ascontiguousarray(recv, np.int64)
    P, E = r.shape
    st = np.zeros(E, np.int32)
    rows = np.zeros(E, np.int32)
    off = np.zeros(P * E, np.int64)
    LL = ctypes.POINTER(ctypes.c_longlong)
    _lib.check(_lib.lib.tamoe_ep_plan(P, E, r.ctypes.data_as(LL), st.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                      rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), off.ctypes.data_as(LL)))
    return st, rows, off.reshape(P, E)


class TAMoELayer:
    """world_size > 1: expert parallelism.  With `nccl_id` (nccl_unique_id() broadcast from one rank) the
    ranks bootstrap over NCCL (one process per GPU); without it the workspace handles are all-gathered over
    torch.distributed (`group`, any backend -- gloo lets several ranks share one GPU)."""

    def __init__(self, cfg: LayerConfig, c_hat=None, device="cuda", nccl_id: bytes = None, group=None):
        self.cfg = cfg
        self.device = torch.device(device)
        c = _Cfg(cfg.P, cfg.S, cfg.d, cfg.d_out, cfg.N, cfg.k, cfg.f, cfg.act, cfg.cap_mode, cfg.capacity_factor,
                 cfg.aux_kind, cfg.aux_weight, cfg.penalty_norm, cfg.temperature, int(cfg.need_dx), cfg.world_size,
                 cfg.rank)
        self._c_hat = np.ascontiguousarray(c_hat, np.float64) if c_hat is not None else None
        h = ctypes.c_void_p()
        chp = self._c_hat.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if self._c_hat is not None else None
        if cfg.world_size > 1 and nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("expert parallelism needs the 128-byte NCCL id from nccl_unique_id()")
            _lib.check(_lib.lib.tamoe_layer_create_ep(ctypes.byref(c), chp, nccl_id, ctypes.byref(h)))
        elif cfg.world_size > 1:
            from .ops import allgather_blobs
            blob = ctypes.create_string_buffer(128)
            _lib.check(_lib.lib.tamoe_layer_create_ep_begin(ctypes.byref(c), chp, ctypes.byref(h), blob))
            try:
                blobs = allgather_blobs(blob.raw, group)
                _lib.check(_lib.lib.tamoe_layer_ep_connect(h, blobs))
            except BaseException:
                _lib.lib.tamoe_layer_destroy(h)
                raise
        else:
            _lib.check(_lib.lib.tamoe_layer_create(ctypes.byref(c), chp, ctypes.byref(h)))
        self._h = h
        E = cfg.experts_local
        bf = dict(dtype=torch.bfloat16, device=self.device)
        # gradient buffers (reused every step)
        self.dwg = torch.zeros(cfg.P, cfg.n_pad, cfg.d, dtype=torch.float32, device=self.device)
        if cfg.f == 0:
            self.dw1 = torch.zeros(E, cfg.d_out, cfg.d, **bf)
            self.dw2 = None
        else:
            self.dw1 = torch.zeros(E, cfg.f, cfg.d, **bf)
            self.dw2 = torch.zeros(E, cfg.d_out, cfg.f, **bf)
        self.dx = torch.zeros(cfg.P * cfg.S, cfg.d, **bf) if cfg.need_dx else None
        self.losses = torch.zeros(2, dtype=torch.float64, device=self.device)

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.lib.tamoe_layer_destroy(self._h)
            self._h = None

    # ------------------------------------------------------------------ parameters
    def init_params(self, seed=0, gate_std=0.02):
        cfg = self.cfg
        g = torch.Generator(device=self.device).manual_seed(seed)
        E = cfg.experts_local
        wg = torch.zeros(cfg.P, cfg.n_pad, cfg.d, dtype=torch.bfloat16, device=self.device)
        wg[:, :cfg.N] = (torch.randn(cfg.P, cfg.N, cfg.d, generator=g, device=self.device) * gate_std).bfloat16()
        if cfg.f == 0:
            w1 = (torch.randn(E, cfg.d_out, cfg.d, generator=g, device=self.device) / cfg.d ** 0.5).bfloat16()
            w2 = None
        else:
            w1 = (torch.randn(E, cfg.f, cfg.d, generator=g, device=self.device) / cfg.d ** 0.5).bfloat16()
            w2 = (torch.randn(E, cfg.d_out, cfg.f, generator=g, device=self.device) / cfg.f ** 0.5).bfloat16()
        return dict(wg=wg, w1=w1, w2=w2)

    def step(self, x, y, params, y_hat=None, stream=None):
        """Forward + task/aux loss + backward.  Gradients land in self.dwg / dw1 / dw2 / dx;
        losses (device fp64[2]: task, aux) in self.losses.  Stream-ordered; no host sync."""
        io = _IO(_ptr(x), _ptr(y), _ptr(params["wg"]), _ptr(params["w1"]), _ptr(params.get("w2")), _ptr(self.dwg),
                 _ptr(self.dw1), _ptr(self.dw2), _ptr(self.dx), _ptr(y_hat), _ptr(self.losses))
        s = stream if stream is not None else torch.cuda.current_stream()
        _lib.check(_lib.lib.tamoe_layer_step(self._h, ctypes.byref(io), ctypes.c_void_p(s.cuda_stream)))
        return self.losses

    def status(self):
        """Wait for the last step; raise ValidationError("non-finite gate logit") if it saw one
        (gate.cpp:16-17).  The next step() raises it too, once the failing step has completed."""
        _lib.check(_lib.lib.tamoe_layer_status(self._h))

    def read(self, what, shape):
        out = np.zeros(shape, dtype=_R_DTYPES[what])
        _lib.check(_lib.lib.tamoe_layer_read(self._h, what, out.ctypes.data_as(ctypes.c_void_p), out.nbytes,
                                             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return out

    def a2a_bytes(self):
        """Off-rank payload bytes of the last step's all-to-alls: dispatch, combine, grad dispatch, grad combine."""
        out = (ctypes.c_longlong * 4)()
        _lib.check(_lib.lib.tamoe_layer_a2a_bytes(self._h, out))
        return list(out)

    def launches_per_step(self) -> int:
        return _lib.lib.tamoe_layer_launches_per_step(self._h)

    def enable_timing(self, on=True):
        _lib.check(_lib.lib.tamoe_layer_enable_timing(self._h, int(on)))

    def timing(self):
        """{launch name: average ms per step} from the CUDA events recorded on the step stream."""
        cap = 32
        names = (ctypes.c_char_p * cap)()
        ms = (ctypes.c_double * cap)()
        n, steps = ctypes.c_int(), ctypes.c_int()
        _lib.check(_lib.lib.tamoe_layer_timing(self._h, names, ms, cap, ctypes.byref(n), ctypes.byref(steps)))
        st = max(steps.value, 1)
        return {names[i].decode(): ms[i] / st for i in range(n.value)}, steps.value

    # ------------------------------------------------------------------ reference-layout converters
    @staticmethod
    def gates_from_reference(gates, n_pad_, device="cuda"):
        """reference gates [P][d][N] -> wg [P, n_pad, d] bf16."""
        g = torch.as_tensor(np.asarray(gates), dtype=torch.float32)
        P, d, N = g.shape
        wg = torch.zeros(P, n_pad_, d, dtype=torch.bfloat16)
        wg[:, :N] = g.transpose(1, 2).bfloat16()
        return wg.to(device)

    @staticmethod
    def linear_from_reference(U, device="cuda"):
        """reference experts U_e [N][d][d_out] -> w1 [N, d_out, d] bf16."""
        return torch.as_tensor(np.asarray(U), dtype=torch.float32).transpose(1, 2).contiguous().bfloat16().to(device)
