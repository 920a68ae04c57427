"""TEST INFRASTRUCTURE ONLY -- ctypes access to the two CPU oracles.

* ``orc``: oracle/build/liboracle.so, the fp64 C restatement of the reference
  hot path (oracle/tamoe_oracle.c).  Always buildable (gcc only).
* ``ref``: oracle/_ref/libtadref.so, the reference library compiled from its
  own sources (oracle/ref.mk).  Present when it was built in the builder
  container (the GPU box receives the prebuilt .so; it never reads
  /root/reference).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this package, and only as the checker.  The product library never loads it.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_longlong, c_ubyte, c_ulonglong, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtadref.so")

_D = POINTER(c_double)
_L = POINTER(c_longlong)
_I = POINTER(c_int)
_U = POINTER(c_ubyte)


def _dp(a):
    return a.ctypes.data_as(_D) if a is not None else None


def _lp(a):
    return a.ctypes.data_as(_L) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(_I)


def _up(a):
    return a.ctypes.data_as(_U)


class OracleError(ValueError):
    pass


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------------------------
class _Layer(ctypes.Structure):
    _fields_ = [("P", c_int), ("S", c_int), ("d", c_int), ("d_out", c_int), ("N", c_int), ("k", c_int),
                ("f", c_int), ("act", c_int), ("cap_mode", c_int), ("cf", c_double), ("aux_kind", c_int),
                ("aux_weight", c_double), ("c_hat", _D), ("penalties", _D)]


class _LayerOut(ctypes.Structure):
    _fields_ = [("probs", _D), ("expert", _I), ("gate", _D), ("score", _D), ("kept", _U), ("counts", _L),
                ("dropped", _L), ("mean_probs", _D), ("y_hat", _D), ("task_loss", c_double),
                ("aux_loss", c_double), ("gate_grads", _D), ("grad_u", _D), ("grad_w1", _D), ("grad_w2", _D),
                ("dx", _D)]


class _Common:
    """Operations shared by the restatement (orc_*) and the reference wrapper (ref_*)."""

    prefix = ""

    def __init__(self, path):
        self.path = path
        self.lib = ctypes.CDLL(path)
        self._err = getattr(self.lib, self.prefix + "last_error")
        self._err.restype = ctypes.c_char_p

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(self._err().decode())

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def softmax_rows(self, logits):
        logits = f64(logits)
        S, N = logits.shape
        out = np.empty_like(logits)
        self._chk(self.fn("softmax_rows")(_dp(logits), S, N, _dp(out)))
        return out

    def gate_forward(self, x, W):
        x, W = f64(x), f64(W)
        S, d = x.shape
        N = W.shape[1]
        out = np.empty((S, N))
        self._chk(self.fn("gate_forward")(_dp(x), _dp(W), S, d, N, _dp(out)))
        return out

    def largest_remainder_round(self, values, target):
        v = f64(values)
        out = np.zeros(len(v), dtype=np.int64)
        self.fn("largest_remainder_round")(_dp(v), len(v), c_longlong(int(target)), _lp(out))
        return out

    def topk_route(self, probs, k, mode=0, cf=1.0, c_hat=None):
        """probs: [P, S, N] (or [S, N] for one process). Returns a dict of arrays shaped [P, ...]."""
        probs = f64(probs)
        if probs.ndim == 2:
            probs = probs[None]
        P, S, N = probs.shape
        ch = f64(c_hat) if c_hat is not None else None
        r = dict(expert=np.zeros((P, S, k), np.int32), gate=np.zeros((P, S, k)), score=np.zeros((P, S, k)),
                 kept=np.zeros((P, S, k), np.uint8), counts=np.zeros((P, N), np.int64),
                 dropped=np.zeros((P, N), np.int64), mean_probs=np.zeros((P, N)))
        self._chk(self.fn("topk_route")(_dp(probs), P, S, N, k, mode, c_double(cf), _dp(ch), _ip(r["expert"]),
                                        _dp(r["gate"]), _dp(r["score"]), _up(r["kept"]), _lp(r["counts"]),
                                        _lp(r["dropped"]), _dp(r["mean_probs"])))
        return r

    def penalty_weights(self, c_hat_row, norm=0, temperature=0.0):
        c = f64(c_hat_row)
        p = np.zeros(len(c))
        self._chk(self.fn("penalty_weights")(_dp(c), len(c), norm, c_double(temperature), _dp(p)))
        return p

    def target_closed_form(self, beta, N, k, S):
        beta = f64(beta)
        P = beta.shape[0]
        out = np.zeros((P, N))
        self._chk(self.fn("target_closed_form")(_dp(beta), P, N, k, S, _dp(out)))
        return out


class Oracle(_Common):
    prefix = "orc_"

    def __init__(self, path=ORACLE_SO):
        super().__init__(path)
        self.lib.orc_loss_balance.restype = c_double
        self.lib.orc_loss_topo.restype = c_double

    def loss_balance(self, counts, mean_probs, S):
        c = np.ascontiguousarray(counts, np.int64)
        m = f64(mean_probs)
        return self.lib.orc_loss_balance(_lp(c), _dp(m), len(c), S)

    def loss_topo(self, counts, mean_probs, penalty, P, S):
        c = np.ascontiguousarray(counts, np.int64)
        m, p = f64(mean_probs), f64(penalty)
        return self.lib.orc_loss_topo(_lp(c), _dp(m), _dp(p), len(c), P, S)

    def grad_aux(self, x, probs, coeff):
        x, probs, coeff = f64(x), f64(probs), f64(coeff)
        S, d = x.shape
        N = probs.shape[1]
        g = np.zeros((d, N))
        self.lib.orc_grad_aux_loss(_dp(x), _dp(probs), _dp(coeff), S, d, N, _dp(g))
        return g

    def topo_coefficients(self, counts, penalty, P, S):
        c = np.ascontiguousarray(counts, np.int64)
        p = f64(penalty)
        out = np.zeros(len(c))
        self.lib.orc_topo_coefficients(_lp(c), _dp(p), len(c), P, S, _dp(out))
        return out

    def balance_coefficients(self, counts, S):
        c = np.ascontiguousarray(counts, np.int64)
        out = np.zeros(len(c))
        self.lib.orc_balance_coefficients(_lp(c), len(c), S, _dp(out))
        return out

    def layer_step(self, x, y, gates, U=None, W1=None, W2=None, k=1, cap_mode=0, cf=1.0, c_hat=None,
                   aux_kind=0, aux_weight=1.0, penalties=None, act=1, want_dx=False):
        """One MoE layer step (trainer.cpp:371-482). x [P,S,d], y [P,S,dout], gates [P,d,N].
        Linear experts: U [N,d,dout].  FFN experts: W1 [N,d,f], W2 [N,f,dout]."""
        x, y, gates = f64(x), f64(y), f64(gates)
        P, S, d = x.shape
        dout = y.shape[2]
        N = gates.shape[2]
        f = 0 if U is not None else W1.shape[2]
        cfg = _Layer(P, S, d, dout, N, k, f, act if f else 0, cap_mode, cf, aux_kind, aux_weight,
                     _dp(f64(c_hat)) if c_hat is not None else None,
                     _dp(f64(penalties)) if penalties is not None else None)
        keep = [c_hat, penalties]
        ch = f64(c_hat) if c_hat is not None else None
        pen = f64(penalties) if penalties is not None else None
        cfg.c_hat, cfg.penalties = _dp(ch), _dp(pen)
        out = dict(probs=np.zeros((P, S, N)), expert=np.zeros((P, S, k), np.int32), gate=np.zeros((P, S, k)),
                   score=np.zeros((P, S, k)), kept=np.zeros((P, S, k), np.uint8), counts=np.zeros((P, N), np.int64),
                   dropped=np.zeros((P, N), np.int64), mean_probs=np.zeros((P, N)), y_hat=np.zeros((P, S, dout)),
                   gate_grads=np.zeros((P, d, N)))
        if f == 0:
            U = f64(U)
            out["grad_u"] = np.zeros_like(U)
        else:
            W1, W2 = f64(W1), f64(W2)
            out["grad_w1"] = np.zeros_like(W1)
            out["grad_w2"] = np.zeros_like(W2)
        if want_dx:
            out["dx"] = np.zeros_like(x)
        o = _LayerOut(_dp(out["probs"]), _ip(out["expert"]), _dp(out["gate"]), _dp(out["score"]),
                      _up(out["kept"]), _lp(out["counts"]), _lp(out["dropped"]), _dp(out["mean_probs"]),
                      _dp(out["y_hat"]), 0.0, 0.0, _dp(out["gate_grads"]), _dp(out.get("grad_u")),
                      _dp(out.get("grad_w1")), _dp(out.get("grad_w2")), _dp(out.get("dx")))
        self._chk(self.lib.orc_layer_step(ctypes.byref(cfg), _dp(x), _dp(y), _dp(gates), _dp(U), _dp(W1), _dp(W2),
                                          ctypes.byref(o)))
        del keep
        out["task_loss"] = o.task_loss
        out["aux_loss"] = o.aux_loss
        return out


class Reference(_Common):
    prefix = "ref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)
        self.lib.ref_loss_balance.restype = c_double
        self.lib.ref_derive_seed.restype = c_ulonglong
        self.lib.ref_derive_seed.argtypes = [c_ulonglong, c_ulonglong]
        self.lib.ref_rng_normal.argtypes = [c_ulonglong, c_int, c_double, _D]
        self.lib.ref_rng_uniform.argtypes = [c_ulonglong, c_int, c_double, c_double, _D]

    # ---- measured-topology pipeline
    def fit_profile(self, samples, P):
        arr = np.asarray(list(samples), dtype=np.float64).reshape(-1, 4)
        src = np.ascontiguousarray(arr[:, 0], np.int32)
        dst = np.ascontiguousarray(arr[:, 1], np.int32)
        mb, us = f64(arr[:, 2]), f64(arr[:, 3])
        a, b = np.zeros((P, P)), np.zeros((P, P))
        self._chk(self.lib.ref_fit_profile(_ip(src), _ip(dst), _dp(mb), _dp(us), int(arr.shape[0]), P, _dp(a), _dp(b)))
        return a, b

    def fill_partial_profile(self, alpha, beta, levels=None, floor=0.1):
        a, b = f64(alpha), f64(beta)
        P = a.shape[0]
        lv = np.ascontiguousarray(levels if levels is not None else [0], np.int32)
        ao, bo = np.zeros((P, P)), np.zeros((P, P))
        self._chk(self.lib.ref_fill_partial_profile(_dp(a), _dp(b), P, _ip(lv), 0 if levels is None else len(lv),
                                                      c_double(floor), _dp(ao), _dp(bo)))
        return ao, bo

    def smooth_profile(self, levels, alpha, beta, floor=0.1):
        a, b = f64(alpha), f64(beta)
        P = a.shape[0]
        lv = np.ascontiguousarray(levels, np.int32)
        ah, bh = np.zeros((P, P)), np.zeros((P, P))
        self._chk(self.lib.ref_smooth_profile(_ip(lv), len(lv), _dp(a), _dp(b), P, c_double(floor), _dp(ah), _dp(bh)))
        return ah, bh

    def device_groups(self, levels, device, P):
        lv = np.ascontiguousarray(levels, np.int32)
        g = np.full(P, -1, np.int32)
        self._chk(self.lib.ref_device_groups(_ip(lv), len(lv), device, _ip(g)))
        return g

    def exchange_cost(self, alpha, beta, c, d, b=2, rounds=0):
        a, bb, cc = f64(alpha), f64(beta), f64(c)
        P, N = cc.shape
        pc, summ = np.zeros((P, P)), np.zeros(4)
        self._chk(self.lib.ref_exchange_cost(_dp(a), _dp(bb), _dp(cc), P, N, d, b, rounds, _dp(pc), _dp(summ)))
        return dict(pair_cost_us=pc, bottleneck_us=summ[0], total_bytes=summ[1], size_exchange_us=summ[2],
                    total_estimate_us=summ[3])

    def rng_normal(self, seed, n, scale=1.0):
        out = np.zeros(n)
        self.lib.ref_rng_normal(seed, n, scale, _dp(out))
        return out

    def rng_uniform(self, seed, n, lo, hi):
        out = np.zeros(n)
        self.lib.ref_rng_uniform(seed, n, lo, hi, _dp(out))
        return out

    def derive_seed(self, seed, stream):
        return int(self.lib.ref_derive_seed(seed, stream))

    def loss_balance(self, counts, mean_probs, S):
        c = np.ascontiguousarray(counts, np.int64)
        m = f64(mean_probs)
        return self.lib.ref_loss_balance(_lp(c), _dp(m), len(c), S)

    def loss_topo(self, counts, mean_probs, penalty, P, S):
        c = np.ascontiguousarray(counts, np.int64)
        m, p = f64(mean_probs), f64(penalty)
        out = c_double()
        self._chk(self.lib.ref_loss_topo(_lp(c), _dp(m), _dp(p), len(c), P, S, ctypes.byref(out)))
        return out.value

    def grad_loss_topo(self, x, probs, counts, mean_probs, penalty, P):
        x, probs, m, p = f64(x), f64(probs), f64(mean_probs), f64(penalty)
        c = np.ascontiguousarray(counts, np.int64)
        S, d = x.shape
        N = probs.shape[1]
        g = np.zeros((d, N))
        self._chk(self.lib.ref_grad_loss_topo(_dp(x), _dp(probs), _lp(c), _dp(m), _dp(p), S, d, N, P, _dp(g)))
        return g

    def grad_loss_balance(self, x, probs, counts, mean_probs):
        x, probs, m = f64(x), f64(probs), f64(mean_probs)
        c = np.ascontiguousarray(counts, np.int64)
        S, d = x.shape
        N = probs.shape[1]
        g = np.zeros((d, N))
        self._chk(self.lib.ref_grad_loss_balance(_dp(x), _dp(probs), _lp(c), _dp(m), S, d, N, _dp(g)))
        return g

    def gen_synthetic(self, seed, P, S, d, d_out, N=4, k=1, clusters=4, separation=3.0, within_std=1.0,
                      noise_std=0.05, map_spread=1.0):
        x = np.zeros((P, S, d))
        y = np.zeros((P, S, d_out))
        means = np.zeros((clusters, d))
        maps = np.zeros((clusters, d, d_out))
        self._chk(self.lib.ref_gen_synthetic(c_ulonglong(seed), P, S, d, d_out, N, k, clusters,
                                             c_double(separation), c_double(within_std), c_double(noise_std),
                                             c_double(map_spread), _dp(x), _dp(y), _dp(means), _dp(maps)))
        return x, y, means, maps

    def train(self, x, y, gates, experts, kind=0, cap_mode=0, cf=1.0, c_hat=None, norm=0, temperature=0.0,
              lr=0.05, steps=1, aux_weight=1.0, switch_step=None, k=1):
        x, y, gates, experts = f64(x), f64(y), f64(gates), f64(experts)
        P, S, d = x.shape
        dout = y.shape[2]
        N = gates.shape[2]
        ch = f64(c_hat) if c_hat is not None else None
        tl, al, dr = np.zeros(steps), np.zeros(steps), np.zeros(steps)
        d0, d1 = np.zeros((P, N)), np.zeros((P, N))
        sec = c_double()
        ss = -(10 ** 7) if switch_step is None else switch_step
        self._chk(self.lib.ref_train(P, S, d, dout, N, k, _dp(x), _dp(y), _dp(gates), _dp(experts), kind, cap_mode,
                                     c_double(cf), _dp(ch), norm, c_double(temperature), c_double(lr), steps,
                                     c_double(aux_weight), ss, _dp(tl), _dp(al), _dp(dr), _dp(d0), _dp(d1),
                                     ctypes.byref(sec)))
        return dict(task_loss=tl, aux_loss=al, dropped_rate=dr, initial_dispatch=d0, final_dispatch=d1,
                    seconds=sec.value)


_ORC = None
_REF = None


def orc() -> Oracle:
    global _ORC
    if _ORC is None:
        _ORC = Oracle()
    return _ORC


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> Reference:
    global _REF
    if _REF is None:
        _REF = Reference()
    return _REF
