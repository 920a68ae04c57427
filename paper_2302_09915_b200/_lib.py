"""ctypes binding of libtamoe.so (include/tamoe.h).

The library is the product: every compute entry point below runs the
sm_100a CUDA kernels.  There is no CPU fallback -- if the shared library is
missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import c_double, c_int, c_longlong, c_void_p, POINTER

_HERE = os.path.dirname(os.path.abspath(__file__))
# TAMOE_LIB: alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("TAMOE_LIB") or os.path.join(_HERE, "lib", "libtamoe.so")


class TamoeError(RuntimeError):
    """Internal error (status 1): CUDA / NCCL / runtime failure."""


class ValidationError(ValueError):
    """Mirrors tad::ValidationError (status 2, reference errors.hpp:11-14)."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make lib` (or __graft_entry__.build()); "
            "the TA-MoE layer has no CPU fallback")
    return ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)


lib = _load()

_P = c_void_p
_D = POINTER(c_double)
_L = POINTER(c_longlong)
_I = POINTER(ctypes.c_int)

# name -> argtypes (restype is always int status except where noted)
SIGNATURES = {
    "tamoe_largest_remainder_round": [_D, c_int, c_longlong, _L],
    "tamoe_penalty_weights": [_D, c_int, c_int, c_double, _D],
    "tamoe_target_closed_form": [_D, c_int, c_int, c_int, c_int, _D],
    "tamoe_capacity_caps": [c_int, c_double, c_int, c_int, c_int, c_int, _D, _L],
    "tamoe_device_payload_tokens": [_D, c_int, c_int, _D],
    "tamoe_fit_profile": [_I, _I, _D, _D, c_int, c_int, _D, _D],
    "tamoe_fill_partial_profile": [_D, _D, c_int, _I, c_int, c_double, _D, _D],
    "tamoe_smooth_profile": [_I, c_int, _D, _D, c_int, c_double, _D, _D, _D, _D],
    "tamoe_exchange_cost": [_D, _D, _D, c_int, c_int, c_int, c_int, c_int, _D, _D],
    "tamoe_p2p_sweep": [_P, c_int, c_int, _D, c_int, c_int, c_int, _D],
    "tamoe_set_link_emulation": [c_int, c_int],
    "tamoe_p2p_probe_create": [c_int, c_int, c_double, POINTER(c_void_p), _P],
    "tamoe_p2p_probe_connect": [_P, _P, c_int],
    "tamoe_p2p_probe_sweep": [_P, _D, c_int, c_int, c_int, _D],
    "tamoe_p2p_probe_destroy": [_P],
    "tamoe_grouped_fwd": [_P, _P, c_int, c_int, c_int, c_int, _P, _P, _P, _P, c_int, _P],
    "tamoe_grouped_dgrad": [_P, _P, c_int, c_int, c_int, c_int, _P, _P, _P, _P, c_int, _P],
    "tamoe_grouped_wgrad": [_P, _P, c_int, c_int, c_int, c_int, _P, _P, _P, _P],
}

for _name, _args in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = c_int

lib.tamoe_last_error.restype = ctypes.c_char_p
lib.tamoe_last_error.argtypes = []
lib.tamoe_version.restype = c_int


def check(status: int) -> None:
    if status == 0:
        return
    msg = lib.tamoe_last_error().decode(errors="replace")
    if status == 2:
        raise ValidationError(msg)
    raise TamoeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib, name)(*args))
