"""Loader for oracle/gate_logits.c (TEST INFRASTRUCTURE -- see oracle/__init__.py).

Compiles the C file with gcc on first use (or when the source is newer than the .so).
Flags: -O2 -ffp-contract=off (no implicit contraction beyond the explicit fmaf), no
-ffast-math, OpenMP over tokens (tokens are independent; the per-(t,e) chain order is fixed).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gate_logits.c")
_SO = os.path.join(_HERE, "liboracle_gate.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                        "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"], check=True)
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_gate_logits.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                            ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
        _lib.oracle_gate_logits.restype = None
    return _lib


def gate_logits(x: np.ndarray, wg: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    wg = np.ascontiguousarray(wg, dtype=np.float32)
    T, d = x.shape
    d2, E = wg.shape
    assert d == d2
    out = np.empty((T, E), dtype=np.float32)
    lib().oracle_gate_logits(x.ctypes.data, wg.ctypes.data, T, d, E, out.ctypes.data)
    return out
