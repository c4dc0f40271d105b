"""ctypes wrapper of oracle/libfemoracle.so (femoracle.c) -- TEST INFRASTRUCTURE.

The CPU restatement of the element kernels used as the parity checker.  Only
tests/, __graft_entry__.smoke() and bench.py's CPU legs may import it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfemoracle.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        d = C.POINTER(C.c_double)
        L.femoracle_assemble.argtypes = [C.c_int, C.c_long, C.c_int, C.c_int, C.c_int, d, d, d, d,
                                         d, d, d, C.c_long, d]
        L.femoracle_assemble.restype = C.c_int
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def assemble(cfg, tabs, coords: np.ndarray, coeffs: np.ndarray) -> np.ndarray:
    """Element matrices [E][n][n] for ``cfg`` (see femoracle.c)."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    E = coords.shape[0]
    A = np.empty((E, cfg.n, cfg.n))
    W = np.ascontiguousarray(tabs.W)
    B = np.ascontiguousarray(tabs.B)
    D = np.ascontiguousarray(tabs.D)
    P = np.ascontiguousarray(tabs.P)
    consts = np.array(list(cfg.consts) + [0.0, 0.0], dtype=np.float64)
    rc = lib().femoracle_assemble(cfg.kind, E, W.shape[0], B.shape[1], P.shape[1], _p(W), _p(B),
                                  _p(D), _p(P), _p(consts), _p(coords), _p(coeffs),
                                  coeffs.shape[1], _p(A))
    if rc != 0:
        raise RuntimeError("femoracle_assemble failed")
    return A
