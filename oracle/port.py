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


# ----------------------------------------------------------------------------
# Element vectors (arity-1 forms, kernel.cpp:369-390), numpy restatement of the
# IR that paper_1604_05872_b200/ir.py builds for them (helmholtz_load,
# hyperelasticity_residual, burgers_residual); pinned to the reference's own
# interpreter (interp.cpp:125-154) by tests/test_oracle.py.
# ----------------------------------------------------------------------------
def _geometry(coords):
    x = coords.reshape(-1, 4, 3)
    J = np.transpose(x[:, 1:, :] - x[:, :1, :], (0, 2, 1))  # J_ab = x_{b+1,a} - x_{0,a}
    det = np.linalg.det(J)
    K = np.linalg.inv(J)                                     # K_ab = dX_a/dx_b
    return K, np.abs(det)


def assemble_vector(cfg, tabs, coords: np.ndarray, coeffs: np.ndarray) -> np.ndarray:
    """Element vectors [E][n]: Helmholtz load b_j = int f phi_j; St Venant--Kirchhoff
    residual r_(c,j) = int (F S) : grad(phi_j e_c); Burgers residual
    r_(c,j) = int (u_c/dt + (u.grad) u_c) phi_j + nu grad u_c . grad phi_j."""
    coords = np.asarray(coords, dtype=np.float64)
    coeffs = np.asarray(coeffs, dtype=np.float64)
    K, adet = _geometry(coords)
    W, B, D, P = tabs.W, tabs.B, tabs.D, tabs.P
    wq = W[None, :] * adet[:, None]                          # [E][Q]
    if cfg.kind == 1:                                         # HELMHOLTZ
        f = coeffs @ P.T                                      # [E][Q]
        return np.einsum("eq,qj->ej", f * wq, B)
    ns = B.shape[1]
    Dx = np.einsum("eab,aqj->eqbj", K, D)                     # physical d/dx_b phi_j
    if cfg.kind == 3:                                         # HYPERELASTICITY
        w = coeffs[:, : 3 * ns].reshape(-1, 3, ns)
        mu = coeffs[:, 3 * ns: 3 * ns + 4] @ P.T
        lam = coeffs[:, 3 * ns + 4: 3 * ns + 8] @ P.T
        F = np.eye(3)[None, None] + np.einsum("ecm,eqbm->eqcb", w, Dx)
        E_ = 0.5 * (np.einsum("eqpa,eqpb->eqab", F, F) - np.eye(3)[None, None])
        trE = np.trace(E_, axis1=2, axis2=3)
        S = lam[..., None, None] * trE[..., None, None] * np.eye(3) + 2.0 * mu[..., None, None] * E_
        Pk = np.einsum("eqcp,eqpb->eqcb", F, S)
        r = np.einsum("eqcb,eqbj,eq->ecj", Pk, Dx, wq)
        return r.reshape(-1, 3 * ns)
    if cfg.kind == 4:                                         # BURGERS
        nu, dt = cfg.consts
        u = coeffs[:, : 3 * ns].reshape(-1, 3, ns)
        uq = np.einsum("ecm,qm->eqc", u, B)
        gu = np.einsum("ecm,eqbm->eqcb", u, Dx)
        adv = uq / dt + np.einsum("eqb,eqcb->eqc", uq, gu)
        r = np.einsum("eqc,qj,eq->ecj", adv, B, wq) + nu * np.einsum("eqcb,eqbj,eq->ecj", gu, Dx, wq)
        return r.reshape(-1, 3 * ns)
    raise ValueError(f"no element-vector form for kind {cfg.kind}")
