"""ORACLE (test infrastructure only): ctypes front of sv_oracle.c.

Applies a logical gate list (workloads/synthetic.py dict format) one gate at a
time in fp64, exactly as each gate's plain definition states (SURVEY §8(c):
psi = G_L ... G_2 G_1 |0...0>). Named gate kinds are expanded here to their
textbook dense matrices; 'diagonal' multiplies each amplitude by its table entry
(sv_oracle.c orc_apply_diagonal); 'swap' is the 4×4 SWAP
permutation. No fusion, no blocking, no reordering.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

SWAP = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=complex)


def build(force: bool = False) -> str:
    """Compile sv_oracle.c with gcc/OpenMP into oracle/liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.POINTER
        L.orc_apply_controlled.argtypes = [ctypes.c_int, P(ctypes.c_double), ctypes.c_int, P(ctypes.c_int),
                                           ctypes.c_int, P(ctypes.c_int), ctypes.c_uint64, P(ctypes.c_double)]
        L.orc_apply_recip_ry.argtypes = [ctypes.c_int, P(ctypes.c_double), ctypes.c_int, ctypes.c_int,
                                         P(ctypes.c_int), ctypes.c_double, ctypes.c_int, ctypes.c_double]
        L.orc_apply_diagonal.argtypes = [ctypes.c_int, P(ctypes.c_double), ctypes.c_int, P(ctypes.c_int),
                                         P(ctypes.c_double)]
        L.orc_recip_s.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_double]
        L.orc_recip_s.restype = ctypes.c_double
        L.orc_marginal.argtypes = [ctypes.c_int, P(ctypes.c_double), ctypes.c_int, P(ctypes.c_int),
                                   P(ctypes.c_double)]
        L.orc_init_zero.argtypes = [ctypes.c_int, P(ctypes.c_double)]
        L.orc_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(lst):
    arr = (ctypes.c_int * max(1, len(lst)))(*lst)
    return arr


def zero_state(n: int) -> np.ndarray:
    psi = np.empty(1 << n, dtype=np.complex128)
    lib().orc_init_zero(n, _dp(psi.view(np.float64)))
    return psi


def n_threads() -> int:
    return lib().orc_num_threads()


def gate_matrix(g: dict) -> np.ndarray:
    """Dense matrix of a dense/controlled/diagonal/swap gate dict (target block only)."""
    kind = g["kind"]
    if kind in ("dense", "controlled"):
        return np.ascontiguousarray(g["data"], dtype=np.complex128)
    if kind == "diagonal":
        return np.diag(np.asarray(g["data"], dtype=np.complex128))
    if kind == "swap":
        return SWAP.copy()
    raise ValueError(kind)


def apply_gate(psi: np.ndarray, n: int, g: dict) -> None:
    """Apply one logical gate in place (psi: complex128 C-contiguous, length 2^n)."""
    assert psi.dtype == np.complex128 and psi.flags.c_contiguous and psi.size == 1 << n
    L = lib()
    fp = _dp(psi.view(np.float64))
    if g["kind"] == "diagonal":
        d = np.ascontiguousarray(g["data"], dtype=np.complex128)
        t = list(g["targets"])
        assert d.size == 1 << len(t)
        rc = L.orc_apply_diagonal(n, fp, len(t), _ip(t), _dp(d.view(np.float64)))
    elif g["kind"] == "recip_ry":
        clock = list(g["controls"])
        rc = L.orc_apply_recip_ry(n, fp, int(g["targets"][0]), len(clock), _ip(clock), float(g["delta"]),
                                  int(g.get("signed", 1)), float(g.get("snap", 0.0)))
    else:
        U = gate_matrix(g)
        t = list(g["targets"])
        c = list(g.get("controls", [])) if g["kind"] == "controlled" else []
        cv = int(g.get("cvals", (1 << len(c)) - 1)) if c else 0
        assert U.shape == (1 << len(t), 1 << len(t))
        rc = L.orc_apply_controlled(n, fp, len(t), _ip(t), len(c), _ip(c), cv, _dp(U.view(np.float64)))
    if rc != 0:
        raise ValueError(f"oracle rejected gate {g['kind']}")


def run(gates, n: int, psi: np.ndarray | None = None) -> np.ndarray:
    """psi = G_L ... G_1 psi0 (psi0 = |0...0> by default)."""
    psi = zero_state(n) if psi is None else np.ascontiguousarray(psi, dtype=np.complex128).copy()
    for g in gates:
        apply_gate(psi, n, g)
    return psi


def marginal(psi: np.ndarray, n: int, qubits) -> np.ndarray:
    out = np.empty(1 << len(qubits))
    rc = lib().orc_marginal(n, _dp(np.ascontiguousarray(psi).view(np.float64)), len(qubits), _ip(list(qubits)),
                            _dp(out))
    if rc != 0:
        raise ValueError("bad marginal")
    return out


def recip_s(m: int, n_c: int, delta: float, signed: int = 1, snap: float = 0.0) -> float:
    return lib().orc_recip_s(m, n_c, delta, signed, snap)
