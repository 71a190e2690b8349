"""Brute-force full-operator simulation for tiny circuits (≤ ~10 qubits), test-only.

Independent of oracle/sv_oracle.c: each gate is embedded as a tensor contraction
(np.tensordot on a [2]*n state tensor) rather than an index loop, and the whole
circuit unitary is the product of the embedded operators. Used to pin the oracle
(SURVEY §8(c) "brute-force full-unitary product on ≤ 6 qubits").
"""
from __future__ import annotations

import numpy as np

from oracle.closed_form import recip_table


def _block_matrix(g: dict):
    """(matrix over qubit list, qubit list) with qubit list[0] = LSB of the matrix index."""
    kind = g["kind"]
    if kind == "dense":
        return np.asarray(g["data"], complex), list(g["targets"])
    if kind == "diagonal":
        return np.diag(np.asarray(g["data"], complex)), list(g["targets"])
    if kind == "swap":
        M = np.zeros((4, 4), complex)
        for i in range(4):
            j = ((i & 1) << 1) | (i >> 1)
            M[j, i] = 1.0
        return M, list(g["targets"])
    if kind == "controlled":
        U = np.asarray(g["data"], complex)
        k = len(g["targets"])
        c = len(g["controls"])
        M = np.eye(1 << (k + c), dtype=complex)
        cv = int(g.get("cvals", (1 << c) - 1))
        lo = cv << k
        M[lo:lo + (1 << k), lo:lo + (1 << k)] = U
        return M, list(g["targets"]) + list(g["controls"])
    if kind == "recip_ry":
        clock = list(g["controls"])
        nc = len(clock)
        s = recip_table(nc, g["delta"], g.get("signed", 1), g.get("snap", 0.0))
        th = 2 * np.arcsin(s)
        M = np.zeros((2 << nc, 2 << nc), complex)
        for m in range(1 << nc):
            c, sn = np.cos(th[m] / 2), np.sin(th[m] / 2)
            i0, i1 = 2 * m, 2 * m + 1           # index = anc + 2*m
            M[i0, i0], M[i0, i1], M[i1, i0], M[i1, i1] = c, -sn, sn, c
        return M, [g["targets"][0]] + clock
    raise ValueError(kind)


def apply(states: np.ndarray, n: int, g: dict) -> np.ndarray:
    """states: (2^n, B) columns; returns gate ⊗ I applied to every column."""
    M, qs = _block_matrix(g)
    k = len(qs)
    B = states.shape[1]
    T = states.reshape([2] * n + [B])           # axis a <-> qubit n-1-a
    Mt = M.reshape([2] * (2 * k))               # out axes (q_{k-1}..q_0), in axes (q_{k-1}..q_0)
    in_axes = [n - 1 - q for q in reversed(qs)]
    R = np.tensordot(Mt, T, axes=(list(range(k, 2 * k)), in_axes))
    # R axes: k output axes (q_{k-1}..q_0) then the remaining state axes in order
    rest = [a for a in range(n + 1) if a not in in_axes]
    order = [None] * (n + 1)
    for i, a in enumerate(in_axes):
        order[a] = i
    for i, a in enumerate(rest):
        order[a] = k + i
    return np.transpose(R, order).reshape(1 << n, B)


def circuit_unitary(gates, n: int) -> np.ndarray:
    U = np.eye(1 << n, dtype=complex)
    for g in gates:
        U = apply(U, n, g)
    return U


def run(gates, n: int, psi0=None) -> np.ndarray:
    psi = np.zeros((1 << n, 1), complex)
    if psi0 is None:
        psi[0, 0] = 1
    else:
        psi[:, 0] = psi0
    for g in gates:
        psi = apply(psi, n, g)
    return psi[:, 0]
