"""Seeded synthetic inputs shared by the oracle tests and the GPU parity tests.

Only random numbers and data layout live here, no HHL/method arithmetic:
complex-Gaussian states, Haar-random unitaries (QR of a complex Gaussian with the
standard phase fix), and random gate lists in the plain-dict gate format below.

Gate dict format (data only; both sides parse it with their own code):
    {"kind": "dense",      "targets": [t0..], "data": (2^k,2^k) complex}
    {"kind": "controlled", "targets": [..], "controls": [..], "cvals": int, "data": (2^k,2^k)}
    {"kind": "diagonal",   "targets": [..], "data": (2^k,) complex}     # diag entries
    {"kind": "recip_ry",   "targets": [anc], "controls": [clock LSB first],
                           "delta": float, "signed": 0|1, "snap": float}
    {"kind": "swap",       "targets": [a, b]}
targets[0] is the least-significant bit of the matrix row/column index; qubit q
is bit q of the amplitude index (little-endian).
"""
from __future__ import annotations

import numpy as np


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def random_state(n: int, seed: int) -> np.ndarray:
    """Normalised complex-Gaussian state of 2^n amplitudes (complex128)."""
    g = rng(seed)
    v = g.standard_normal(1 << n) + 1j * g.standard_normal(1 << n)
    return v / np.linalg.norm(v)


def haar_unitary(k: int, g: np.random.Generator) -> np.ndarray:
    """Haar-random 2^k × 2^k unitary (QR of a complex Gaussian, R-diagonal phase fix)."""
    d = 1 << k
    z = (g.standard_normal((d, d)) + 1j * g.standard_normal((d, d))) / np.sqrt(2)
    q, r = np.linalg.qr(z)
    ph = np.diag(r) / np.abs(np.diag(r))
    return q * ph[None, :]


def random_phases(k: int, g: np.random.Generator) -> np.ndarray:
    return np.exp(2j * np.pi * g.random(1 << k))


def random_gate(width: int, g: np.random.Generator, kinds=("dense", "controlled", "diagonal", "swap"),
                kmax: int = 3, diag_kmax: int = 4) -> dict:
    kind = kinds[g.integers(len(kinds))]
    if kind == "swap":
        a, b = g.choice(width, 2, replace=False)
        return {"kind": "swap", "targets": [int(a), int(b)]}
    if kind == "diagonal":
        k = int(g.integers(1, min(diag_kmax, width) + 1))
        t = [int(x) for x in g.choice(width, k, replace=False)]
        return {"kind": "diagonal", "targets": t, "data": random_phases(k, g)}
    if kind == "controlled" and width >= 2:
        k = int(g.integers(1, min(kmax, width - 1) + 1))
        c = int(g.integers(1, min(3, width - k) + 1))
        q = [int(x) for x in g.choice(width, k + c, replace=False)]
        return {"kind": "controlled", "targets": q[:k], "controls": q[k:],
                "cvals": int(g.integers(1 << c)), "data": haar_unitary(k, g)}
    k = int(g.integers(1, min(kmax, width) + 1))
    t = [int(x) for x in g.choice(width, k, replace=False)]
    return {"kind": "dense", "targets": t, "data": haar_unitary(k, g)}


def random_circuit(width: int, n_gates: int, seed: int, **kw) -> list:
    g = rng(seed)
    return [random_gate(width, g, **kw) for _ in range(n_gates)]


def basis_circuit(width: int, n_gates: int, seed: int) -> list:
    """Random 1q/2q basis-gate stream (Fig. 2-like transpiled shape):
    1q gates are Haar U(2), 2q gates are CX with random control/target."""
    g = rng(seed)
    cx = np.array([[1, 0, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0], [0, 1, 0, 0]], dtype=complex)
    out = []
    for _ in range(n_gates):
        if width >= 2 and g.random() < 0.43:
            a, b = (int(x) for x in g.choice(width, 2, replace=False))
            # matrix index bit0 = targets[0] = control a, bit1 = target b
            out.append({"kind": "dense", "targets": [a, b], "data": cx.copy()})
        else:
            out.append({"kind": "dense", "targets": [int(g.integers(width))], "data": haar_unitary(1, g)})
    return out
