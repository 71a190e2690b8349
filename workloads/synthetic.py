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


def pad_brickwork(pad_qubits, layers: int = 8, seed: int = 2402) -> list:
    """SURVEY §8(d) padded stress circuits, the pad part: `layers` brickwork layers on the pad qubits,
    each a Haar U(2) on every pad qubit (QR of a complex Gaussian) then CZ on alternating neighbouring
    pairs (offset 0 on even layers, 1 on odd layers)."""
    g = rng(seed)
    cz = np.array([1, 1, 1, -1], dtype=complex)
    out = []
    for layer in range(layers):
        for q in pad_qubits:
            out.append({"kind": "dense", "targets": [int(q)], "data": haar_unitary(1, g)})
        for i in range(layer % 2, len(pad_qubits) - 1, 2):
            out.append({"kind": "diagonal", "targets": [int(pad_qubits[i]), int(pad_qubits[i + 1])], "data": cz.copy()})
    return out


def padded_circuit(gates15: list, n15: int, n: int, layers: int = 8):
    """P_n stress circuit: the n15-qubit gate list placed on a seeded random injective map
    of its qubits into n physical qubits (seed 2402 + n), plus brickwork layers on the n - n15 pad
    qubits. Returns (gates, qubit_map, pad_qubits): circuit qubit q of the small list -> qubit_map[q].
    Its final state is the tensor product of the two factors' states, permuted (the tensor-factor pin)."""
    g = rng(2402 + n)
    perm = [int(x) for x in g.permutation(n)]
    qmap = perm[:n15]
    pad = sorted(perm[n15:])

    def remap(x):
        y = dict(x)
        y["targets"] = [qmap[q] for q in x["targets"]]
        if "controls" in x:
            y["controls"] = [qmap[q] for q in x["controls"]]
        return y
    return [remap(x) for x in gates15] + pad_brickwork(pad, layers), qmap, pad


def tensor_factor_amplitudes(psi_small: np.ndarray, qmap, psi_pad: np.ndarray, pad, idx) -> np.ndarray:
    """psi_full[i] = psi_small[bits of i at qmap] * psi_pad[bits of i at pad] (layout bookkeeping only)."""
    idx = np.asarray(idx, dtype=np.int64)
    a = np.zeros_like(idx)
    for j, q in enumerate(qmap):
        a |= ((idx >> q) & 1) << j
    b = np.zeros_like(idx)
    for j, q in enumerate(pad):
        b |= ((idx >> q) & 1) << j
    return psi_small[a] * psi_pad[b]
